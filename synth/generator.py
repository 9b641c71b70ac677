"""Seeded, bit-stable synthetic inputs (DESIGN.md §"Input recipe").

Everything here is INPUT construction: counter vectors F shaped like the
paper's four workload classes (Table `classification`
L610-625), the partition tables (Table `search-space` L556-566 and the
flexible 8-GPC splits of L500/L794), power-cap grids and random-structured
coefficient tables. No basis function, model term, objective or search lives
here; the oracle and the CUDA path each implement those on their own.

Randomness: a splitmix64 stream (Steele et al.), vectorised in numpy uint64
arithmetic, so the bytes are identical on every machine and numpy version.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

G_FULL = 8  # GPCs of the unpartitioned chip = the RPerf normalisation point

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


class SplitMix64:
    """Counter-based splitmix64: output k of seed s is mix(s + (k+1)*golden)."""

    def __init__(self, seed: int):
        self.state = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
        self.counter = 0

    def next_u64(self, n: int) -> np.ndarray:
        with np.errstate(over="ignore"):
            k = np.arange(self.counter + 1, self.counter + 1 + n, dtype=np.uint64)
            z = self.state + k * _GOLDEN
            z = (z ^ (z >> np.uint64(30))) * _M1
            z = (z ^ (z >> np.uint64(27))) * _M2
            z = z ^ (z >> np.uint64(31))
        self.counter += n
        return z

    def uniform(self, n: int) -> np.ndarray:
        """n doubles in [0, 1) with 53 random bits each."""
        return (self.next_u64(n) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


# ---------------------------------------------------------------------------
# Workload classes (SURVEY.md §8(d) feature table), percent.
# (lo, hi) for F1..F5; tensor share of F1 for TI only.
CLASS_RANGES: Dict[str, Dict[str, Tuple[float, float]]] = {
    "TI": {"F1": (60, 95), "F2": (20, 60), "F3": (5, 40), "F4": (40, 95), "F5": (10, 50), "T": (0.5, 1.0)},
    "CI": {"F1": (50, 95), "F2": (10, 60), "F3": (5, 40), "F4": (40, 95), "F5": (30, 90), "T": (0.0, 0.0)},
    "MI": {"F1": (5, 45), "F2": (60, 98), "F3": (50, 95), "F4": (5, 50), "F5": (30, 90), "T": (0.0, 0.0)},
    "US": {"F1": (1, 25), "F2": (1, 30), "F3": (0, 20), "F4": (20, 90), "F5": (5, 40), "T": (0.0, 0.0)},
}
CLASSES = ("TI", "CI", "MI", "US")

# Class shares. `paper` = Table `classification` counts 7/6/5/6 of 24.
MIXES: Dict[str, Dict[str, float]] = {
    "paper": {"TI": 7 / 24, "CI": 6 / 24, "MI": 5 / 24, "US": 6 / 24},
    "rodinia": {"TI": 0.0, "CI": 4 / 13, "MI": 3 / 13, "US": 6 / 13},
    "dl": {"TI": 0.7, "CI": 0.1, "MI": 0.2, "US": 0.0},
    "npb": {"TI": 0.0, "CI": 0.5, "MI": 0.4, "US": 0.1},
}

# Where a TI job's tensor share lands: F6 mixed (tf32/h/fp16/bf16gemm, 4 of 7),
# F7 double (tdgemm, 1 of 7), F8 integer (igemm4/8, 2 of 7) -- PAPER.md L598-604, L618.
_TENSOR_SLOTS = ((4 / 7, 5), (5 / 7, 6), (1.0, 7))


def make_features(n: int, seed: int, mix: str = "paper",
                  classes: Optional[Sequence[str]] = None) -> Tuple[np.ndarray, List[str]]:
    """float32 F[n][8] (percent, order F1..F8 as PAPER.md L531) and class labels.

    Eight uniforms are drawn per job whatever its class, so job k's bytes
    depend only on (seed, k, mix).
    """
    rng = SplitMix64(seed)
    u = rng.uniform(8 * n).reshape(n, 8) if n else np.zeros((0, 8))
    shares = MIXES[mix]
    cum = np.cumsum([shares[c] for c in CLASSES])
    F = np.zeros((n, 8), dtype=np.float64)
    labels: List[str] = []
    for k in range(n):
        if classes is not None:
            cl = classes[k]
        else:
            idx = int(np.searchsorted(cum, u[k, 0] * cum[-1], side="right"))
            cl = CLASSES[min(idx, 3)]
        r = CLASS_RANGES[cl]
        for f, name in enumerate(("F1", "F2", "F3", "F4", "F5")):
            lo, hi = r[name]
            F[k, f] = lo + (hi - lo) * u[k, 1 + f]
        tlo, thi = r["T"]
        if thi > 0:
            t = (tlo + (thi - tlo) * u[k, 6]) * F[k, 0]
            for bound, col in _TENSOR_SLOTS:
                if u[k, 7] < bound:
                    F[k, col] = t
                    break
        labels.append(cl)
    return F.astype(np.float32), labels


def tie_stress_features(n: int, seed: int, frac: float = 0.25, mix: str = "paper") -> np.ndarray:
    """A queue where ~frac of the jobs are exact copies of another job (exact model ties)."""
    F, _ = make_features(n, seed, mix)
    rng = SplitMix64(seed ^ 0x5EED)
    u = rng.uniform(2 * n).reshape(n, 2)
    for k in range(n):
        if u[k, 0] < frac:
            src = int(u[k, 1] * n) % n
            F[k] = F[src]
    return F


# ---------------------------------------------------------------------------
# Partition tables (state order = the tie-break order).

@dataclass
class Problem:
    """The searchable space + model coefficients; field names mirror cosched_desc."""
    name: str
    n_slots: int
    gpcs_total: int
    state_gpcs: np.ndarray   # int32 [n_states][n_slots]
    state_mem: np.ndarray    # int32 [n_states]  0 shared, 1 private
    state_slice: np.ndarray  # int32 [n_states][n_slots]
    slices: List[Tuple[int, int]]  # slice id -> (gpcs, mem)
    caps_w: np.ndarray       # float32 [n_caps], ascending
    coef_c: np.ndarray = field(default=None)  # float32 [n_caps][n_slices][6]
    coef_d: np.ndarray = field(default=None)  # float32 [n_caps][n_slices][3]
    objective: int = 2
    alpha: float = 0.2

    @property
    def n_states(self) -> int:
        return int(self.state_gpcs.shape[0])

    @property
    def n_slices(self) -> int:
        return len(self.slices)

    @property
    def n_caps(self) -> int:
        return int(self.caps_w.shape[0])

    @property
    def n_configs(self) -> int:
        return self.n_states * self.n_caps


def _compositions(total: int, parts: int) -> List[Tuple[int, ...]]:
    if parts == 1:
        return [(total,)] if total >= 1 else []
    out = []
    for first in range(total - parts + 1, 0, -1):  # descending lexicographic
        for rest in _compositions(total - first, parts - 1):
            out.append((first,) + rest)
    return out


def partition_table(name: str):
    """(n_slots, gpcs_total, [(gpcs tuple, mem)] in canonical order).

    a100_paper: S1..S4 of Table `search-space`, 7 usable GPCs (L283).
    b200:       (7,1),(6,2),...,(1,7) shared then private (flexible splits, L500/L794).
    b200_3way:  the 21 compositions of 8 into 3 parts, descending lex, x {shared, private}.
    solo:       one job on the unpartitioned chip (normalisation point, L410/L444).
    """
    if name in ("a100_paper", "a100_50w", "a100_p1"):
        states = [((4, 3), 0), ((3, 4), 0), ((4, 3), 1), ((3, 4), 1)]
        return 2, 7, states
    if name == "b200":
        st = [((g, G_FULL - g), m) for m in (0, 1) for g in range(7, 0, -1)]
        return 2, 8, st
    if name == "b200_3way":
        comps = _compositions(G_FULL, 3)
        st = [(c, m) for m in (0, 1) for c in comps]
        return 3, 8, st
    if name == "solo":
        return 1, 8, [((8,), 0)]
    raise KeyError(name)


def cap_grid(name: str) -> np.ndarray:
    grids = {
        "a100_paper": [150, 170, 190, 210, 230, 250],      # PAPER.md L565 ("230 250" typo read as two caps)
        "a100_50w": [50, 100, 150, 200, 250],              # BASELINE.json 50 W steps
        "a100_230": [230],                                 # Problem 1 at P = 230 W
        "c10": list(range(550, 1001, 50)),                 # B200-like, 10 caps @ 50 W
        "c21": list(range(500, 1001, 25)),                 # B200-like, 21 caps @ 25 W
        "c1_900": [900],
        "c1_1000": [1000],
    }
    return np.asarray(grids[name], dtype=np.float32)


def _slices_for(states) -> List[Tuple[int, int]]:
    used = sorted({(g, m) for gp, m in states for g in gp}, key=lambda x: (x[1], x[0]))
    used = [s for s in used if s != (G_FULL, 0)]
    return used + [(G_FULL, 0)]  # the baseline slice (full chip, shared) is always last


def make_coefficients(slices: List[Tuple[int, int]], caps_w: np.ndarray, seed: int,
                      jitter: float = 0.10, mirror_ties: bool = False) -> Tuple[np.ndarray, np.ndarray]:
    """Random-structured C[n_caps][n_slices][6], D[..][3] (SURVEY.md §8(d) coefficient recipe).

    For slice (g, mem) at cap P: x = g/G_full, y = P/P_max, bw = 1 (shared) or g/G_full (private):
      C = (-(1-x*y), -(1-x*y^1.5), -0.05(1-bw), 0.05(1-x), -0.2(1-x), 1)
      D = (-0.45, -0.05, 0) shared, (-0.05, 0, 0) private      (private mitigates interference)
    then a +-jitter multiplicative draw per entry. The baseline slice (G_full, shared) at
    P_max is exactly C = e6, D = 0 (reading R11: a least-squares fit to targets == 1
    with a constant column). These numbers are synthetic, not hardware claims.
    """
    n_caps, n_sl = len(caps_w), len(slices)
    pmax = float(np.max(caps_w))
    C = np.zeros((n_caps, n_sl, 6), dtype=np.float64)
    D = np.zeros((n_caps, n_sl, 3), dtype=np.float64)
    for p in range(n_caps):
        y = float(caps_w[p]) / pmax
        for s, (g, m) in enumerate(slices):
            x = g / G_FULL
            bw = 1.0 if m == 0 else x
            C[p, s] = (-(1 - x * y), -(1 - x * y ** 1.5), -0.05 * (1 - bw),
                       0.05 * (1 - x), -0.2 * (1 - x), 1.0)
            D[p, s] = (-0.45, -0.05, 0.0) if m == 0 else (-0.05, 0.0, 0.0)
    rng = SplitMix64(seed)
    jc = 1.0 + jitter * (2.0 * rng.uniform(C.size).reshape(C.shape) - 1.0)
    jd = 1.0 + jitter * (2.0 * rng.uniform(D.size).reshape(D.shape) - 1.0)
    C *= jc
    D *= jd
    base = slices.index((G_FULL, 0))
    C[n_caps - 1, base] = (0, 0, 0, 0, 0, 1)
    D[n_caps - 1, base] = (0, 0, 0)
    if mirror_ties:
        idx = {sl: i for i, sl in enumerate(slices)}
        for (g, m), i in idx.items():
            mirror = (G_FULL - g, m)
            if g < G_FULL - g and mirror in idx:
                C[:, idx[mirror]] = C[:, i]
                D[:, idx[mirror]] = D[:, i]
    return C.astype(np.float32), D.astype(np.float32)


def make_problem(table: str, caps: str, coef_seed: int, objective: int = 2, alpha: float = 0.2,
                 jitter: float = 0.10, mirror_ties: bool = False) -> Problem:
    n_slots, gtot, states = partition_table(table)
    slices = _slices_for(states)
    sidx = {sl: i for i, sl in enumerate(slices)}
    gp = np.asarray([s[0] for s in states], dtype=np.int32).reshape(len(states), n_slots)
    mem = np.asarray([s[1] for s in states], dtype=np.int32)
    ssl = np.asarray([[sidx[(g, m)] for g in s[0]] for (s, m) in zip(states, mem)],
                     dtype=np.int32).reshape(len(states), n_slots)
    caps_w = cap_grid(caps)
    C, D = make_coefficients(slices, caps_w, coef_seed, jitter=jitter, mirror_ties=mirror_ties)
    return Problem(name=f"{table}x{caps}", n_slots=n_slots, gpcs_total=gtot, state_gpcs=gp,
                   state_mem=mem, state_slice=ssl, slices=slices, caps_w=caps_w,
                   coef_c=C, coef_d=D, objective=objective, alpha=alpha)


# ---------------------------------------------------------------------------
# BASELINE.json configs (SURVEY.md §8(d) "Configs restated").

BENCH_CONFIGS = {
    "C1": dict(n_jobs=2, table="a100_paper", caps="a100_50w", classes=("TI", "MI"), mix="paper", k=1),
    "C2": dict(n_jobs=8, table="b200", caps="c10", mix="paper", k=4),
    "C3": dict(n_jobs=1000, table="b200", caps="c10", mix="paper", k=500),
    "C4": dict(n_jobs=10000, table="b200", caps="c21", mix="paper", k=5000),
    "C5": dict(n_jobs=2000, table="b200_3way", caps="c21", mix="paper", k=666),
}
_CFG_NUM = {"C1": 1, "C2": 2, "C3": 3, "C4": 4, "C5": 5}


def bench_config(name: str, seed_offset: int = 0, alpha: float = 0.2, objective: int = 2):
    """(problem, F float32[n][8]) for a BASELINE.json config; seeds 1000+k / 2000+k (+offset)."""
    spec = BENCH_CONFIGS[name]
    k = _CFG_NUM[name]
    prob = make_problem(spec["table"], spec["caps"], coef_seed=2000 + k + seed_offset,
                        objective=objective, alpha=alpha)
    F, _ = make_features(spec["n_jobs"], seed=1000 + k + seed_offset, mix=spec["mix"],
                         classes=spec.get("classes"))
    return prob, F
