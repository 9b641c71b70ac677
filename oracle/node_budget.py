"""CPU oracle of node-level power budgeting -- TEST
INFRASTRUCTURE ONLY (tests/, smoke(), bench.py's cpu_baseline leg).

The job manager sets the power caps of a node's GPUs (PAPER.md L165, L400, L782,
L844): given the sets allocated to the G GPUs of a node and the node budget
P_node, choose one cap per GPU (and, per GPU, the best partition state at that
cap) -- reading R23:
  thr_g(p)  = max over states s with Fairness(S_g, s, p) > alpha of Throughput(S_g, s, p)
              (lowest s on ties; -inf when no state is feasible at p);
  Problem 1: maximise  sum_g thr_g(p_g)                subject to sum_g P(p_g) <= P_node;
  Problem 2: maximise  sum_g thr_g(p_g) / sum_g P(p_g) subject to sum_g P(p_g) <= P_node.
Both are a multiple-choice knapsack on the cap grid; with integer-watt caps the
exact optimum is a dynamic programme over the total power in units of the
caps' gcd: best[b] = max over p of best_prev[b - u(p)] + thr_g(p). FP64 here.
"""
from __future__ import annotations

import math
from functools import reduce
from typing import List, Sequence, Tuple

import numpy as np


def frontier(orc, rows) -> Tuple[np.ndarray, np.ndarray]:
    """(thr[n_caps], state[n_caps]) of one set: the best feasible Throughput per cap."""
    pb = orc.pb
    _, fair, thr, feas, _ = orc.eval_set(rows)
    nc = pb.n_caps
    best = np.full(nc, -math.inf)
    arg = np.full(nc, -1, dtype=np.int64)
    for s in range(pb.n_states):
        for p in range(nc):
            c = s * nc + p
            if feas[c] and thr[c] > best[p]:
                best[p] = thr[c]
                arg[p] = s
    return best, arg


def cap_units(caps_w) -> Tuple[int, np.ndarray]:
    w = [int(round(float(c))) for c in caps_w]
    if any(abs(float(c) - x) > 0 for c, x in zip(caps_w, w)):
        raise ValueError("caps must be integer watts")
    g = reduce(math.gcd, w)
    return g, np.array([x // g for x in w], dtype=np.int64)


def solve_node(fronts: Sequence[np.ndarray], caps_w, node_w: float, objective: int):
    """(objective value, caps per GPU) of one node by the DP (-inf, [] if infeasible)."""
    unit, u = cap_units(caps_w)
    U = int(math.floor(node_w / unit + 1e-9))
    best = np.full(U + 1, -math.inf)
    best[0] = 0.0
    choice = []
    for f in fronts:
        new = np.full(U + 1, -math.inf)
        ch = np.full(U + 1, -1, dtype=np.int64)
        for p in range(len(u)):
            if f[p] == -math.inf or u[p] > U:
                continue
            cand = np.full(U + 1, -math.inf)
            cand[u[p]:] = best[:U + 1 - u[p]] + f[p]
            better = cand > new  # strict: the lowest cap index wins ties
            new = np.where(better, cand, new)
            ch = np.where(better, p, ch)
        best = new
        choice.append(ch)
    if objective == 1:
        vals = best
    else:
        vals = np.where(np.arange(U + 1) > 0, best / (np.arange(U + 1) * unit), -math.inf)
    if not np.any(vals > -math.inf):
        return -math.inf, []
    b = int(np.argmax(vals))  # the lowest total power on ties
    val = float(vals[b])
    caps = []
    for ch in reversed(choice):
        p = int(ch[b])
        caps.append(p)
        b -= int(u[p])
    return val, caps[::-1]


def brute_node(fronts, caps_w, node_w, objective):
    """Exhaustive enumeration of every cap combination (tiny nodes only)."""
    import itertools
    best, arg = -math.inf, []
    for combo in itertools.product(range(len(caps_w)), repeat=len(fronts)):
        P = sum(float(caps_w[p]) for p in combo)
        if P > node_w + 1e-9:
            continue
        t = sum(f[p] for f, p in zip(fronts, combo))
        if t == -math.inf:
            continue
        v = t if objective == 1 else t / P
        if v > best:
            best, arg = v, list(combo)
    return best, arg
