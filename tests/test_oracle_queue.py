"""Pins of the oracle's queue-level parts: set enumeration (colex ids), the
best set, exact allocation and greedy allocation -- against brute force over
tiny queues and the closed-form counts (BASELINE.json north_star: the number
of pairings of 2n jobs is (2n-1)!!)."""
import itertools
import math

import numpy as np
import pytest

import oracle
from oracle import Oracle
from synth import make_features, make_problem


@pytest.mark.parametrize("k", [1, 2, 3])
def test_colex_unrank_is_a_bijection_in_colex_order(k):
    for n in range(k, 13):
        combos = sorted(itertools.combinations(range(n), k), key=lambda c: c[::-1])  # colex
        assert oracle.n_sets(n, k) == len(combos) == math.comb(n, k)
        for sid, c in enumerate(combos):
            assert oracle.unrank(n, k, sid) == c


def test_unrank_rejects_out_of_range():
    with pytest.raises(ValueError):
        oracle.unrank(5, 2, 10)
    with pytest.raises(ValueError):
        oracle.unrank(5, 2, -1)


def test_score_range_matches_per_set_search():
    """score_range walks sets in colex order; each entry equals the per-set search of its jobs."""
    pb = make_problem("b200", "c10", coef_seed=5, alpha=0.6)
    F, _ = make_features(14, seed=5)
    jobs = np.array([3, 1, 4, 1, 5, 9, 2, 6, 5, 3, 5, 8], dtype=np.int32)  # rows may repeat
    o = Oracle(pb)
    cfg, obj = o.score_range(F, jobs)
    assert len(cfg) == math.comb(12, 2)
    for sid, (a, b) in enumerate(sorted(itertools.combinations(range(12), 2), key=lambda c: c[::-1])):
        c, ob = o.best_config([F[jobs[a]], F[jobs[b]]])
        assert (c, ob) == (cfg[sid], obj[sid])
    # a sub-range gives the same entries
    c2, o2 = o.score_range(F, jobs, first=17, count=20)
    assert np.array_equal(c2, cfg[17:37]) and np.array_equal(o2, obj[17:37])
    assert (cfg == -1).any() and (cfg >= 0).any()   # alpha 0.6 mixes feasible and infeasible


def test_best_set_brute_force():
    pb = make_problem("b200_3way", "c10", coef_seed=6, alpha=0.2)
    F, _ = make_features(9, seed=6)
    o = Oracle(pb)
    best = (-math.inf, -1)
    for sid, t in enumerate(sorted(itertools.combinations(range(9), 3), key=lambda c: c[::-1])):
        c, ob = o.best_config([F[i] for i in t])
        if c >= 0 and ob > best[0]:
            best = (ob, sid)
    st, sid, cfg, ob = o.best_set(F)
    assert st == oracle.OK and (ob, sid) == best


def _double_factorial(m):
    return math.prod(range(m, 0, -2)) if m > 0 else 1


@pytest.mark.parametrize("n", [2, 4, 6, 8, 10, 12])
def test_number_of_pairings(n):
    """(2k-1)!! perfect matchings of 2k jobs; 105 for the 8-job queue of BASELINE.json config 2."""
    so = np.ones(math.comb(n, 2))
    st, rank, ids, tot, nm = oracle.exact_allocation(n, 2, so)
    assert nm == _double_factorial(n - 1)
    if n == 8:
        assert nm == 105


@pytest.mark.parametrize("n", [3, 6, 9, 12])
def test_number_of_triple_partitions(n):
    k = n // 3
    so = np.ones(math.comb(n, 3))
    st, rank, ids, tot, nm = oracle.exact_allocation(n, 3, so)
    assert nm == math.factorial(n) // (math.factorial(k) * 6 ** k)


def _brute_partitions(n, k):
    """Independent construction: every permutation cut into k-blocks, canonicalised,
    deduplicated, ordered lexicographically by the canonical block list (which is the
    lowest-free-job-first, partners-ascending order)."""
    seen = set()
    for perm in itertools.permutations(range(n)):
        blocks = tuple(sorted(tuple(sorted(perm[i:i + k])) for i in range(0, n, k)))
        seen.add(blocks)
    return sorted(seen)


def _colex_id(t):
    return sum(math.comb(v, i + 1) for i, v in enumerate(sorted(t)))


@pytest.mark.parametrize("n,k,seed", [(6, 2, 1), (8, 2, 2), (8, 2, 3), (6, 3, 4), (9, 3, 5)])
def test_exact_allocation_brute_force(n, k, seed):
    table = "b200" if k == 2 else "b200_3way"
    pb = make_problem(table, "c10", coef_seed=100 + seed, alpha=0.62 if k == 2 else 0.3)
    F, _ = make_features(n, seed=100 + seed)
    o = Oracle(pb)
    cfg, obj = o.score_range(F)
    parts = _brute_partitions(n, k)
    best = (-math.inf, None, None)
    for r, blocks in enumerate(parts):
        vals = [obj[_colex_id(b)] for b in blocks]
        if any(v == -math.inf for v in vals):
            continue
        w = 0.0
        for v in vals:
            w += v
        if w > best[0]:
            best = (w, r, [_colex_id(b) for b in blocks])
    st, rank, ids, tot, nm = oracle.exact_allocation(n, k, obj)
    assert nm == len(parts)
    if best[1] is None:
        assert st == oracle.INFEASIBLE and rank == -1
    else:
        assert st == oracle.OK and rank == best[1] and tot == best[0] and ids == best[2]


def test_exact_allocation_ties_and_infeasible():
    # all equal -> the first partition (rank 0): {0,1},{2,3},{4,5}
    so = np.full(15, 1.0)
    st, rank, ids, tot, nm = oracle.exact_allocation(6, 2, so)
    assert rank == 0 and ids == [_colex_id((0, 1)), _colex_id((2, 3)), _colex_id((4, 5))]
    # forbid {0,1}: first remaining is {0,2},{1,3},{4,5}  (rank 3: partners of 0 ascending, 3 matchings each)
    so[_colex_id((0, 1))] = -math.inf
    st, rank, ids, tot, nm = oracle.exact_allocation(6, 2, so)
    assert rank == 3 and ids[0] == _colex_id((0, 2))
    assert oracle.exact_allocation(4, 2, np.full(6, -math.inf))[0] == oracle.INFEASIBLE


def test_greedy_is_exact_on_planted_instance():
    """When one perfect matching's sets dominate every other set, greedy finds exactly it."""
    n = 10
    rng = np.random.default_rng(3)
    perm = rng.permutation(n)
    so = rng.uniform(0.1, 1.0, math.comb(n, 2))
    planted = [tuple(sorted(perm[i:i + 2])) for i in range(0, n, 2)]
    for t, v in zip(planted, [5, 4, 3, 2, 1.5]):
        so[_colex_id(t)] = v
    got = oracle.greedy_allocation(n, 2, so, 5)
    assert got == [_colex_id(t) for t in planted]
    st, rank, ids, tot, nm = oracle.exact_allocation(n, 2, so)
    assert sorted(ids) == sorted(got)


def test_greedy_properties():
    pb = make_problem("b200", "c10", coef_seed=8, alpha=0.62)
    F, _ = make_features(40, seed=8)
    cfg, obj = Oracle(pb).score_range(F)
    k = 20
    got = oracle.greedy_allocation(40, 2, obj, k)
    used = set()
    prev = math.inf
    for sid in got:
        j = oracle.unrank(40, 2, sid)
        assert not used & set(j) and obj[sid] > -math.inf
        assert obj[sid] <= prev
        # sid is the max over sets disjoint from the earlier picks (ties -> lowest id)
        cands = [(obj[t], -t) for t in range(len(obj))
                 if obj[t] > -math.inf and not used & set(oracle.unrank(40, 2, t))]
        assert max(cands) == (obj[sid], -sid)
        used |= set(j)
        prev = obj[sid]
    # maximal: no remaining feasible set is disjoint from the chosen ones (unless k reached)
    if len(got) < k:
        for t in range(len(obj)):
            if obj[t] > -math.inf:
                assert used & set(oracle.unrank(40, 2, t))


def test_all_cores_split_equals_single_process():
    """tests/oracle_parallel.py only splits the work: identical results to one process."""
    from oracle_parallel import score_range_all_cores
    for table, n in (("b200", 57), ("b200_3way", 23)):
        pb = make_problem(table, "c10", coef_seed=9)
        F, _ = make_features(n, seed=9)
        cfg1, obj1 = Oracle(pb).score_range(F)
        cfg2, obj2, _ = score_range_all_cores(pb, F, procs=3)
        assert np.array_equal(cfg1, cfg2) and np.array_equal(obj1, obj2)
        cfg3, obj3, _ = score_range_all_cores(pb, F, first=100, count=333, procs=2)
        assert np.array_equal(cfg3, cfg1[100:433]) and np.array_equal(obj3, obj1[100:433])
