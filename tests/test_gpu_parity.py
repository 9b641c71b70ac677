"""GPU (CUDA path through the C-ABI) vs the FP64 oracle, on seeded synthetic inputs.

Bar: chosen config / set / allocation indices equal to the oracle's up to the
tie-aware rule of tests/parity.py (objectives within 1e-5 relative); integer
outputs (set ids, unranking, counts, statuses) bit-exact.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from oracle import Oracle  # noqa: E402
from synth import bench_config, make_features, make_problem, tie_stress_features  # noqa: E402
from parity import TAU_OBJ, accept_set, check_sets, replay_greedy  # noqa: E402


@pytest.fixture(scope="module")
def cs():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2405_03838_b200 as cs
    return cs


def _run(cs, pb, F, jobs=None, variant=None):
    s = cs.Scheduler(pb)
    if variant is not None:
        s.set_variant(variant)
    Fd = torch.from_numpy(np.ascontiguousarray(F)).cuda()
    Jd = None if jobs is None else torch.from_numpy(np.ascontiguousarray(jobs, dtype=np.int32)).cuda()
    obj, cfg = s.score_all(Fd, Jd)
    torch.cuda.synchronize()
    return s, obj.cpu().numpy(), cfg.cpu().numpy()


def _full_parity(cs, pb, F, jobs=None, variant=None):
    s, obj_g, cfg_g = _run(cs, pb, F, jobs, variant)
    n = F.shape[0] if jobs is None else len(jobs)
    o = Oracle(pb)
    cfg_o, obj_o = o.score_range(F, jobs)
    assert len(cfg_g) == len(cfg_o)
    mism = np.nonzero(cfg_g != cfg_o)[0]
    # where the index agrees the objective must agree to 1e-5 relative
    same = (cfg_g == cfg_o) & (cfg_o >= 0)
    rel = np.abs(obj_g[same].astype(np.float64) - obj_o[same]) / np.abs(obj_o[same])
    assert rel.max(initial=0) <= TAU_OBJ, rel.max()
    assert np.all(obj_g[cfg_g < 0] == -np.inf)
    # index disagreements must be ties under the tie-aware rule
    exact, fails = check_sets(o, F, jobs, mism, cfg_g[mism], obj_g[mism], n, pb.n_slots)
    assert not fails, fails[:5]
    return s, obj_g, cfg_g, cfg_o, obj_o, len(mism)


# ---- configs C1-C3 exhaustively ------------------------------------------------

def test_c1_single_pair(cs):
    pb, F = bench_config("C1")
    s, obj_g, cfg_g, cfg_o, obj_o, nm = _full_parity(cs, pb, F)
    assert nm == 0 and cfg_g[0] == cfg_o[0]
    d = s.best_config(0)
    o = Oracle(pb)
    _, fair, thr, _, rp = o.eval_set([F[0], F[1]])
    c = d["cfg"]
    assert np.allclose(d["rperf"], rp[c], atol=1e-5) and abs(d["throughput"] - thr[c]) < 1e-5
    assert abs(d["fairness"] - fair[c]) < 1e-5
    st, sid, cfg, ob = s.best_set()
    assert (st, sid, cfg) == (0, 0, cfg_o[0])


def test_c2_pairs_best_set_and_exact_allocation(cs):
    pb, F = bench_config("C2")
    s, obj_g, cfg_g, cfg_o, obj_o, nm = _full_parity(cs, pb, F)
    st, sid, cfg, ob = s.best_set()
    ost, osid, ocfg, oob = Oracle(pb).best_set(F)
    assert st == ost == 0
    assert sid == osid or obj_o[sid] >= oob * (1 - TAU_OBJ)
    # exact allocation over the 105 pairings (BASELINE.json config 2)
    st, ids, cfgs, tot = s.best_allocation(4)
    ost, rank, oids, otot, nmatch = oracle.exact_allocation(8, 2, obj_o)
    assert nmatch == 105 and st == ost == 0
    w_gpu_by_oracle = sum(obj_o[i] for i in ids)
    assert ids == oids or w_gpu_by_oracle >= otot * (1 - TAU_OBJ)
    assert abs(tot - otot) <= TAU_OBJ * abs(otot)
    assert sorted(sum((list(oracle.unrank(8, 2, i)) for i in ids), [])) == list(range(8))
    assert cfgs == [int(cfg_g[i]) for i in ids]


@pytest.mark.parametrize("variant", [0, 1])
def test_c3_all_pairs(cs, variant):
    pb, F = bench_config("C3")
    s, obj_g, cfg_g, cfg_o, obj_o, nm = _full_parity(cs, pb, F, variant=variant)
    assert nm <= len(cfg_g) * 1e-3  # index disagreements are rare (and all were ties)
    st, sid, cfg, ob = s.best_set()
    best_o = obj_o.max()
    assert st == 0 and obj_o[sid] >= best_o * (1 - TAU_OBJ)


def test_c3_greedy_allocation(cs):
    pb, F = bench_config("C3")
    s, obj_g, cfg_g = _run(cs, pb, F)
    st, ids, cfgs, tot = s.best_allocation(500)
    assert st == 0 and len(ids) == 500
    _, obj_o = Oracle(pb).score_range(F)
    ok, why = replay_greedy(1000, 2, obj_o, ids)
    assert ok, why
    assert cfgs == [int(cfg_g[i]) for i in ids]
    gk = [obj_g[i] for i in ids]
    assert all(a >= b for a, b in zip(gk, gk[1:]))


@pytest.mark.parametrize("batch", ["3000", "20000", "100000"])
@pytest.mark.parametrize("table,n,k", [("b200", 600, 300), ("b200_3way", 120, 40)])
def test_greedy_many_batches_and_endgame(cs, batch, table, n, k, monkeypatch):
    """Small greedy batches (COSCHED_GREEDY_BATCH) force many histogram batches, the
    alive-scaled batch sizing and the endgame enumeration of the free jobs' sets: the
    picks must still replay the oracle's sequential greedy exactly (tie-aware)."""
    monkeypatch.setenv("COSCHED_GREEDY_BATCH", batch)
    pb = make_problem(table, "c21", coef_seed=81, alpha=0.2)
    F, _ = make_features(n, seed=81)
    ns = pb.n_slots
    s, obj_g, cfg_g = _run(cs, pb, F)
    st, ids, cfgs, tot = s.best_allocation(k)
    _, obj_o = Oracle(pb).score_range(F)
    ok, why = replay_greedy(n, ns, obj_o, ids)
    assert ok, why
    # as many picks as the oracle's greedy finds (it stops only when no disjoint feasible set is left)
    ref = oracle.greedy_allocation(n, ns, obj_o, k)
    assert len(ids) == len(ref), (len(ids), len(ref))


# ---- edge cases ----------------------------------------------------------------------

@pytest.mark.parametrize("n", [2, 3, 31, 33, 65, 127, 130])
def test_ragged_queue_sizes(cs, n):
    pb = make_problem("b200", "c21", coef_seed=50 + n, alpha=0.62)
    F, _ = make_features(n, seed=50 + n)
    for variant in (0, 1):
        _full_parity(cs, pb, F, variant=variant)


def test_empty_and_single_job_queue(cs):
    pb = make_problem("b200", "c10", coef_seed=3)
    F, _ = make_features(1, seed=3)
    s, obj_g, cfg_g = _run(cs, pb, F)
    assert len(cfg_g) == 0
    st, sid, cfg, ob = s.best_set()
    assert st == 2 and sid == -1


def test_all_infeasible(cs):
    pb = make_problem("b200", "c10", coef_seed=4, alpha=10.0)
    F, _ = make_features(40, seed=4)
    s, obj_g, cfg_g = _run(cs, pb, F)
    assert (cfg_g == -1).all() and np.all(obj_g == -np.inf)
    assert s.best_set()[0] == 2
    assert s.best_allocation(20)[0] == 2


def test_jobs_indirection_with_repeats(cs):
    pb = make_problem("b200", "c21", coef_seed=7, alpha=0.6)
    F, _ = make_features(50, seed=7)
    jobs = np.array([(i * 7) % 50 for i in range(70)], dtype=np.int32)  # repeats rows
    _full_parity(cs, pb, F, jobs)


def test_tie_stress_duplicates(cs):
    """Duplicated jobs create exact ties between mirrored states: the lowest config must win."""
    pb = make_problem("b200", "c21", coef_seed=8, alpha=0.2, mirror_ties=True)
    F = tie_stress_features(120, seed=8, frac=0.25)
    for variant in (0, 1):
        s, obj_g, cfg_g, cfg_o, obj_o, nm = _full_parity(cs, pb, F, variant=variant)


def test_problem1_one_cap(cs):
    pb = make_problem("b200", "c1_900", coef_seed=9, objective=1, alpha=0.3)
    F, _ = make_features(90, seed=9)
    _full_parity(cs, pb, F)


def test_alpha_zero_and_high(cs):
    for alpha in (0.0, 0.7):
        pb = make_problem("b200", "c10", coef_seed=10, alpha=alpha)
        F, _ = make_features(80, seed=10)
        _full_parity(cs, pb, F)


def test_triples_small(cs):
    pb = make_problem("b200_3way", "c21", coef_seed=11, alpha=0.2)
    F, _ = make_features(24, seed=11)
    s, obj_g, cfg_g, cfg_o, obj_o, nm = _full_parity(cs, pb, F)
    st, ids, cfgs, tot = s.best_allocation(8)  # greedy (24 > 15)
    ok, why = replay_greedy(24, 3, obj_o, ids)
    assert ok, why


def test_triples_exact_allocation(cs):
    pb = make_problem("b200_3way", "c10", coef_seed=12, alpha=0.2)
    F, _ = make_features(9, seed=12)
    s, obj_g, cfg_g, cfg_o, obj_o, nm = _full_parity(cs, pb, F)
    st, ids, cfgs, tot = s.best_allocation(3)
    ost, rank, oids, otot, nmatch = oracle.exact_allocation(9, 3, obj_o)
    assert nmatch == 280 and st == ost == 0
    assert ids == oids or sum(obj_o[i] for i in ids) >= otot * (1 - TAU_OBJ)


@pytest.mark.parametrize("table", ["b200", "b200_3way"])
def test_tiny_fairness_margins(cs, table):
    """Margins RPerf - alpha of 1e-20..1e-30 (alpha = 0, constant-only C rows): the
    scaled margins flush them to 0 (infeasible, inside tau_f), and the tiled scorers
    never mistake a tiny positive margin for the objective."""
    pb = make_problem(table, "c10", coef_seed=14, alpha=0.0)
    rng = np.random.default_rng(14)
    vals = np.array([1e-20, 1e-30, 3e-38, 0.5, 2.0, 1e-6], dtype=np.float32)
    C = np.zeros_like(pb.coef_c)
    C[..., 5] = vals[rng.integers(0, len(vals), size=C.shape[:2])]
    C[:, -1, :] = pb.coef_c[:, -1, :]  # keep the baseline slice
    pb.coef_c = C
    pb.coef_d = np.zeros_like(pb.coef_d)
    F, _ = make_features(70 if table == "b200" else 20, seed=14)
    r0 = _full_parity(cs, pb, F, variant=0)
    r1 = _full_parity(cs, pb, F, variant=1)
    assert np.array_equal(r0[2], r1[2]) and np.array_equal(r0[1], r1[1])


def test_solo_normalisation(cs):
    """A solo job on the full chip at P_max has RPerf exactly 1 (C = e6, D = 0)."""
    pb = make_problem("solo", "c10", coef_seed=13, objective=1, alpha=0.0)
    F, _ = make_features(64, seed=13)
    s, obj_g, cfg_g, cfg_o, obj_o, nm = _full_parity(cs, pb, F)
    for sid in (0, 17, 63):
        d = s.best_config(sid)
        if d["cap"] == pb.n_caps - 1:
            assert d["rperf"][0] == 1.0


def test_validation_errors(cs):
    pb = make_problem("b200", "c10", coef_seed=14)
    F, _ = make_features(20, seed=14)
    for row, col, val, code in [(5, 0, 0.001, 13), (7, 3, 150.0, 14), (9, 2, float("nan"), 14)]:
        G = F.copy()
        G[row, col] = val
        G[row + 3, 0] = 0.0  # a later bad job must not win
        s = cs.Scheduler(pb)
        s.score_all(torch.from_numpy(G).cuda())
        with pytest.raises(cs.CoschedError) as e:
            s.best_set()
        assert e.value.status == code and f"job {row}" in str(e.value)
        assert Oracle.validate_features(G)[0] == code


def test_create_validation(cs):
    bad = make_problem("b200", "c10", coef_seed=1)
    bad.state_gpcs = bad.state_gpcs.copy()
    bad.state_gpcs[0, 0] = 6
    with pytest.raises(cs.CoschedError) as e:
        cs.Scheduler(bad)
    assert e.value.status == 11 and Oracle(bad).validate()[0] == 11
    bad = make_problem("b200", "c10", coef_seed=1)
    bad.state_slice = bad.state_slice.copy()
    bad.state_slice[2, 1] = 40
    with pytest.raises(cs.CoschedError) as e:
        cs.Scheduler(bad)
    assert e.value.status == 12


# ---- multi-GPU sharding on one GPU (fake ranks) ---------------------------------------

@pytest.mark.parametrize("W", [2, 3, 4, 8])
def test_fake_ranks_equal_single_rank(cs, W):
    pb = make_problem("b200", "c21", coef_seed=15, alpha=0.3)
    F, _ = make_features(301, seed=15)
    s1, obj1, cfg1 = _run(cs, pb, F)
    key1 = s1.local_best_key()
    Fd = torch.from_numpy(F).cuda()
    keys, objs, cfgs = [], [], []
    for r in range(W):
        s = cs.Scheduler(pb)
        s.set_shard_view(r, W)
        o, c = s.score_all(Fd)
        keys.append(s.local_best_key())
        objs.append(o.cpu().numpy())
        cfgs.append(c.cpu().numpy())
    assert max(keys) == key1
    assert np.array_equal(np.concatenate(cfgs), cfg1)
    assert np.array_equal(np.concatenate(objs), obj1)


# ---- full-size configs: sampled parity --------------------------------------------------

def test_c4_full_size_sampled(cs):
    pb, F = bench_config("C4")
    s, obj_g, cfg_g = _run(cs, pb, F)
    n = 10000
    rng = np.random.default_rng(2024)
    sample = np.unique(np.concatenate([rng.integers(0, len(cfg_g), 3000), [0, len(cfg_g) - 1]]))
    o = Oracle(pb)
    exact, fails = check_sets(o, F, None, sample, cfg_g[sample], obj_g[sample], n, 2)
    assert not fails, fails[:5]
    assert exact >= 0.99 * len(sample)
    st, sid, cfg, ob = s.best_set()
    # best_set reports the winner's exact FP32 argmax: >= the tiled choice's objective, within tau/2
    assert st == 0 and sid == int(np.argmax(obj_g)) and obj_g.max() <= ob <= obj_g.max() * (1 + TAU_OBJ / 2)
    exact, fails = check_sets(o, F, None, [sid], [cfg], [ob], n, 2)
    assert not fails, fails


def test_c5_triples_sampled(cs):
    pb, F = bench_config("C5")
    s, obj_g, cfg_g = _run(cs, pb, F)
    rng = np.random.default_rng(2025)
    sample = np.unique(rng.integers(0, len(cfg_g), 400))
    exact, fails = check_sets(Oracle(pb), F, None, sample, cfg_g[sample], obj_g[sample], 2000, 3)
    assert not fails, fails[:5]
    st, sid, cfg, ob = s.best_set()
    assert st == 0 and sid == int(np.argmax(obj_g)) and obj_g.max() <= ob <= obj_g.max() * (1 + TAU_OBJ / 2)


def _parity_every_set(pb, F, obj_g, cfg_g, cfg_o, obj_o, n, n_slots):
    """Every set against the oracle: equal config and objective within tau, else the
    tie-aware rule with the conditioning bands (tests/parity.py)."""
    same = (cfg_g == cfg_o) & (cfg_o >= 0)
    off = np.zeros(len(cfg_g), bool)
    off[same] = np.abs(obj_g[same].astype(np.float64) - obj_o[same]) > TAU_OBJ * np.abs(obj_o[same])
    check = np.nonzero((cfg_g != cfg_o) | off)[0]
    assert np.all(obj_g[(cfg_g < 0)] == -np.inf)
    exact, fails = check_sets(Oracle(pb), F, None, check, cfg_g[check], obj_g[check], n, n_slots)
    assert not fails, fails[:5]
    return len(check)


def test_c4_every_set_against_oracle_on_all_host_cores(cs):
    """BASELINE config 4 at full size: all 49,995,000 pairs x 294 configs (1.47e10
    candidates) by the FP64 oracle on every host core (tests/oracle_parallel.py),
    against the CUDA path's per-set choices, and the queue's best set inside the
    oracle's tied set (P:L663 exhaustive search, P:L843 queue-level choice)."""
    from oracle_parallel import score_range_all_cores
    pb, F = bench_config("C4")
    s, obj_g, cfg_g = _run(cs, pb, F)
    st, sid, cfg, ob = s.best_set()
    cfg_o, obj_o, cores = score_range_all_cores(pb, F)
    n_checked = _parity_every_set(pb, F, obj_g, cfg_g, cfg_o, obj_o, 10000, 2)
    assert n_checked <= 1e-3 * len(cfg_g)
    best_o = obj_o.max()
    assert st == 0 and obj_o[sid] >= best_o * (1 - TAU_OBJ) and abs(ob - obj_o[sid]) <= TAU_OBJ * obj_o[sid]
    print(f"C4: {len(cfg_g)} sets on {cores} cores, {n_checked} index/objective disagreements, all ties")


def test_triples_n200_every_set_against_oracle(cs):
    """Full exhaustive triple parity at N = 200 (C(200,3) = 1,313,400 triples x 882
    configs): every tile shape of the triple scorer (diagonal, last-j1-block, whole)
    against the FP64 oracle on every set."""
    from oracle_parallel import score_range_all_cores
    pb = make_problem("b200_3way", "c21", coef_seed=2005)
    F, _ = make_features(200, seed=1005)
    s, obj_g, cfg_g = _run(cs, pb, F)
    cfg_o, obj_o, _ = score_range_all_cores(pb, F)
    n_checked = _parity_every_set(pb, F, obj_g, cfg_g, cfg_o, obj_o, 200, 3)
    assert n_checked <= 1e-3 * len(cfg_g)
    st, sid, cfg, ob = s.best_set()
    assert st == 0 and obj_o[sid] >= obj_o.max() * (1 - TAU_OBJ)


@pytest.mark.parametrize("k", [1, 37, 60])
def test_greedy_partial_and_ties(cs, k):
    pb = make_problem("b200", "c21", coef_seed=16, alpha=0.3, mirror_ties=True)
    F = tie_stress_features(120, seed=16, frac=0.25)
    s, obj_g, cfg_g = _run(cs, pb, F)
    st, ids, cfgs, tot = s.best_allocation(k)
    assert st == 0 and len(ids) == k
    _, obj_o = Oracle(pb).score_range(F)
    ok, why = replay_greedy(120, 2, obj_o, ids)
    assert ok, why


@pytest.mark.parametrize("n_slots,n", [(2, 700), (2, 1501), (3, 150)])
def test_fast_scorer_equals_generic(cs, n_slots, n):
    """The tiled scorers reproduce the one-thread-per-set reference kernel on every set
    (same canonical FP32 evaluation order; they can differ only at objective near-ties
    below the packed objective's quantum, where both choices are accepted)."""
    table = "b200" if n_slots == 2 else "b200_3way"
    pb = make_problem(table, "c21", coef_seed=60 + n, alpha=0.62 if n_slots == 2 else 0.3)
    F, _ = make_features(n, seed=60 + n)
    s0, obj0, cfg0 = _run(cs, pb, F, variant=0)
    s1, obj1, cfg1 = _run(cs, pb, F, variant=1)
    same = (cfg0 == cfg1) & ((obj0 == obj1) | ((cfg0 < 0) & (cfg1 < 0)))
    assert same.mean() >= 1 - 1e-6, (np.nonzero(~same)[0][:10], cfg0[~same][:10], cfg1[~same][:10])
    assert s0.local_best_key() == s1.local_best_key()


@pytest.mark.parametrize("split", ["1", "2", "4", "15"])
@pytest.mark.parametrize("W", [1, 3])
def test_pair_tail_split_units(cs, split, W, monkeypatch):
    """The pair scorer's last-round tiles split into 1, 2, 4 or 15 stage groups per
    tile (units merged per pair by atomicMax, then resolved by k_pairs_merge_finish)
    give the generic kernel's results on every set of every fake rank (n = 1501: 24
    column tiles, 300 tiles, a ragged last column; 15 stages of 20 configs)."""
    monkeypatch.setenv("COSCHED_PAIR_SPLIT", split)
    pb = make_problem("b200", "c21", coef_seed=71, alpha=0.5)
    F, _ = make_features(1501, seed=71)
    for r in range(W):
        res = []
        for variant in (0, 1):
            s = cs.Scheduler(pb)
            s.set_variant(variant)
            s.set_shard_view(r, W)
            obj, cfg = s.score_all(torch.from_numpy(F).cuda())
            torch.cuda.synchronize()
            res.append((obj.cpu().numpy(), cfg.cpu().numpy(), s.local_best_key()))
        (o0, c0, k0), (o1, c1, k1) = res
        same = (c0 == c1) & ((o0 == o1) | ((c0 < 0) & (c1 < 0)))
        assert same.mean() >= 1 - 1e-6 and k0 == k1, (r, np.nonzero(~same)[0][:10])


@pytest.mark.parametrize("table,n", [("b200", 300), ("b200_3way", 60)])
def test_best_set_detail_from_basis_equals_projection(cs, table, n):
    """With the tiled scorers the step projects no ka / kb rows: best_set's detail is
    evaluated from the basis rows and the coefficient tables. It must give exactly the
    config and objective that best_config (which projects ka / kb on demand and reads
    them) and the generic scorer give."""
    pb = make_problem(table, "c21", coef_seed=91, alpha=0.2)
    F, _ = make_features(n, seed=91)
    s, obj_g, cfg_g = _run(cs, pb, F)
    st, sid, cfg, obj = s.best_set()
    assert st == 0 and cfg == int(cfg_g[sid]) and obj == float(obj_g[sid])
    d = s.best_config(sid)
    assert d["cfg"] == cfg and d["obj"] == obj
    s0, obj0, cfg0 = _run(cs, pb, F, variant=0)
    st0, sid0, c0, o0 = s0.best_set()
    assert (sid0, c0, o0) == (sid, cfg, obj)


def test_one_rank_nccl_communicator_matches_no_comm(cs):
    """Every collective path (best-set u64 max all-reduce, greedy min/max + histogram
    all-reduces and per-batch all-gathers) run through a real one-rank NCCL communicator
    returns exactly what the communicator-free path returns."""
    for name, k in (("C3", 500), ("C2", 4)):
        pb, F = bench_config(name)
        a = cs.Scheduler(pb)
        b = cs.Scheduler(pb)
        b.set_comm(cs.get_unique_id(), 0, 1)
        Fd = torch.from_numpy(F).cuda()
        oa, ca = a.score_all(Fd)
        ob, cb = b.score_all(Fd)
        torch.cuda.synchronize()
        assert torch.equal(ca, cb) and torch.equal(oa, ob)
        assert a.best_set() == b.best_set()
        assert a.best_allocation(k) == b.best_allocation(k)
    pb = make_problem("b200_3way", "c21", coef_seed=11, alpha=0.2)
    F, _ = make_features(60, seed=11)
    a, b = cs.Scheduler(pb), cs.Scheduler(pb)
    b.set_comm(cs.get_unique_id(), 0, 1)
    for s in (a, b):
        s.score_all(torch.from_numpy(F).cuda())
    assert a.best_allocation(20) == b.best_allocation(20)


@pytest.mark.parametrize("table,n,k", [("b200", 300, 150), ("b200_3way", 45, 15)])
def test_greedy_fallback_rounds_match_sorted_scan(cs, table, n, k, monkeypatch):
    """With a communicator, a batch larger than the per-rank capacity switches the greedy to
    the locally-dominant-rounds fallback; forcing it (COSCHED_GREEDY_BATCH_CAP) must give the
    same picks as the sorted scan (both are the exact sequential greedy)."""
    pb = make_problem(table, "c10", coef_seed=121, alpha=0.2)
    F, _ = make_features(n, seed=122)
    a = cs.Scheduler(pb)
    a.score_all(torch.from_numpy(F).cuda())
    ref = a.best_allocation(k)
    monkeypatch.setenv("COSCHED_GREEDY_BATCH_CAP", "64")
    b = cs.Scheduler(pb)
    b.set_comm(cs.get_unique_id(), 0, 1)
    b.score_all(torch.from_numpy(F).cuda())
    got = b.best_allocation(k)
    assert b.greedy_rounds > 1 and got == ref


@pytest.mark.parametrize("W", [3, 8])
@pytest.mark.parametrize("table", ["b200", "b200_3way"])
def test_fake_ranks_hill_truth_and_triples(cs, W, table):
    """Sharded by W fake ranks, the hill-climbing outputs and the triple scorer's outputs are
    bit-identical to one rank, and the ground-truth summary sums over the shards."""
    from synth.ground_truth import B200
    pb = make_problem(table, "c10", coef_seed=16, alpha=0.25)
    F, _ = make_features(120 if table == "b200" else 40, seed=16)
    Fd = torch.from_numpy(F).cuda()
    for mode in (0, 1):
        ref = cs.Scheduler(pb)
        ref.set_search(mode, 2, 3)
        o1, c1 = ref.score_all(Fd)
        o1, c1 = o1.cpu().numpy(), c1.cpu().numpy()
        _, sm1 = ref.evaluate_truth(Fd, B200)
        objs, cfgs, n_cmp, n_vio, lsum = [], [], 0, 0, 0.0
        for r in range(W):
            s = cs.Scheduler(pb)
            s.set_search(mode, 2, 3)
            s.set_shard_view(r, W)
            o, c = s.score_all(Fd)
            objs.append(o.cpu().numpy())
            cfgs.append(c.cpu().numpy())
            _, sm = s.evaluate_truth(Fd, B200)
            n_cmp += sm["n_compared"]
            n_vio += sm["n_violations"]
            if sm["n_compared"]:
                lsum += sm["n_compared"] * math.log(sm["geomean_prop_over_best"])
        assert np.array_equal(np.concatenate(cfgs), c1) and np.array_equal(np.concatenate(objs), o1)
        assert n_cmp == sm1["n_compared"] and n_vio == sm1["n_violations"]
        assert abs(math.exp(lsum / n_cmp) - sm1["geomean_prop_over_best"]) <= 1e-9


# ---- hand-derived golden examples through the CUDA path --------------------------

def _golden_problem(g, objective, alpha):
    from synth import Problem
    p = g["problem"]
    return Problem(name="hand", n_slots=p["n_slots"], gpcs_total=p["gpcs_total"],
                   state_gpcs=np.array(p["state_gpcs"], dtype=np.int32),
                   state_mem=np.array(p["state_mem"], dtype=np.int32),
                   state_slice=np.array(p["state_slice"], dtype=np.int32),
                   slices=[(0, 0)] * len(p["coef_c"][0]),
                   caps_w=np.array(p["caps_w"], dtype=np.float32),
                   coef_c=np.array(p["coef_c"], dtype=np.float32),
                   coef_d=np.array(p["coef_d"], dtype=np.float32),
                   objective=objective, alpha=alpha)


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("case", range(5))
def test_hand_triple_on_gpu(cs, golden, case, variant):
    """tests/golden/hand_triple_example.json (three slots, two partners under one D):
    the CUDA path's choice, objective and RPerfs equal the hand-derived values."""
    g = golden("hand_triple_example.json")
    ch = g["choices_by_hand"][case]
    pb = _golden_problem(g, ch["objective"], ch["alpha"])
    F = np.array([g["features"][k] for k in g["queue"]], np.float32)
    s, obj_g, cfg_g = _run(cs, pb, F, variant=variant)
    assert cfg_g[0] == ch["cfg"], ch["why"]
    if ch["obj"] is None:
        assert obj_g[0] == -np.inf
        return
    assert abs(obj_g[0] - ch["obj"]) <= 1e-6 * ch["obj"]
    d = s.best_config(0)
    row = g["per_config_by_hand"][ch["cfg"]]
    assert d["cfg"] == ch["cfg"]
    assert np.allclose(d["rperf"], row["rperf"], rtol=0, atol=1e-6)
    assert abs(d["throughput"] - row["throughput"]) <= 1e-6 and abs(d["fairness"] - row["fairness"]) <= 1e-6


def test_tensor_sum_boundary_on_gpu(cs):
    """Reading R24: the kernel decides F6+F7+F8 <= 100 on the FP32 sum, like the oracle."""
    pb = make_problem("b200", "c10", coef_seed=14)
    F, _ = make_features(4, seed=14)
    F[2, 5:8] = [33.33333206176758, 33.33333206176758, 33.33333969116211]  # FP32 sum == 100, FP64 > 100
    F[2, 0] = 90.0
    s = cs.Scheduler(pb)
    s.score_all(torch.from_numpy(F).cuda())
    assert s.best_set()[0] in (0, 2) and Oracle.validate_features(F)[0] == 0
    F[2, 7] = np.nextafter(np.float32(F[2, 7]), np.float32(200))
    s.score_all(torch.from_numpy(F).cuda())
    with pytest.raises(cs.CoschedError) as e:
        s.best_set()
    assert e.value.status == 14 and Oracle.validate_features(F)[0] == 14
