"""GPU: the split best-set calls and the step timing events of the C-ABI
(include/cosched.h cosched_best_set_begin / _end, cosched_last_step_ms), against
the one-call cosched_best_set and the FP64 oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from synth import bench_config, make_features, make_problem  # noqa: E402


@pytest.fixture(scope="module")
def cs():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2405_03838_b200 as cs
    return cs


def test_best_set_begin_end_equals_best_set(cs):
    pb, F = bench_config("C3")
    s = cs.Scheduler(pb)
    Fd = torch.from_numpy(F).cuda()
    s.score_all(Fd)
    one = s.best_set()
    s.score_all(Fd)
    s.best_set_begin()
    two = s.best_set_end()
    assert one == two
    ms = s.last_step_ms()
    assert 0.0 < ms < 1e3
    # the winner is the oracle's best set (tie-aware: its objective within 1e-5)
    _, obj_o = oracle.Oracle(pb).score_range(F)
    assert two[0] == 0 and obj_o[two[1]] >= obj_o.max() * (1 - 1e-5)


def test_best_set_end_without_begin_is_a_state_error(cs):
    pb = make_problem("b200", "c10", coef_seed=3, alpha=0.2)
    F, _ = make_features(40, seed=3)
    s = cs.Scheduler(pb)
    s.score_all(torch.from_numpy(F).cuda())
    with pytest.raises(cs.CoschedError) as e:
        s.best_set_end()
    assert cs.STATUS[e.value.status] == "E_STATE"
    with pytest.raises(cs.CoschedError):
        s.last_step_ms()  # no completed best_set after this score_all


def test_last_step_ms_brackets_the_step(cs):
    """The library's events sit inside the caller's: the step's device time is at
    most the time between events recorded before score_all and after best_set_begin."""
    pb, F = bench_config("C3")
    s = cs.Scheduler(pb)
    Fd = torch.from_numpy(F).cuda()
    st = torch.cuda.current_stream()
    for _ in range(2):
        s.score_all(Fd, stream=st)
        s.best_set()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    s.score_all(Fd, stream=st)
    s.best_set_begin()
    e1.record(st)
    s.best_set_end()
    e1.synchronize()
    inner, outer = s.last_step_ms(), e0.elapsed_time(e1)
    assert 0.0 < inner <= outer + 1e-3


def test_consecutive_steps_on_one_handle_match_fresh_handles(cs):
    """The pair scorer's stage-split merge area keeps step-tagged entries between
    calls (never reset): back-to-back queues on one handle -- with tail tiles, the
    second queue having pairs infeasible where the first had feasible ones -- must
    give exactly what fresh handles give."""
    pb = make_problem("b200", "c21", coef_seed=97, alpha=0.6)
    F1, _ = make_features(2000, seed=97)   # 32 column blocks: 528 tiles, a stage-split tail
    F2, _ = make_features(2000, seed=98)
    shared = cs.Scheduler(pb)
    for F in (F1, F2, F1):
        Fd = torch.from_numpy(F).cuda()
        o1, c1 = shared.score_all(Fd)
        o1, c1 = o1.cpu().numpy().copy(), c1.cpu().numpy().copy()
        fresh = cs.Scheduler(pb)
        o2, c2 = fresh.score_all(Fd)
        assert np.array_equal(c1, c2.cpu().numpy())
        assert np.array_equal(o1, o2.cpu().numpy())
        assert shared.best_set() == fresh.best_set()
    # the two queues really differ in feasibility somewhere (the stale-entry case)
    Fa, Fb = torch.from_numpy(F1).cuda(), torch.from_numpy(F2).cuda()
    _, ca = cs.Scheduler(pb).score_all(Fa)
    _, cb = cs.Scheduler(pb).score_all(Fb)
    assert ((ca.cpu().numpy() >= 0) != (cb.cpu().numpy() >= 0)).any()


def test_prep_scorer_split_only_on_request(cs):
    """cosched_last_timings needs cosched_set_timing(h, 1) for that step (its events
    cost the PDL overlap, so the default step records none)."""
    pb, F = bench_config("C3")
    s = cs.Scheduler(pb)
    Fd = torch.from_numpy(F).cuda()
    s.score_all(Fd)
    with pytest.raises(cs.CoschedError) as e:
        s.last_timings()
    assert cs.STATUS[e.value.status] == "E_STATE"
    s.set_timing(True)
    s.score_all(Fd)
    prep, score, total = s.last_timings()
    assert 0.0 < prep < total and 0.0 < score < total and prep + score <= total + 1e-3
    s.set_timing(False)
    s.score_all(Fd)
    with pytest.raises(cs.CoschedError):
        s.last_timings()
