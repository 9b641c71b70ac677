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
