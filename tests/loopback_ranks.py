"""W cosched ranks as W threads of one process on one GPU, every collective
through the loopback NCCL stand-in (tests/loopback/, COSCHED_NCCL_LIB).
TEST INFRASTRUCTURE: run by tests/test_gpu_loopback.py in a fresh process.

For each case the W-rank results must equal the communicator-free W = 1 run:
the sharded per-set outputs (concatenated in rank order) bit-identical, the
best set (all-reduce u64 max), the greedy allocation (min/max/histogram
all-reduces + per-batch all-gathers, or the locally-dominant rounds fallback),
the exact allocation, and the ground-truth summary (f64 sum all-reduce; sums
regroup by rank, so equal to 1e-12 relative)."""
import json
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_03838_b200 as cs  # noqa: E402
from synth import bench_config, make_features, make_problem  # noqa: E402
from synth.ground_truth import B200  # noqa: E402


def one_rank(pb, Fd, uid, r, W, k, truth, out, errs):
    try:
        torch.cuda.set_device(0)
        st = torch.cuda.Stream()
        s = cs.Scheduler(pb)
        if uid is not None:
            s.set_comm(uid, r, W)
        with torch.cuda.stream(st):
            obj, cfg = s.score_all(Fd, stream=st)
        st.synchronize()
        res = {"obj": obj.cpu().numpy().copy(), "cfg": cfg.cpu().numpy().copy(), "best": s.best_set()}
        res["alloc"] = s.best_allocation(k)
        if truth:
            with torch.cuda.stream(st):
                _, summ = s.evaluate_truth(Fd, B200, stream=st)
            res["truth"] = summ
        res["first"], res["count"] = s.first, s.count
        out[r] = res
    except Exception as e:  # noqa: BLE001 -- reported by the main thread
        errs.append((r, repr(e)))


def run_case(pb, F, W, k, truth):
    print(f"case {pb.name} n={F.shape[0]} W={W} k={k}", file=sys.stderr, flush=True)
    Fd = torch.from_numpy(np.ascontiguousarray(F)).cuda()
    torch.cuda.synchronize()
    ref = {}
    one_rank(pb, Fd, None, 0, 1, k, truth, ref, [])
    uid = cs.get_unique_id()
    out, errs = [None] * W, []
    th = [threading.Thread(target=one_rank, args=(pb, Fd, uid, r, W, k, truth, out, errs)) for r in range(W)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    R = ref[0]
    firsts = [o["first"] for o in out]
    assert firsts == sorted(firsts) and sum(o["count"] for o in out) == R["count"]
    assert np.array_equal(np.concatenate([o["cfg"] for o in out]), R["cfg"])
    assert np.array_equal(np.concatenate([o["obj"] for o in out]), R["obj"])
    for o in out:
        assert o["best"] == R["best"], (o["best"], R["best"])
        assert o["alloc"] == R["alloc"], (o["alloc"][:2], R["alloc"][:2])
        if truth:
            a, b = o["truth"], R["truth"]
            assert a["n_compared"] == b["n_compared"] and a["n_violations"] == b["n_violations"]
            for key in ("geomean_prop_over_best", "geomean_worst_over_best"):
                assert abs(a[key] - b[key]) <= 1e-12 * abs(b[key]), (key, a[key], b[key])
    return {"W": W, "sets": int(R["count"]), "best": list(R["best"]), "n_picks": len(R["alloc"][1])}


def main():
    import faulthandler
    faulthandler.dump_traceback_later(400, exit=True)  # a hang prints every thread's stack
    W = int(sys.argv[1])
    report = []
    pb, F = bench_config("C3")
    report.append(run_case(pb, F, W, 500, True))                    # pairs: best set, sorted-scan greedy, truth
    pb, F = bench_config("C2")
    report.append(run_case(pb, F, W, 4, False))                     # exact allocation over 105 matchings
    pb = make_problem("b200_3way", "c21", coef_seed=11, alpha=0.2)
    F, _ = make_features(60, seed=11)
    report.append(run_case(pb, F, W, 20, True))                     # triples
    os.environ["COSCHED_GREEDY_BATCH_CAP"] = "64"                     # force the locally-dominant fallback
    pb = make_problem("b200", "c10", coef_seed=121, alpha=0.2)
    F, _ = make_features(300, seed=121)
    report.append(run_case(pb, F, W, 150, False))
    pb = make_problem("b200_3way", "c10", coef_seed=121, alpha=0.2)
    F, _ = make_features(45, seed=121)
    report.append(run_case(pb, F, W, 15, False))
    print(json.dumps(report))


if __name__ == "__main__":
    main()
