"""World-size-2 CPU test (gloo) of the multi-GPU host logic: each rank takes
its shard from the C-ABI (cosched_shard_range_for), scores it (here with the
oracle, standing in for the GPU), packs the argmax key with cosched_pack_key
and all-reduces it (MAX). The reduced key must equal the single-rank search,
and the shards must cover every set exactly once."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_slots, n_jobs, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_2405_03838_b200 as cs
    from synth import make_features, make_problem
    table = "b200" if n_slots == 2 else "b200_3way"
    pb = make_problem(table, "c10", coef_seed=77, alpha=0.5)
    F, _ = make_features(n_jobs, seed=77)
    first, count = cs.shard_range_for(n_jobs, n_slots, rank, world)
    o = oracle.Oracle(pb)
    cfg, obj = o.score_range(F, None, first, count)
    key = 0
    for k in range(count):
        if cfg[k] >= 0:
            key = max(key, cs.pack_key(float(np.float32(obj[k])), first + k))
    # u64 max through a signed int64 all-reduce: flip the top bit
    t = torch.tensor([key ^ (1 << 63)], dtype=torch.uint64).view(torch.int64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    red = int(t.view(torch.uint64).item()) ^ (1 << 63)
    cnt = torch.tensor([count], dtype=torch.int64)
    dist.all_reduce(cnt)
    if rank == 0:
        q.put((red, int(cnt.item())))
    dist.destroy_process_group()


@pytest.mark.parametrize("n_slots,n_jobs", [(2, 61), (3, 23)])
def test_two_rank_argmax(n_slots, n_jobs):
    import oracle
    import paper_2405_03838_b200 as cs
    from paper_2405_03838_b200 import build
    from synth import make_features, make_problem
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_slots, n_jobs, q)) for r in range(2)]
    for p in procs:
        p.start()
    red, cnt = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    table = "b200" if n_slots == 2 else "b200_3way"
    pb = make_problem(table, "c10", coef_seed=77, alpha=0.5)
    F, _ = make_features(n_jobs, seed=77)
    st, sid, cfg, ob = oracle.Oracle(pb).best_set(F)
    assert cnt == cs.n_sets(n_jobs, n_slots)
    assert red == cs.pack_key(float(np.float32(ob)), sid)
