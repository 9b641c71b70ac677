"""The C-ABI library loads and exports every symbol include/cosched.h declares;
its host-only helpers (no CUDA) behave; compute entry points fail loudly
without a GPU (no CPU fallback)."""
import ctypes
import itertools
import math
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def cs():
    from paper_2405_03838_b200 import build
    build.build()
    import paper_2405_03838_b200 as cs
    return cs


def _declared():
    src = open(os.path.join(ROOT, "include", "cosched.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cosched_[a-z_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported(cs):
    from paper_2405_03838_b200 import _lib
    L = _lib.load()
    names = _declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(L, n), n
    assert sorted(n for n, _, _ in _lib.SIGNATURES) == names


def test_host_helpers_match_the_oracle(cs):
    import oracle
    for k in (1, 2, 3):
        for n in (k, 5, 11):
            assert cs.n_sets(n, k) == math.comb(n, k)
            for sid in range(math.comb(n, k)):
                assert cs.unrank(n, k, sid) == oracle.unrank(n, k, sid)
    assert cs.n_sets(2000, 3) == 1331334000 and cs.n_sets(10000, 2) == 49995000


def test_key_order(cs):
    rng = np.random.default_rng(0)
    objs = np.concatenate([rng.normal(size=50).astype(np.float32), np.float32([0.0, -0.0, 1e-30, 3.0])])
    ids = rng.integers(0, 2 ** 31, len(objs))
    keys = [cs.pack_key(float(o), int(i)) for o, i in zip(objs, ids)]
    for (o1, i1, k1), (o2, i2, k2) in itertools.combinations(zip(objs, ids, keys), 2):
        if o1 != o2 or (o1 == 0 and np.signbit(o1) != np.signbit(o2)):
            assert (k1 > k2) == (o1 > o2 or (o1 == o2 and not np.signbit(o1)))
        else:
            assert (k1 > k2) == (i1 < i2)
    for o, i, k in zip(objs, ids, keys):
        oo, ii = cs.unpack_key(k)
        assert ii == i and (oo == o)
    assert cs.unpack_key(0) == (-math.inf, -1)


@pytest.mark.parametrize("n,k", [(10000, 2), (2000, 3), (1000, 2), (7, 2), (3, 3), (1, 2)])
def test_shards_partition_whole_columns(cs, n, k):
    total = math.comb(n, k) if n >= k else 0
    for W in (1, 2, 3, 4, 8):
        nxt = 0
        sizes = []
        for r in range(W):
            a, b = cs.shard_range_for(n, k, r, W)
            assert a == nxt
            nxt = a + b
            sizes.append(b)
            if b:
                # whole columns: the shard starts at C(b_r, k) for an integer b_r
                cols = [c for c in range(n + 1) if math.comb(c, k) == a]
                assert cols
        assert nxt == total
        if total >= 1000 * W and k == 2:
            # pairs: whole 64-column blocks (cosched.h), chosen to balance the scorer's
            # modelled time -- per-rank tile counts within two column blocks' tiles
            bounds = [next(c for c in range(n + 1) if math.comb(c, 2) >= a) for a in
                      [sum(sizes[:r]) for r in range(W)]] + [n]
            assert all(b % 64 == 0 for b in bounds[1:-1])
            nb = -(-n // 64)
            blk = [-(-b // 64) for b in bounds]
            tiles = [blk[r + 1] * (blk[r + 1] + 1) // 2 - blk[r] * (blk[r] + 1) // 2 for r in range(W)]
            assert sum(tiles) == nb * (nb + 1) // 2
            assert max(tiles) - min(tiles) <= 2 * nb
        if total >= 1000 * W and k == 3:
            # triples balance the scorer's 64 x 64 tiles per plane (cosched.h): per-rank
            # tile counts within one plane's tiles of each other
            def plane_tiles(j):
                t = -(-j // 64)
                return t * (t + 1) // 2
            cols = [next(c for c in range(n + 1) if math.comb(c, 3) >= a) for a in
                    [sum(sizes[:r]) for r in range(W)]] + [n]
            tiles = [sum(plane_tiles(j) for j in range(max(cols[r], 1), cols[r + 1])) for r in range(W)]
            assert max(tiles) - min(tiles) <= 2 * plane_tiles(n - 1)


def test_compute_fails_loudly_without_gpu(cs):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from synth import make_problem
    with pytest.raises(cs.CoschedError) as e:
        cs.Scheduler(make_problem("b200", "c10", coef_seed=1))
    assert e.value.status == 20
