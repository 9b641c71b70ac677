"""The seeded input generator: bit-stability and table invariants (BASELINE.json:
every partition split sums to the chip's GPC count)."""
import hashlib
import math

import numpy as np

from synth import SplitMix64, bench_config, make_features, make_problem, partition_table


def test_splitmix64_reference_values():
    # splitmix64 with seed 0: first outputs of the reference algorithm (Steele, Lea, Flood 2014)
    r = SplitMix64(0)
    assert [int(x) for x in r.next_u64(3)] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_features_deterministic_and_valid():
    a, la = make_features(500, seed=1234)
    b, lb = make_features(500, seed=1234)
    assert a.tobytes() == b.tobytes() and la == lb
    assert a.dtype == np.float32 and a.shape == (500, 8)
    assert (a >= 0).all() and (a <= 100).all() and (a[:, 0] > 0.01).all()
    assert ((a[:, 5] + a[:, 6]) + a[:, 7] <= 100).all()
    assert set(la) == {"TI", "CI", "MI", "US"}
    c, _ = make_features(500, seed=1235)
    assert c.tobytes() != a.tobytes()


def test_tables_sum_to_gpc_total():
    for name, n_states in [("a100_paper", 4), ("b200", 14), ("b200_3way", 42), ("solo", 1)]:
        k, g, states = partition_table(name)
        assert len(states) == n_states
        for gp, m in states:
            assert len(gp) == k and sum(gp) == g and min(gp) >= 1 and m in (0, 1)
    # 21 compositions of 8 into 3 positive parts = C(7,2)
    k, g, st = partition_table("b200_3way")
    assert len({s for s, m in st}) == math.comb(7, 2)


def test_bench_configs_shapes():
    sizes = {"C1": (2, 20), "C2": (8, 140), "C3": (1000, 140), "C4": (10000, 294), "C5": (2000, 882)}
    for name, (n, ncfg) in sizes.items():
        pb, F = bench_config(name)
        assert F.shape == (n, 8) and pb.n_configs == ncfg
        assert pb.coef_c.shape == (pb.n_caps, pb.n_slices, 6) and pb.coef_d.shape == (pb.n_caps, pb.n_slices, 3)
    pb, F = bench_config("C1")
    assert pb.n_slots == 2 and pb.gpcs_total == 7


def test_baseline_slice_is_e6():
    pb = make_problem("b200", "c21", coef_seed=2004)
    base = pb.slices.index((8, 0))
    assert list(pb.coef_c[-1, base]) == [0, 0, 0, 0, 0, 1] and list(pb.coef_d[-1, base]) == [0, 0, 0]
