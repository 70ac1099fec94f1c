"""Host-side pieces of bench.py (no GPU): the partition fixture generator it
uses on the product path matches the reference fixture (tests/support.hpp:89-105)."""
import numpy as np


def test_bench_partition_matches_reference_fixture(oracle):
    import bench
    for n, ns, seed in ((14336, 8, 6000), (1408, 4, 6003), (12, 4, 6)):
        assert np.array_equal(bench.balanced_partition(n, ns, seed), oracle.random_balanced_partition(n, ns, seed))


def test_layer_roofline_numbers():
    import bench
    pk = {"hbm_gbs": 6552.6, "bf16_tflops_sustained": 1430.8, "source": "measured"}
    r = bench.layer_roofline(4096, 8, 1.0, pk, 64)
    # k=8 -> TC bound, 1.009 ms
    assert r["bound"] == "tensor" and abs(r["t_roofline_ms"] - 1.009) < 0.01
    r2 = bench.layer_roofline(4096, 2, 1.0, pk, 64)
    assert r2["bound"] == "hbm" and abs(r2["t_roofline_ms"] - 0.44) < 0.02
