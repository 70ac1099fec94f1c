"""GPU calibration path through the C-ABI against the
reference (oracle/_ref) and its numpy restatements."""
import math

import numpy as np
import pytest

from gpu_util import bf16_round, make_layer, toy_setup
from oracle_lib import np_binarize_topk, np_coactivation

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda(cuda_lib):
    import torch
    return torch


def _ref_or_oracle_activations(oracle, d, ff, e, x):
    """|a| rows (collect_activation_matrix); the oracle's toy_ffn_forward
    activations are pinned bit for bit to the reference in test_calib_host."""
    return np.stack([np.abs(oracle.toy_ffn_forward(d, ff, *e, x[b])[1]) for b in range(x.shape[0])])


@pytest.mark.parametrize("B", [1, 130, 300])
def test_collect_activations_vs_oracle(oracle, torch_cuda, B):
    torch = torch_cuda
    from paper_2510_19366_b200.calibrate import collect_activations
    E, S, d, ff = 2, 4, 256, 512
    experts, parts, wr, x = toy_setup(oracle, E, S, d, ff, B)
    L = make_layer(experts, parts, wr, S, "bf16", k_max=4, max_tokens=max(B, 8))
    xb = bf16_round(x)
    for e in range(E):
        act = collect_activations(L, e, torch.from_numpy(xb).cuda().to(torch.bfloat16)).cpu().numpy()
        want = _ref_or_oracle_activations(oracle, d, ff, tuple(bf16_round(a) for a in experts[e]), xb)
        # bf16 operands, fp32 accumulation: scale-aware tolerance per row
        rms = np.sqrt((want.astype(np.float64) ** 2).mean(axis=1, keepdims=True))
        assert (np.abs(act - want) <= 2e-2 * (rms + np.abs(want))).all()
        assert (act >= 0).all()
    L.close()


@pytest.mark.parametrize("k_a", [1, 5, 64, 203])
def test_binarize_topk_exact(torch_cuda, k_a):
    torch = torch_cuda
    from paper_2510_19366_b200.calibrate import binarize_topk
    rng = np.random.default_rng(k_a)
    rows, cols = 97, 203
    for act in (rng.random((rows, cols), dtype=np.float32),
                (rng.integers(0, 5, size=(rows, cols)) * 0.5).astype(np.float32),  # heavy ties
                np.zeros((rows, cols), np.float32)):
        bits = binarize_topk(torch.from_numpy(act).cuda(), k_a).cpu().numpy()
        assert np.array_equal(bits, np_binarize_topk(act, k_a))


@pytest.mark.parametrize("rows,cols", [(300, 512), (77, 203), (1, 8)])
def test_coactivation_exact(torch_cuda, rows, cols):
    torch = torch_cuda
    from paper_2510_19366_b200.calibrate import coactivation
    rng = np.random.default_rng(rows)
    bits = (rng.random((rows, cols)) < 0.3).astype(np.uint8)
    co = coactivation(torch.from_numpy(bits).cuda()).cpu().numpy().view(np.uint32)
    assert np.array_equal(co, np_coactivation(bits))


def test_calibration_pipeline_mixtral_expert(torch_cuda):
    """collect -> binarize -> co-activation for one Mixtral expert (d=4096,
    ffn=14336) on 512 calibration tokens; spot-checked against numpy."""
    torch = torch_cuda
    import bench
    from paper_2510_19366_b200.calibrate import binarize_topk, coactivation, collect_activations
    L, xs = bench.build_layer(0, 512, 2)
    act = collect_activations(L, 3, xs[0])
    k_a = 1434  # 10% of the neurons
    bits = binarize_topk(act, k_a)
    co = coactivation(bits)
    torch.cuda.synchronize()
    b = bits.cpu().numpy()
    assert (b.sum(axis=1) == k_a).all()
    a = act.cpu().numpy()
    assert np.array_equal(b[:8], np_binarize_topk(a[:8], k_a))
    rng = np.random.default_rng(0)
    ii, jj = rng.integers(0, 14336, 64), rng.integers(0, 14336, 64)
    c = co.cpu().numpy().view(np.uint32)
    bb = b.astype(np.int64)
    for i, j in zip(ii, jj):
        assert c[i, j] == int(bb[:, i] @ bb[:, j])
    assert np.array_equal(np.diag(c), b.sum(axis=0).astype(np.uint32))
    L.close()


def test_perf_table_measured_loads_in_reference(oracle, torch_cuda, tmp_path):
    torch = torch_cuda
    from oracle_lib import RefLib, have_ref
    from paper_2510_19366_b200.calibrate import measure_perf_table, write_perf_table
    E, S, d, ff = 4, 4, 256, 512
    experts, parts, wr, x = toy_setup(oracle, E, S, d, ff, 8)
    L = make_layer(experts, parts, wr, S, "bf16", k_max=8, max_tokens=512)
    cells = measure_perf_table(L, [32, 128, 512], [1, 2, 4, 8], steps=5)
    write_perf_table(tmp_path / "perf.csv", cells)
    lat = {(b, k): s for b, k, s in cells}
    assert all(s > 0 for s in lat.values())
    if have_ref():
        cost, nb, nk = RefLib().perf_table_eval(tmp_path / "perf.csv", 128, 4)
        assert (nb, nk) == (3, 4) and math.isclose(cost, lat[(128, 4)], rel_tol=1e-6)
    L.close()


def test_acceptance_c4_gating_fidelity_on_gpu(ref, torch_cuda):
    """Acceptance C4 (tests/acceptance.cpp:166-206) through the GPU pipeline:
    binarize_topk -> coactivation -> select_gate_neurons -> gating_fidelity,
    every stage equal to the reference; saturated gates (r = group size) give
    fidelity exactly 1 for every k, planted clusters recall >= 0.95 with r = 1."""
    torch = torch_cuda
    from paper_2510_19366_b200.calibrate import binarize_topk, coactivation, gating_fidelity, select_gate_neurons
    for trial in range(20):
        rng = np.random.default_rng(4000 + trial)  # shapes only (the reference draws its own with mt19937_64)
        n = int(rng.integers(2, 6))
        group = int(rng.integers(2, 7))
        cols, rows = n * group, int(rng.integers(8, 33))
        m = ref.random_matrix(rows, cols, 9000 + trial)
        part = ref.random_balanced_partition(cols, n, 9500 + trial)
        k_a = ref.default_binarize_count(cols)
        md = torch.from_numpy(m).cuda()
        bits = binarize_topk(md, k_a)
        assert np.array_equal(bits.cpu().numpy(), ref.binarize_topk(m, k_a))
        co = coactivation(bits)
        co_ref = ref.coactivation(bits.cpu().numpy(), k_a)
        assert np.array_equal(co.cpu().numpy().view(np.uint32), co_ref)
        gates = select_gate_neurons(co, part, n, group)
        assert gates == ref.select_gate_neurons(co_ref, part, n, group)
        for k in range(1, n + 1):
            f = gating_fidelity(md, part, n, gates, k)
            assert f == ref.gating_fidelity(m, part, n, gates, group, k) == 1.0
    recalls = []
    for trial in range(20):
        m, part = ref.planted_cluster(64, 4, 8, 10000 + trial)
        md = torch.from_numpy(m).cuda()
        bits = binarize_topk(md, ref.default_binarize_count(m.shape[1]))
        co = coactivation(bits)
        gates = select_gate_neurons(co, part, 4, 1)
        assert gates == ref.select_gate_neurons(co.cpu().numpy().view(np.uint32), part, 4, 1)
        f = gating_fidelity(md, part, 4, gates, 1)
        assert f == ref.gating_fidelity(m, part, 4, gates, 1, 1)
        recalls.append(f)
    assert min(recalls) >= 0.95


def test_gate_selection_and_fidelity_mixtral_expert(oracle, torch_cuda):
    """The proxy-gate pipeline at the Mixtral expert shape (14336 neurons, 8
    sub-experts of 1792) on 512 calibration tokens: gates equal the reference's
    select_gate_neurons on the same co-activation matrix; fidelity equals the
    reference's on the same activations (when the reference build is present)."""
    torch = torch_cuda
    import bench
    from oracle_lib import RefLib, have_ref
    from paper_2510_19366_b200.calibrate import (binarize_topk, coactivation, collect_activations, gating_fidelity,
                                                select_gate_neurons)
    L, xs = bench.build_layer(0, 512, 2)
    act = collect_activations(L, 2, xs[0])
    co = coactivation(binarize_topk(act, 1434))
    part = bench.balanced_partition(14336, 8, 6002)
    gates = select_gate_neurons(co, part, 8, 4)
    assert all(len(g) == 4 and g == sorted(g) and all(part[j] == s for j in g) for s, g in enumerate(gates))
    f = gating_fidelity(act, part, 8, gates, 2)
    assert 0.0 <= f <= 1.0
    if have_ref():
        r = RefLib()
        c = co.cpu().numpy().view(np.uint32)
        assert gates == r.select_gate_neurons(c, part, 8, 4)
        assert f == r.gating_fidelity(act.cpu().numpy(), part, 8, gates, 4, 2)
    L.close()
