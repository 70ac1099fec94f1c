"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Contract (BASELINE north_star): selected sub-expert indices
and bucket offsets bit-exact (tokens whose oracle k-th/(k+1)-th logit gap is
< 1e-6 are counted separately); outputs within 1e-5 * (1 + |y|) in fp32 mode
and 2e-2 * (1 + |y|) in bf16 mode (against the oracle run on bf16-rounded
weights and inputs).
"""
import math
from pathlib import Path

import numpy as np
import pytest

from gpu_util import (U32, bf16_ok, bf16_round, close_mask, make_layer, out_ok, routing_agreement,
                      torch_layer_reference, toy_setup)

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"
TOL_F32, TOL_BF16 = 1e-5, 2e-2


@pytest.fixture(scope="module")
def torch_cuda(cuda_lib):
    import torch
    return torch


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


# ------------------------------------------------------------ C1 toy (golden)

@pytest.mark.parametrize("mode", ["softmax_renorm", "unit"])
def test_c1_fp32_against_reference_golden(oracle, torch_cuda, mode):
    torch = torch_cuda
    E, S, d, ff, T, K = 8, 4, 512, 1024, 256, 4
    g = np.load(GOLD / "c1_toy.npz")
    experts, parts, wr, x = toy_setup(oracle, E, S, d, ff, T)
    L = make_layer(experts, parts, wr, S, "f32", weights=mode, k_max=K, max_tokens=T)
    xd = torch.from_numpy(x).cuda()
    y, sel, w, off = L.forward(xd, k=K, return_routing=True)
    torch.cuda.synchronize()
    assert np.array_equal(_u32(sel), g["sel"])  # routing bit-exact (golden has no near ties)
    assert np.array_equal(_u32(off), g["offsets"])
    yh = y.cpu().numpy()
    if mode == "softmax_renorm":
        assert np.allclose(w.cpu().numpy(), g["w"], rtol=1e-6, atol=1e-7)
        assert close_mask(yh, g["y_w"], TOL_F32).all()
    else:
        assert (w.cpu().numpy() == 1.0).all()
        assert close_mask(yh[:64], g["y_u"], TOL_F32).all()


def test_c1_bf16_tensor_core_path(oracle, torch_cuda):
    torch = torch_cuda
    E, S, d, ff, T, K = 8, 4, 512, 1024, 256, 4
    experts, parts, wr, x = toy_setup(oracle, E, S, d, ff, T)
    L = make_layer(experts, parts, wr, S, "bf16", k_max=K, max_tokens=T)
    xb = bf16_round(x)
    xd = torch.from_numpy(xb).cuda().to(torch.bfloat16)
    y, sel, w, off = L.forward(xd, k=K, return_routing=True)
    logits = oracle.router_logits(xb, wr, T, d, E * S)
    osel, ow, gap = oracle.route(logits, K, K, 1)
    bad, ties = routing_agreement(_u32(sel), osel, gap, np.full(T, K))
    assert not bad, f"routing mismatch outside near-ties: {bad[:5]}"
    _, ooff, _, _ = oracle.bucket(_u32(sel), E * S)
    assert np.array_equal(_u32(off), ooff)
    ex_b = [tuple(bf16_round(a) for a in e) for e in experts]
    yo = oracle.layer_forward(ex_b, parts, S, xb, _u32(sel), w.cpu().numpy(), 1)
    yh = y.float().cpu().numpy()
    ok = bf16_ok(yh, yo)
    assert ok.all(), f"{(~ok).sum()} elements off"


# ------------------------------------------------------------ Mixtral shape

@pytest.mark.parametrize("k", [2, 3, 4, 6, 8, 10, 12, 14, 16])
def test_mixtral_layer_bf16_k_sweep(oracle, torch_cuda, k, mixtral):
    torch = torch_cuda
    L, x_dev, xb, wr, parts, ex_nm_b, logits = mixtral
    E, S, d, ff, T = 8, 8, 4096, 14336, x_dev.shape[0]
    y, sel, w, off = L.forward(x_dev, k=k, return_routing=True)
    torch.cuda.synchronize()
    osel, ow, gap = oracle.route(logits, k, L.k_max, 1)
    gsel = _u32(sel)
    bad, ties = routing_agreement(gsel, osel, gap, np.full(T, k))
    nres, near = L.route_stats()
    print(f"k={k}: near-ties {ties}/{T} (GPU count {near}), re-selected from exact logits {nres}")
    assert not bad, f"routing mismatch outside near-ties at tokens {bad[:5]}"
    assert near == ties
    _, ooff, _, _ = oracle.bucket(gsel, E * S)
    assert np.array_equal(_u32(off), ooff)
    if ties == 0:
        _, ooff2, _, _ = oracle.bucket(osel, E * S)
        assert np.array_equal(_u32(off), ooff2)
    # outputs on a fixed 32-token subsample
    sub = np.linspace(0, T - 1, 32).astype(np.int64)
    yo = oracle.layer_forward(ex_nm_b, parts, S, xb[sub], gsel[sub], w.cpu().numpy()[sub], 1, layout=1)
    yh = y.float().cpu().numpy()[sub]
    assert close_mask(yh, yo, TOL_BF16).all()  # the north_star form, 2e-2 * (1 + |y|)
    ok = bf16_ok(yh, yo)  # and the scale-aware form (stricter at this scale)
    assert ok.all(), f"{(~ok).sum()} off"


@pytest.fixture(scope="module")
def mixtral(oracle, torch_cuda):
    """Mixtral-8x7B layer shape: W_gate/W_up U(-1,1)/sqrt(d),
    W_down U(-1,1)/sqrt(ffn), W_r U(-1,1)/sqrt(d) fp32, x U(-1,1); counter-based
    synthetic stream on both sides (bit-identical)."""
    torch = torch_cuda
    from paper_2510_19366_b200 import MoeLayer, synth_fill
    E, S, d, ff, T = 8, 8, 4096, 14336, 4096
    L = MoeLayer(E, S, d, ff, dtype="bf16", k_max=16, max_tokens=T)
    parts = [oracle.random_balanced_partition(ff, S, 6000 + e) for e in range(E)]
    ex_nm_b = []
    buf = torch.empty(d * ff, dtype=torch.float32, device="cuda")
    for e in range(E):
        ws = []
        for m, (seed, scale) in enumerate(((100 + 3 * e, 1 / math.sqrt(d)), (101 + 3 * e, 1 / math.sqrt(d)),
                                           (102 + 3 * e, 1 / math.sqrt(ff)))):
            t = torch.empty(d * ff, dtype=torch.float32, device="cuda")
            synth_fill(t, seed, scale)
            ws.append(t)
        L.set_partition(e, parts[e])
        L.load_expert(e, *ws)
        # oracle side: neuron-major gate/up (same numbers, contiguous per neuron), bf16-rounded
        wg = bf16_round(oracle.synth_t(100 + 3 * e, d, ff, 1 / math.sqrt(d)))
        wu = bf16_round(oracle.synth_t(101 + 3 * e, d, ff, 1 / math.sqrt(d)))
        wd = bf16_round(oracle.synth(102 + 3 * e, d * ff, 1 / math.sqrt(ff)))
        if e == 0:  # the two generators agree bit for bit
            assert np.array_equal(ws[2].cpu().numpy(), oracle.synth(102, d * ff, 1 / math.sqrt(ff)))
        ex_nm_b.append((wg, wu, wd))
        del ws
    del buf
    wr = oracle.synth(7, d * E * S, 1 / math.sqrt(d))
    L.set_router(wr)
    xt = torch.empty((T, d), dtype=torch.bfloat16, device="cuda")
    synth_fill(xt, 11, 1.0)
    xb = bf16_round(oracle.synth(11, T * d, 1.0)).reshape(T, d)
    assert np.array_equal(xt.float().cpu().numpy(), xb)
    logits = oracle.router_logits(xb, wr, T, d, E * S)
    yield L, xt, xb, wr, parts, ex_nm_b, logits
    L.close()


# ------------------------------------------------------------ edge cases

@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("T", [1, 31, 33, 100])
def test_ragged_tokens_and_per_token_k(oracle, torch_cuda, dtype, T):
    torch = torch_cuda
    E, S, d, ff = 4, 4, 128, 256
    experts, parts, wr, x = toy_setup(oracle, E, S, d, ff, T, seed_x=T)
    L = make_layer(experts, parts, wr, S, dtype, k_max=16, max_tokens=128)
    rng = np.random.default_rng(T)
    kpt = rng.integers(1, 17, T).astype(np.uint32)
    xin = x if dtype == "f32" else bf16_round(x)
    xd = torch.from_numpy(xin).cuda().to(L.torch_dtype)
    y, sel, w, off = L.forward(xd, k_per_token=torch.from_numpy(kpt.astype(np.int32)), return_routing=True)
    L.check_errors()
    logits = oracle.router_logits(xin, wr, T, d, E * S)
    osel, ow, gap = oracle.route(logits, 0, 16, 1, k_per_token=kpt)
    bad, _ = routing_agreement(_u32(sel), osel, gap, kpt)
    assert not bad
    exs = experts if dtype == "f32" else [tuple(bf16_round(a) for a in e) for e in experts]
    yo = oracle.layer_forward(exs, parts, S, xin, _u32(sel), w.cpu().numpy(), 1)
    assert out_ok(y.float().cpu().numpy(), yo, dtype).all()


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_all_subexperts_and_k1(oracle, torch_cuda, dtype):
    torch = torch_cuda
    E, S, d, ff, T = 2, 8, 64, 128, 40
    experts, parts, wr, x = toy_setup(oracle, E, S, d, ff, T)
    L = make_layer(experts, parts, wr, S, dtype, weights="unit", k_max=16, max_tokens=T)
    xin = x if dtype == "f32" else bf16_round(x)
    xd = torch.from_numpy(xin).cuda().to(L.torch_dtype)
    exs = experts if dtype == "f32" else [tuple(bf16_round(a) for a in e) for e in experts]
    for k in (1, 16):
        y, sel, w, off = L.forward(xd, k=k, return_routing=True)
        if k == 16:  # every sub-expert of every expert: the full toy_ffn_forward sum
            assert (_u32(sel) == np.arange(16)).all()
            for t in range(T):
                want = sum(oracle.toy_ffn_forward(d, ff, *exs[e], xin[t])[0].astype(np.float64) for e in range(E))
                assert out_ok(y[t].float().cpu().numpy()[None], want[None], dtype).all()
        yo = oracle.layer_forward(exs, parts, S, xin, _u32(sel), w.cpu().numpy(), 0)
        assert out_ok(y.float().cpu().numpy(), yo, dtype).all()


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_dropin_partitioned_forward_acceptance_c1(oracle, torch_cuda, dtype):
    """tests/acceptance.cpp:69-100 through the GPU: one expert, explicit active
    sets (forward_selected, unit weights) == partitioned_forward / toy_ffn_forward."""
    torch = torch_cuda
    from paper_2510_19366_b200 import MoeLayer
    rng = np.random.default_rng(1)
    for trial in range(12):
        n = (2, 4, 8)[trial % 3]
        d = int(rng.integers(1, 65))
        ff = int(n + rng.integers(0, 129 - n))
        e = oracle.random_expert(d, ff, 5000 + trial)
        p = oracle.random_balanced_partition(ff, n, 6000 + trial)
        T = 5
        x = oracle.uniform_pm1(1000 + trial, T * d).reshape(T, d)
        if dtype == "bf16":
            x = bf16_round(x)
            e = tuple(bf16_round(a) for a in e)
        L = MoeLayer(1, n, d, ff, dtype=dtype, weights="unit", k_max=n, max_tokens=T)
        L.set_partition(0, p)
        L.load_expert(0, *e)
        sel = np.full((T, n), U32, np.uint32)
        actives = [list(range(n)), [], [trial % n], sorted({0, n - 1}), list(range(0, n, 2))]
        for t, act in enumerate(actives):
            sel[t, :len(act)] = act
        y = L.forward_selected(torch.from_numpy(x).cuda().to(L.torch_dtype),
                               torch.from_numpy(sel.view(np.int32))).float().cpu().numpy()
        for t, act in enumerate(actives):
            want = oracle.partitioned_forward(d, ff, *e, n, p, x[t], act)
            assert out_ok(y[t][None], want[None], dtype).all(), (trial, t)
        full, _ = oracle.toy_ffn_forward(d, ff, *e, x[0])
        assert out_ok(y[0][None], full[None], dtype).all()
        assert not y[1].any()  # empty active set -> exactly zero (tests/test_expert.cpp:90-96)
        L.close()


def test_validation_errors(oracle, torch_cuda):
    torch = torch_cuda
    from paper_2510_19366_b200 import MoeLayer, ValidationError
    E, S, d, ff, T = 2, 4, 32, 64, 8
    experts, parts, wr, x = toy_setup(oracle, E, S, d, ff, T)
    L = MoeLayer(E, S, d, ff, dtype="f32", k_max=4, max_tokens=T)
    xd = torch.from_numpy(x).cuda()
    with pytest.raises(ValidationError):  # not ready
        L.forward(xd, k=2)
    with pytest.raises(ValidationError):  # unbalanced partition
        L.set_partition(0, np.r_[np.zeros(40), np.arange(24) % 4].astype(np.uint32))
    with pytest.raises(ValidationError):  # wrong width
        L.set_partition(0, parts[0][:60])
    bad = experts[0][0].copy()
    bad[3] = np.nan
    with pytest.raises(ValidationError):  # non-finite weight (inc/expert.hpp:34)
        L.load_expert(0, bad, experts[0][1], experts[0][2])
    for e in range(E):
        L.set_partition(e, parts[e])
        L.load_expert(e, *experts[e])
    with pytest.raises(ValidationError):  # router missing
        L.forward(xd, k=2)
    L.set_router(wr)
    for k in (0, 5):
        with pytest.raises(ValidationError):  # k_active out of range (inc/gating.hpp:131-134)
            L.forward(xd, k=k)
    with pytest.raises(ValidationError):
        L.forward_host(x, k_per_token=np.array([1, 2, 3, 4, 5, 1, 1, 1], np.uint32))
    xn = x.copy()
    xn[2, 3] = np.inf
    with pytest.raises(ValidationError):  # non-finite input (inc/expert.hpp:55-57)
        L.forward_host(xn, k=2)
    sel = np.full((T, 4), U32, np.uint32)
    sel[0, :2] = [3, 3]  # duplicate (inc/expert.hpp:117)
    L.forward_selected(xd, torch.from_numpy(sel.view(np.int32)))
    with pytest.raises(ValidationError):
        L.check_errors()
    y = L.forward_host(x, k=2)  # layer still usable after errors
    assert np.isfinite(y).all()


def test_host_path_matches_device_path(oracle, torch_cuda):
    torch = torch_cuda
    E, S, d, ff, T = 4, 4, 128, 256, 64
    experts, parts, wr, x = toy_setup(oracle, E, S, d, ff, T)
    L = make_layer(experts, parts, wr, S, "f32", k_max=8, max_tokens=T)
    yd = L.forward(torch.from_numpy(x).cuda(), k=3).cpu().numpy()
    yh, sel, w, off = L.forward_host(x, k=3, return_routing=True)
    assert np.array_equal(yd, yh)  # deterministic: same kernels, same order


def test_files_path(oracle, ref, torch_cuda, tmp_path):
    """MPEX + NDJSON written by the reference, loaded by the layer."""
    torch = torch_cuda
    from paper_2510_19366_b200 import MoeLayer
    E, S, d, ff, T = 3, 4, 16, 32, 10
    experts, parts, wr, x = toy_setup(oracle, E, S, d, ff, T)
    pm = tmp_path / "map.ndjson"
    for e in range(E):
        ref.save_toy_expert(tmp_path / f"e{e}.mpex", d, ff, *experts[e])
        ref.append_partition_doc(pm, e, S, parts[e], truncate=(e == 0))
    L = MoeLayer(E, S, d, ff, dtype="f32", k_max=4, max_tokens=T)
    L.load_partition_map(pm)
    for e in range(E):
        L.load_expert_file(e, tmp_path / f"e{e}.mpex")
    L.set_router(wr)
    y, sel, w, off = L.forward(torch.from_numpy(x).cuda(), k=3, return_routing=True)
    yo = oracle.layer_forward(experts, parts, S, x, _u32(sel), w.cpu().numpy(), 1)
    assert close_mask(y.cpu().numpy(), yo, TOL_F32).all()


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_proxy_router(oracle, torch_cuda, dtype):
    torch = torch_cuda
    E, S, d, ff, T, K = 2, 4, 64, 128, 48, 3
    experts, parts, wr, x = toy_setup(oracle, E, S, d, ff, T)
    members = [[np.flatnonzero(p == s).tolist() for s in range(S)] for p in parts]
    gates = [members[e][s][:4] for e in range(E) for s in range(S)]
    L = make_layer(experts, parts, None, S, dtype, k_max=K, max_tokens=T, router="proxy")
    for e in range(E):
        L.set_gates(e, 4, gates[e * S:(e + 1) * S])
    xin = x if dtype == "f32" else bf16_round(x)
    y, sel, w, off = L.forward(torch.from_numpy(xin).cuda().to(L.torch_dtype), k=K, return_routing=True)
    scores = oracle.proxy_router_scores(experts, S, gates, xin)
    osel, ow, gap = oracle.route(scores, K, K, 1)
    bad, ties = routing_agreement(_u32(sel), osel, gap, np.full(T, K))
    assert not bad


def test_synth_fill_matches_oracle(oracle, torch_cuda):
    torch = torch_cuda
    from paper_2510_19366_b200 import synth_fill
    t = synth_fill(torch.empty(100003, dtype=torch.float32, device="cuda"), 42, 0.125, first=17)
    assert np.array_equal(t.cpu().numpy(), oracle.synth(42, 100003, 0.125, first=17))
    b = synth_fill(torch.empty(1000, dtype=torch.bfloat16, device="cuda"), 42, 0.125, first=17)
    assert np.array_equal(b.float().cpu().numpy(), bf16_round(oracle.synth(42, 1000, 0.125, first=17)))


def test_profiling_stage_times(oracle, torch_cuda):
    torch = torch_cuda
    E, S, d, ff, T = 4, 4, 128, 256, 64
    experts, parts, wr, x = toy_setup(oracle, E, S, d, ff, T)
    L = make_layer(experts, parts, wr, S, "bf16", k_max=8, max_tokens=T)
    L.set_profiling(True)
    n0 = L.launch_count()
    L.forward(torch.from_numpy(x).cuda().to(torch.bfloat16), k=4)
    st = L.stage_times()
    assert set(st) == {"router", "bucket", "dispatch", "gemm1", "gemm2", "combine"}
    # the bucketing runs inside the tensor-core router's fused epilogue here,
    # and at this decode-size batch (gemm1 gathers its rows from x) so do the
    # permutation tables: no dispatch launch
    assert st["bucket"][1] == 0 and st["router"][1] == 2
    assert st["dispatch"][1] == 0
    assert all(v[0] > 0 for name, v in st.items() if v[1])
    assert L.launch_count() - n0 == sum(v[1] for v in st.values()) == 5


def test_tensor_core_router_logit_error(oracle, torch_cuda, mixtral):
    """Accuracy of the split-bf16 tensor-core router vs the fp64 oracle logits:
    every logit must sit inside the per-token certification bound the routing
    epilogue uses (router_tc.cu: depth 2^-23 max|W_r| sum|x_t| + 2^-23
    max|logit_t|), which is what makes the re-selection of uncertain tokens
    exact."""
    import ctypes as C
    torch = torch_cuda
    from debug_tc import as_tensor
    from paper_2510_19366_b200 import _lib
    L, x_dev, xb, wr, parts, ex_nm_b, logits = mixtral
    L.route(x_dev, k=8)
    torch.cuda.synchronize()
    lib = _lib.load()
    lib.mp_debug_router_partials.argtypes = [C.c_void_p, C.POINTER(C.c_void_p)] + [C.POINTER(C.c_uint32)] * 4
    p, ks, T, npad, nf = C.c_void_p(), C.c_uint32(), C.c_uint32(), C.c_uint32(), C.c_uint32()
    _lib.check(lib.mp_debug_router_partials(L.h, C.byref(p), C.byref(ks), C.byref(T), C.byref(npad), C.byref(nf)))
    part = as_tensor(p.value, (ks.value, T.value, npad.value), torch.float64).cpu().numpy()
    got = part.sum(axis=0)[:, :logits.shape[1]]
    err = np.abs(got - logits)
    depth = 256  # 4096 tokens: 256-deep chunks (router_tc.cu plan_router_tc)
    bound = (depth * 2.0 ** -23 * np.abs(wr).max() * np.abs(xb).sum(axis=1, dtype=np.float64))[:, None] \
        + 2.0 ** -23 * np.abs(logits).max(axis=1, keepdims=True)
    print(f"router logit error: max {err.max():.3g}, p99 {np.quantile(err, 0.99):.3g} (K splits {ks.value}); "
          f"max error / bound {(err / bound).max():.3g}; {nf.value}/{T.value} tokens re-selected from fp64 logits")
    assert (err <= bound).all()


@pytest.mark.parametrize("k", [1, 2, 8, "mixed"])
def test_mixtral_all_tokens_vs_torch(oracle, torch_cuda, k, mixtral):
    """Every token of the Mixtral-shape layer against the PyTorch fp32 reference
    (the oracle runs on a subsample only: 1.45 s per (token, expert) call)."""
    torch = torch_cuda
    from paper_2510_19366_b200 import synth_fill
    L, x_dev, xb, wr, parts, ex_nm_b, logits = mixtral
    E, S, d, ff, T = 8, 8, 4096, 14336, x_dev.shape[0]
    if k == "mixed":  # SURVEY 8(d) C5 tiers {2,4,8,16}, pmf {.25,.35,.25,.15}
        rng = np.random.default_rng(13)
        kpt = rng.choice([2, 4, 8, 16], size=T, p=[0.25, 0.35, 0.25, 0.15]).astype(np.int32)
        y, sel, w, off = L.forward(x_dev, k_per_token=torch.from_numpy(kpt), return_routing=True)
    else:
        y, sel, w, off = L.forward(x_dev, k=k, return_routing=True)
    torch.cuda.synchronize()
    gsel = _u32(sel).astype(np.int64)
    gsel[gsel == U32] = -1

    def gen(e):
        out = []
        for m, (seed, scale, shape) in enumerate(((100 + 3 * e, 1 / math.sqrt(d), (d, ff)),
                                                   (101 + 3 * e, 1 / math.sqrt(d), (d, ff)),
                                                   (102 + 3 * e, 1 / math.sqrt(ff), (ff, d)))):
            t = torch.empty(d * ff, dtype=torch.float32, device="cuda")
            synth_fill(t, seed, scale)
            out.append(t.bfloat16().float().view(*shape))
        return out

    want = torch_layer_reference(torch, gen, parts, S, d, xb, gsel, w.cpu().numpy())
    ok = bf16_ok(y.float().cpu().numpy(), want)
    assert ok.all(), f"{(~ok).sum()} elements off in {np.unique(np.nonzero(~ok)[0]).size} tokens"


def test_fused_residual(oracle, torch_cuda):
    """mp_layer_set_residual: forward returns x + MoE(x) (layer-stack step,
    SURVEY 8(d) C3) with the residual as the combine's accumulator start."""
    torch = torch_cuda
    E, S, d, ff, T, K = 4, 4, 256, 512, 96, 4
    experts, parts, wr, x = toy_setup(oracle, E, S, d, ff, T)
    L = make_layer(experts, parts, wr, S, "bf16", k_max=K, max_tokens=T)
    xd = torch.from_numpy(bf16_round(x)).cuda().to(torch.bfloat16)
    y0 = L.forward(xd, k=K).float()
    L.set_residual(True)
    y1 = L.forward(xd, k=K).float()
    want = (xd.float() + y0).cpu().numpy()
    assert bf16_ok(y1.cpu().numpy(), want).all()
    assert not torch.equal(y1, y0)
    L.set_residual(False)
    assert torch.equal(L.forward(xd, k=K).float(), y0)
    L.close()
    Lf = make_layer(experts, parts, wr, S, "f32", k_max=K, max_tokens=T)
    from paper_2510_19366_b200 import ValidationError
    with pytest.raises(ValidationError, match="bf16"):
        Lf.set_residual(True)
    Lf.close()


@pytest.mark.parametrize("k", [1, 4, 7])
def test_router_exact_reselection_window(oracle, torch_cuda, k, monkeypatch):
    """The fused routing epilogue re-selects near-tie tokens from exact fp64
    logits over the uncertainty window.  Widening the guard by 0.05 sends most
    tokens down that path; routing must still equal the oracle bit for bit
    (outside the 1e-6 near-tie window) and the bucket offsets must match."""
    torch = torch_cuda
    monkeypatch.setenv("MOEPRISM_ROUTER_GUARD", "0.05")
    E, S, d, ff, T = 8, 4, 512, 1024, 256
    experts, parts, wr, x = toy_setup(oracle, E, S, d, ff, T)
    L = make_layer(experts, parts, wr, S, "bf16", k_max=8, max_tokens=T)
    xb = bf16_round(x)
    y, sel, w, off = L.forward(torch.from_numpy(xb).cuda().to(torch.bfloat16), k=k, return_routing=True)
    torch.cuda.synchronize()
    nf, near = L.route_stats()
    logits = oracle.router_logits(xb, wr, T, d, E * S)
    osel, ow, gap = oracle.route(logits, k, 8, 1)
    print(f"k={k}: {nf}/{T} tokens re-selected from exact logits, {near} near ties")
    assert nf > T // 4
    assert near == int((gap < 1e-6).sum())
    bad, ties = routing_agreement(_u32(sel), osel, gap, np.full(T, k))
    assert not bad, f"routing mismatch at tokens {bad[:5]}"
    _, ooff, _, _ = oracle.bucket(_u32(sel), E * S)
    assert np.array_equal(_u32(off), ooff)
    assert np.allclose(w.cpu().numpy()[:, :k], ow[:, :k], rtol=1e-5, atol=1e-6)
    L.close()


def test_forward_host_batches_pipelined(oracle, torch_cuda):
    """mp_layer_forward_host_batches == per-batch device forwards, bit for bit,
    for ragged batch sizes (uploads / compute / downloads overlapped)."""
    torch = torch_cuda
    E, S, d, ff = 4, 4, 256, 512
    experts, parts, wr, x = toy_setup(oracle, E, S, d, ff, 8)
    L = make_layer(experts, parts, wr, S, "bf16", k_max=4, max_tokens=96)
    sizes = [96, 17, 64, 1, 80, 33, 96]
    xs = [torch.from_numpy(bf16_round(oracle.uniform_pm1(50 + i, n * d))).reshape(n, d).to(torch.bfloat16).pin_memory()
          for i, n in enumerate(sizes)]
    ys = L.forward_host_batches(xs, k=3)
    for xh, yh in zip(xs, ys):
        yd = L.forward(xh.cuda(), k=3)
        assert torch.equal(yd.cpu(), yh)
    ys2 = L.forward_host_batches(xs[:2], k=3)  # a second call reuses the slots
    assert all(torch.equal(a, b) for a, b in zip(ys2, ys[:2]))
    L.close()


def test_forward_is_cuda_graph_capturable(oracle, torch_cuda):
    """The stream-ordered forward (router, fused routing epilogue, bulk
    dispatch, grouped GEMMs, combine, shared-expert fork/join) captures into a
    CUDA graph; replays equal eager forwards bit for bit (decode serving)."""
    torch = torch_cuda
    E, S, d, ff, T = 4, 4, 256, 512, 48
    experts, parts, wr, x = toy_setup(oracle, E, S, d, ff, T)
    L = make_layer(experts, parts, wr, S, "bf16", k_max=4, max_tokens=T)
    L.set_shared_expert(*(oracle.random_expert(d, 256, 9)), gate=oracle.uniform_pm1(3, d, 0.1))
    xs = [torch.from_numpy(bf16_round(oracle.uniform_pm1(60 + i, T * d))).reshape(T, d).cuda().to(torch.bfloat16)
          for i in range(2)]
    ys = [torch.empty_like(xs[0]) for _ in range(2)]
    want = [L.forward(xs[i], k=3).clone() for i in range(2)]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        L.forward(xs[0], k=3, y=ys[0])  # warm-up on the capture stream
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(2):
                L.forward(xs[i], k=3, y=ys[i])
    for _ in range(3):
        ys[0].zero_()
        ys[1].zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(ys[0], want[0]) and torch.equal(ys[1], want[1])
    L.close()


@pytest.mark.parametrize("k", [2, 4, 8])
def test_gemm_schedules_agree(oracle, torch_cuda, k, mixtral):
    """The three GEMM schedules (CTA pairs with swapped-operand remainder
    tiles, CTA pairs with plain 256-row remainders, 1-SM 128-row tiles) give
    the same layer output; buckets with partial last tiles of every size class
    occur at these bucket sizes."""
    import ctypes as C
    torch = torch_cuda
    from paper_2510_19366_b200 import _lib
    L, x_dev, *_ = mixtral
    lib = _lib.load()
    lib.mp_debug_set_tile_mode.argtypes = [C.c_void_p, C.c_int]
    outs = {}
    try:
        for mode in (2, 3, 1):  # pairs + swapped tails, pairs plain, 1-SM
            _lib.check(lib.mp_debug_set_tile_mode(L.h, mode))
            y, sel, w, off = L.forward(x_dev, k=k, return_routing=True)
            torch.cuda.synchronize()
            outs[mode] = y.float().cpu().numpy()
    finally:
        _lib.check(lib.mp_debug_set_tile_mode(L.h, 0))
    cnt = np.diff(off.cpu().numpy().view(np.uint32).astype(np.int64))
    assert ((cnt % 256) > 0).any()  # remainder tiles
    assert ((cnt % 128) > 0).any()
    ref = outs[3]
    for mode, y in outs.items():
        ok = bf16_ok(y, ref)
        assert ok.all(), f"mode {mode}: {(~ok).sum()} elements off"


@pytest.mark.parametrize("T,d", [(1, 512), (37, 512), (300, 512), (560, 512), (777, 512), (37, 768), (560, 768),
                                 (300, 576), (560, 640)])
def test_pair_swapped_tails_ragged(oracle, torch_cuda, T, d):
    """CTA pairs with swapped-operand remainder tiles on ragged buckets against
    the oracle: every remainder class (< 32, 32..255 rows, with and without
    full tiles before them, an odd N-tile count at d = 768, exact multiples;
    d = 576 / 640: K not a multiple of the 128-deep pair k-block, the last one
    half zero-filled by the TMA); routing bit-exact, outputs within the bf16
    tolerance."""
    import ctypes as C
    torch = torch_cuda
    from paper_2510_19366_b200 import _lib
    E, S, ff, K = 4, 4, 1024, 8
    experts, parts, wr, x = toy_setup(oracle, E, S, d, ff, T, seed_x=T)
    L = make_layer(experts, parts, wr, S, "bf16", k_max=K, max_tokens=T)
    lib = _lib.load()
    lib.mp_debug_set_tile_mode.argtypes = [C.c_void_p, C.c_int]
    _lib.check(lib.mp_debug_set_tile_mode(L.h, 2))
    xb = bf16_round(x)
    y, sel, w, off = L.forward(torch.from_numpy(xb).cuda().to(torch.bfloat16), k=K, return_routing=True)
    L.check_errors()
    logits = oracle.router_logits(xb, wr, T, d, E * S)
    osel, ow, gap = oracle.route(logits, K, K, 1)
    bad, _ = routing_agreement(_u32(sel), osel, gap, np.full(T, K, np.uint32))
    assert not bad
    cnt = np.diff(off.cpu().numpy().view(np.uint32).astype(np.int64))
    assert cnt.sum() == T * K
    exs = [tuple(bf16_round(a) for a in e) for e in experts]
    yo = oracle.layer_forward(exs, parts, S, xb, _u32(sel), w.cpu().numpy(), 1)
    assert out_ok(y.float().cpu().numpy(), yo, "bf16").all()
    L.close()


def test_zero_tokens(oracle, torch_cuda, mixtral):
    """An empty batch is a no-op: (0, d) output, no error, no launches."""
    torch = torch_cuda
    L, x_dev, *_ = mixtral
    n0 = L.launch_count()
    y = L.forward(x_dev[:0], k=8)
    torch.cuda.synchronize()
    assert tuple(y.shape) == (0, x_dev.shape[1])
    assert L.launch_count() == n0


def test_shared_scratch_layers(oracle, torch_cuda):
    """MP_LAYER_SHARED_SCRATCH: layers with the same shapes share the token
    scratch (x_perm / h / o) from a per-device pool; a two-layer stack run on
    one stream gives the same outputs as two layers with private scratch, and
    closing one sharer leaves the other working."""
    torch = torch_cuda
    from paper_2510_19366_b200 import MoeLayer
    from paper_2510_19366_b200._lib import MP_LAYER_SHARED_SCRATCH
    E, S, d, ff, T, K = 4, 4, 256, 512, 96, 4
    layers = {}
    for shared in (False, True):
        ls = []
        for l in range(2):
            experts, parts, wr, _ = toy_setup(oracle, E, S, d, ff, T, seed_w=7000 + 10 * l, seed_r=70 + l)
            L = MoeLayer(E, S, d, ff, dtype="bf16", k_max=K, max_tokens=T,
                         flags=MP_LAYER_SHARED_SCRATCH if shared else 0)
            for e in range(E):
                L.set_partition(e, parts[e])
                L.load_expert(e, *experts[e])
            L.set_router(wr)
            L.set_residual(True)
            ls.append(L)
        layers[shared] = ls
    x = torch.from_numpy(bf16_round(oracle.uniform_pm1(3, T * d).reshape(T, d))).cuda().to(torch.bfloat16)

    def stack(ls):
        y = x
        for L in ls:
            y = L.forward(y, k=K)
        return y

    assert torch.equal(stack(layers[True]), stack(layers[False]))
    layers[True][0].close()
    assert torch.equal(layers[True][1].forward(x, k=K), layers[False][1].forward(x, k=K))
    for ls in layers.values():
        for L in ls:
            L.close()
