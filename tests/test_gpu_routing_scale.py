"""Routing exactness at any input scale (the routing contract of SURVEY 8(c)).

The tensor-core router certifies each token with a per-token error bound
(router_tc.cu: chunk depth * 2^-23 * max|W_r| * sum|x_t| + 2^-23 * max|logit_t|)
and re-selects every uncertain token from exact fp64 logits.  These tests push
the inputs where a fixed absolute guard would break: hidden states scaled by
10 and 100, outlier channels with |x| ~ 500, router weights giving logits
beyond +-64, and all of them at once.  Selected ids must equal the fp64
oracle's bit for bit (tokens whose oracle k-th/(k+1)-th gap is < 1e-6 are
near ties: counted, and the GPU's own near-tie count must equal the oracle's),
bucket offsets must be bit-exact, and the softmax-renormalised weights must
match.  Both routing paths are covered: the fused routing epilogue of
mp_layer_forward and the separate top-k + fixup kernels of mp_layer_route, at
a prefill batch (256-deep router chunks) and a decode batch (64-deep chunks).
"""
import math

import numpy as np
import pytest

from gpu_util import bf16_round, routing_agreement

pytestmark = pytest.mark.gpu

E, S, D, FF = 8, 8, 4096, 1024  # the Mixtral router shape (d=4096, 64 sub-experts), small experts
G = E * S
KS = [1, 2, 3, 6, 8, 10, 12, 14, 16]


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


def _inputs(oracle, case, T):
    x = oracle.uniform_pm1(11 + T, T * D).reshape(T, D).astype(np.float32)
    wr = oracle.uniform_pm1(7, D * G, 1.0 / math.sqrt(D))
    rng = np.random.default_rng(5)
    if case in ("x10", "x100", "all"):
        x = x * (100.0 if case != "x10" else 10.0)
    if case in ("outliers", "all"):
        ch = np.array([3, 77, 1000, 2048, 4095])
        x[:, ch] = 500.0 * np.where(rng.random((T, ch.size)) < 0.5, -1.0, 1.0)
    if case in ("big_logits", "all"):
        wr = wr * 256.0  # logits ~ U(-1,1)-weighted sums with |logit| well beyond 64
    return bf16_round(x), wr.astype(np.float32)


@pytest.fixture(scope="module")
def layer(torch_cuda_mod):
    torch = torch_cuda_mod
    from paper_2510_19366_b200 import MoeLayer, synth_fill
    L = MoeLayer(E, S, D, FF, dtype="bf16", k_max=16, max_tokens=4096)
    buf = [torch.empty(D * FF, dtype=torch.float32, device="cuda") for _ in range(3)]
    for e in range(E):
        for m in range(3):
            synth_fill(buf[m], 300 + 3 * e + m, 1.0 / math.sqrt(D if m < 2 else FF))
        L.set_partition(e, np.arange(FF, dtype=np.uint32) % S)
        L.load_expert(e, *buf)
    yield L
    L.close()


@pytest.fixture(scope="module")
def torch_cuda_mod(cuda_lib):
    import torch
    return torch


@pytest.mark.parametrize("T", [4096, 64])
@pytest.mark.parametrize("case", ["x10", "x100", "outliers", "big_logits", "all"])
def test_routing_bit_exact_at_scale(oracle, torch_cuda_mod, layer, case, T):
    torch = torch_cuda_mod
    L = layer
    x, wr = _inputs(oracle, case, T)
    L.set_router(wr)
    logits = oracle.router_logits(x, wr, T, D, G)
    xd = torch.from_numpy(x).cuda().to(torch.bfloat16)
    assert np.array_equal(xd.float().cpu().numpy(), x)
    amax = np.abs(logits).max()
    # the router's per-token certification bound (router_tc.cu), 256-deep chunks at most
    bound = (256 * 2.0 ** -23 * np.abs(wr).max() * np.abs(x).sum(axis=1, dtype=np.float64))[:, None] \
        + 2.0 ** -23 * np.abs(logits).max(axis=1, keepdims=True)
    report = []
    for k in KS:
        osel, ow, gap = oracle.route(logits, k, 16, 1)
        o_ties = int((gap < 1e-6).sum())
        # fused routing epilogue (forward)
        y, sel, w, off = L.forward(xd, k=k, return_routing=True)
        nres, near = L.route_stats()
        gsel = _u32(sel)
        bad, ties = routing_agreement(gsel, osel, gap, np.full(T, k))
        assert not bad, f"{case} T={T} k={k}: forward routing differs at tokens {bad[:5]}"
        assert near == o_ties, f"{case} T={T} k={k}: near ties {near} vs oracle {o_ties}"
        _, ooff, _, _ = oracle.bucket(gsel, G)
        assert np.array_equal(_u32(off), ooff)
        if ties == 0:
            assert np.array_equal(_u32(off), oracle.bucket(osel, G)[1])
        # weights: floating point, from the tensor-core logits (error <= the
        # certification bound, relative weight error <= 2 x that)
        wg = w.cpu().numpy()
        ok_t = np.array([np.array_equal(gsel[t, :k], osel[t, :k]) for t in range(T)])
        assert (np.abs(wg[ok_t, :k] - ow[ok_t, :k]) <= (4 * bound[ok_t] + 1e-6) * np.abs(ow[ok_t, :k]) + 1e-9).all()
        assert np.isfinite(y.float().cpu().numpy()).all()
        # separate top-k + exact fixup kernels (route)
        sel2, w2 = L.route(xd, k=k)
        nres2, near2 = L.route_stats()
        bad2, _ = routing_agreement(_u32(sel2), osel, gap, np.full(T, k))
        assert not bad2, f"{case} T={T} k={k}: route() differs at tokens {bad2[:5]}"
        assert near2 == o_ties
        report.append(f"k={k}: re-selected {nres}/{T}, near ties {near}")
    print(f"{case} T={T} max|logit| {amax:.1f}: " + "; ".join(report))


def test_routing_per_token_k_at_scale(oracle, torch_cuda_mod, layer):
    """Mixed-QoS tiers (per-token k) with scaled inputs and outliers."""
    torch = torch_cuda_mod
    T = 2048
    x, wr = _inputs(oracle, "all", T)
    layer.set_router(wr)
    logits = oracle.router_logits(x, wr, T, D, G)
    kpt = np.random.default_rng(13).choice([1, 2, 3, 4, 8, 11, 16], size=T).astype(np.uint32)
    osel, ow, gap = oracle.route(logits, 0, 16, 1, k_per_token=kpt)
    y, sel, w, off = layer.forward(torch.from_numpy(x).cuda().to(torch.bfloat16),
                                   k_per_token=torch.from_numpy(kpt.astype(np.int32)), return_routing=True)
    layer.check_errors()
    bad, ties = routing_agreement(_u32(sel), osel, gap, kpt)
    assert not bad
    assert np.array_equal(_u32(off), oracle.bucket(_u32(sel), G)[1])
    assert layer.route_stats()[1] == int((gap < 1e-6).sum())
