"""Proxy-gate router (reference proxy_scores + select_topk_subexperts,
inc/gating.hpp:107-145) on the GPU, against the oracle restatement
(orc_proxy_router_scores: the activation of every gate neuron computed like
inc/expert.hpp:62-75, the double mean of |a| over the sub-expert's gates).

Two device paths, both certified (proxy.cu):
  * exact fp64 gate activations in the reference's order (fp32 layers);
  * tensor-core gate/up columns with a per-neuron error bound and exact fp64
    re-selection of uncertain tokens (bf16 layers at serving shapes).
Selected ids are bit-exact outside the 1e-6 near-tie window; the GPU's
near-tie count equals the oracle's.  Acceptance C4 (tests/acceptance.cpp:
166-205, tests/test_gating.cpp:167-175) is replayed through mp_layer_route:
planted clusters, gates from the reference's select_gate_neurons, recall >= 0.95.
"""
import math

import numpy as np
import pytest

from gpu_util import bf16_round, routing_agreement

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda_mod(cuda_lib):
    import torch
    return torch


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


def _gates(oracle, parts, S, r, seed):
    """r gate neurons per sub-expert: ascending members chosen at random."""
    rng = np.random.default_rng(seed)
    out = []
    for p in parts:
        for s in range(S):
            mem = np.flatnonzero(p == s)
            out.append(sorted(rng.choice(mem, size=min(r, mem.size), replace=False).tolist()))
    return out


@pytest.fixture(scope="module")
def mixtral_proxy(oracle, torch_cuda_mod):
    """Mixtral layer shape in proxy-router mode (bf16: the tensor-core path),
    r = 4 gate neurons per sub-expert (the reference default, inc/gating.hpp:25).
    The oracle gets compact neuron-major experts holding only the gate neurons
    (a neuron's activation depends on its own columns only)."""
    torch = torch_cuda_mod
    from paper_2510_19366_b200 import MoeLayer, synth_fill
    E, S, d, ff, r = 8, 8, 4096, 14336, 4
    L = MoeLayer(E, S, d, ff, dtype="bf16", router="proxy", k_max=16, max_tokens=1024)
    parts = [oracle.random_balanced_partition(ff, S, 6000 + e) for e in range(E)]
    gates = _gates(oracle, parts, S, r, 21)
    compact, cgates = [], []
    for e in range(E):
        ws = []
        for m, (seed, scale) in enumerate(((100 + 3 * e, 1 / math.sqrt(d)), (101 + 3 * e, 1 / math.sqrt(d)),
                                           (102 + 3 * e, 1 / math.sqrt(ff)))):
            t = torch.empty(d * ff, dtype=torch.float32, device="cuda")
            synth_fill(t, seed, scale)
            ws.append(t)
        L.set_partition(e, parts[e])
        L.load_expert(e, *ws)
        ids = sorted({j for s in range(S) for j in gates[e * S + s]})
        pos = {j: q for q, j in enumerate(ids)}
        # neuron-major rows of the gate neurons
        wg = oracle.synth_t(100 + 3 * e, d, ff, 1 / math.sqrt(d)).reshape(ff, d)[ids]
        wu = oracle.synth_t(101 + 3 * e, d, ff, 1 / math.sqrt(d)).reshape(ff, d)[ids]
        compact.append((np.ascontiguousarray(wg), np.ascontiguousarray(wu), None))
        cgates += [[pos[j] for j in gates[e * S + s]] for s in range(S)]
        L.set_gates(e, r, gates[e * S:(e + 1) * S])
        del ws
    yield L, compact, cgates, d
    L.close()


def _oracle_scores(oracle, compact, cgates, S, x):
    import ctypes as C
    from oracle_lib import _csr, _ptr_array
    E = len(compact)
    T, d = x.shape
    ffc = compact[0][0].shape[0]
    off, ids = _csr(cgates)
    out = np.empty(T * E * S, np.float64)
    oracle._check(oracle.L.orc_proxy_router_scores(E, S, d, ffc, _ptr_array([c[0] for c in compact], None),
                                                   _ptr_array([c[1] for c in compact], None), 1, off, ids, T,
                                                   np.ascontiguousarray(x, np.float32).reshape(-1), out))
    return out.reshape(T, E * S)


@pytest.mark.parametrize("T,scale", [(1024, 1.0), (64, 1.0), (1024, 100.0)])
def test_proxy_router_mixtral_shape(oracle, torch_cuda_mod, mixtral_proxy, T, scale):
    torch = torch_cuda_mod
    L, compact, cgates, d = mixtral_proxy
    x = bf16_round(oracle.uniform_pm1(77 + T, T * d, scale).reshape(T, d))
    scores = _oracle_scores(oracle, compact, cgates, 8, x)
    xd = torch.from_numpy(x).cuda().to(torch.bfloat16)
    for k in (1, 2, 4, 8, 13, 16):
        osel, ow, gap = oracle.route(scores, k, 16, 1)
        sel, w = L.route(xd, k=k)
        nres, near = L.route_stats()
        bad, ties = routing_agreement(_u32(sel), osel, gap, np.full(T, k))
        assert not bad, f"T={T} x{scale} k={k}: proxy routing differs at tokens {bad[:5]}"
        assert near == ties, (near, ties)
        print(f"proxy T={T} x{scale} k={k}: re-selected {nres}/{T}, near ties {near}")
    # the full layer forward in proxy mode routes the same way
    y, sel, w, off = L.forward(xd, k=4, return_routing=True)
    osel, ow, gap = oracle.route(scores, 4, 16, 1)
    bad, _ = routing_agreement(_u32(sel), osel, gap, np.full(T, 4))
    assert not bad
    assert np.array_equal(_u32(off), oracle.bucket(_u32(sel), 64)[1])
    assert np.isfinite(y.float().cpu().numpy()).all()


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_proxy_router_small_exact_and_tc(oracle, torch_cuda_mod, dtype):
    """Toy shape, both dtypes (f32: exact fp64 path; bf16 d % 8 == 0: tensor
    cores), per-token k, weights against the oracle's softmax renormalisation."""
    torch = torch_cuda_mod
    from gpu_util import make_layer, toy_setup
    E, S, d, ff, T = 4, 4, 256, 512, 200
    experts, parts, wr, x = toy_setup(oracle, E, S, d, ff, T)
    gates = _gates(oracle, parts, S, 4, 3)
    L = make_layer(experts, parts, None, S, dtype, k_max=8, max_tokens=T, router="proxy")
    for e in range(E):
        L.set_gates(e, 4, gates[e * S:(e + 1) * S])
    xin = x if dtype == "f32" else bf16_round(x)
    scores = oracle.proxy_router_scores(experts, S, gates, xin)
    kpt = np.random.default_rng(2).integers(1, 9, T).astype(np.uint32)
    osel, ow, gap = oracle.route(scores, 0, 8, 1, k_per_token=kpt)
    sel, w = L.route(torch.from_numpy(xin).cuda().to(L.torch_dtype), k_per_token=torch.from_numpy(kpt.astype(np.int32)))
    L.check_errors()
    bad, ties = routing_agreement(_u32(sel), osel, gap, kpt)
    assert not bad
    assert L.route_stats()[1] == ties
    if dtype == "f32":  # exact path: the oracle's scores, hence its weights
        assert np.allclose(w.cpu().numpy(), ow, rtol=1e-6, atol=1e-8)
    L.close()


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_acceptance_c4_planted_clusters_through_layer_route(ref, oracle, torch_cuda_mod, dtype):
    """Acceptance C4's planted clusters (tests/acceptance.cpp:190-204) routed by
    the layer itself in proxy mode: one expert of 32 neurons in 4 contiguous
    sub-experts, token t = one-hot input e_t, w_gate = 30 (SiLU(30) = 30 to
    1e-11), w_up[t][j] = m[t][j] / SiLU(30), so the layer's gate activations
    are the planted matrix.  Gates from the reference's select_gate_neurons
    (r = 1); the layer's top-1 must equal the oracle's proxy selection and its
    recall against the true sub-expert norms must reach the reference's >= 0.95
    (and equal the reference's gating_fidelity)."""
    torch = torch_cuda_mod
    from paper_2510_19366_b200 import MoeLayer
    min_recall = 1.0
    for trial in range(20):
        m, part = ref.planted_cluster(64, 4, 8, 10000 + trial)
        k_a = ref.default_binarize_count(m.shape[1])
        co = ref.coactivation(ref.binarize_topk(m, k_a), k_a)
        gates = ref.select_gate_neurons(co, part, 4, 1)
        T, ff = m.shape
        d = T
        silu30 = 30.0 / (1.0 + math.exp(-30.0))
        wg = np.full((d, ff), 30.0, np.float32)
        wu = (m / silu30).astype(np.float32)          # row i = token i's input channel
        wd = np.zeros((ff, d), np.float32)
        L = MoeLayer(1, 4, d, ff, dtype=dtype, router="proxy", k_max=4, max_tokens=T)
        L.set_partition(0, part)
        L.load_expert(0, wg, wu, wd)
        L.set_gates(0, 1, gates)
        x = np.eye(T, dtype=np.float32)
        sel, w = L.route(torch.from_numpy(x).cuda().to(L.torch_dtype), k=1)
        gsel = _u32(sel)[:, 0]
        scores = oracle.proxy_router_scores([(wg, wu, wd)], 4, gates, x)
        osel, _, gap = oracle.route(scores, 1, 4, 1)
        assert np.array_equal(gsel, osel[:, 0])
        norms = np.stack([m[:, part == s].astype(np.float64).sum(axis=1) for s in range(4)], axis=1)
        truth = norms.argmax(axis=1)
        recall = float((gsel == truth).mean())
        assert recall == ref.gating_fidelity(m, part, 4, gates, 1, 1)
        min_recall = min(min_recall, recall)
        L.close()
    print(f"C4 planted through mp_layer_route ({dtype}): min recall {min_recall}")
    assert min_recall >= 0.95
