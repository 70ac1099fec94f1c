"""Randomised layer shapes against the oracle (GPU): expert / sub-expert
counts, ragged d and d_ff (not multiples of the tile sizes), ragged batches,
scalar and per-token k, both dtypes and both weight modes.  Routing must be
bit-exact (outside the 1e-6 near-tie window), bucket offsets bit-exact, and
the output within the dtype's tolerance — the same contract as
test_gpu_layer.py, over shapes no fixed test pins."""
from __future__ import annotations

import numpy as np
import pytest

from gpu_util import U32, bf16_round, make_layer, out_ok, routing_agreement, toy_setup

pytestmark = pytest.mark.gpu


def _u32(t):
    return t.cpu().numpy().view(np.uint32) if t.dtype.itemsize == 4 else t.cpu().numpy().astype(np.uint32)


@pytest.mark.parametrize("seed", range(64))
def test_random_layer_config(oracle, cuda_lib, seed):
    import torch
    rng = np.random.default_rng(7000 + seed)
    E = int(rng.integers(1, 9))
    S = int(rng.integers(1, 9))
    if seed % 7 == 3:  # > 128 sub-experts: the router's column split, the 8-chunk top-k
        E, S = int(rng.integers(33, 65)), 4
    d = int(rng.choice([40, 64, 96, 136, 200, 256, 312]))
    ff = int(rng.integers(S, 300))
    T = int(rng.integers(1, 1500 if seed % 5 == 0 else 300))  # crosses the 2 / 8 / 32-token routing CTAs
    dtype = "bf16" if seed % 3 else "f32"
    weights = "unit" if seed % 4 == 1 else "softmax_renorm"
    G = E * S
    k_max = int(min(16, G))
    experts, parts, wr, x = toy_setup(oracle, E, S, d, ff, T, seed_x=seed, seed_r=seed + 3, seed_w=9000 + 10 * seed,
                                      seed_p=9500 + 10 * seed, contiguous=bool(seed % 2))
    L = make_layer(experts, parts, wr, S, dtype, weights=weights, k_max=k_max, max_tokens=max(T, 1))
    try:
        xin = x if dtype == "f32" else bf16_round(x)
        xd = torch.from_numpy(np.ascontiguousarray(xin)).cuda().to(L.torch_dtype)
        if seed % 2:
            kpt = rng.integers(1, k_max + 1, T).astype(np.uint32)
            y, sel, w, off = L.forward(xd, k_per_token=torch.from_numpy(kpt.astype(np.int32)), return_routing=True)
            k_arg = 0
        else:
            k = int(rng.integers(1, k_max + 1))
            kpt = np.full(T, k, np.uint32)
            y, sel, w, off = L.forward(xd, k=k, return_routing=True)
            k_arg = k
        L.check_errors()
        torch.cuda.synchronize()
        logits = oracle.router_logits(xin, wr, T, d, G)
        wm = 0 if weights == "unit" else 1
        if k_arg:
            osel, ow, gap = oracle.route(logits, k_arg, k_max, wm)
        else:
            osel, ow, gap = oracle.route(logits, 0, k_max, wm, k_per_token=kpt)
        gsel = _u32(sel)
        bad, _ = routing_agreement(gsel, osel, gap, kpt)
        assert not bad, f"E={E} S={S} d={d} ff={ff} T={T}: routing mismatch at {bad[:5]}"
        _, ooff, _, _ = oracle.bucket(gsel, G)
        assert np.array_equal(_u32(off), ooff)
        exs = experts if dtype == "f32" else [tuple(bf16_round(a) for a in e) for e in experts]
        yo = oracle.layer_forward(exs, parts, S, xin, gsel, w.cpu().numpy(), wm)
        ok = out_ok(y.float().cpu().numpy(), yo, dtype)
        assert ok.all(), f"E={E} S={S} d={d} ff={ff} T={T} {dtype} {weights}: {(~ok).sum()} elements off"
    finally:
        L.close()
