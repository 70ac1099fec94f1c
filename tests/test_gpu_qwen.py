"""GPU parity at the Qwen1.5-MoE-A2.7B layer shape (BASELINE configs[3],
SURVEY 8(d) C4): d=2048, 60 routed experts of ffn=1408 split into S=4
sub-experts (w=352, padded to 384 in the GEMM layout), E*S=240, plus the
always-on shared expert (ffn=5632, weight sigmoid(x . w_sg)).  Decode batch
(T=64) against the CPU oracle on every token; prefill (T=8192) routing
bit-exact on every token and outputs against the PyTorch fp32 reference on
every token."""
import math

import numpy as np
import pytest

from gpu_util import U32, bf16_ok, bf16_round, close_mask, routing_agreement, torch_layer_reference

pytestmark = pytest.mark.gpu
E, S, D, FF, FF_SH = 60, 4, 2048, 1408, 5632
TOL_BF16 = 2e-2


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


def _seeds(e):
    return ((300 + 3 * e, 1 / math.sqrt(D)), (301 + 3 * e, 1 / math.sqrt(D)), (302 + 3 * e, 1 / math.sqrt(FF)))


@pytest.fixture(scope="module")
def qwen(oracle, cuda_lib):
    import torch
    from paper_2510_19366_b200 import MoeLayer, synth_fill
    L = MoeLayer(E, S, D, FF, dtype="bf16", k_max=16, max_tokens=8192)
    parts = [oracle.random_balanced_partition(FF, S, 6000 + e) for e in range(E)]
    for e in range(E):
        ws = []
        for seed, scale in _seeds(e):
            t = torch.empty(D * FF, dtype=torch.float32, device="cuda")
            ws.append(synth_fill(t, seed, scale))
        L.set_partition(e, parts[e])
        L.load_expert(e, *ws)
    sh = []
    for seed, scale, n in ((900, 1 / math.sqrt(D), D * FF_SH), (901, 1 / math.sqrt(D), D * FF_SH),
                           (902, 1 / math.sqrt(FF_SH), FF_SH * D)):
        t = torch.empty(n, dtype=torch.float32, device="cuda")
        sh.append(synth_fill(t, seed, scale))
    gate = oracle.synth(903, D, 1 / math.sqrt(D))
    L.set_shared_expert(*sh, gate=gate)
    del sh
    wr = oracle.synth(17, D * E * S, 1 / math.sqrt(D))
    L.set_router(wr)
    yield L, parts, wr, gate
    L.close()


def _gen(torch, synth_fill):
    def gen(e):
        out = []
        for (seed, scale), shape in zip(_seeds(e), ((D, FF), (D, FF), (FF, D))):
            t = torch.empty(D * FF, dtype=torch.float32, device="cuda")
            synth_fill(t, seed, scale)
            out.append(t.bfloat16().float().view(*shape))
        return out
    return gen


_EXPERTS = []


def _oracle_experts(oracle):
    """bf16-rounded oracle weights, neuron-major gate/up (layout 1), built once."""
    if not _EXPERTS:
        for e in range(E):
            (sg, cg), (su, cu), (sd, cd) = _seeds(e)
            _EXPERTS.append((bf16_round(oracle.synth_t(sg, D, FF, cg)), bf16_round(oracle.synth_t(su, D, FF, cu)),
                             bf16_round(oracle.synth(sd, D * FF, cd))))
    return _EXPERTS


@pytest.mark.parametrize("k,T", [(4, 64), (8, 64), (16, 64), (8, 1), (8, 3), (16, 129)])
def test_qwen_decode_batch_vs_oracle(oracle, qwen, k, T):
    """Decode batches (64 tokens, and ragged 1 / 3 / 129 crossing the 2-token
    routing CTAs and the 128-token router tiles): routing bit-exact, bucket
    offsets bit-exact, every token's output (routed + shared) against the
    oracle on bf16-rounded inputs."""
    import torch
    L, parts, wr, gate = qwen
    x = torch.empty((T, D), dtype=torch.bfloat16, device="cuda")
    from paper_2510_19366_b200 import synth_fill
    synth_fill(x, 19, 1.0)
    xb = bf16_round(oracle.synth(19, T * D, 1.0)).reshape(T, D)
    y, sel, w, off = L.forward(x, k=k, return_routing=True)
    torch.cuda.synchronize()
    logits = oracle.router_logits(xb, wr, T, D, E * S)
    osel, ow, gap = oracle.route(logits, k, 16, 1)
    gsel = _u32(sel)
    bad, ties = routing_agreement(gsel, osel, gap, np.full(T, k))
    assert not bad, f"routing mismatch at tokens {bad[:5]}"
    _, ooff, _, _ = oracle.bucket(gsel, E * S)
    assert np.array_equal(_u32(off), ooff)
    experts = _oracle_experts(oracle)
    yo = oracle.layer_forward(experts, parts, S, xb, gsel, w.cpu().numpy(), 1, layout=1).astype(np.float64)
    shg = bf16_round(oracle.synth(900, D * FF_SH, 1 / math.sqrt(D)))
    shu = bf16_round(oracle.synth(901, D * FF_SH, 1 / math.sqrt(D)))
    shd = bf16_round(oracle.synth(902, FF_SH * D, 1 / math.sqrt(FF_SH)))
    yo += oracle.shared_expert_forward(D, FF_SH, shg, shu, shd, gate, xb)
    yh = y.float().cpu().numpy()
    assert close_mask(yh, yo, TOL_BF16).all()
    ok = bf16_ok(yh, yo)
    assert ok.all(), f"{(~ok).sum()} elements off"


def test_qwen_prefill_all_tokens(oracle, qwen):
    """T=8192 prefill at k=8: routing bit-exact on every token; every output
    row against the PyTorch fp32 reference (routed + shared expert)."""
    import torch
    from paper_2510_19366_b200 import synth_fill
    L, parts, wr, gate = qwen
    T, k = 8192, 8
    x = torch.empty((T, D), dtype=torch.bfloat16, device="cuda")
    synth_fill(x, 23, 1.0)
    xb = bf16_round(oracle.synth(23, T * D, 1.0)).reshape(T, D)
    y, sel, w, off = L.forward(x, k=k, return_routing=True)
    torch.cuda.synchronize()
    logits = oracle.router_logits(xb, wr, T, D, E * S)
    osel, ow, gap = oracle.route(logits, k, 16, 1)
    gsel = _u32(sel)
    bad, ties = routing_agreement(gsel, osel, gap, np.full(T, k))
    assert not bad, f"routing mismatch at tokens {bad[:5]}"
    print(f"Qwen prefill: near-ties {ties}/{T}")
    _, ooff, _, _ = oracle.bucket(gsel, E * S)
    assert np.array_equal(_u32(off), ooff)
    s64 = gsel.astype(np.int64)
    s64[s64 == U32] = -1
    want = torch_layer_reference(torch, _gen(torch, synth_fill), parts, S, D, xb, s64, w.cpu().numpy())
    # shared expert in torch fp32: h = bf16(silu(x Wg) * (x Wu)), o = bf16(h Wd), weight sigmoid(x . gate)
    shw = []
    for seed, scale, shape in ((900, 1 / math.sqrt(D), (D, FF_SH)), (901, 1 / math.sqrt(D), (D, FF_SH)),
                               (902, 1 / math.sqrt(FF_SH), (FF_SH, D))):
        t = torch.empty(D * FF_SH, dtype=torch.float32, device="cuda")
        synth_fill(t, seed, scale)
        shw.append(t.bfloat16().float().view(*shape))
    xt = torch.from_numpy(xb).cuda()
    h = (torch.nn.functional.silu(xt @ shw[0]) * (xt @ shw[1])).bfloat16().float()
    o = (h @ shw[2]).bfloat16().float()
    sg = torch.sigmoid(xt @ torch.from_numpy(gate).cuda())
    want = want + (o * sg[:, None]).cpu().numpy()
    ok = bf16_ok(y.float().cpu().numpy(), want)
    assert ok.all(), f"{(~ok).sum()} elements off in {np.unique(np.nonzero(~ok)[0]).size} tokens"


def test_shared_expert_validation(cuda_lib):
    import torch
    from paper_2510_19366_b200 import MoeLayer, ValidationError
    L = MoeLayer(2, 2, 64, 128, dtype="f32", k_max=2, max_tokens=8)
    w = np.zeros(64 * 256, np.float32)
    with pytest.raises(ValidationError, match="bf16"):
        L.set_shared_expert(w, w, w)
    L.close()
    L = MoeLayer(2, 2, 64, 128, dtype="bf16", k_max=2, max_tokens=8)
    bad = w.copy()
    bad[3] = np.inf
    with pytest.raises(ValidationError, match="not finite"):
        L.set_shared_expert(bad, w, w)
    L.set_shared_expert(w, w, w)
    with pytest.raises(ValidationError, match="already"):
        L.set_shared_expert(w, w, w)
    L.close()
