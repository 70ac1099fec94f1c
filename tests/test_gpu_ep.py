"""Expert-parallel kernels (mp_ep_plan / mp_ep_pack / mp_ep_combine) and the
role-split layers on one GPU: world=1 loopback must equal the single layer
bit for bit; an emulated world=2 (both ranks in this process, the all-to-all
done by slicing) must match the single layer within bf16 tolerance."""
import math

import numpy as np
import pytest

from gpu_util import bf16_ok

pytestmark = pytest.mark.gpu
E, S, D, FF, T, K_MAX = 4, 4, 256, 512, 96, 8


def _setup(oracle, E=E):
    experts = [tuple(a / np.float32(math.sqrt(D if i < 2 else FF)) for i, a in enumerate(oracle.random_expert(D, FF, 70 + e)))
               for e in range(E)]
    parts = [oracle.random_balanced_partition(FF, S, 80 + e) for e in range(E)]
    wr = oracle.uniform_pm1(7, D * E * S, 1.0 / math.sqrt(D))
    return experts, parts, wr


def _ops(world, rank, experts, parts, wr):
    from paper_2510_19366_b200.ep import CudaEpOps
    E = len(experts)
    ops = CudaEpOps(E, S, D, FF, rank, world, dtype="bf16", k_max=K_MAX, max_tokens=T, device=0)
    for e in range(E):
        ops.set_partition(e, parts[e])
        ops.load_expert(e, *experts[e])
    ops.set_router(wr)
    return ops


def test_ep_world1_loopback_bitwise(oracle, cuda_lib):
    import torch
    from paper_2510_19366_b200 import MoeLayer
    from paper_2510_19366_b200.ep import ExpertParallelLayer
    experts, parts, wr = _setup(oracle)
    x = torch.from_numpy(oracle.uniform_pm1(5, T * D).reshape(T, D)).cuda().to(torch.bfloat16)
    ref = MoeLayer(E, S, D, FF, dtype="bf16", k_max=K_MAX, max_tokens=T)
    for e in range(E):
        ref.set_partition(e, parts[e])
        ref.load_expert(e, *experts[e])
    ref.set_router(wr)
    kpt = torch.from_numpy(np.random.default_rng(0).choice([1, 2, 4, 8], size=T).astype(np.int32)).cuda()
    y_ref = ref.forward(x, k_per_token=kpt)
    layer = ExpertParallelLayer(_ops(1, 0, experts, parts, wr))
    y = layer.forward(x, k_per_token=kpt)
    torch.cuda.synchronize()
    assert torch.equal(y, y_ref)


@pytest.mark.parametrize("E", [4, 3])  # E=3: sub-expert-granularity sharding (6 of 12 sub-experts per rank)
def test_ep_world2_emulated(oracle, cuda_lib, E):
    import torch
    from paper_2510_19366_b200 import MoeLayer
    experts, parts, wr = _setup(oracle, E)
    ref = MoeLayer(E, S, D, FF, dtype="bf16", k_max=K_MAX, max_tokens=T)
    for e in range(E):
        ref.set_partition(e, parts[e])
        ref.load_expert(e, *experts[e])
    ref.set_router(wr)
    ranks = [_ops(2, r, experts, parts, wr) for r in range(2)]
    xs = [torch.from_numpy(oracle.uniform_pm1(9 + r, T * D).reshape(T, D)).cuda().to(torch.bfloat16) for r in range(2)]
    k = 6
    sends, counts = [], []
    for r, ops in enumerate(ranks):
        sel, w = ops.route(xs[r], k, None)
        c = ops.plan(sel)
        counts.append(c)
        sends.append(ops.pack(xs[r], sel, w, sum(c)))
        # dedup: each (token, destination rank) appears once
        s = sel.cpu().numpy().view(np.uint32)
        dests = sum(len({int(g) // (E * S // 2) for g in row if g != 0xFFFFFFFF}) for row in s)
        assert dests == sum(c)
    # emulated all-to-all: rank q receives the q-th segment of every rank's send
    def seg(r, q):
        off = sum(counts[r][:q])
        return slice(off, off + counts[r][q])
    parts_out = {}
    for q, ops in enumerate(ranks):
        rx = torch.cat([sends[r][0][seg(r, q)] for r in range(2)])
        rs = torch.cat([sends[r][1][seg(r, q)] for r in range(2)])
        rw = torch.cat([sends[r][2][seg(r, q)] for r in range(2)])
        part = ops.experts(rx, rs, rw)
        o = 0
        for r in range(2):
            n = counts[r][q]
            parts_out[(r, q)] = part[o:o + n]
            o += n
    for r, ops in enumerate(ranks):
        back = torch.cat([parts_out[(r, q)] for q in range(2)])
        y = ops.combine(back, T)
        y_ref = ref.forward(xs[r], k=k)
        torch.cuda.synchronize()
        assert bf16_ok(y.float().cpu().numpy(), y_ref.float().cpu().numpy()).all()
    for ops in ranks:
        ops.close()


def test_ep_nccl_collectives_world1(oracle, cuda_lib):
    """The NCCL exchange path itself (all_to_all_single of counts, bf16 rows,
    int32 metadata and the partials) in a 1-rank NCCL process group: equal to
    the single layer bit for bit, like the copy loopback."""
    import socket
    import torch
    import torch.distributed as dist
    from paper_2510_19366_b200 import MoeLayer
    from paper_2510_19366_b200.ep import ExpertParallelLayer
    if dist.is_initialized():
        pytest.skip("a process group is already initialised")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        experts, parts, wr = _setup(oracle)
        x = torch.from_numpy(oracle.uniform_pm1(6, T * D).reshape(T, D)).cuda().to(torch.bfloat16)
        ref = MoeLayer(E, S, D, FF, dtype="bf16", k_max=K_MAX, max_tokens=T)
        for e in range(E):
            ref.set_partition(e, parts[e])
            ref.load_expert(e, *experts[e])
        ref.set_router(wr)
        y_ref = ref.forward(x, k=4)
        layer = ExpertParallelLayer(_ops(1, 0, experts, parts, wr), force_collectives=True)
        y = layer.forward(x, k=4)
        torch.cuda.synchronize()
        assert torch.equal(y, y_ref)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("residual", [False, True])
def test_ep_cpp_nccl_transport_world1(oracle, cuda_lib, residual):
    """The production path: mp_ep_forward (C++ host, the library's own NCCL
    communicator, grouped ncclSend/ncclRecv all-to-allv) in a 1-rank world,
    bit-identical to the single layer over several calls (buffer reuse) and
    per-token k.  With the residual, the expert-parallel combine adds x to the
    bf16 partial of each rank (the single layer adds it inside its fp32
    accumulator), so the reference is bf16(x + bf16(MoE(x))), bit for bit."""
    import torch
    from paper_2510_19366_b200 import MoeLayer
    from paper_2510_19366_b200.ep import NcclExpertParallelLayer
    experts, parts, wr = _setup(oracle)
    ref = MoeLayer(E, S, D, FF, dtype="bf16", k_max=K_MAX, max_tokens=T)
    for e in range(E):
        ref.set_partition(e, parts[e])
        ref.load_expert(e, *experts[e])
    ref.set_router(wr)
    ops = _ops(1, 0, experts, parts, wr)
    layer = NcclExpertParallelLayer(ops, residual=residual)
    for i, Tn in enumerate((T, 17, 1, T)):
        x = torch.from_numpy(oracle.uniform_pm1(50 + i, Tn * D).reshape(Tn, D)).cuda().to(torch.bfloat16)
        kpt = torch.from_numpy(np.random.default_rng(i).choice([1, 2, 4, 8], size=Tn).astype(np.int32)).cuda()
        for kk, kp in ((4, None), (0, kpt)):
            y_ref = ref.forward(x, k=kk, k_per_token=kp)
            if residual:
                y_ref = (x.float() + y_ref.float()).to(torch.bfloat16)
            y = layer.forward(x, k=kk, k_per_token=kp)
            torch.cuda.synchronize()
            assert torch.equal(y, y_ref), (Tn, kk)
        sent, recv = layer.last_counts()
        assert sent == [Tn] and recv == [Tn]
    ops.close()
    ref.close()
