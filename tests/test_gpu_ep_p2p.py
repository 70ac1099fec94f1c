"""Peer-memory expert parallelism (PeerExpertParallelLayer): two processes
share the GPU, exchange CUDA IPC handles over gloo and write each other's
receive / return buffers directly (the code path NVLink peers take).  Each
rank's output must match the single full layer within bf16 tolerance, and
equal the NCCL-style path (same kernels, same order) bit for bit."""
import math
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
S, D, FF, T, K_MAX = 4, 256, 512, 96, 8


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir, E):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle_lib import Oracle
    from paper_2510_19366_b200 import MoeLayer
    from paper_2510_19366_b200.ep import CudaEpOps, ExpertParallelLayer, PeerExpertParallelLayer
    o = Oracle()
    experts = [tuple(a / np.float32(math.sqrt(D if i < 2 else FF)) for i, a in enumerate(o.random_expert(D, FF, 70 + e)))
               for e in range(E)]
    parts = [o.random_balanced_partition(FF, S, 80 + e) for e in range(E)]
    wr = o.uniform_pm1(7, D * E * S, 1.0 / math.sqrt(D))

    def make_ops():
        ops = CudaEpOps(E, S, D, FF, rank, world, dtype="bf16", k_max=K_MAX, max_tokens=T, device=0)
        for e in range(E):
            ops.set_partition(e, parts[e])
            ops.load_expert(e, *experts[e])
        ops.set_router(wr)
        return ops

    x = torch.from_numpy(o.uniform_pm1(9 + rank, T * D).reshape(T, D)).cuda().to(torch.bfloat16)
    kpt = torch.from_numpy(np.random.default_rng(rank).choice([1, 2, 4, 8], size=T).astype(np.int32)).cuda()
    peer = PeerExpertParallelLayer(make_ops())
    y_peer = peer.forward(x, k_per_token=kpt)
    y_peer2 = peer.forward(x, k_per_token=kpt)  # buffers reused across layers / steps
    nccl_style = ExpertParallelLayer(make_ops())
    y_a2a = nccl_style.forward(x, k_per_token=kpt)
    ref = MoeLayer(E, S, D, FF, dtype="bf16", k_max=K_MAX, max_tokens=T)
    for e in range(E):
        ref.set_partition(e, parts[e])
        ref.load_expert(e, *experts[e])
    ref.set_router(wr)
    y_ref = ref.forward(x, k_per_token=kpt)
    torch.cuda.synchronize()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), peer=y_peer.float().cpu().numpy(),
             peer2=y_peer2.float().cpu().numpy(), a2a=y_a2a.float().cpu().numpy(), ref=y_ref.float().cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("E", [4, 3])  # 3: sub-expert-granularity sharding
def test_peer_memory_ep_two_processes_one_gpu(cuda_lib, tmp_path, E):
    import torch.multiprocessing as mp
    from gpu_util import bf16_ok
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path), E), nprocs=2, join=True)
    for r in range(2):
        res = np.load(tmp_path / f"rank{r}.npz")
        assert np.array_equal(res["peer"], res["a2a"])
        assert np.array_equal(res["peer"], res["peer2"])
        assert bf16_ok(res["peer"], res["ref"]).all()
