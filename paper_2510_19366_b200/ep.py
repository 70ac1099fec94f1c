"""Expert parallelism across GPUs: one process per GPU, the
parent experts sharded over the ranks, NCCL all-to-all(v) for the token
dispatch and the partial-output return.

Per layer and rank (T local tokens):
  1. route      replicated router-only layer: sel, w [T x k_max] (global ids)
  2. plan       mp_ep_plan: destination ranks per token (dedup), send counts
  3. pack       mp_ep_pack: each token row once per destination rank, with its
                selection in that rank's local ids and its combine weights
  4. exchange   all_to_all_single of counts, rows and metadata (NCCL/NVLink)
  5. experts    experts-only layer: mp_layer_forward_selected on the received
                rows -> one weighted partial per (token, rank)
  6. return     all_to_all_single of the partials back to the token owners
  7. combine    mp_ep_combine: y[t] = sum of partials in ascending rank order

PyTorch is the plumbing (process group, NCCL collectives, buffers); every
data-path computation runs in libmoeprism_b200.so.  The exchange logic is
backend-agnostic (``ops``) so the multi-process protocol is also exercised by
world-size-2 gloo tests on CPU with the oracle standing in for the kernels.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

from . import _lib
from ._lib import MP_DTYPE_BF16, MP_LAYER_EXPERTS_ONLY, MP_LAYER_ROUTER_ONLY, check
from .layer import MoeLayer, _ptr, _stream_handle


def _dist():
    import torch.distributed as dist
    return dist


class CudaEpOps:
    """The data-path steps on the GPU, through the C-ABI."""

    def __init__(self, E, S, d, ff, rank, world, dtype="bf16", k_max=16, max_tokens=4096, device=0):
        import torch
        self.torch = torch
        self.rank, self.world, self.d, self.k_max = rank, world, d, k_max
        G = E * S
        if G % world:
            raise ValueError(f"{G} sub-experts do not shard evenly over {world} ranks")
        # contiguous sub-expert ranges: whole experts when E % world == 0, else
        # sub-expert granularity (the boundary expert is held by both ranks)
        self.per_rank = G // world
        self.first_e = (self.per_rank * rank) // S
        self.last_e = (self.per_rank * (rank + 1) - 1) // S
        self.epr = self.last_e - self.first_e + 1
        self.router = MoeLayer(E, S, d, ff, dtype=dtype, k_max=k_max, max_tokens=max_tokens, device=device,
                               flags=MP_LAYER_ROUTER_ONLY)
        self.local = MoeLayer(self.epr, S, d, ff, dtype=dtype, weights="softmax_renorm", k_max=k_max,
                              max_tokens=max_tokens * world, device=device, flags=MP_LAYER_EXPERTS_ONLY)
        self.dtype = self.router.torch_dtype
        h = C.c_void_p()
        check(_lib.load().mp_ep_create_subexpert(world, rank, self.per_rank, S, d, k_max, max_tokens,
                                                 1 if self.dtype == torch.bfloat16 else 0, device, C.byref(h)))
        self.ep = h

    def route(self, x, k, k_per_token):
        return self.router.route(x, k=k, k_per_token=k_per_token)

    def plan(self, sel):
        counts = (C.c_uint32 * self.world)()
        check(_lib.load().mp_ep_plan(self.ep, _ptr(sel), sel.shape[0], counts, _stream_handle(None)))
        return [int(c) for c in counts]

    def pack(self, x, sel, w, n_send):
        torch = self.torch
        send_x = torch.empty((n_send, self.d), dtype=self.dtype, device=x.device)
        send_sel = torch.empty((n_send, self.k_max), dtype=torch.int32, device=x.device)
        send_w = torch.empty((n_send, self.k_max), dtype=torch.float32, device=x.device)
        check(_lib.load().mp_ep_pack(self.ep, _ptr(x), _ptr(sel), _ptr(w), x.shape[0], _ptr(send_x), _ptr(send_sel),
                                     _ptr(send_w), _stream_handle(None)))
        return send_x, send_sel, send_w

    def experts(self, recv_x, recv_sel, recv_w):
        if recv_x.shape[0] == 0:
            return recv_x.new_empty((0, self.d))
        return self.local.forward_selected(recv_x, recv_sel, recv_w)

    def combine(self, back, T):
        y = back.new_empty((T, self.d))
        check(_lib.load().mp_ep_combine(self.ep, _ptr(back), T, _ptr(y), _stream_handle(None)))
        return y

    # weights: experts are addressed by their GLOBAL id; non-owned ones are skipped
    def owns(self, e):
        return self.first_e <= e <= self.last_e

    def load_expert(self, e, wg, wu, wd):
        if self.owns(e):
            self.local.load_expert(e - self.first_e, wg, wu, wd)

    def set_partition(self, e, assignment):
        if self.owns(e):
            self.local.set_partition(e - self.first_e, assignment)

    def set_router(self, w_r):
        self.router.set_router(w_r)

    def close(self):
        if getattr(self, "ep", None):
            _lib.load().mp_ep_destroy(self.ep)
            self.ep = None
        self.router.close()
        self.local.close()


class ExpertParallelLayer:
    """A MoE-Prism layer sharded expert-parallel over the process group."""

    def __init__(self, ops, group=None, force_collectives=False):
        self.ops = ops
        self.group = group
        # run the NCCL collectives even in a 1-rank group (tests the exchange
        # path on one GPU); otherwise a 1-rank group short-cuts to copies
        self.force = force_collectives

    def _collective(self):
        dist = _dist()
        return dist.is_initialized() and (self.force or dist.get_world_size(self.group) > 1)

    def _a2a(self, out, inp, out_splits, in_splits):
        dist = _dist()
        if self._collective():
            dist.all_to_all_single(out, inp, output_split_sizes=out_splits, input_split_sizes=in_splits,
                                   group=self.group)
        else:
            out.copy_(inp)
        return out

    def exchange_counts(self, counts, device):
        import torch
        dist = _dist()
        send = torch.tensor(counts, dtype=torch.int64, device=device)
        if self._collective():
            recv = torch.empty_like(send)
            dist.all_to_all_single(recv, send, group=self.group)
            return [int(v) for v in recv.tolist()]
        return list(counts)

    def forward(self, x, k: int = 0, k_per_token=None, return_routing: bool = False):
        import torch
        ops = self.ops
        T = x.shape[0]
        sel, w = ops.route(x, k, k_per_token)
        counts = ops.plan(sel)
        send_x, send_sel, send_w = ops.pack(x, sel, w, sum(counts))
        recv_counts = self.exchange_counts(counts, x.device)
        n_recv = sum(recv_counts)
        recv_x = self._a2a(send_x.new_empty((n_recv, send_x.shape[1])), send_x, recv_counts, counts)
        # selection + weights in one message: [rows x 2*k_max] int32 (weights bit-cast)
        meta = torch.cat([send_sel, send_w.view(torch.int32)], dim=1).contiguous()
        recv_meta = self._a2a(meta.new_empty((n_recv, meta.shape[1])), meta, recv_counts, counts)
        kk = send_sel.shape[1]
        recv_sel = recv_meta[:, :kk].contiguous()
        recv_w = recv_meta[:, kk:].contiguous().view(torch.float32)
        part = ops.experts(recv_x, recv_sel, recv_w)
        back = self._a2a(part.new_empty((sum(counts), part.shape[1])), part.contiguous(), counts, recv_counts)
        y = ops.combine(back, T)
        if return_routing:
            return y, sel, w, counts, recv_counts
        return y


class NcclExpertParallelLayer:
    """The production expert-parallel layer: the whole per-layer sequence
    (route, plan, count exchange, pack, NCCL all-to-allv dispatch, experts,
    NCCL return, deterministic combine) runs in C++ inside
    libmoeprism_b200.so (mp_ep_forward) on a communicator the library owns.
    Python only hands the 128-byte NCCL unique id from rank 0 to the others
    (torch.distributed object broadcast) -- the exchange itself never touches
    torch.distributed, and each layer costs one host synchronisation (the
    count matrix)."""

    def __init__(self, ops, group=None, residual: bool = False):
        import torch
        self.ops, self.torch = ops, torch
        self.lib = _lib.load()
        self.flags = _lib.MP_EP_RESIDUAL if residual else 0
        uid = (C.c_uint8 * _lib.MP_EP_NCCL_ID_BYTES)()
        dist = _dist() if ops.world > 1 else None
        if ops.rank == 0:
            check(self.lib.mp_ep_nccl_unique_id(uid))
        if dist is not None and dist.is_initialized():
            box = [bytes(uid)]
            dist.broadcast_object_list(box, src=0, group=group)
            uid = (C.c_uint8 * _lib.MP_EP_NCCL_ID_BYTES).from_buffer_copy(box[0])
        check(self.lib.mp_ep_nccl_init(ops.ep, uid))

    def forward(self, x, k: int = 0, k_per_token=None, y=None, stream=None):
        torch, ops = self.torch, self.ops
        T = x.shape[0]
        if y is None:
            y = torch.empty((T, ops.d), dtype=ops.dtype, device=x.device)
        kpt = None if k_per_token is None else k_per_token.to(device=x.device, dtype=torch.int32).contiguous()
        check(self.lib.mp_ep_forward(ops.ep, ops.router.h, ops.local.h, _ptr(x), T, _ptr(kpt), k, _ptr(y), self.flags,
                                     _stream_handle(stream)))
        return y

    def last_counts(self):
        """(rows sent to each rank, rows received from each rank) of the last forward."""
        s = (C.c_uint32 * self.ops.world)()
        r = (C.c_uint32 * self.ops.world)()
        check(self.lib.mp_ep_last_counts(self.ops.ep, s, r))
        return list(s), list(r)


class PeerExpertParallelLayer:
    """Expert parallelism with both exchanges as peer-memory stores instead of
    NCCL all-to-alls: the pack kernel writes every token row straight into the
    destination rank's receive buffer (CUDA IPC mapping; NVLink between the
    GPUs of a node) and the return kernel writes the expert partials straight
    back into the source ranks' return buffers.  Host-side, per layer: one
    all-gather of the world x world plan and two barriers (every rank's writes
    complete before the readers launch)."""

    def __init__(self, ops, group=None, max_recv_rows=None):
        import torch
        self.ops, self.group = ops, group
        self.lib = _lib.load()
        dist = _dist()
        world = ops.world
        max_recv = max_recv_rows or ops.local.max_tokens
        handles = (C.c_uint8 * 256)()
        check(self.lib.mp_ep_p2p_setup(ops.ep, max_recv, handles))
        mine = bytes(handles)
        if dist.is_initialized() and dist.get_world_size(group) > 1:
            gathered = [None] * world
            dist.all_gather_object(gathered, mine, group=group)
        else:
            gathered = [mine]
        allh = (C.c_uint8 * (256 * world)).from_buffer_copy(b"".join(gathered))
        check(self.lib.mp_ep_p2p_open(ops.ep, allh))
        self.torch = torch

    def _sync(self):
        dist = _dist()
        self.torch.cuda.current_stream().synchronize()
        if dist.is_initialized() and dist.get_world_size(self.group) > 1:
            dist.barrier(group=self.group)

    def _plan_matrix(self, counts):
        dist = _dist()
        if dist.is_initialized() and dist.get_world_size(self.group) > 1:
            gathered = [None] * self.ops.world
            dist.all_gather_object(gathered, list(counts), group=self.group)
        else:
            gathered = [list(counts)]
        return [c for row in gathered for c in row]

    def forward(self, x, k: int = 0, k_per_token=None):
        torch, ops, lib = self.torch, self.ops, self.lib
        T = x.shape[0]
        sel, w = ops.route(x, k, k_per_token)
        counts = ops.plan(sel)
        mat = (C.c_uint32 * (ops.world * ops.world))(*self._plan_matrix(counts))
        n_recv = C.c_uint32()
        stream = _stream_handle(None)
        check(lib.mp_ep_p2p_pack(ops.ep, _ptr(x), _ptr(sel), _ptr(w), T, mat, C.byref(n_recv), stream))
        self._sync()  # every rank's rows are in place
        rx, rs, rw = C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(lib.mp_ep_p2p_recv_buffers(ops.ep, C.byref(rx), C.byref(rs), C.byref(rw)))
        part = torch.empty((max(n_recv.value, 1), ops.d), dtype=ops.dtype, device=x.device)
        if n_recv.value:
            check(lib.mp_layer_forward_selected(ops.local.h, rx, n_recv.value, rs, rw, _ptr(part), None, stream))
        check(lib.mp_ep_p2p_return(ops.ep, _ptr(part), n_recv.value, stream))
        self._sync()  # every partial is back at its source
        y = torch.empty((T, ops.d), dtype=ops.dtype, device=x.device)
        check(lib.mp_ep_p2p_combine(ops.ep, T, _ptr(y), stream))
        return y
