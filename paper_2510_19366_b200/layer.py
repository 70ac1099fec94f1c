"""Python mirror of the C++ host API (include/moeprism/moe_layer.hpp) over the
C-ABI, used by the tests and bench.py.  Device buffers are torch tensors
(PyTorch is plumbing here: memory, streams); every computation happens in the
CUDA kernels of libmoeprism_b200.so.

Reference interfaces mirrored:
  MoeLayer.forward           <- partitioned_forward composed over the selected
                                sub-experts + the router (inc/expert.hpp:101)
  MoeLayer.forward_selected  <- partitioned_forward with explicit active sets
  MoeLayer.route             <- select_topk_subexperts (inc/gating.hpp:129)
  MoeLayer.load_expert_file  <- load_toy_expert (inc/io.hpp:225)
  MoeLayer.load_partition_map<- read_ndjson + partition_doc_from_json
                                (inc/serde.hpp:113-151)
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import (MP_DTYPE_BF16, MP_DTYPE_F32, MP_ROUTER_LINEAR, MP_ROUTER_PROXY, MP_SEL_NONE,
                   MP_WEIGHT_SOFTMAX_RENORM, MP_WEIGHT_UNIT, LayerDesc, check)

_DTYPES = {"f32": MP_DTYPE_F32, "fp32": MP_DTYPE_F32, "float32": MP_DTYPE_F32, "bf16": MP_DTYPE_BF16,
           "bfloat16": MP_DTYPE_BF16}
_ROUTERS = {"linear": MP_ROUTER_LINEAR, "proxy": MP_ROUTER_PROXY}
_WEIGHTS = {"unit": MP_WEIGHT_UNIT, "softmax_renorm": MP_WEIGHT_SOFTMAX_RENORM}


def _torch():
    import torch
    return torch


def _ptr(a) -> Optional[int]:
    """Address of a torch tensor (host or device) or numpy array; None passes NULL."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def _stream_handle(stream) -> Optional[int]:
    if stream is None:
        torch = _torch()
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


class MoeLayer:
    def __init__(self, n_experts: int, n_subexperts: int, d_model: int, d_ff: int, dtype: str = "bf16",
                 router: str = "linear", weights: str = "softmax_renorm", k_max: int = 16,
                 max_tokens: int = 4096, device: int = 0, flags: int = 0):
        self.lib = _lib.load()
        self.E, self.S, self.d, self.ff = n_experts, n_subexperts, d_model, d_ff
        self.G = n_experts * n_subexperts
        self.dtype_code = _DTYPES[dtype]
        self.k_max, self.max_tokens, self.device = k_max, max_tokens, device
        desc = LayerDesc(n_experts, n_subexperts, d_model, d_ff, self.dtype_code, _ROUTERS[router], _WEIGHTS[weights],
                         k_max, max_tokens, device, flags)
        h = C.c_void_p()
        check(self.lib.mp_layer_create(C.byref(desc), C.byref(h)))
        self.h = h

    # ---------------------------------------------------------------- setup
    @property
    def torch_dtype(self):
        torch = _torch()
        return torch.bfloat16 if self.dtype_code == MP_DTYPE_BF16 else torch.float32

    def load_expert(self, e: int, w_gate, w_up, w_down):
        """MPEX layout fp32: w_gate, w_up d x ff row-major; w_down ff x d (host numpy or torch, any device)."""
        keep = [self._f32(w) for w in (w_gate, w_up, w_down)]
        check(self.lib.mp_layer_load_expert(self.h, e, *(_ptr(w) for w in keep)))

    def load_expert_file(self, e: int, path):
        check(self.lib.mp_layer_load_expert_file(self.h, e, str(path).encode()))

    def set_partition(self, e: int, assignment, n_sub: Optional[int] = None):
        a = np.ascontiguousarray(assignment, np.uint32)
        check(self.lib.mp_layer_set_partition(self.h, e, self.S if n_sub is None else n_sub,
                                              a.ctypes.data if a.size else None, a.size))

    def load_partition_map(self, path):
        check(self.lib.mp_layer_load_partition_map(self.h, str(path).encode()))

    def set_router(self, w_r):
        """w_r: d x (E*S) row-major fp32 (host or device)."""
        w = self._f32(w_r)
        check(self.lib.mp_layer_set_router(self.h, _ptr(w)))

    def set_shared_expert(self, w_gate, w_up, w_down, gate=None):
        """Always-on shared expert (Qwen1.5-MoE style): y += sigmoid(x . gate) * ffn(x).
        MPEX layout fp32 (w_gate, w_up d x ff_sh; w_down ff_sh x d); gate d fp32 or None (weight 1)."""
        keep = [self._f32(w) for w in (w_gate, w_up, w_down)]
        g = None if gate is None else self._f32(gate)
        ff_sh = (keep[0].size if isinstance(keep[0], np.ndarray) else keep[0].numel()) // self.d
        check(self.lib.mp_layer_set_shared_expert(self.h, ff_sh, *(_ptr(w) for w in keep), _ptr(g)))

    def set_residual(self, on: bool = True):
        """Fused residual: forward returns x + MoE(x) (bf16 layers; y must not alias x)."""
        check(self.lib.mp_layer_set_residual(self.h, int(on)))

    def enable_offload(self, cache_units: int, monolithic: bool = False):
        """Sub-expert offload cache (moe_layer.h): weights to pinned host memory,
        a device LRU cache of cache_units units (sub-experts, or whole experts)."""
        check(self.lib.mp_layer_enable_offload(self.h, self.S if monolithic else 1, cache_units))

    def offload_stats(self):
        """(hits, misses, bytes_h2d, last forward's requested units, last forward's misses)."""
        h, m, b = C.c_uint64(), C.c_uint64(), C.c_uint64()
        n, lm = C.c_uint32(), C.c_uint32()
        units = np.zeros(self.G, np.uint32)
        check(self.lib.mp_layer_offload_stats(self.h, C.byref(h), C.byref(m), C.byref(b), units.ctypes.data, self.G,
                                              C.byref(n), C.byref(lm)))
        return h.value, m.value, b.value, units[:n.value].copy(), lm.value

    def set_gates(self, e: int, r: int, gates: Sequence[Sequence[int]]):
        off = np.zeros(len(gates) + 1, np.uint32)
        for s, g in enumerate(gates):
            off[s + 1] = off[s] + len(g)
        ids = np.ascontiguousarray(np.concatenate([np.asarray(g, np.uint32) for g in gates]), np.uint32)
        check(self.lib.mp_layer_set_gates(self.h, e, r, off.ctypes.data, ids.ctypes.data))

    @staticmethod
    def _f32(w):
        if isinstance(w, np.ndarray):
            return np.ascontiguousarray(w, np.float32)
        torch = _torch()
        return w.to(torch.float32).contiguous()

    # ---------------------------------------------------------------- forward
    def forward(self, x, k: int = 0, k_per_token=None, y=None, return_routing: bool = False, stream=None):
        """x: (T, d) cuda tensor of the layer dtype.  Returns y (and sel, w, offsets)."""
        torch = _torch()
        T = x.shape[0]
        if y is None:
            y = torch.empty((T, self.d), dtype=self.torch_dtype, device=x.device)
        sel = w = off = None
        if return_routing:
            sel = torch.empty((T, self.k_max), dtype=torch.int32, device=x.device)
            w = torch.empty((T, self.k_max), dtype=torch.float32, device=x.device)
            off = torch.empty(self.G + 1, dtype=torch.int32, device=x.device)
        kpt = None if k_per_token is None else k_per_token.to(device=x.device, dtype=torch.int32).contiguous()
        check(self.lib.mp_layer_forward(self.h, _ptr(x), T, _ptr(kpt), k, _ptr(y), _ptr(sel), _ptr(w), _ptr(off),
                                        _stream_handle(stream)))
        if return_routing:
            return y, sel, w, off
        return y

    def forward_host(self, x: np.ndarray, k: int = 0, k_per_token=None, return_routing: bool = False, stream=None):
        """Host buffers in / out (x: numpy float32, or torch pinned bf16/f32)."""
        torch = _torch()
        T = x.shape[0]
        if isinstance(x, np.ndarray):
            y = np.empty((T, self.d), np.float32)
        else:
            y = torch.empty((T, self.d), dtype=x.dtype, pin_memory=x.is_pinned())
        sel = w = off = None
        if return_routing:
            sel = np.empty((T, self.k_max), np.uint32)
            w = np.empty((T, self.k_max), np.float32)
            off = np.empty(self.G + 1, np.uint32)
        kpt = None if k_per_token is None else np.ascontiguousarray(k_per_token, np.uint32)
        check(self.lib.mp_layer_forward_host(self.h, _ptr(x), T, _ptr(kpt), k, _ptr(y), _ptr(sel), _ptr(w),
                                             _ptr(off), _stream_handle(stream)))
        return (y, sel, w, off) if return_routing else y

    def forward_host_batches(self, xs, k: int, ys=None, stream=None):
        """Pipelined forwards over host batches (pinned torch tensors): uploads,
        compute and downloads of neighbouring batches overlap.  Returns ys."""
        torch = _torch()
        if ys is None:
            ys = [torch.empty((x.shape[0], self.d), dtype=x.dtype, pin_memory=x.is_pinned()) for x in xs]
        n = len(xs)
        xp = (C.c_void_p * n)(*[x.data_ptr() for x in xs])
        yp = (C.c_void_p * n)(*[y.data_ptr() for y in ys])
        nt = (C.c_uint32 * n)(*[x.shape[0] for x in xs])
        check(self.lib.mp_layer_forward_host_batches(self.h, n, xp, nt, k, yp, _stream_handle(stream)))
        return ys

    def forward_selected(self, x, sel, w=None, y=None, return_offsets: bool = False, stream=None):
        """Explicit selection (T x k_max global ids, MP_SEL_NONE padded); w None = unit weights."""
        torch = _torch()
        T = x.shape[0]
        if y is None:
            y = torch.empty((T, self.d), dtype=self.torch_dtype, device=x.device)
        off = torch.empty(self.G + 1, dtype=torch.int32, device=x.device) if return_offsets else None
        sel = sel.to(device=x.device, dtype=torch.int32).contiguous()
        if w is not None:
            w = w.to(device=x.device, dtype=torch.float32).contiguous()
        check(self.lib.mp_layer_forward_selected(self.h, _ptr(x), T, _ptr(sel), _ptr(w), _ptr(y), _ptr(off),
                                                 _stream_handle(stream)))
        return (y, off) if return_offsets else y

    def route(self, x, k: int = 0, k_per_token=None, stream=None):
        torch = _torch()
        T = x.shape[0]
        sel = torch.empty((T, self.k_max), dtype=torch.int32, device=x.device)
        w = torch.empty((T, self.k_max), dtype=torch.float32, device=x.device)
        kpt = None if k_per_token is None else k_per_token.to(device=x.device, dtype=torch.int32).contiguous()
        check(self.lib.mp_layer_route(self.h, _ptr(x), T, _ptr(kpt), k, _ptr(sel), _ptr(w), _stream_handle(stream)))
        return sel, w

    def route_stats(self, stream=None):
        """(tokens re-selected from exact fp64 logits, near ties with exact gap < 1e-6) of the last forward."""
        r, n = C.c_uint32(), C.c_uint32()
        check(self.lib.mp_layer_route_stats(self.h, C.byref(r), C.byref(n), _stream_handle(stream)))
        return r.value, n.value

    def check_errors(self, stream=None):
        check(self.lib.mp_layer_check_errors(self.h, _stream_handle(stream)))

    # ---------------------------------------------------------------- profiling
    def set_profiling(self, on: bool):
        check(self.lib.mp_layer_set_profiling(self.h, int(on)))

    def reset_stage_times(self):
        check(self.lib.mp_layer_reset_stage_times(self.h))

    def stage_times(self):
        names = C.create_string_buffer(256)
        ms = (C.c_double * 16)()
        launches = (C.c_uint64 * 16)()
        n = C.c_uint32()
        check(self.lib.mp_layer_stage_times(self.h, names, 256, ms, launches, C.byref(n), 16))
        keys = names.value.decode().split(",")
        return {keys[i]: (ms[i], launches[i]) for i in range(n.value)}

    def launch_count(self) -> int:
        return int(self.lib.mp_layer_launch_count(self.h))

    def close(self):
        if getattr(self, "h", None):
            self.lib.mp_layer_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def synth_fill(t, seed: int, scale: float = 1.0, first: int = 0, stream=None):
    """Fill a cuda tensor (float32 / bfloat16) with the counter-based synthetic
    stream (bit-identical to oracle orc_synth_fill)."""
    torch = _torch()
    code = MP_DTYPE_BF16 if t.dtype == torch.bfloat16 else MP_DTYPE_F32
    check(_lib.load().mp_synth_fill(t.data_ptr(), code, t.numel(), seed, first, scale, _stream_handle(stream)))
    return t


def read_mpex(path):
    """load_toy_expert (inc/io.hpp:225-251) through the library's own reader."""
    L = _lib.load()
    d, ff = C.c_uint32(), C.c_uint32()
    check(L.mp_format_read_mpex(str(path).encode(), C.byref(d), C.byref(ff), None, None, None))
    ws = [np.empty(d.value * ff.value, np.float32) for _ in range(3)]
    check(L.mp_format_read_mpex(str(path).encode(), C.byref(d), C.byref(ff), *(w.ctypes.data for w in ws)))
    return d.value, ff.value, ws


def read_partition_doc(path, index: int = 0):
    """Document `index` of an NDJSON partition map -> (expert_id, n_sub, assignment, r, gates, n_docs)."""
    L = _lib.load()
    nd, eid, ns, n, r, ng = C.c_size_t(), C.c_uint64(), C.c_uint32(), C.c_size_t(), C.c_uint32(), C.c_size_t()
    args = (C.byref(nd), C.byref(eid), C.byref(ns), C.byref(n))
    check(L.mp_format_read_partition_doc(str(path).encode(), index, *args, None, C.byref(r), C.byref(ng), None, None))
    a = np.empty(max(n.value, 1), np.uint32)
    off = np.empty(ns.value + 1, np.uint32)
    ids = np.empty(max(ng.value, 1), np.uint32)
    check(L.mp_format_read_partition_doc(str(path).encode(), index, *args, a.ctypes.data, C.byref(r), C.byref(ng),
                                         off.ctypes.data, ids.ctypes.data))
    gates = [ids[off[s]:off[s + 1]].tolist() for s in range(ns.value)] if r.value else None
    return eid.value, ns.value, a[:n.value], r.value, gates, nd.value


def validate_partition(n_sub: int, assignment):
    a = np.ascontiguousarray(assignment, np.uint32)
    check(_lib.load().mp_validate_partition(n_sub, a.ctypes.data if a.size else None, a.size))


__all__ = ["MoeLayer", "synth_fill", "read_mpex", "read_partition_doc", "validate_partition", "MP_SEL_NONE"]
