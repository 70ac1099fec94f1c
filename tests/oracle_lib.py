"""ctypes bindings to the parity oracle (test infrastructure only).

* ``Oracle``  -> oracle/liboracle.so, the C restatement (oracle/moe_oracle.c)
* ``RefLib``  -> oracle/_ref/libmoeprism_ref.so, the reference headers compiled
  verbatim (oracle/ref_shim.cpp); absent when it was never built.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
ORACLE_SO = ROOT / "oracle" / "liboracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "libmoeprism_ref.so"

U32 = 0xFFFFFFFF

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_sz = C.c_size_t


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _ptr_array(arrays, ctype):
    arr = (C.c_void_p * len(arrays))()
    for i, a in enumerate(arrays):
        arr[i] = a.ctypes.data_as(C.c_void_p)
    return arr


def _csr(gates):
    off = np.zeros(len(gates) + 1, np.uint32)
    for n, g in enumerate(gates):
        off[n + 1] = off[n] + len(g)
    ids = np.ascontiguousarray(np.concatenate([np.asarray(g, np.uint32) for g in gates]) if gates else np.zeros(0, np.uint32), np.uint32)
    return off, ids


class Oracle:
    """The C restatement.  Every method mirrors a reference function."""

    def __init__(self, path: Path = ORACLE_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built; run `make -C oracle`")
        L = self.L = C.CDLL(str(path))
        L.orc_last_error.restype = C.c_char_p
        L.orc_mt64_draw.argtypes = [C.c_uint64, _sz, _u64p]
        L.orc_mt_uniform_pm1.argtypes = [C.c_uint64, _sz, C.c_double, _f32p]
        L.orc_random_expert.argtypes = [_sz, _sz, C.c_uint64, _f32p, _f32p, _f32p]
        L.orc_random_balanced_partition.argtypes = [_sz, C.c_uint32, C.c_uint64, _u32p]
        L.orc_contiguous_partition.argtypes = [_sz, C.c_uint32, _u32p]
        L.orc_synth_fill.argtypes = [C.c_uint64, C.c_uint64, _sz, C.c_double, _f32p]
        L.orc_synth_fill_t.argtypes = [C.c_uint64, _sz, _sz, C.c_double, _f32p]
        L.orc_silu.restype = C.c_double
        L.orc_silu.argtypes = [C.c_double]
        L.orc_toy_ffn_forward.argtypes = [_sz, _sz, _f32p, _f32p, _f32p, _f32p, _sz, _f32p, _f32p]
        L.orc_validate_partition.argtypes = [C.c_uint32, _sz, _u32p]
        L.orc_partitioned_forward.argtypes = [_sz, _sz, _f32p, _f32p, _f32p, C.c_uint32, _sz, _u32p,
                                              _f32p, _sz, _u32p, _sz, _f32p]
        L.orc_proxy_scores.argtypes = [_f32p, _sz, C.c_uint32, C.c_uint32, _u32p, _u32p, _f64p]
        L.orc_select_topk.argtypes = [_f64p, _sz, C.c_uint32, _u32p, C.POINTER(C.c_double)]
        L.orc_router_logits.argtypes = [_sz, _sz, _sz, _f32p, _f32p, _f64p]
        L.orc_route.argtypes = [_sz, _sz, _f64p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_int, _u32p, _f32p, C.c_void_p]
        L.orc_bucket.argtypes = [_sz, _sz, C.c_uint32, _u32p, _u32p, _u32p, _u32p, _u32p]
        L.orc_layer_forward.argtypes = [_sz, _sz, _sz, _sz, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_int, _sz, _f32p, C.c_uint32, _u32p, _f32p, C.c_int, _f32p, C.c_int]
        L.orc_proxy_router_scores.argtypes = [_sz, _sz, _sz, _sz, C.c_void_p, C.c_void_p, C.c_int, _u32p, _u32p,
                                              _sz, _f32p, _f64p]

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.L.orc_last_error().decode())

    # -- generators ------------------------------------------------------
    def mt64_draw(self, seed, n):
        out = np.empty(n, np.uint64)
        self.L.orc_mt64_draw(seed, n, out)
        return out

    def uniform_pm1(self, seed, n, scale=1.0):
        out = np.empty(n, np.float32)
        self.L.orc_mt_uniform_pm1(seed, n, scale, out)
        return out

    def random_expert(self, d, ff, seed):
        wg, wu, wd = (np.empty(d * ff, np.float32) for _ in range(3))
        self._check(self.L.orc_random_expert(d, ff, seed, wg, wu, wd))
        return wg, wu, wd

    def random_balanced_partition(self, n, n_sub, seed):
        out = np.empty(n, np.uint32)
        self._check(self.L.orc_random_balanced_partition(n, n_sub, seed, out))
        return out

    def contiguous_partition(self, n, n_sub):
        out = np.empty(max(n, 1), np.uint32)
        self._check(self.L.orc_contiguous_partition(n, n_sub, out))
        return out[:n]

    def synth(self, seed, n, scale=1.0, first=0):
        out = np.empty(n, np.float32)
        self.L.orc_synth_fill(seed, first, n, scale, out)
        return out

    def synth_t(self, seed, rows, cols, scale=1.0):
        out = np.empty(rows * cols, np.float32)
        self.L.orc_synth_fill_t(seed, rows, cols, scale, out)
        return out

    # -- expert / routing --------------------------------------------------
    def silu(self, x):
        return self.L.orc_silu(x)

    def toy_ffn_forward(self, d, ff, wg, wu, wd, x):
        y = np.empty(d, np.float32)
        a = np.empty(ff, np.float32)
        self._check(self.L.orc_toy_ffn_forward(d, ff, wg, wu, wd, np.ascontiguousarray(x, np.float32), len(x), y, a))
        return y, a

    def shared_expert_forward(self, d, ff_sh, wg, wu, wd, gate, x):
        """Restated shared (always-on) expert, Qwen1.5-MoE style (
        no reference counterpart): sigmoid(x . gate) * toy_ffn_forward(x)
        (inc/expert.hpp:79-96), gate dot product in double, i ascending.
        Returns float64 (T, d); gate None = weight 1."""
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty(x.shape, np.float64)
        for t in range(x.shape[0]):
            y, _ = self.toy_ffn_forward(d, ff_sh, wg, wu, wd, x[t])
            s = 1.0 if gate is None else 1.0 / (1.0 + np.exp(-np.dot(x[t].astype(np.float64), gate.astype(np.float64))))
            out[t] = s * y.astype(np.float64)
        return out

    def partitioned_forward(self, d, ff, wg, wu, wd, n_sub, assignment, x, active):
        y = np.empty(d, np.float32)
        act = np.ascontiguousarray(np.asarray(active, np.uint32).reshape(-1))
        if act.size == 0:
            act = np.zeros(1, np.uint32)
            n_act = 0
        else:
            n_act = act.size
        x = np.ascontiguousarray(x, np.float32)
        self._check(self.L.orc_partitioned_forward(d, ff, wg, wu, wd, n_sub, len(assignment),
                                                   np.ascontiguousarray(assignment, np.uint32), x, len(x), act, n_act, y))
        return y

    def validate_partition(self, n_sub, assignment):
        a = np.ascontiguousarray(assignment, np.uint32)
        self._check(self.L.orc_validate_partition(n_sub, len(a), a if len(a) else np.zeros(1, np.uint32)))

    def proxy_scores(self, act, gates, r):
        off, ids = _csr(gates)
        out = np.empty(len(gates), np.float64)
        self._check(self.L.orc_proxy_scores(np.ascontiguousarray(act, np.float32), len(act), len(gates), r, off,
                                            ids if ids.size else np.zeros(1, np.uint32), out))
        return out

    def select_topk(self, scores, k, with_gap=False):
        s = np.ascontiguousarray(scores, np.float64)
        out = np.empty(max(k, 1), np.uint32)
        gap = C.c_double()
        self._check(self.L.orc_select_topk(s, len(s), k, out, C.byref(gap)))
        return (out[:k], gap.value) if with_gap else out[:k]

    def router_logits(self, x, wr, T, d, G):
        out = np.empty(T * G, np.float64)
        self._check(self.L.orc_router_logits(T, d, G, np.ascontiguousarray(x, np.float32).reshape(-1),
                                             np.ascontiguousarray(wr, np.float32).reshape(-1), out))
        return out.reshape(T, G)

    def route(self, logits, k, k_max, mode, k_per_token=None):
        logits = np.ascontiguousarray(logits, np.float64)
        T, G = logits.shape
        sel = np.empty(T * k_max, np.uint32)
        w = np.empty(T * k_max, np.float32)
        gap = np.empty(T, np.float64)
        kpt = None
        if k_per_token is not None:
            kpt = np.ascontiguousarray(k_per_token, np.uint32)
        self._check(self.L.orc_route(T, G, logits.reshape(-1), kpt.ctypes.data if kpt is not None else None,
                                     k, k_max, mode, sel, w, gap.ctypes.data))
        return sel.reshape(T, k_max), w.reshape(T, k_max), gap

    def bucket(self, sel, G):
        sel = np.ascontiguousarray(sel, np.uint32)
        T, k_max = sel.shape
        counts = np.empty(G, np.uint32)
        offsets = np.empty(G + 1, np.uint32)
        n = int((sel != U32).sum())
        perm = np.empty(max(n, 1), np.uint32)
        slot = np.empty(T * k_max, np.uint32)
        self._check(self.L.orc_bucket(T, G, k_max, sel.reshape(-1), counts, offsets, perm, slot))
        return counts, offsets, perm[:n], slot.reshape(T, k_max)

    def layer_forward(self, experts, assignments, S, x, sel, w, mode, layout=0, nthreads=None):
        """experts: list of (wg, wu, wd) float32 flat arrays; layout 0 = MPEX
        (d x ff gate/up), 1 = neuron-major (ff x d gate/up)."""
        E = len(experts)
        x = np.ascontiguousarray(x, np.float32)
        T, d = x.shape
        ff = assignments[0].size
        sel = np.ascontiguousarray(sel, np.uint32)
        w = np.ascontiguousarray(w, np.float32)
        k_max = sel.shape[1]
        y = np.empty((T, d), np.float32)
        wg = _ptr_array([e[0] for e in experts], None)
        wu = _ptr_array([e[1] for e in experts], None)
        wd = _ptr_array([e[2] for e in experts], None)
        asg = _ptr_array([np.ascontiguousarray(a, np.uint32) for a in assignments], None)
        nthreads = nthreads or os.cpu_count() or 1
        self._check(self.L.orc_layer_forward(E, S, d, ff, wg, wu, wd, asg, layout, T, x.reshape(-1), k_max,
                                             sel.reshape(-1), w.reshape(-1), mode, y.reshape(-1), nthreads))
        return y

    def proxy_router_scores(self, experts, S, gates, x, layout=0):
        """gates: list over global sub-expert g of ascending neuron ids within expert g // S."""
        E = len(experts)
        x = np.ascontiguousarray(x, np.float32)
        T, d = x.shape
        ff = experts[0][0].size // d
        off, ids = _csr(gates)
        out = np.empty(T * E * S, np.float64)
        wg = _ptr_array([e[0] for e in experts], None)
        wu = _ptr_array([e[1] for e in experts], None)
        self._check(self.L.orc_proxy_router_scores(E, S, d, ff, wg, wu, layout, off, ids, T, x.reshape(-1), out))
        return out.reshape(T, E * S)


class RefLib:
    """The reference headers compiled verbatim (oracle/_ref)."""

    def __init__(self, path: Path = REF_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (reference sources absent?)")
        L = self.L = C.CDLL(str(path))
        L.ref_last_error.restype = C.c_char_p
        L.ref_mt64_draw.argtypes = [C.c_uint64, _sz, _u64p]
        L.ref_uniform01.argtypes = [C.c_uint64, _sz, _f64p]
        L.ref_random_expert.argtypes = [_sz, _sz, C.c_uint64, _f32p, _f32p, _f32p]
        L.ref_random_balanced_partition.argtypes = [_sz, C.c_uint32, C.c_uint64, _u32p]
        L.ref_contiguous_partition.argtypes = [_sz, C.c_uint32, _u32p]
        L.ref_validate_partition.argtypes = [C.c_uint32, _sz, _u32p]
        L.ref_toy_ffn_forward.argtypes = [_sz, _sz, _f32p, _f32p, _f32p, _f32p, _sz, _f32p, _f32p]
        L.ref_partitioned_forward.argtypes = [_sz, _sz, _f32p, _f32p, _f32p, C.c_uint32, _sz, _u32p,
                                              _f32p, _sz, _u32p, _sz, _f32p]
        L.ref_proxy_scores.argtypes = [_f32p, _sz, C.c_uint32, C.c_uint32, _u32p, _u32p, _f64p]
        L.ref_select_topk.argtypes = [_f64p, _sz, C.c_uint32, _u32p]
        L.ref_save_toy_expert.argtypes = [C.c_char_p, _sz, _sz, _f32p, _f32p, _f32p]
        L.ref_collect_activation_matrix.argtypes = [_sz, _sz, _f32p, _f32p, _f32p, _sz, _f32p, _f32p]
        L.ref_binarize_topk.argtypes = [_f32p, _sz, _sz, _sz, C.c_void_p]
        L.ref_coactivation.argtypes = [C.c_void_p, _sz, _sz, _sz, _u32p]
        L.ref_save_activation_matrix.argtypes = [C.c_char_p, _sz, _sz, _f32p]
        L.ref_offload_replay.argtypes = [C.c_uint32, C.c_uint32, _sz, _u32p, _u32p, _u64p]
        L.ref_default_binarize_count.argtypes = [_sz]
        L.ref_default_binarize_count.restype = _sz
        L.ref_random_matrix.argtypes = [_sz, _sz, C.c_uint64, _f32p]
        L.ref_planted_cluster.argtypes = [_sz, C.c_uint32, _sz, C.c_uint64, _f32p, _u32p]
        L.ref_select_gate_neurons.argtypes = [_u32p, _sz, C.c_uint32, _u32p, C.c_uint32, _u32p, _u32p]
        L.ref_gating_fidelity.argtypes = [_f32p, _sz, _sz, C.c_uint32, _u32p, C.c_uint32, _u32p, _u32p, C.c_uint32,
                                          C.POINTER(C.c_double)]
        L.ref_load_activation_matrix.argtypes = [C.c_char_p, C.POINTER(_sz), C.POINTER(_sz), C.c_void_p]
        L.ref_perf_table_eval.argtypes = [C.c_char_p, C.c_uint64, C.c_uint32, C.POINTER(C.c_double), C.POINTER(_sz),
                                          C.POINTER(_sz)]
        L.ref_load_toy_expert.argtypes = [C.c_char_p, C.POINTER(_sz), C.POINTER(_sz), C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_append_partition_doc.argtypes = [C.c_char_p, C.c_uint64, C.c_uint32, _sz, _u32p, C.c_double, C.c_uint64, C.c_int]
        L.ref_append_partition_gates_doc.argtypes = [C.c_char_p, C.c_uint64, C.c_uint32, _sz, _u32p, C.c_uint32,
                                                     _u32p, _u32p, C.c_int]
        L.ref_read_partition_doc.argtypes = [C.c_char_p, _sz, C.POINTER(C.c_uint64), C.POINTER(C.c_uint32),
                                             C.POINTER(_sz), C.c_void_p, C.POINTER(_sz)]
        L.ref_layer_create.restype = C.c_void_p
        L.ref_layer_create.argtypes = [_sz, _sz, _sz, _sz, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_layer_destroy.argtypes = [C.c_void_p]
        L.ref_layer_route.argtypes = [C.c_void_p, _sz, _f32p, _f32p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_int,
                                      _u32p, _f32p]
        L.ref_layer_forward.argtypes = [C.c_void_p, _sz, _f32p, C.c_uint32, _u32p, _f32p, C.c_int, _f32p, C.c_int]

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.L.ref_last_error().decode())

    def mt64_draw(self, seed, n):
        out = np.empty(n, np.uint64)
        self.L.ref_mt64_draw(seed, n, out)
        return out

    def uniform01(self, seed, n):
        out = np.empty(n, np.float64)
        self.L.ref_uniform01(seed, n, out)
        return out

    def random_expert(self, d, ff, seed):
        wg, wu, wd = (np.empty(d * ff, np.float32) for _ in range(3))
        self._check(self.L.ref_random_expert(d, ff, seed, wg, wu, wd))
        return wg, wu, wd

    def random_balanced_partition(self, n, n_sub, seed):
        out = np.empty(n, np.uint32)
        self._check(self.L.ref_random_balanced_partition(n, n_sub, seed, out))
        return out

    # -- calibration --------------------------------------
    def collect_activation_matrix(self, d, ff, wg, wu, wd, x):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty((x.shape[0], ff), np.float32)
        self._check(self.L.ref_collect_activation_matrix(d, ff, wg, wu, wd, x.shape[0], x.reshape(-1), out.reshape(-1)))
        return out

    def binarize_topk(self, act, k_a):
        act = np.ascontiguousarray(act, np.float32)
        bits = np.empty(act.shape, np.uint8)
        self._check(self.L.ref_binarize_topk(act.reshape(-1), act.shape[0], act.shape[1], k_a, bits.ctypes.data))
        return bits

    def coactivation(self, bits, k_a):
        bits = np.ascontiguousarray(bits, np.uint8)
        co = np.empty((bits.shape[1], bits.shape[1]), np.uint32)
        self._check(self.L.ref_coactivation(bits.ctypes.data, bits.shape[0], bits.shape[1], k_a, co.reshape(-1)))
        return co

    def save_activation_matrix(self, path, act):
        act = np.ascontiguousarray(act, np.float32)
        self._check(self.L.ref_save_activation_matrix(str(path).encode(), act.shape[0], act.shape[1], act.reshape(-1)))

    def load_activation_matrix(self, path):
        r, c = _sz(), _sz()
        self._check(self.L.ref_load_activation_matrix(str(path).encode(), C.byref(r), C.byref(c), None))
        out = np.empty((r.value, c.value), np.float32)
        self._check(self.L.ref_load_activation_matrix(str(path).encode(), C.byref(r), C.byref(c), out.ctypes.data))
        return out

    def offload_replay(self, n_units, capacity, steps):
        """Per-step miss counts of cache_step (inc/offload.hpp:202-255) over
        the request sets `steps` (each ascending), cold start."""
        off = np.zeros(len(steps) + 1, np.uint32)
        for i, st in enumerate(steps):
            off[i + 1] = off[i] + len(st)
        ids = np.ascontiguousarray(np.concatenate([np.asarray(st, np.uint32) for st in steps]), np.uint32)
        out = np.zeros(len(steps), np.uint64)
        self._check(self.L.ref_offload_replay(n_units, capacity, len(steps), off, ids, out))
        return out

    def default_binarize_count(self, cols):
        return int(self.L.ref_default_binarize_count(cols))

    def random_matrix(self, rows, cols, seed):
        out = np.empty((rows, cols), np.float32)
        self._check(self.L.ref_random_matrix(rows, cols, seed, out.reshape(-1)))
        return out

    def planted_cluster(self, tokens, n_sub, group, seed):
        m = np.empty((tokens, n_sub * group), np.float32)
        a = np.empty(n_sub * group, np.uint32)
        self._check(self.L.ref_planted_cluster(tokens, n_sub, group, seed, m.reshape(-1), a))
        return m, a

    def select_gate_neurons(self, co, assignment, n_sub, r):
        co = np.ascontiguousarray(co, np.uint32)
        a = np.ascontiguousarray(assignment, np.uint32)
        off = np.zeros(n_sub + 1, np.uint32)
        ids = np.zeros(max(a.size, 1), np.uint32)
        self._check(self.L.ref_select_gate_neurons(co.reshape(-1), a.size, n_sub, a, r, off, ids))
        return [ids[off[q]:off[q + 1]].tolist() for q in range(n_sub)]

    def gating_fidelity(self, act, assignment, n_sub, gates, r, k):
        act = np.ascontiguousarray(act, np.float32)
        a = np.ascontiguousarray(assignment, np.uint32)
        off = np.zeros(n_sub + 1, np.uint32)
        for q, g in enumerate(gates):
            off[q + 1] = off[q] + len(g)
        ids = np.ascontiguousarray(np.concatenate([np.asarray(g, np.uint32) for g in gates]), np.uint32)
        out = C.c_double()
        self._check(self.L.ref_gating_fidelity(act.reshape(-1), act.shape[0], act.shape[1], n_sub, a, r, off, ids, k,
                                               C.byref(out)))
        return out.value

    def perf_table_eval(self, path, batch, k):
        """load_perf_table (with its grid / monotonicity validation) + eval_cost."""
        cost, nb, nk = C.c_double(), _sz(), _sz()
        self._check(self.L.ref_perf_table_eval(str(path).encode(), batch, k, C.byref(cost), C.byref(nb), C.byref(nk)))
        return cost.value, nb.value, nk.value

    def contiguous_partition(self, n, n_sub):
        out = np.empty(max(n, 1), np.uint32)
        self._check(self.L.ref_contiguous_partition(n, n_sub, out))
        return out[:n]

    def validate_partition(self, n_sub, assignment):
        a = np.ascontiguousarray(assignment, np.uint32)
        self._check(self.L.ref_validate_partition(n_sub, len(a), a if len(a) else np.zeros(1, np.uint32)))

    def toy_ffn_forward(self, d, ff, wg, wu, wd, x):
        y = np.empty(d, np.float32)
        a = np.empty(ff, np.float32)
        self._check(self.L.ref_toy_ffn_forward(d, ff, wg, wu, wd, np.ascontiguousarray(x, np.float32), len(x), y, a))
        return y, a

    def shared_expert_forward(self, d, ff_sh, wg, wu, wd, gate, x):
        """Restated shared (always-on) expert, Qwen1.5-MoE style (
        no reference counterpart): sigmoid(x . gate) * toy_ffn_forward(x)
        (inc/expert.hpp:79-96), gate dot product in double, i ascending.
        Returns float64 (T, d); gate None = weight 1."""
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty(x.shape, np.float64)
        for t in range(x.shape[0]):
            y, _ = self.toy_ffn_forward(d, ff_sh, wg, wu, wd, x[t])
            s = 1.0 if gate is None else 1.0 / (1.0 + np.exp(-np.dot(x[t].astype(np.float64), gate.astype(np.float64))))
            out[t] = s * y.astype(np.float64)
        return out

    def partitioned_forward(self, d, ff, wg, wu, wd, n_sub, assignment, x, active):
        y = np.empty(d, np.float32)
        act = np.ascontiguousarray(np.asarray(active, np.uint32).reshape(-1))
        n_act = act.size
        if n_act == 0:
            act = np.zeros(1, np.uint32)
        x = np.ascontiguousarray(x, np.float32)
        self._check(self.L.ref_partitioned_forward(d, ff, wg, wu, wd, n_sub, len(assignment),
                                                   np.ascontiguousarray(assignment, np.uint32), x, len(x), act, n_act, y))
        return y

    def proxy_scores(self, act, gates, r):
        off, ids = _csr(gates)
        out = np.empty(len(gates), np.float64)
        self._check(self.L.ref_proxy_scores(np.ascontiguousarray(act, np.float32), len(act), len(gates), r, off,
                                            ids if ids.size else np.zeros(1, np.uint32), out))
        return out

    def select_topk(self, scores, k):
        s = np.ascontiguousarray(scores, np.float64)
        out = np.empty(max(k, 1), np.uint32)
        self._check(self.L.ref_select_topk(s, len(s), k, out))
        return out[:k]

    def save_toy_expert(self, path, d, ff, wg, wu, wd):
        self._check(self.L.ref_save_toy_expert(str(path).encode(), d, ff, wg, wu, wd))

    def load_toy_expert(self, path):
        d, ff = _sz(), _sz()
        self._check(self.L.ref_load_toy_expert(str(path).encode(), C.byref(d), C.byref(ff), None, None, None))
        wg, wu, wd = (np.empty(d.value * ff.value, np.float32) for _ in range(3))
        self._check(self.L.ref_load_toy_expert(str(path).encode(), C.byref(d), C.byref(ff),
                                               wg.ctypes.data, wu.ctypes.data, wd.ctypes.data))
        return d.value, ff.value, wg, wu, wd

    def append_partition_doc(self, path, expert_id, n_sub, assignment, cost=0.0, seed=0, truncate=False):
        a = np.ascontiguousarray(assignment, np.uint32)
        self._check(self.L.ref_append_partition_doc(str(path).encode(), expert_id, n_sub, len(a), a, cost, seed,
                                                    int(truncate)))

    def append_partition_gates_doc(self, path, expert_id, n_sub, assignment, r, gates, truncate=False):
        a = np.ascontiguousarray(assignment, np.uint32)
        off, ids = _csr(gates)
        self._check(self.L.ref_append_partition_gates_doc(str(path).encode(), expert_id, n_sub, len(a), a, r, off,
                                                          ids, int(truncate)))

    def read_partition_doc(self, path, index):
        eid, ns, n, nd = C.c_uint64(), C.c_uint32(), _sz(), _sz()
        self._check(self.L.ref_read_partition_doc(str(path).encode(), index, C.byref(eid), C.byref(ns), C.byref(n),
                                                  None, C.byref(nd)))
        a = np.empty(n.value, np.uint32)
        self._check(self.L.ref_read_partition_doc(str(path).encode(), index, C.byref(eid), C.byref(ns), C.byref(n),
                                                  a.ctypes.data, C.byref(nd)))
        return eid.value, ns.value, a, nd.value


class RefLayer:
    """Reference CPU layer: verbatim partitioned_forward calls (oracle/_ref)."""

    def __init__(self, ref: RefLib, experts, assignments, S):
        self.ref = ref
        E = len(experts)
        d = None
        ff = assignments[0].size
        self.d_ff = ff
        self._keep = [experts, assignments]
        wg = _ptr_array([e[0] for e in experts], None)
        wu = _ptr_array([e[1] for e in experts], None)
        wd = _ptr_array([e[2] for e in experts], None)
        asg = _ptr_array([np.ascontiguousarray(a, np.uint32) for a in assignments], None)
        self._keep.append(asg)
        d = experts[0][0].size // ff
        self.d = d
        self.h = ref.L.ref_layer_create(E, S, d, ff, wg, wu, wd, asg)

    def route(self, x, wr, k, k_max, mode, k_per_token=None):
        x = np.ascontiguousarray(x, np.float32)
        T = x.shape[0]
        sel = np.empty(T * k_max, np.uint32)
        w = np.empty(T * k_max, np.float32)
        kpt = np.ascontiguousarray(k_per_token, np.uint32) if k_per_token is not None else None
        self.ref._check(self.ref.L.ref_layer_route(self.h, T, x.reshape(-1), np.ascontiguousarray(wr, np.float32).reshape(-1),
                                                   kpt.ctypes.data if kpt is not None else None, k, k_max, mode, sel, w))
        return sel.reshape(T, k_max), w.reshape(T, k_max)

    def forward(self, x, sel, w, mode, nthreads=1):
        x = np.ascontiguousarray(x, np.float32)
        T = x.shape[0]
        y = np.empty((T, self.d), np.float32)
        sel = np.ascontiguousarray(sel, np.uint32)
        self.ref._check(self.ref.L.ref_layer_forward(self.h, T, x.reshape(-1), sel.shape[1], sel.reshape(-1),
                                                     np.ascontiguousarray(w, np.float32).reshape(-1), mode,
                                                     y.reshape(-1), nthreads))
        return y

    def __del__(self):
        try:
            self.ref.L.ref_layer_destroy(self.h)
        except Exception:
            pass


def have_ref() -> bool:
    return REF_SO.exists()


# ---- numpy restatements of the calibration helpers (the checker where the
# reference build is absent; pinned against it in tests/test_oracle.py) ----

def np_binarize_topk(act, k_a):
    """binarize_topk (inc/activation.hpp:213-240): per row the k_a largest
    magnitudes, ties broken by lower column index."""
    act = np.asarray(act, np.float32)
    rows, cols = act.shape
    if not 1 <= k_a <= cols:
        raise OracleError(1, f"k_a = {k_a} out of range [1, {cols}]")
    bits = np.zeros((rows, cols), np.uint8)
    idx = np.arange(cols)
    for r in range(rows):
        order = np.lexsort((idx, -act[r].astype(np.float64)))
        bits[r, order[:k_a]] = 1
    return bits


def np_coactivation(bits):
    """coactivation (inc/activation.hpp:242-266): C = B^T B over the 0/1 mask."""
    b = np.asarray(bits, np.int64)
    return (b.T @ b).astype(np.uint32)
