"""Calibration tools around the layer, all compute on the GPU
through the C-ABI (libmoeprism_b200.so):

  collect_activations <- collect_activation_matrix (inc/expert.hpp:137-151)
  binarize_topk       <- binarize_topk             (inc/activation.hpp:213-240)
  coactivation        <- coactivation              (inc/activation.hpp:242-266)
  select_gate_neurons <- select_gate_neurons       (inc/gating.hpp:72-103)
  gating_fidelity     <- gating_fidelity           (inc/gating.hpp:149-174)
  write_mpam/read_mpam<- save_/load_activation_matrix (inc/io.hpp:147-200)
  measure_perf_table  -> the "batch,k,latency_s" CSV that load_perf_table
                         (inc/perfmodel.hpp:122-201) reads: the measured cost
                         C(|Q_m|, m) of the QoS scheduler

  python -m paper_2510_19366_b200.calibrate perf-table --out perf.csv
"""
from __future__ import annotations

import argparse
import ctypes as C
import math
import sys
from typing import Iterable, List, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import check


def _torch():
    import torch
    return torch


def _stream(stream=None):
    torch = _torch()
    return torch.cuda.current_stream().cuda_stream if stream is None else getattr(stream, "cuda_stream", stream)


def collect_activations(layer, e: int, x, stream=None):
    """|a| of expert e for every calibration row of x (B x d cuda tensor of the
    layer dtype): B x d_ff fp32, original neuron order."""
    torch = _torch()
    B = x.shape[0]
    act = torch.empty((B, layer.ff), dtype=torch.float32, device=x.device)
    check(_lib.load().mp_layer_collect_activations(layer.h, e, x.data_ptr(), B, act.data_ptr(), _stream(stream)))
    return act


def binarize_topk(act, k_a: int, stream=None):
    """Per row the k_a largest magnitudes -> 1 (ties: lower column), uint8."""
    torch = _torch()
    act = act.contiguous()
    rows, cols = act.shape
    bits = torch.empty((rows, cols), dtype=torch.uint8, device=act.device)
    check(_lib.load().mp_binarize_topk(act.data_ptr(), rows, cols, k_a, bits.data_ptr(), _stream(stream)))
    return bits


def coactivation(bits, stream=None):
    """co[i][j] = #rows with bits i and j set (cols x cols, int64 view of u32)."""
    torch = _torch()
    bits = bits.contiguous()
    rows, cols = bits.shape
    co = torch.empty((cols, cols), dtype=torch.int32, device=bits.device)
    check(_lib.load().mp_coactivation(bits.data_ptr(), rows, cols, co.data_ptr(), _stream(stream)))
    return co


def select_gate_neurons(co, assignment, n_sub: int, r: int, stream=None):
    """select_gate_neurons (inc/gating.hpp:72-103) on a device co-activation
    matrix; returns the per-sub-expert ascending gate neuron lists."""
    a = np.ascontiguousarray(assignment, np.uint32)
    dim = a.size
    off = np.zeros(n_sub + 1, np.uint32)
    ids = np.zeros(max(dim, 1), np.uint32)
    check(_lib.load().mp_select_gate_neurons(co.data_ptr(), dim, n_sub, a.ctypes.data, r, off.ctypes.data,
                                            ids.ctypes.data, _stream(stream)))
    return [ids[off[q]:off[q + 1]].tolist() for q in range(n_sub)]


def gating_fidelity(act, assignment, n_sub: int, gates, k: int, stream=None) -> float:
    """gating_fidelity (inc/gating.hpp:149-174) over a device activation matrix."""
    a = np.ascontiguousarray(assignment, np.uint32)
    off = np.zeros(n_sub + 1, np.uint32)
    for q, g in enumerate(gates):
        off[q + 1] = off[q] + len(g)
    ids = np.ascontiguousarray(np.concatenate([np.asarray(g, np.uint32) for g in gates]), np.uint32)
    out = C.c_double()
    act = act.contiguous()
    check(_lib.load().mp_gating_fidelity(act.data_ptr(), act.shape[0], act.shape[1], n_sub, a.ctypes.data,
                                        off.ctypes.data, ids.ctypes.data, k, C.byref(out), _stream(stream)))
    return out.value


def write_mpam(path, act: np.ndarray):
    a = np.ascontiguousarray(act, np.float32)
    check(_lib.load().mp_format_write_mpam(str(path).encode(), a.shape[0], a.shape[1], a.ctypes.data))


def read_mpam(path) -> np.ndarray:
    L = _lib.load()
    r, c = C.c_uint32(), C.c_uint32()
    check(L.mp_format_read_mpam(str(path).encode(), C.byref(r), C.byref(c), None))
    out = np.empty((r.value, c.value), np.float32)
    check(L.mp_format_read_mpam(str(path).encode(), C.byref(r), C.byref(c), out.ctypes.data))
    return out


# ---------------------------------------------------------------- perf table

def measure_perf_table(layer, batches: Sequence[int], ks: Sequence[int], steps: int = 20, warmup: int = 3,
                       seed: int = 77) -> List[Tuple[int, int, float]]:
    """Layer-forward latency (seconds, CUDA events, inputs resident) on the
    batch x k grid, returned as (batch, k, latency_s) cells satisfying the
    reference table's monotonicity (inc/perfmodel.hpp:63-72): latency must not
    decrease along either axis, so measurement noise below the previous cell
    is lifted to it (the running-max envelope; the raw value is never lowered)."""
    torch = _torch()
    from .layer import synth_fill
    raw = {}
    for b in batches:
        x = synth_fill(torch.empty((b, layer.d), dtype=layer.torch_dtype, device="cuda"), seed + b, 1.0)
        y = torch.empty_like(x)
        for k in ks:
            for _ in range(warmup):
                layer.forward(x, k=k, y=y)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(steps):
                layer.forward(x, k=k, y=y)
            e1.record()
            torch.cuda.synchronize()
            raw[(b, k)] = e0.elapsed_time(e1) / steps / 1e3
    return monotone_cells(raw, batches, ks)


def monotone_cells(raw, batches, ks) -> List[Tuple[int, int, float]]:
    bs, kk = sorted(set(batches)), sorted(set(ks))
    lat = np.array([[raw[(b, k)] for k in kk] for b in bs], np.float64)
    lat = np.maximum.accumulate(np.maximum.accumulate(lat, axis=0), axis=1)
    return [(b, k, float(lat[i, j])) for i, b in enumerate(bs) for j, k in enumerate(kk)]


def write_perf_table(path, cells: Iterable[Tuple[int, int, float]]):
    """CSV, header 'batch,k,latency_s' (proj/README.md:126-129)."""
    with open(path, "w") as f:
        f.write("batch,k,latency_s\n")
        for b, k, s in cells:
            if not (s > 0 and math.isfinite(s)):
                raise ValueError(f"latency of cell ({b}, {k}) must be positive and finite")
            f.write(f"{int(b)},{int(k)},{s:.9g}\n")


def _main(argv=None):
    ap = argparse.ArgumentParser(prog="python -m paper_2510_19366_b200.calibrate")
    sub = ap.add_subparsers(dest="cmd", required=True)
    pt = sub.add_parser("perf-table", help="measure the Mixtral-shape layer and write batch,k,latency_s")
    pt.add_argument("--out", required=True)
    pt.add_argument("--batches", default="64,256,1024,4096")
    pt.add_argument("--ks", default="1,2,4,8,16")
    pt.add_argument("--steps", type=int, default=20)
    args = ap.parse_args(argv)
    sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parent.parent))
    import bench
    batches = [int(v) for v in args.batches.split(",")]
    ks = [int(v) for v in args.ks.split(",")]
    layer, _ = bench.build_layer(0, max(batches), max(ks))
    cells = measure_perf_table(layer, batches, ks, steps=args.steps)
    write_perf_table(args.out, cells)
    layer.close()
    print(f"wrote {len(cells)} cells to {args.out}")


if __name__ == "__main__":
    _main()
