#!/usr/bin/env python
"""bench.py -- MoE-Prism sub-expert MoE-layer forward on B200.

Metric (BASELINE.json): MoE-layer tokens/sec vs active sub-experts k, with the
tensor-core / HBM roofline fraction.  Workload (BASELINE configs[1], SURVEY
8(d) C2): Mixtral-8x7B layer shape, bf16, d=4096, ffn=14336, 8 experts x 8
sub-experts (w=1792), 4096 tokens per GPU, random-init weights from the
counter-based synthetic stream.  A step = one layer forward over the 4096
tokens (router -> bucket -> dispatch -> grouped SwiGLU GEMMs -> combine).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--k 8] [--impl reference]

N>1 runs under torchrun (one process per GPU, NCCL).  Timing: W warm-up
steps, then K steps bracketed by barrier + cuda synchronize, CUDA events on
the launching stream, max over ranks.  L2: inputs rotate over 8 x buffers
(268 MB) and the weights are 2.8 GB, both far above the 126 MB L2.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "MoE-layer tokens/sec vs active sub-experts k (1/2/4/8 B200); % TC/HBM roofline"
E, S, D, FF = 8, 8, 4096, 14336
W_SUB = FF // S
N_XBUF = 8


def peaks():
    p = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        j = json.loads(f.read_text())
        p.update({k: j[k] for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained") if k in j})
        p["source"] = "measured"
    return p


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.samples, self.proc, self.thread = index, [], None, None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 8:
                self.samples.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({n for s in self.samples for n, v in zip(names, s[4:8]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples),
                "power_w_max": max((float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()),
                                   default=None)}


def dist_setup(n_gpus, force=False):
    """force: a 1-rank NCCL process group even without torchrun (exercises the
    multi-rank code path -- barriers, max over ranks, the NCCL exchange -- on
    one GPU)."""
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif force:
        import socket
        import torch.distributed as dist
        torch.cuda.set_device(0)
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def _dist_on():
    import torch.distributed as dist
    return dist.is_available() and dist.is_initialized()


def barrier(world):
    if _dist_on():
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v, world):
    if not _dist_on():
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def build_layer(local, T, k_max):
    import torch
    from paper_2510_19366_b200 import MoeLayer, synth_fill
    L = MoeLayer(E, S, D, FF, dtype="bf16", router="linear", weights="softmax_renorm", k_max=k_max, max_tokens=T,
                 device=local)
    buf = [torch.empty(D * FF, dtype=torch.float32, device="cuda") for _ in range(3)]
    for e in range(E):
        for m, (seed, scale) in enumerate(((100 + 3 * e, 1 / math.sqrt(D)), (101 + 3 * e, 1 / math.sqrt(D)),
                                           (102 + 3 * e, 1 / math.sqrt(FF)))):
            synth_fill(buf[m], seed, scale)
        L.set_partition(e, balanced_partition(FF, S, 6000 + e))
        L.load_expert(e, *buf)
    del buf
    wr = torch.empty(D * E * S, dtype=torch.float32, device="cuda")
    synth_fill(wr, 7, 1 / math.sqrt(D))
    L.set_router(wr)
    xs = []
    for i in range(N_XBUF):
        x = torch.empty((T, D), dtype=torch.bfloat16, device="cuda")
        synth_fill(x, 11 + 1000 * i, 1.0)
        xs.append(x)
    torch.cuda.synchronize()
    return L, xs


def build_ep_layer(local, rank, world, T, k_max=16, transport="nccl", force_collectives=False):
    """Expert-parallel layer: E/world parent experts on this rank,
    the router replicated.  transport "nccl": the C++ host path (mp_ep_forward,
    the library's own NCCL communicator); "torch": the same protocol driven
    from Python with torch.distributed all-to-alls; "p2p": peer-memory stores."""
    import torch
    from paper_2510_19366_b200 import synth_fill
    from paper_2510_19366_b200.ep import CudaEpOps, ExpertParallelLayer, NcclExpertParallelLayer
    if (E * S) % world:
        raise SystemExit(f"--gpus {world} must divide the {E * S} sub-experts")
    ops = CudaEpOps(E, S, D, FF, rank, world, dtype="bf16", k_max=k_max, max_tokens=T, device=local)
    buf = [torch.empty(D * FF, dtype=torch.float32, device="cuda") for _ in range(3)]
    for e in range(E):
        if not ops.owns(e):
            continue
        for m, (seed, scale) in enumerate(((100 + 3 * e, 1 / math.sqrt(D)), (101 + 3 * e, 1 / math.sqrt(D)),
                                           (102 + 3 * e, 1 / math.sqrt(FF)))):
            synth_fill(buf[m], seed, scale)
        ops.set_partition(e, balanced_partition(FF, S, 6000 + e))
        ops.load_expert(e, *buf)
    del buf
    wr = torch.empty(D * E * S, dtype=torch.float32, device="cuda")
    synth_fill(wr, 7, 1 / math.sqrt(D))
    ops.set_router(wr)
    xs = []
    for i in range(N_XBUF):
        x = torch.empty((T, D), dtype=torch.bfloat16, device="cuda")
        synth_fill(x, 11 + 1000 * i + 100000 * rank, 1.0)
        xs.append(x)
    torch.cuda.synchronize()
    if transport == "p2p":
        from paper_2510_19366_b200.ep import PeerExpertParallelLayer
        return PeerExpertParallelLayer(ops), ops, xs
    if transport == "torch":
        return ExpertParallelLayer(ops, force_collectives=force_collectives), ops, xs
    return NcclExpertParallelLayer(ops), ops, xs


def bench_stack_ep(pk, local, rank, world, n_layers=32, T=4096, ks=(2, 8), steps=10):
    """BASELINE configs[2] / SURVEY 8(d) C3: the Mixtral 32-layer MoE stack,
    expert-parallel over the ranks (E*S/world sub-experts of every layer per
    GPU, 90/world GB of weights), x_{l+1} = x_l + MoE_l(x_l) with the residual
    fused into the combine, T tokens per GPU (weak scaling).  Every layer runs
    through mp_ep_forward on one shared expert-parallel handle (one NCCL
    communicator); the layers' token scratch is shared (MP_LAYER_SHARED_SCRATCH)."""
    import ctypes as C
    import torch
    from paper_2510_19366_b200 import MoeLayer, _lib, synth_fill
    from paper_2510_19366_b200._lib import (MP_EP_RESIDUAL, MP_LAYER_EXPERTS_ONLY, MP_LAYER_ROUTER_ONLY,
                                            MP_LAYER_SHARED_SCRATCH, check)
    from paper_2510_19366_b200.layer import _ptr, _stream_handle
    lib = _lib.load()
    G = E * S
    per_rank = G // world
    first_e, last_e = per_rank * rank // S, (per_rank * (rank + 1) - 1) // S
    k_max = max(ks)
    routers, experts = [], []
    buf = [torch.empty(D * FF, dtype=torch.float32, device="cuda") for _ in range(3)]
    for l in range(n_layers):
        R = MoeLayer(E, S, D, FF, dtype="bf16", k_max=k_max, max_tokens=T, device=local,
                     flags=MP_LAYER_ROUTER_ONLY)
        X = MoeLayer(last_e - first_e + 1, S, D, FF, dtype="bf16", weights="softmax_renorm", k_max=k_max,
                     max_tokens=T * world, device=local, flags=MP_LAYER_EXPERTS_ONLY | MP_LAYER_SHARED_SCRATCH)
        for e in range(first_e, last_e + 1):
            for m, (seed, scale) in enumerate(((100 + 3 * e, 1 / math.sqrt(D)), (101 + 3 * e, 1 / math.sqrt(D)),
                                               (102 + 3 * e, 1 / math.sqrt(FF)))):
                synth_fill(buf[m], seed + 7919 * l, scale)
            X.set_partition(e - first_e, balanced_partition(FF, S, 6000 + e + 64 * l))
            X.load_expert(e - first_e, *buf)
        synth_fill(buf[0][:D * G], 7 + 7919 * l, 1 / math.sqrt(D))
        R.set_router(buf[0][:D * G])
        routers.append(R)
        experts.append(X)
    del buf
    ep = C.c_void_p()
    check(lib.mp_ep_create_subexpert(world, rank, per_rank, S, D, k_max, T, 1, local, C.byref(ep)))
    uid = (C.c_uint8 * 128)()
    if rank == 0:
        check(lib.mp_ep_nccl_unique_id(uid))
    if _dist_on():
        import torch.distributed as dist
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=0)
        uid = (C.c_uint8 * 128).from_buffer_copy(box[0])
    check(lib.mp_ep_nccl_init(ep, uid))
    xa = torch.empty((T, D), dtype=torch.bfloat16, device="cuda")
    synth_fill(xa, 11 + 100000 * rank, 1.0)
    xb = torch.empty_like(xa)
    out = []
    for k in ks:
        def step(i, k=k):
            x, y = xa, xb
            for R, X in zip(routers, experts):
                check(lib.mp_ep_forward(ep, R.h, X.h, _ptr(x), T, None, k, _ptr(y), MP_EP_RESIDUAL,
                                        _stream_handle(None)))
                x, y = y, x
        ms = time_steps(step, steps, 3, world)
        F = n_layers * 6.0 * D * W_SUB * T * k * world
        B = n_layers * (G * 3.0 * D * W_SUB * 2 + 2.0 * T * world * D * 2)
        r = roofline_fb(F, B, ms, {**pk, "bf16_tflops_sustained": pk["bf16_tflops_sustained"] * world,
                                   "hbm_gbs": pk["hbm_gbs"] * world})
        out.append({"k": k, "tokens_per_s": world * T / (ms * 1e-3), "ms_per_pass": ms, "roofline": r})
    lib.mp_ep_destroy(ep)
    for L in routers + experts:
        L.close()
    torch.cuda.synchronize()
    return {"workload": f"Mixtral-8x7B {n_layers}-layer MoE stack, expert-parallel over {world} GPU(s) (BASELINE "
                        f"configs[2]), {T} tokens per GPU (weak), residual fused, C++ NCCL transport "
                        "(mp_ep_forward), shared layer scratch",
            "weights_gb_per_gpu": n_layers * per_rank * 3 * D * W_SUB * 2 / 1e9, "sweep": out}


def balanced_partition(n, n_sub, seed):
    """testsupport::random_balanced_partition (tests/support.hpp:89-105): seeded
    Fisher-Yates (mt19937_64 + uniform_index) dealt round-robin."""
    import numpy as np
    rng = _MT64(seed)
    order = list(range(n))
    for i in range(n - 1, 0, -1):
        j = rng.uniform_index(i + 1)
        order[i], order[j] = order[j], order[i]
    a = np.empty(n, np.uint32)
    for i, o in enumerate(order):
        a[o] = i % n_sub
    return a


class _MT64:
    """std::mt19937_64 (fixture generation for the partition layout only)."""

    def __init__(self, seed):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.idx = 312

    def next(self):
        M = 0xFFFFFFFFFFFFFFFF
        if self.idx >= 312:
            mt = self.mt
            for i in range(312):
                x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                mt[i] = mt[(i + 156) % 312] ^ xa
            self.idx = 0
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000 & M
        y ^= (y << 37) & 0xFFF7EEE000000000 & M
        y ^= y >> 43
        return y & M

    def uniform_index(self, n):
        M = 0xFFFFFFFFFFFFFFFF
        limit = M - M % n
        while True:
            x = self.next()
            if x < limit:
                return x % n


def layer_roofline(T, k, ms, pk, touched_groups):
    """t_roofline = max(F / P_tc, B / BW); F = 6 d w T k expert flops,
    B = touched sub-expert weights (3 d w bf16 each) + x in + y out."""
    F = 6.0 * D * W_SUB * T * k
    B = touched_groups * 3.0 * D * W_SUB * 2 + 2.0 * T * D * 2
    t_tc = F / (pk["bf16_tflops_sustained"] * 1e12)
    t_hbm = B / (pk["hbm_gbs"] * 1e9)
    t_roof = max(t_tc, t_hbm)
    return {"bound": "tensor" if t_tc >= t_hbm else "hbm", "t_roofline_ms": t_roof * 1e3, "t_measured_ms": ms,
            "frac": (t_roof * 1e3) / ms, "tc_util": (F / (ms * 1e-3)) / (pk["bf16_tflops_sustained"] * 1e12),
            "peak_tflops": pk["bf16_tflops_sustained"], "peak_gbs": pk["hbm_gbs"], "peak_source": pk["source"]}


def roofline_fb(F, B, ms, pk):
    """t_roofline = max(F / P_tc, B / BW) for F flops and B algorithmic bytes."""
    t_tc = F / (pk["bf16_tflops_sustained"] * 1e12)
    t_hbm = B / (pk["hbm_gbs"] * 1e9)
    t_roof = max(t_tc, t_hbm)
    return {"bound": "tensor" if t_tc >= t_hbm else "hbm", "t_roofline_ms": t_roof * 1e3, "t_measured_ms": ms,
            "frac": (t_roof * 1e3) / ms, "tc_util": (F / (ms * 1e-3)) / (pk["bf16_tflops_sustained"] * 1e12)}


def bench_stack(pk, n_layers=32, T=4096, ks=(2, 8), steps=10):
    """BASELINE configs[2] / SURVEY 8(d) C3 on one GPU: a Mixtral-shape 32-layer
    MoE stack, x_{l+1} = x_l + MoE_l(x_l) (residual fused into each layer's
    combine), 32 independently seeded layers (90 GB of bf16 weights)."""
    import torch
    from paper_2510_19366_b200 import MoeLayer, synth_fill
    layers = []
    buf = [torch.empty(D * FF, dtype=torch.float32, device="cuda") for _ in range(3)]
    for l in range(n_layers):
        L = MoeLayer(E, S, D, FF, dtype="bf16", k_max=max(ks), max_tokens=T)
        for e in range(E):
            for m, (seed, scale) in enumerate(((100 + 3 * e, 1 / math.sqrt(D)), (101 + 3 * e, 1 / math.sqrt(D)),
                                               (102 + 3 * e, 1 / math.sqrt(FF)))):
                synth_fill(buf[m], seed + 7919 * l, scale)
            L.set_partition(e, balanced_partition(FF, S, 6000 + e + 64 * l))
            L.load_expert(e, *buf)
        synth_fill(buf[0][:D * E * S], 7 + 7919 * l, 1 / math.sqrt(D))
        L.set_router(buf[0][:D * E * S])
        L.set_residual(True)
        layers.append(L)
    del buf
    xa = torch.empty((T, D), dtype=torch.bfloat16, device="cuda")
    synth_fill(xa, 11, 1.0)
    xb = torch.empty_like(xa)
    out = []
    for k in ks:
        def step(i, k=k):
            x, y = xa, xb
            for L in layers:
                L.forward(x, k=k, y=y)
                x, y = y, x
        ms = time_steps(step, steps, 3, 1)
        F = n_layers * 6.0 * D * W_SUB * T * k
        B = n_layers * (E * S * 3.0 * D * W_SUB * 2 + 2.0 * T * D * 2)
        out.append({"k": k, "tokens_per_s": T / (ms * 1e-3), "ms_per_pass": ms,
                    "roofline": roofline_fb(F, B, ms, pk)})
    for L in layers:
        L.close()
    torch.cuda.synchronize()
    return {"workload": f"Mixtral-8x7B {n_layers}-layer MoE stack on 1 GPU (BASELINE configs[2] at N=1), "
                        f"{T} tokens, residual x + MoE(x) fused, independently seeded layers",
            "weights_gb": n_layers * E * S * 3 * D * W_SUB * 2 / 1e9, "sweep": out}


QW = {"E": 60, "S": 4, "d": 2048, "ff": 1408, "ff_sh": 5632}


def build_qwen_layer(max_tokens):
    """The Qwen1.5-MoE-A2.7B-shape layer of BASELINE configs[3] (random init,
    counter-based stream): 60 experts x 4 sub-experts + the shared expert."""
    import torch
    from paper_2510_19366_b200 import MoeLayer, synth_fill
    q = QW
    Eq, Sq, d, ff, ffs = q["E"], q["S"], q["d"], q["ff"], q["ff_sh"]
    L = MoeLayer(Eq, Sq, d, ff, dtype="bf16", k_max=16, max_tokens=max_tokens)
    buf = [torch.empty(d * ff, dtype=torch.float32, device="cuda") for _ in range(3)]
    for e in range(Eq):
        for m, (seed, scale) in enumerate(((300 + 3 * e, 1 / math.sqrt(d)), (301 + 3 * e, 1 / math.sqrt(d)),
                                           (302 + 3 * e, 1 / math.sqrt(ff)))):
            synth_fill(buf[m], seed, scale)
        L.set_partition(e, balanced_partition(ff, Sq, 6000 + e))
        L.load_expert(e, *buf)
    sh = [synth_fill(torch.empty(d * ffs, dtype=torch.float32, device="cuda"), 900 + m,
                     1 / math.sqrt(ffs if m == 2 else d)) for m in range(3)]
    gate = synth_fill(torch.empty(d, dtype=torch.float32, device="cuda"), 903, 1 / math.sqrt(d))
    L.set_shared_expert(*sh, gate=gate)
    wr = synth_fill(torch.empty(d * Eq * Sq, dtype=torch.float32, device="cuda"), 17, 1 / math.sqrt(d))
    L.set_router(wr)
    del buf, sh
    return L


def bench_qwen(pk, steps=30):
    """BASELINE configs[3] / SURVEY 8(d) C4: Qwen1.5-MoE-A2.7B layer shape (60
    experts x 4 sub-experts of w=352, E*S=240, plus the always-on shared expert
    ffn=5632 with a sigmoid gate), decode T=64 and prefill T=8192."""
    import numpy as np
    import torch
    from paper_2510_19366_b200 import MoeLayer, synth_fill
    q = QW
    Eq, Sq, d, ff, ffs = q["E"], q["S"], q["d"], q["ff"], q["ff_sh"]
    w = ff // Sq
    L = build_qwen_layer(8192)
    out = []
    for T in (64, 8192):
        xs = [synth_fill(torch.empty((T, d), dtype=torch.bfloat16, device="cuda"), 19 + 1000 * i, 1.0)
              for i in range(4)]
        y = torch.empty((T, d), dtype=torch.bfloat16, device="cuda")
        for k in (4, 8, 16):
            _, _, _, off = L.forward(xs[0], k=k, return_routing=True)
            touched = int((np.diff(off.cpu().numpy().view(np.uint32).astype(np.int64)) > 0).sum())
            ms = time_steps(lambda i, k=k: L.forward(xs[i % 4], k=k, y=y), steps, 3, 1)
            F = 6.0 * d * w * T * k + 6.0 * d * ffs * T
            B = touched * 3.0 * d * w * 2 + 3.0 * d * ffs * 2 + 2.0 * T * d * 2
            st = stage_profile([L], lambda x, kk, kpt, y=y: L.forward(x, k=kk, y=y), xs, k)
            # routed GEMMs against their bound (CUDA-event stage times on the
            # forward's stream; the shared expert runs concurrently on a side
            # stream, so these include its contention): TFLOP/s of 4 d w T k /
            # 2 d w T k at prefill, GB/s of the touched weights at decode
            gr = {}
            for name, fl, wb in (("gemm1", 4.0 * d * w * T * k, touched * 2.0 * d * w * 2),
                                 ("gemm2", 2.0 * d * w * T * k, touched * 1.0 * d * w * 2)):
                t = st.get(name, 0.0)
                if t <= 0:
                    continue
                if fl / (pk["bf16_tflops_sustained"] * 1e12) >= wb / (pk["hbm_gbs"] * 1e9):
                    a = fl / (t * 1e-3) / 1e12
                    gr[name] = {"bound": "tensor", "achieved": a, "unit": "TFLOP/s", "ms": t,
                                "frac": a / pk["bf16_tflops_sustained"]}
                else:
                    a = wb / (t * 1e-3) / 1e9
                    gr[name] = {"bound": "hbm", "achieved": a, "unit": "GB/s", "ms": t, "frac": a / pk["hbm_gbs"]}
            out.append({"tokens": T, "k": k, "tokens_per_s": T / (ms * 1e-3), "ms_per_step": ms,
                        "touched_subexperts": touched, "roofline": roofline_fb(F, B, ms, pk),
                        "stages_ms": st, "routed_gemm_roofline": gr})
        del xs
    L.close()
    torch.cuda.synchronize()
    return {"workload": "Qwen1.5-MoE-A2.7B layer shape bf16 (BASELINE configs[3]): d=2048, 60 experts x 4 "
                        "sub-experts (w=352, GEMM-padded to 384) + shared expert ffn=5632 (sigmoid gate); "
                        "flops/bytes counted at w=352", "sweep": out}


def bench_mixed_qos_32k(L32, pk, steps=10):
    """BASELINE configs[4] / SURVEY 8(d) C5 on one GPU: 32768 tokens with
    per-token elastic k from the 4 SLO tiers {2,4,8,16} (pmf .25/.35/.25/.15)."""
    import numpy as np
    import torch
    from paper_2510_19366_b200 import synth_fill
    T = 32768
    xs = [synth_fill(torch.empty((T, D), dtype=torch.bfloat16, device="cuda"), 5011 + i, 1.0) for i in range(2)]
    rng = np.random.default_rng(13)
    kpt = torch.from_numpy(rng.choice([2, 4, 8, 16], size=T, p=[0.25, 0.35, 0.25, 0.15]).astype(np.int32)).cuda()
    y = torch.empty((T, D), dtype=torch.bfloat16, device="cuda")
    ms = time_steps(lambda i: L32.forward(xs[i % 2], k_per_token=kpt, y=y), steps, 3, 1)
    kk = float(kpt.float().mean().item())
    F = 6.0 * D * W_SUB * T * kk
    B = E * S * 3.0 * D * W_SUB * 2 + 2.0 * T * D * 2
    del xs
    return {"workload": "mixed-QoS batch (BASELINE configs[4]) at N=1: 32768 tokens, Mixtral layer shape, "
                        "per-token k tiers {2,4,8,16} pmf {.25,.35,.25,.15} seed 13",
            "mean_k": kk, "tokens_per_s": T / (ms * 1e-3), "ms_per_step": ms, "roofline": roofline_fb(F, B, ms, pk)}


def bench_c1_gpu(pk, steps=50):
    """BASELINE configs[0] / SURVEY 8(d) C1 on the GPU: the toy layer (8 experts
    x 4 sub-experts, d=512, ffn=1024, k=4, 256 tokens), fp32 (reference-exact
    mode) and bf16, weights U(-1,1) from the counter-based stream."""
    import torch
    from paper_2510_19366_b200 import MoeLayer, synth_fill
    Ec, Sc, dc, ffc, Tc, kc = 8, 4, 512, 1024, 256, 4
    out = {}
    for dt in ("f32", "bf16"):
        L = MoeLayer(Ec, Sc, dc, ffc, dtype=dt, k_max=kc, max_tokens=Tc)
        buf = [torch.empty(dc * ffc, dtype=torch.float32, device="cuda") for _ in range(3)]
        for e in range(Ec):
            for m in range(3):
                synth_fill(buf[m], 5000 + 3 * e + m, 1.0)
            L.set_partition(e, balanced_partition(ffc, Sc, 6000 + e))
            L.load_expert(e, *buf)
        L.set_router(synth_fill(torch.empty(dc * Ec * Sc, dtype=torch.float32, device="cuda"), 7, 1 / math.sqrt(dc)))
        xs = [synth_fill(torch.empty((Tc, dc), dtype=L.torch_dtype, device="cuda"), 11 + i, 1.0) for i in range(4)]
        y = torch.empty((Tc, dc), dtype=L.torch_dtype, device="cuda")
        ms = time_steps(lambda i: L.forward(xs[i % 4], k=kc, y=y), steps, 3, 1)
        out[dt] = {"tokens_per_s": Tc / (ms * 1e-3), "ms_per_step": ms}
        L.close()
    return {"workload": "C1 toy layer (BASELINE configs[0]) on the GPU: 8 experts x 4 sub-experts, d=512, "
                        "ffn=1024, k=4, 256 tokens; fp32 = reference-exact fp64-accumulating SIMT path, "
                        "bf16 = tcgen05 path (launch-bound at this size)", **out}


def bench_proxy(pk, T=4096, k=8, r=4, steps=30):
    """the proxy-gate router at the Mixtral layer shape (r = 4
    gate neurons per sub-expert, E*S*r = 256 gate neurons): tensor-core
    gate/up columns with certified selection.  Route-only and full-layer
    times, and how many tokens the certification sent to the exact pass."""
    import numpy as np
    import torch
    from paper_2510_19366_b200 import MoeLayer, synth_fill
    L = MoeLayer(E, S, D, FF, dtype="bf16", router="proxy", k_max=16, max_tokens=T)
    buf = [torch.empty(D * FF, dtype=torch.float32, device="cuda") for _ in range(3)]
    rng = np.random.default_rng(21)
    for e in range(E):
        for m, (seed, scale) in enumerate(((100 + 3 * e, 1 / math.sqrt(D)), (101 + 3 * e, 1 / math.sqrt(D)),
                                           (102 + 3 * e, 1 / math.sqrt(FF)))):
            synth_fill(buf[m], seed, scale)
        part = balanced_partition(FF, S, 6000 + e)
        L.set_partition(e, part)
        L.load_expert(e, *buf)
        L.set_gates(e, r, [sorted(rng.choice(np.flatnonzero(part == s), r, replace=False).tolist())
                           for s in range(S)])
    del buf
    xs = [synth_fill(torch.empty((T, D), dtype=torch.bfloat16, device="cuda"), 11 + 1000 * i, 1.0) for i in range(4)]
    y = torch.empty((T, D), dtype=torch.bfloat16, device="cuda")
    ms_route = time_steps(lambda i: L.route(xs[i % 4], k=k), steps, 3, 1)
    resel, near = L.route_stats()
    ms_fwd = time_steps(lambda i: L.forward(xs[i % 4], k=k, y=y), steps, 3, 1)
    L.close()
    torch.cuda.synchronize()
    F = 3 * 2.0 * 2 * E * S * r * D * T  # three bf16 planes of the 2 E S r gate/up columns
    return {"workload": f"proxy-gate router, Mixtral layer shape, {E * S * r} gate neurons (r={r}), T={T}, k={k}",
            "route_ms": ms_route, "route_tokens_per_s": T / (ms_route * 1e-3), "route_tc_tflops": F / (ms_route * 1e-3) / 1e12,
            "forward_ms": ms_fwd, "forward_tokens_per_s": T / (ms_fwd * 1e-3),
            "reselected_exact": resel, "near_ties_lt_1e-6": near}


def bench_offload(T=16, k=2, cache_units=32, steps=20):
    """SURVEY 8(f).4 at the Mixtral shape: decode batches of T tokens on a
    layer whose packed weights live in pinned host memory, with a device
    cache of `cache_units` of the 64 sub-experts (LRU, cache_step semantics);
    misses are real host->device copies."""
    import time
    import torch
    L, xs = build_layer(0, T, k)
    L.enable_offload(cache_units)
    y = torch.empty((T, D), dtype=torch.bfloat16, device="cuda")
    for i in range(3):
        L.forward(xs[i % N_XBUF][:T], k=k, y=y)
    torch.cuda.synchronize()
    h0, m0, b0, _, _ = L.offload_stats()
    t0 = time.perf_counter()
    for i in range(steps):
        L.forward(xs[i % N_XBUF][:T], k=k, y=y)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    h1, m1, b1, _, _ = L.offload_stats()
    L.close()
    return {"workload": f"Mixtral-shape layer with weights offloaded to pinned host memory, device cache of "
                        f"{cache_units}/64 sub-experts (LRU), decode batches of {T} tokens, k={k}; wall clock "
                        "(each forward synchronises to read its bucket sizes)",
            "tokens_per_s": steps * T / dt, "ms_per_step": 1e3 * dt / steps,
            "hit_ratio": (h1 - h0) / max(1, (h1 - h0) + (m1 - m0)), "h2d_gb_per_s": (b1 - b0) / dt / 1e9,
            "h2d_mb_per_step": (b1 - b0) / steps / 1e6}


def bench_calibration(pk, B=4096, k_a=1434, steps=5):
    """SURVEY 8(f).2 on the GPU at the Mixtral expert shape: the activation
    profile of one expert on B calibration tokens (collect_activation_matrix),
    its top-k_a binarisation and the 14336 x 14336 co-activation counts."""
    import torch
    from paper_2510_19366_b200.calibrate import binarize_topk, coactivation, collect_activations
    L, xs = build_layer(0, B, 2)
    act = collect_activations(L, 0, xs[0])
    bits = binarize_topk(act, k_a)
    co = coactivation(bits)
    t_act = time_steps(lambda i: collect_activations(L, i % E, xs[i % N_XBUF]), steps, 2, 1)
    t_bin = time_steps(lambda i: binarize_topk(act, k_a), steps, 2, 1)
    t_co = time_steps(lambda i: coactivation(bits), steps, 2, 1)
    f_act = 4.0 * B * D * FF
    f_co = 2.0 * FF * FF * B
    out = {"workload": f"activation profile of one Mixtral expert (d=4096, ffn=14336) on {B} calibration tokens, "
                       f"top-{k_a} binarisation, {FF}x{FF} co-activation counts",
           "collect_ms": t_act, "collect_tflops": f_act / (t_act * 1e-3) / 1e12,
           "binarize_ms": t_bin, "binarize_gbs": B * FF * 5 / (t_bin * 1e-3) / 1e9,
           "coactivation_ms": t_co, "coactivation_tflops": f_co / (t_co * 1e-3) / 1e12,
           "peak_tflops": pk["bf16_tflops_sustained"]}
    del act, bits, co
    L.close()
    torch.cuda.synchronize()
    return out


def time_steps(fn, steps, warmup, world):
    import torch
    for i in range(warmup):
        fn(i)
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(steps):
        fn(i)
    e1.record(st)
    torch.cuda.synchronize()
    barrier(world)
    ms = e0.elapsed_time(e1) / steps
    return max_over_ranks(ms, world)


def stage_profile(layers, fwd, xs, k, reps=20, kpt=None):
    """Per-stage device time per step (CUDA events on the launching stream)."""
    import torch
    for L in layers:
        L.reset_stage_times()
        L.set_profiling(True)
    for i in range(reps):
        fwd(xs[i % len(xs)], k, kpt)
    torch.cuda.synchronize()
    out = {}
    for L in layers:
        L.set_profiling(False)
        for name, (ms, n) in L.stage_times().items():
            if n:
                out[name] = out.get(name, 0.0) + ms / reps
    return out


def kernel_roofline(stage_ms_per_step, T, k, pk, touched_groups):
    """The dominant kernel's roofline: gemm1 (SwiGLU) at TC-bound k, against the
    sustained bf16 peak; algorithmic flops = 4 d w T k per launch."""
    g1 = stage_ms_per_step.get("gemm1", 0.0)
    g2 = stage_ms_per_step.get("gemm2", 0.0)
    name = "gemm1" if g1 >= g2 else "gemm2"
    ms = max(g1, g2)
    flops = (4.0 if name == "gemm1" else 2.0) * D * W_SUB * T * k
    wbytes = touched_groups * (2 if name == "gemm1" else 1) * D * W_SUB * 2.0
    abytes = T * k * D * 2.0 + T * k * W_SUB * 2.0
    t_tc = flops / (pk["bf16_tflops_sustained"] * 1e12)
    t_hbm = (wbytes + abytes) / (pk["hbm_gbs"] * 1e9)
    traffic = None
    # DRAM bytes of the kernel per launch from the committed ncu --set full
    # capture of the same workload (tests/probes/ncu_summary.py)
    prof = ROOT / "profiles" / "ncu_summary_r02af.json"
    if prof.exists():
        try:
            j = json.loads(prof.read_text())
            traffic = j.get(name, {}).get(f"dram_bytes_k{k}")
        except Exception:
            traffic = None
    if t_tc >= t_hbm:
        ach = flops / (ms * 1e-3) / 1e12
        return {"kernel": name, "bound": "tensor", "achieved": ach, "peak": pk["bf16_tflops_sustained"],
                "unit": "TFLOP/s", "frac": ach / pk["bf16_tflops_sustained"], "traffic": traffic,
                "algorithmic_flops": flops, "launch_ms": ms, "peak_source": pk["source"] + " sustained"}
    ach = (wbytes + abytes) / (ms * 1e-3) / 1e9
    return {"kernel": name, "bound": "hbm", "achieved": ach, "peak": pk["hbm_gbs"], "unit": "GB/s",
            "frac": ach / pk["hbm_gbs"], "traffic": traffic, "algorithmic_bytes": wbytes + abytes, "launch_ms": ms,
            "peak_source": pk["source"]}


def stage_rooflines(stage_ms, T, k, pk):
    """Every stage against its bound (SURVEY 8(d) per-kernel bytes): router,
    dispatch and combine in HBM GB/s of algorithmic bytes, the two GEMMs in
    TFLOP/s -- the north_star's "tensor-pipe utilisation for the GEMMs and
    achieved HBM GB/s for routing, permute and combine, each against peak".
    Stage times are CUDA-event times per step on the forward's stream."""
    G = E * S
    b = 2.0  # bf16
    algo = {
        "router": ("hbm", T * D * b + 4.0 * D * G + 8.0 * T * k),   # x in, W_r, sel/w out
        "dispatch": ("hbm", T * D * b + T * k * D * b),             # x in, k bucket rows out
        "combine": ("hbm", T * k * D * b + 4.0 * T * k + T * D * b),  # partials + weights in, y out
        "gemm1": ("tensor", 4.0 * D * W_SUB * T * k),
        "gemm2": ("tensor", 2.0 * D * W_SUB * T * k),
    }
    out = {}
    for name, (bound, work) in algo.items():
        ms = stage_ms.get(name)
        if not ms:
            continue
        if bound == "hbm":
            ach = work / (ms * 1e-3) / 1e9
            out[name] = {"bound": "hbm", "ms": ms, "algorithmic_bytes": work, "achieved": ach, "unit": "GB/s",
                         "frac": ach / pk["hbm_gbs"]}
        else:
            ach = work / (ms * 1e-3) / 1e12
            out[name] = {"bound": "tensor", "ms": ms, "algorithmic_flops": work, "achieved": ach,
                         "unit": "TFLOP/s", "frac": ach / pk["bf16_tflops_sustained"]}
    return out


def cpu_reference_sample(k, T_sample, nthreads, seed_tokens=11):
    """The reference CPU path (oracle/_ref = reference headers compiled
    verbatim): router restated in double + select_topk_subexperts +
    partitioned_forward per selected sub-expert, std::thread over tokens."""
    import numpy as np
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import Oracle, RefLayer, RefLib, have_ref
    orc = Oracle()
    if have_ref():
        ref = RefLib()
        kind = "reference"
    else:
        ref = None
        kind = "port"
    experts = [(orc.synth(100 + 3 * e, D * FF, 1 / math.sqrt(D)), orc.synth(101 + 3 * e, D * FF, 1 / math.sqrt(D)),
                orc.synth(102 + 3 * e, D * FF, 1 / math.sqrt(FF))) for e in range(E)]
    parts = [orc.random_balanced_partition(FF, S, 6000 + e) for e in range(E)]
    wr = orc.synth(7, D * E * S, 1 / math.sqrt(D))
    x = orc.synth(seed_tokens, T_sample * D, 1.0).reshape(T_sample, D)
    if kind == "reference":
        rl = RefLayer(ref, experts, parts, S)
        t0 = time.perf_counter()
        sel, w = rl.route(x, wr, k, 16, 1)
        y = rl.forward(x, sel, w, 1, nthreads=nthreads)
        dt = time.perf_counter() - t0
    else:
        t0 = time.perf_counter()
        logits = orc.router_logits(x, wr, T_sample, D, E * S)
        sel, w, _ = orc.route(logits, k, 16, 1)
        y = orc.layer_forward(experts, parts, S, x, sel, w, 1, nthreads=nthreads)
        dt = time.perf_counter() - t0
    assert np.isfinite(y).all()
    return T_sample / dt, kind, dt


def cpu_reference_c1(nthreads):
    """BASELINE configs[0] / SURVEY 8(d) C1 timed in full on the reference CPU
    path: toy layer fp32, 8 experts x 4 sub-experts, d=512, ffn=1024, k=4,
    256 tokens (reference fixtures: random_expert, random_balanced_partition,
    W_r = U(-1,1)/sqrt(d), x = U(-1,1))."""
    import numpy as np
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import Oracle, RefLayer, RefLib, have_ref
    orc = Oracle()
    Ec, Sc, dc, ffc, Tc, kc = 8, 4, 512, 1024, 256, 4
    experts = [orc.random_expert(dc, ffc, 5000 + e) for e in range(Ec)]
    parts = [orc.random_balanced_partition(ffc, Sc, 6000 + e) for e in range(Ec)]
    wr = orc.uniform_pm1(7, dc * Ec * Sc, 1.0 / math.sqrt(dc))
    x = orc.uniform_pm1(11, Tc * dc).reshape(Tc, dc)
    t0 = time.perf_counter()
    if have_ref():
        rl = RefLayer(RefLib(), experts, parts, Sc)
        sel, w = rl.route(x, wr, kc, kc, 1)
        y = rl.forward(x, sel, w, 1, nthreads=nthreads)
        kind = "reference"
    else:
        logits = orc.router_logits(x, wr, Tc, dc, Ec * Sc)
        sel, w, _ = orc.route(logits, kc, kc, 1)
        y = orc.layer_forward(experts, parts, Sc, x, sel, w, 1, nthreads=nthreads)
        kind = "port"
    dt = time.perf_counter() - t0
    assert np.isfinite(y).all()
    return {"value": Tc / dt, "unit": "tokens/s", "cores": nthreads, "kind": kind, "seconds": dt,
            "sample": "C1 toy layer in full: 256 tokens, k=4, 8x4 sub-experts, d=512, ffn=1024, fp32"}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference_arm(args, world, rank):
    if rank != 0:
        return
    nthreads = os.cpu_count() or 1
    # a step = one bounded sample: one token per host thread (~1.45 s per
    # (token, sub-expert) reference call at this shape)
    T_sample = nthreads
    vals = []
    kind = None
    for i in range(args.warmup + args.steps):
        v, kind, dt = cpu_reference_sample(args.k, T_sample, nthreads, seed_tokens=11 + i)
        if i >= args.warmup:
            vals.append(v)
    v = statistics.mean(vals)
    cfg = workload_config(args, world)
    line = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * T_sample / v, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": cfg, "impl": "reference",
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": nthreads, "kind": kind,
                             "sample": f"{T_sample} tokens per step (one per thread), k={args.k}, "
                                       f"Mixtral layer shape fp32 weights; CPU {cpu_model()}"},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


def workload_config(args, world):
    return {"workload": "Mixtral-8x7B MoE layer shape bf16 (BASELINE configs[1]): d=4096, ffn=14336, "
                        "8 experts x 8 sub-experts (w=1792), linear fp32 router, softmax-renormalised top-k",
            "d_model": D, "d_ff": FF, "experts": E, "subexperts_per_expert": S, "tokens_per_gpu": args.tokens,
            "k": args.k, "global_tokens": args.tokens * world,
            "parallelism": ((f"ep{world} (experts sharded, "
                             + {"p2p": "peer-memory stores", "torch": "torch.distributed NCCL all-to-all",
                                "nccl": "C++ host, NCCL all-to-allv (mp_ep_forward)"}[args.ep_transport] + ")")
                            if world > 1 or args.force_ep else "single"),
            "l2": f"x rotates over {N_XBUF} buffers ({N_XBUF * args.tokens * D * 2 / 1e6:.0f} MB) + 2.8 GB weights, "
                  "both > 126 MB L2"}


def use_ep_flag(args, world):
    return world > 1 or args.force_ep


_OUT = None


def emit(line):
    """The one JSON line on stdout (bench contract); everything else the
    process prints -- NCCL's version banner, library diagnostics -- goes to
    stderr (main() moves fd 1 there)."""
    print(json.dumps(line), file=_OUT or sys.stdout, flush=True)


def main():
    global _OUT
    sys.stdout.flush()
    _OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    sys.stdout = sys.stderr
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--tokens", type=int, default=4096)
    ap.add_argument("--sweep", default=",".join(str(k) for k in range(2, 17)))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--force-ep", action="store_true", help="run the expert-parallel path even at N=1 (loopback)")
    ap.add_argument("--force-dist", action="store_true",
                    help="N=1 with a 1-rank NCCL process group and the expert-parallel path through real NCCL "
                         "collectives (the multi-rank code path on one GPU)")
    ap.add_argument("--ep-transport", default="nccl", choices=["nccl", "torch", "p2p"],
                    help="N>1 token exchange: the C++ NCCL path (mp_ep_forward, default), the same protocol with "
                         "torch.distributed all-to-alls, or direct peer-memory stores (CUDA IPC / NVLink)")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the other BASELINE configs (Qwen shape, 32-layer stack, 32k mixed-QoS batch) "
                         "and the calibration timing")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.force_dist:
        args.force_ep = True
    world, rank, local = dist_setup(args.gpus, force=args.force_dist)
    if args.impl == "reference":
        run_reference_arm(args, world, rank)
        if _dist_on():
            import torch.distributed as dist
            dist.destroy_process_group()
        return

    import numpy as np
    import torch
    pk = peaks()
    T = args.tokens
    sweep = [int(v) for v in args.sweep.split(",") if v]
    use_ep = world > 1 or args.force_ep
    extras = not args.no_extras and world == 1 and not use_ep_flag(args, world)
    if not use_ep:
        L, xs = build_layer(local, max(T, 32768) if extras else T, k_max=16)
        xs = [x[:T] for x in xs] if extras and T < 32768 else xs
        layers = [L]

        def fwd(x, k, kpt, y=None):
            return L.forward(x, k=k, k_per_token=kpt, y=y)
    else:
        ep_layer, ops, xs = build_ep_layer(local, rank, world, T, transport=args.ep_transport,
                                           force_collectives=args.force_dist)
        layers = [ops.router, ops.local]

        def fwd(x, k, kpt, y=None):
            if args.ep_transport == "nccl":
                return ep_layer.forward(x, k=k, k_per_token=kpt, y=y)
            return ep_layer.forward(x, k=k, k_per_token=kpt)
    touched = E * S // world  # sub-experts whose weights this GPU streams (all receive tokens at 4096/GPU)

    def step(i, k=args.k, kpt=None):
        fwd(xs[i % N_XBUF], k, kpt, ybuf)

    ybuf = torch.empty((T, D), dtype=torch.bfloat16, device="cuda")
    clocks = ClockSampler(local)
    clocks.start()
    n0 = sum(x.launch_count() for x in layers)
    ms = time_steps(step, args.steps, args.warmup, world)
    launches = (sum(x.launch_count() for x in layers) - n0) // (args.steps + args.warmup) * args.steps
    if use_ep:
        # plan (4 kernels), pack, combine (+ the count kernel of mp_ep_forward / the
        # peer-memory return kernel) per step
        launches += (6 if args.ep_transport == "torch" else 7) * args.steps
    value = world * T / (ms * 1e-3)
    # steady state: a driver run of a few steps sits at burst clocks; the
    # serving figure is a long loop under the 1000 W cap
    steady = None
    if args.steps < 300:
        n_ss = 600
        ms_ss = time_steps(step, n_ss, 3, world)
        steady = {"steps": n_ss, "ms_per_step": ms_ss, "value": world * T / (ms_ss * 1e-3), "unit": "tokens/s",
                  "layer_roofline": layer_roofline(T, args.k, ms_ss, pk, touched)}

    # per-stage device times (CUDA events on the forward's stream), the sweep
    sweep_out = []
    stages_main = None
    for k in sweep + ["mixed"]:
        kpt = None
        kk = k
        if k == "mixed":
            rng = np.random.default_rng(13)
            kpt = torch.from_numpy(rng.choice([2, 4, 8, 16], size=T, p=[0.25, 0.35, 0.25, 0.15]).astype(np.int32))
            kpt = kpt.cuda()
            kk = float(kpt.float().mean().item())
        msk = time_steps(lambda i: step(i, k=0 if kpt is not None else k, kpt=kpt), max(args.steps // 2, 10), 3,
                         world)
        per_step = stage_profile(layers, fwd, xs, 0 if kpt is not None else k, kpt=kpt)
        resel, near = layers[0].route_stats()  # the last forward's routing (4096 tokens)
        ent = {"k": k, "tokens_per_s": world * T / (msk * 1e-3), "ms_per_step": msk,
               "layer_roofline": layer_roofline(T, kk, msk, pk, touched), "stages_ms": per_step,
               "routing": {"tokens": T, "reselected_exact": resel, "near_ties_lt_1e-6": near}}
        if k != "mixed":
            ent["kernel_roofline"] = kernel_roofline(per_step, T, k, pk, touched)
        sweep_out.append(ent)
        if k == args.k:
            stages_main = per_step
    if stages_main is None:
        stages_main = stage_profile(layers, fwd, xs, args.k)

    # e2e: public API with HOST buffers (pinned), H2D of x + D2H of y per step
    xh = [xs[i].cpu().pin_memory() for i in range(2)]
    yh = torch.empty((T, D), dtype=torch.bfloat16).pin_memory()
    from paper_2510_19366_b200 import _lib
    lib = _lib.load()
    if not use_ep:
        # the public pipelined host API: every step uploads its x and downloads
        # its y (pinned host buffers); copies of neighbouring steps overlap the
        # compute (mp_layer_forward_host_batches)
        yh2 = [yh, torch.empty((T, D), dtype=torch.bfloat16).pin_memory()]

        def e2e_run(n):
            L.forward_host_batches([xh[i % 2] for i in range(n)], args.k, ys=[yh2[i % 2] for i in range(n)])
        path = "mp_layer_forward_host_batches (C-ABI), pinned host x/y, copies pipelined against compute"
    else:
        xd = torch.empty((T, D), dtype=torch.bfloat16, device="cuda")

        def e2e_step(i):
            xd.copy_(xh[i % 2], non_blocking=True)
            y = fwd(xd, args.k, None)
            yh.copy_(y, non_blocking=True)
            torch.cuda.current_stream().synchronize()
        path = "ExpertParallelLayer.forward with pinned host x/y copied in/out"

    n_e2e = max(args.steps // 2, 10)
    if not use_ep:
        e2e_run(3)  # warm-up
        torch.cuda.synchronize()
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        e2e_run(n_e2e)  # synchronises (all downloads done) before returning
        e1.record(st)
        torch.cuda.synchronize()
        ms_e2e = e0.elapsed_time(e1) / n_e2e
    else:
        ms_e2e = time_steps(e2e_step, n_e2e, 3, world)
    e2e = {"value": world * T / (ms_e2e * 1e-3), "unit": "tokens/s", "h2d_bytes_per_step": T * D * 2,
           "d2h_bytes_per_step": T * D * 2, "ms_per_step": ms_e2e, "path": path}
    clk = clocks.stop()  # sampled across the main timed loop, the k sweep and the e2e loop

    other = None
    if use_ep and not args.no_extras:
        # C3: the 32-layer stack, expert-parallel over the ranks (C5's mixed-QoS
        # tiers at 4096 tokens per GPU are the sweep's "mixed" entry)
        for x in layers:
            x.close()
        ops.close()
        layers = []
        torch.cuda.empty_cache()
        other = {"stack32_ep": bench_stack_ep(pk, local, rank, world)}
    if extras:
        other = {"mixed_qos_32k": bench_mixed_qos_32k(L, pk)}
        other["qwen"] = bench_qwen(pk)
        other["c1_toy_gpu"] = bench_c1_gpu(pk)
        other["proxy_router"] = bench_proxy(pk)
        L.close()
        layers = []
        torch.cuda.empty_cache()
        other["stack32"] = bench_stack(pk)
        other["calibration"] = bench_calibration(pk)
        other["offload"] = bench_offload()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        nthreads = os.cpu_count() or 1
        try:
            v, kind, dt = cpu_reference_sample(args.k, nthreads, nthreads)
            cpu = {"value": v, "unit": "tokens/s", "cores": nthreads, "kind": kind,
                   "sample": f"{nthreads} tokens (one per thread), k={args.k}, Mixtral layer shape, fp32 weights, "
                             f"{dt:.1f} s; CPU {cpu_model()}"}
            v1, kind1, dt1 = cpu_reference_sample(args.k, 1, 1, seed_tokens=12)
            cpu["one_thread"] = {"value": v1, "unit": "tokens/s", "cores": 1, "kind": kind1,
                                 "sample": f"1 token, k={args.k}, Mixtral layer shape, {dt1:.1f} s"}
            cpu["c1_full"] = {"threads_1": cpu_reference_c1(1), f"threads_{nthreads}": cpu_reference_c1(nthreads)}
        except Exception as exc:  # report, never fabricate
            cpu = {"value": None, "unit": "tokens/s", "cores": nthreads, "kind": None, "sample": f"failed: {exc}"}

    if rank == 0:
        main_k = next((s for s in sweep_out if s["k"] == args.k), None)
        line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic (counter-based U(-1,1) stream; random-init weights of the Mixtral layer shape)",
                "config": workload_config(args, world),
                "roofline": kernel_roofline(stages_main, T, args.k, pk, touched),
                "layer_roofline": layer_roofline(T, args.k, ms, pk, touched),
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
                "stages_ms": stages_main, "sweep": sweep_out, "steady_state": steady}
        if not use_ep:
            line["stage_roofline"] = stage_rooflines(stages_main, T, args.k, pk)
        if other:
            line["other_configs"] = other
        if main_k:
            line["roofline"] = main_k.get("kernel_roofline", line["roofline"])
        emit(line)
    for x in layers:
        x.close()
    if _dist_on():
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
