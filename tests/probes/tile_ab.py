"""In-process A/B of the grouped-GEMM kernels (1-SM 128-row tiles vs CTA-pair
256-row tiles, with / without the M=128 tail MMA): alternating blocks of
steps, median per mode of the layer step and of the gemm1 / gemm2 stage
times (CUDA events), with the SM clock (NVML) sampled after each block --
robust to the power-cap clock drift that makes separate runs incomparable."""
import ctypes as C, statistics, sys
import torch
sys.path.insert(0, '.')
import bench
from paper_2510_19366_b200 import _lib
try:
    import pynvml
    pynvml.nvmlInit()
    hnd = pynvml.nvmlDeviceGetHandleByIndex(0)
    clock = lambda: pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM)
except Exception:
    clock = lambda: 0
L, xs = bench.build_layer(0, 4096, 16)
lib = _lib.load()
lib.mp_debug_set_tile_mode.argtypes = [C.c_void_p, C.c_int]
y = torch.empty((4096, bench.D), dtype=torch.bfloat16, device='cuda')
names = {1: "128-row", 2: "pair", 3: "pair-no-tail128", 4: "pair-tail128-both"}
modes = [int(a) for a in (sys.argv[2] if len(sys.argv) > 2 else "1,2,3").split(",")]
for k in [int(a) for a in (sys.argv[1] if len(sys.argv) > 1 else "2,4,8,16").split(",")]:
    res = {m: {"step": [], "gemm1": [], "gemm2": [], "mhz": []} for m in modes}
    for rep in range(int(sys.argv[3]) if len(sys.argv) > 3 else 6):
        for mode in modes:
            _lib.check(lib.mp_debug_set_tile_mode(L.h, mode))
            ms = bench.time_steps(lambda i: L.forward(xs[i % 8], k=k, y=y), 20, 3, 1)
            res[mode]["mhz"].append(clock())
            st = bench.stage_profile([L], lambda x, kk, kpt: L.forward(x, k=kk, y=y), xs, k, reps=10)
            res[mode]["step"].append(ms)
            res[mode]["gemm1"].append(st["gemm1"])
            res[mode]["gemm2"].append(st["gemm2"])
    line = f"k={k}:"
    for m in modes:
        r = {a: statistics.median(b) for a, b in res[m].items()}
        line += f" | {names[m]} step {r['step']:.3f} g1 {r['gemm1']:.3f} g2 {r['gemm2']:.3f} ms @{r['mhz']:.0f}MHz"
    print(line, flush=True)
