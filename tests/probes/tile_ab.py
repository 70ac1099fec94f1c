"""In-process A/B of the grouped-GEMM schedules with TIME and ENERGY per step.
Under the 1000 W cap the clock follows power, so wall time alone is noisy
across blocks; energy per step (NVML total energy) is the power-robust
metric: at the cap, throughput ~ P_cap / energy_per_step.
  python tests/probes/tile_ab.py <k-list> <mode-list> [reps] [steps-per-block] [qwen]
modes: 1 128-row 1-SM, 2 pairs (modes 4-7 of round 1 -- tail / split / merged / wide
remainders -- were removed after measuring slower); "qwen": the Qwen layer at T=8192 instead of Mixtral T=4096"""
import ctypes as C, statistics, sys
import torch
sys.path.insert(0, '.')
import bench
from paper_2510_19366_b200 import _lib
import pynvml
pynvml.nvmlInit()
hnd = pynvml.nvmlDeviceGetHandleByIndex(0)
if len(sys.argv) > 5 and sys.argv[5] == "qwen":
    from paper_2510_19366_b200 import synth_fill
    T = 8192
    L = bench.build_qwen_layer(T)
    xs = [synth_fill(torch.empty((T, bench.QW["d"]), dtype=torch.bfloat16, device="cuda"), 19 + i, 1.0)
          for i in range(8)]
else:
    T = 4096
    L, xs = bench.build_layer(0, T, 16)
lib = _lib.load()
lib.mp_debug_set_tile_mode.argtypes = [C.c_void_p, C.c_int]
y = torch.empty_like(xs[0])
names = {0: "auto", 1: "128-row", 2: "pair", 3: "pair", 4: "pair-tail128", 5: "split", 6: "pair-merged", 7: "pair-wide"}
ks = [int(a) for a in sys.argv[1].split(",")]
modes = [int(a) for a in sys.argv[2].split(",")]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 6
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 40
for k in ks:
    res = {m: {"ms": [], "mj": [], "mhz": []} for m in modes}
    for rep in range(reps):
        for mode in modes:
            _lib.check(lib.mp_debug_set_tile_mode(L.h, mode))
            for i in range(3):
                L.forward(xs[i % 8], k=k, y=y)
            torch.cuda.synchronize()
            e0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(hnd)
            ms = bench.time_steps(lambda i: L.forward(xs[i % 8], k=k, y=y), steps, 0, 1)
            e1 = pynvml.nvmlDeviceGetTotalEnergyConsumption(hnd)
            res[mode]["ms"].append(ms)
            res[mode]["mj"].append((e1 - e0) / steps)
            res[mode]["mhz"].append(pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM))
    line = f"k={k}:"
    for m in modes:
        r = {a: statistics.median(b) for a, b in res[m].items()}
        line += f" | {names[m]} {r['ms']:.3f} ms {r['mj']:.0f} mJ/step @{r['mhz']:.0f}MHz"
    print(line, flush=True)
