"""In-process A/B of the grouped-GEMM kernels (1-SM 128-row tiles vs CTA-pair
256-row tiles): alternating blocks of steps, median per mode -- robust to the
power-cap clock drift that makes separate runs incomparable."""
import ctypes as C, statistics, sys
import torch
sys.path.insert(0, '.')
import bench
from paper_2510_19366_b200 import _lib
L, xs = bench.build_layer(0, 4096, 16)
lib = _lib.load()
lib.mp_debug_set_tile_mode.argtypes = [C.c_void_p, C.c_int]
y = torch.empty((4096, bench.D), dtype=torch.bfloat16, device='cuda')
for k in [int(a) for a in (sys.argv[1] if len(sys.argv) > 1 else "2,4,8,16").split(",")]:
    res = {1: [], 2: []}
    for rep in range(6):
        for mode in (1, 2):
            _lib.check(lib.mp_debug_set_tile_mode(L.h, mode))
            ms = bench.time_steps(lambda i: L.forward(xs[i % 8], k=k, y=y), 20, 3, 1)
            res[mode].append(ms)
    m1, m2 = statistics.median(res[1]), statistics.median(res[2])
    print(f"k={k}: 128-row {m1:.3f} ms | pair {m2:.3f} ms | pair/128 {m2 / m1:.3f}", flush=True)
