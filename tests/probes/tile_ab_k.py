"""In-process A/B of the GEMM kernels per k (Mixtral T=4096 or Qwen prefill):
1-SM 128-row tiles (mode 1) vs CTA pairs with swapped remainders (mode 2),
alternating blocks of steps, median ms per step.
  python tests/probes/tile_ab_k.py [mixtral|qwen] [k-list] [steps]"""
import ctypes as C, json, statistics, sys
import torch
sys.path.insert(0, '.')
import bench
from paper_2510_19366_b200 import _lib, synth_fill
shape = sys.argv[1] if len(sys.argv) > 1 else "mixtral"
ks = [int(a) for a in (sys.argv[2] if len(sys.argv) > 2 else "2,3,4,5,6,7,8,9,10,11,12,13,14,15,16").split(",")]
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 30
if shape == "qwen":
    T = 8192
    L = bench.build_qwen_layer(T)
    d = bench.QW["d"]
    xs = [synth_fill(torch.empty((T, d), dtype=torch.bfloat16, device='cuda'), 19 + i, 1.0) for i in range(4)]
else:
    T, d = 4096, bench.D
    L, xs = bench.build_layer(0, T, 16)
y = torch.empty((T, d), dtype=torch.bfloat16, device='cuda')
lib = _lib.load()
lib.mp_debug_set_tile_mode.argtypes = [C.c_void_p, C.c_int]
for k in ks:
    res = {1: [], 2: []}
    for rep in range(int(__import__("os").environ.get("REPS", "4"))):
        for mode in (1, 2) if rep % 2 == 0 else (2, 1):
            _lib.check(lib.mp_debug_set_tile_mode(L.h, mode))
            res[mode].append(bench.time_steps(lambda i: L.forward(xs[i % len(xs)], k=k, y=y), steps, 3, 1))
    _lib.check(lib.mp_debug_set_tile_mode(L.h, 0))
    auto = bench.time_steps(lambda i: L.forward(xs[i % len(xs)], k=k, y=y), steps, 3, 1)
    m1, m2 = statistics.median(res[1]), statistics.median(res[2])
    print(json.dumps({"shape": shape, "k": k, "ms_1sm": round(m1, 4), "ms_pairs": round(m2, 4),
                      "pairs_over_1sm": round(m2 / m1, 3), "ms_auto": round(auto, 4)}), flush=True)
