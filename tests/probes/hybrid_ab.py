"""In-process A/B of the GEMM schedules (1-SM 128-row tiles / CTA pairs /
hybrid) on the Mixtral layer at several k: python tests/probes/hybrid_ab.py [steps] [reps]"""
import ctypes as C, json, statistics, sys
import torch
sys.path.insert(0, '.')
import bench
from paper_2510_19366_b200 import _lib
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 60
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
L, xs = bench.build_layer(0, 4096, 16)
lib = _lib.load()
lib.mp_debug_set_tile_mode.argtypes = [C.c_void_p, C.c_int]
y = torch.empty((4096, bench.D), dtype=torch.bfloat16, device='cuda')
for k in (4, 5, 6, 8, 10, 12, 16):
    res = {}
    for rep in range(reps):
        for mode, name in ((1, "128"), (2, "pairs"), (3, "hybrid")):
            _lib.check(lib.mp_debug_set_tile_mode(L.h, mode))
            ms = bench.time_steps(lambda i: L.forward(xs[i % 8], k=k, y=y), steps, 5, 1)
            res.setdefault(name, []).append(ms)
    _lib.check(lib.mp_debug_set_tile_mode(L.h, 0))
    auto = bench.time_steps(lambda i: L.forward(xs[i % 8], k=k, y=y), steps, 5, 1)
    print(json.dumps({"k": k, **{n: round(statistics.median(v), 4) for n, v in res.items()}, "auto": round(auto, 4)}),
          flush=True)
