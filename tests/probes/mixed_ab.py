import sys, statistics, numpy as np, torch, ctypes as C
sys.path.insert(0, '.')
import bench
from paper_2510_19366_b200 import _lib
L, xs = bench.build_layer(0, 4096, 16)
lib = _lib.load(); lib.mp_debug_set_tile_mode.argtypes = [C.c_void_p, C.c_int]
rng = np.random.default_rng(13)
kpt = torch.from_numpy(rng.choice([2, 4, 8, 16], size=4096, p=[0.25, 0.35, 0.25, 0.15]).astype(np.int32)).cuda()
y = torch.empty((4096, bench.D), dtype=torch.bfloat16, device='cuda')
res = {m: [] for m in (1, 3, 7, 0)}
for rep in range(6):
    for m in res:
        _lib.check(lib.mp_debug_set_tile_mode(L.h, m))
        res[m].append(bench.time_steps(lambda i: L.forward(xs[i % 8], k_per_token=kpt, y=y), 40, 3, 1))
print({m: round(statistics.median(v), 4) for m, v in res.items()})
