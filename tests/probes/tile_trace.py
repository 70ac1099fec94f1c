"""Per-tile MMA-phase timing of the CTA-pair kernel (MP_PAIR_TRACE=1 build):
full 256-row tiles vs M=128 tail tiles.  MOEPRISM_TC_TRACE=1."""
import ctypes as C, sys, numpy as np, torch
sys.path.insert(0, '.')
import bench
from paper_2510_19366_b200 import _lib
L, xs = bench.build_layer(0, 4096, 16)
lib = _lib.load()
lib.mp_debug_gemm_trace.argtypes = [C.c_int, C.c_void_p, C.c_uint32]
N = (4096 + 128 * 128 * 4) // 4
for k in [int(a) for a in sys.argv[1].split(",")]:
    for i in range(3):
        L.forward(xs[i], k=k)
    torch.cuda.synchronize()
    for which, name in ((0, 'gemm1'), (1, 'gemm2')):
        tr = np.zeros((N, 4), np.uint64)
        _lib.check(lib.mp_debug_gemm_trace(which, tr.ctypes.data, N))
        rec = tr[1024:].reshape(-1, 4)
        rec = rec[rec[:, 2] > 0]
        for tail in (0, 1):
            r = rec[rec[:, 3] == tail]
            if len(r):
                print(f"k={k} {name} {'tail ' if tail else 'full '}: tiles {len(r)}  MMA-phase cycles mean {r[:, 2].mean():.0f} "
                      f"p50 {np.median(r[:, 2]):.0f}  operand waits mean {r[:, 1].mean():.0f}", flush=True)
