"""Per-tile MMA-phase timing of the CTA-pair kernel (MP_PAIR_TRACE=1 build):
full 256-row tiles vs M=128 tail tiles vs extended (merged-remainder) tiles.
MOEPRISM_TC_TRACE=1, MOEPRISM_LIB=tests/probes/libmoeprism_trace.so."""
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
        for kind, lab in ((0, 'full '), (1, 'tail '), (2, 'ext  '), (3, 'wide ')):
            r = rec[rec[:, 3] == kind]
            if len(r):
                print(f"k={k} {name} {lab}: tiles {len(r)}  MMA-phase cycles mean {r[:, 2].mean():.0f} "
                      f"p50 {np.median(r[:, 2]):.0f}  operand waits mean {r[:, 1].mean():.0f}", flush=True)
        lead = tr[:512].reshape(-1, 4)
        lead = lead[lead[:, 0] > 0]
        print(f"k={k} {name} leaders: total cycles mean {lead[:, 0].mean():.0f} max {lead[:, 0].max():.0f}  "
              f"accumulator waits mean {lead[:, 1].mean():.0f}  operand waits mean {lead[:, 2].mean():.0f}  "
              f"tiles mean {lead[:, 3].mean():.1f}", flush=True)
        ep = tr[512:1024].reshape(-1, 4)
        ep = ep[ep[:, 3] > 0]
        if len(ep):
            print(f"k={k} {name} epilogue (warp 2/CTA): busy/tile {(ep[:, 0] / ep[:, 3]).mean():.0f}  "
                  f"ext part/tile {(ep[:, 1] / ep[:, 3]).mean():.0f}  tfull waits/tile {(ep[:, 2] / ep[:, 3]).mean():.0f}",
                  flush=True)
