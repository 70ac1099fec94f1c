"""MMA-issuer timing breakdown of the tcgen05 grouped GEMMs (diagnostic).
Run with MOEPRISM_TC_TRACE=1.  python tests/probes/gemm_trace.py [k-list] [qwen T]"""
import ctypes as C, sys, numpy as np, torch
sys.path.insert(0, '.')
import bench
from paper_2510_19366_b200 import _lib
if len(sys.argv) > 2 and sys.argv[2] == "qwen":
    from paper_2510_19366_b200 import synth_fill
    T = int(sys.argv[3]) if len(sys.argv) > 3 else 8192
    L = bench.build_qwen_layer(T)
    xs = [synth_fill(torch.empty((T, bench.QW["d"]), dtype=torch.bfloat16, device="cuda"), 19 + i, 1.0)
          for i in range(3)]
else:
    L, xs = bench.build_layer(0, 4096, 16)
lib = _lib.load()
lib.mp_debug_gemm_trace.argtypes = [C.c_int, C.c_void_p, C.c_uint32]
for k in [int(a) for a in (sys.argv[1] if len(sys.argv) > 1 else "2,8,16").split(",")]:
    for i in range(3):
        L.forward(xs[i], k=k)
    torch.cuda.synchronize()
    for which, name in ((0, 'gemm1'), (1, 'gemm2')):
        tr = np.zeros((148, 4), np.uint64)
        _lib.check(lib.mp_debug_gemm_trace(which, tr.ctypes.data, 148))
        tr = tr[tr[:, 0] > 0]  # CTA-pair kernel: leaders only
        tot, wacc, wfull, tiles = (tr[:, i].astype(np.float64) for i in range(4))
        print(f"k={k} {name}: cycles max {tot.max():.0f} mean {tot.mean():.0f} | wait accumulator {100*wacc.sum()/tot.sum():.1f}% "
              f"| wait smem stage {100*wfull.sum()/tot.sum():.1f}% | tiles/CTA {tiles.min():.0f}-{tiles.max():.0f} "
              f"| CTA imbalance {(tot.max()-tot.mean())/tot.max()*100:.1f}%")
