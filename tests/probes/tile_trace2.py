"""Per-tile MMA-phase timing of the CTA-pair kernel with swapped remainder
tiles (MP_PAIR_TRACE=1 build): full 256-row tiles vs swapped tiles by token
columns, leader totals, epilogue busy time.
  MOEPRISM_TC_TRACE=1 MOEPRISM_TC_TILE=256 MOEPRISM_LIB=tests/probes/libmoeprism_trace.so \\
  python tests/probes/tile_trace2.py mixtral 8 | qwen 8192 8"""
import ctypes as C, sys, numpy as np, torch
sys.path.insert(0, '.')
import bench
from paper_2510_19366_b200 import _lib, synth_fill
if sys.argv[1] == "qwen":
    T, k = int(sys.argv[2]), int(sys.argv[3])
    L = bench.build_qwen_layer(T)
    xs = [synth_fill(torch.empty((T, bench.QW["d"]), dtype=torch.bfloat16, device='cuda'), 19 + i, 1.0) for i in range(3)]
    fwd = lambda x: L.forward(x, k=k)
else:
    T, k = 4096, int(sys.argv[2])
    L, xs = bench.build_layer(0, 4096, 16)
    fwd = lambda x: L.forward(x, k=k)
lib = _lib.load()
lib.mp_debug_gemm_trace.argtypes = [C.c_int, C.c_void_p, C.c_uint32]
N = (4096 + 128 * 128 * 4) // 4
for i in range(3):
    fwd(xs[i])
torch.cuda.synchronize()
for which, name in ((0, 'gemm1'), (1, 'gemm2')):
    tr = np.zeros((N, 4), np.uint64)
    _lib.check(lib.mp_debug_gemm_trace(which, tr.ctypes.data, N))
    rec = tr[1024:].reshape(-1, 4)
    rec = rec[rec[:, 2] > 0]
    for nt in sorted(set(rec[:, 3].tolist())):
        kind = "full" if nt == 0 else (f"twin Nt={nt - 256}" if nt >= 256 and nt != 256 else f"swapped Nt={nt}")
        r = rec[rec[:, 3] == nt]
        print(f"{name} {kind}: tiles {len(r)}  MMA-phase cycles mean "
              f"{r[:, 2].mean():.0f} p50 {np.median(r[:, 2]):.0f}  operand waits mean {r[:, 1].mean():.0f}", flush=True)
    lead = tr[:512].reshape(-1, 4)
    lead = lead[lead[:, 0] > 0]
    print(f"{name} leaders: total cycles mean {lead[:, 0].mean():.0f} max {lead[:, 0].max():.0f}  "
          f"accumulator waits mean {lead[:, 1].mean():.0f}  operand waits mean {lead[:, 2].mean():.0f}  "
          f"tiles mean {lead[:, 3].mean():.1f}", flush=True)
    ep = tr[512:1024].reshape(-1, 4)
    ep = ep[ep[:, 3] > 0]
    if len(ep):
        print(f"{name} epilogue (warp 2/CTA): busy/tile {(ep[:, 0] / ep[:, 3]).mean():.0f}  "
              f"tfull waits/tile {(ep[:, 2] / ep[:, 3]).mean():.0f}", flush=True)
