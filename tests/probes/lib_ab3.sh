#!/bin/bash
# Alternating-process A/B/C of library builds: tests/probes/lib_ab3.sh "libA libB libC" [k-list] [tile-mode]
LIBS=$1; KS=${2:-8,16}; TM=${3:-256}
for rep in 1 2 3; do
  for lib in $LIBS; do
    MOEPRISM_LIB=$lib MOEPRISM_TC_TILE=$TM python - "$KS" <<'PY' 2>&1 | sed "s|^|$(basename $lib) |"
import sys, statistics, torch
sys.path.insert(0, '.')
import bench
L, xs = bench.build_layer(0, 4096, 16)
y = torch.empty((4096, bench.D), dtype=torch.bfloat16, device='cuda')
for k in [int(a) for a in sys.argv[1].split(',')]:
    ms = bench.time_steps(lambda i: L.forward(xs[i % 8], k=k, y=y), 40, 5, 1)
    st = bench.stage_profile([L], lambda x, kk, kpt: L.forward(x, k=kk, y=y), xs, k, reps=20)
    print(f"k={k} step {ms:.3f} g1 {st['gemm1']:.3f} g2 {st['gemm2']:.3f}")
PY
  done
done
