#!/bin/bash
# Alternating-process A/B of an environment knob on the Mixtral layer:
#   bash tests/probes/env_ab.sh "VAR=a VAR=b" [k-list] [reps]
VARIANTS=$1; KS=${2:-4,8,16}; REPS=${3:-3}
for rep in $(seq $REPS); do
  for v in $VARIANTS; do
    env $v python - "$KS" <<'PY' 2>&1 | sed "s|^|$v |"
import sys, torch
sys.path.insert(0, '.')
import bench
L, xs = bench.build_layer(0, 4096, 16)
y = torch.empty((4096, bench.D), dtype=torch.bfloat16, device='cuda')
for k in [int(a) for a in sys.argv[1].split(',')]:
    ms = bench.time_steps(lambda i: L.forward(xs[i % 8], k=k, y=y), 100, 5, 1)
    st = bench.stage_profile([L], lambda x, kk, kpt: L.forward(x, k=kk, y=y), xs, k, reps=20)
    print(f"k={k} step {ms:.3f} g1 {st['gemm1']:.3f} g2 {st['gemm2']:.3f}")
PY
  done
done
