#!/bin/bash
# Alternating-process A/B of two library builds on Mixtral (T=4096, k=2/8) and
# Qwen (decode 64 / prefill 8192, k=8): step ms and routing stats.
#   bash tests/probes/lib_ab_qm.sh "libA libB" [reps]
LIBS=$1; REPS=${2:-3}
for rep in $(seq $REPS); do
  for lib in $LIBS; do
    MOEPRISM_LIB=$lib python - <<'PY' 2>&1 | sed "s|^|$(basename $lib) |"
import sys, torch
sys.path.insert(0, '.')
import bench
from paper_2510_19366_b200 import synth_fill
L, xs = bench.build_layer(0, 4096, 16)
y = torch.empty((4096, bench.D), dtype=torch.bfloat16, device='cuda')
for k in (2, 8):
    ms = bench.time_steps(lambda i: L.forward(xs[i % 8], k=k, y=y), 100, 5, 1)
    print(f"mixtral k={k} step {ms:.4f} routing {L.route_stats()}")
L.close()
Q = bench.build_qwen_layer(8192)
for T in (64, 8192):
    qx = [synth_fill(torch.empty((T, 2048), dtype=torch.bfloat16, device='cuda'), 19 + i, 1.0) for i in range(4)]
    qy = torch.empty((T, 2048), dtype=torch.bfloat16, device='cuda')
    ms = bench.time_steps(lambda i: Q.forward(qx[i % 4], k=8, y=qy), 100 if T > 64 else 300, 5, 1)
    print(f"qwen T={T} k=8 step {ms:.4f} routing {Q.route_stats()}")
PY
  done
done
