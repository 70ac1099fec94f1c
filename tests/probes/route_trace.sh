#!/bin/bash
# Routing-kernel phase trace (route_bucket_kernel, MP_ROUTE_TRACE=1 build in
# tests/probes/libmoeprism_rtrace.so): Qwen decode / prefill and Mixtral k=8.
#   bash tests/probes/route_trace.sh   (on the GPU box)
for T in 64 8192; do
  echo "== qwen T=$T k=8"
  MOEPRISM_LIB=tests/probes/libmoeprism_rtrace.so python tests/probes/profile_qwen.py $T 8 1 2>&1 | grep -v "^done" | tail -4
done
echo "== mixtral T=4096 k=8"
MOEPRISM_LIB=tests/probes/libmoeprism_rtrace.so python tests/probes/profile_step.py 8 1 2>&1 | tail -4
