#!/bin/bash
# gemm1 A rows gathered from x by TMA gather4 (no x_perm) vs the materialised
# x_perm (MOEPRISM_GATHER=0).
for v in "MOEPRISM_GATHER=0" "MOEPRISM_GATHER=1"; do
  echo "== $v"; env $v python tests/probes/mixtral_quick.py 100; env $v python tests/probes/qwen_quick.py 100
done
