#!/bin/bash
# CTA pairs with swapped-operand remainder tiles vs plain 256-row remainders
# vs 1-SM 128-row tiles vs auto (Mixtral T=4096 k=2/4/8/16, Qwen decode /
# prefill): bash tests/probes/swap_ab.sh [steps]
steps=${1:-100}
for v in "MOEPRISM_TC_TILE=auto" "MOEPRISM_TC_TILE=256" "MOEPRISM_TC_TILE=256-plain" "MOEPRISM_TC_TILE=128"; do
  echo "== $v"; env $v python tests/probes/mixtral_quick.py $steps; env $v python tests/probes/qwen_quick.py $steps
done
