#!/bin/bash
# Qwen decode / prefill A/B of the W1 tail + W2 trim (MOEPRISM_W1_TAIL) and the
# decode W2 map's L2 promotion (MOEPRISM_W2D_PROMO).
for v in "MOEPRISM_W1_TAIL=0" "MOEPRISM_W2D_PROMO=256" "MOEPRISM_W2D_PROMO=0" "MOEPRISM_W2D_PROMO=64"; do
  echo "== $v"; env $v python tests/probes/qwen_quick.py 100
done
