#!/bin/bash
# A/B of the grid-barrier bucket bases + CTA-wide split sums in route_bucket
# (MOEPRISM_GRID_SCAN=0 / MOEPRISM_PARTIALS_REDUCE_ABOVE=8 = the previous chain).
for v in "MOEPRISM_GRID_SCAN=0 MOEPRISM_PARTIALS_REDUCE_ABOVE=8" "MOEPRISM_GRID_SCAN=1"; do
  echo "== $v"; env $v python tests/probes/qwen_quick.py 100; env $v python tests/probes/mixtral_quick.py 100
done
