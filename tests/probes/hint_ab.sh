#!/bin/bash
for h in 0 1 0 1; do
  MOEPRISM_TC_TRACE=1 MOEPRISM_TC_HINTS=$h python tests/probes/gemm_trace.py 2>/dev/null | sed "s/^/hints=$h /" | grep "k=8"
done
