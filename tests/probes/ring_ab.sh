#!/bin/bash
# A/B of the GEMM operand ring depths (NA A-stages x 16 KB, NB B-stages x 32 KB).
for v in v44 v54 v43 v34 v44 v54; do
  MOEPRISM_LIB=tests/probes/libmoeprism_$v.so MOEPRISM_TC_TRACE=1 python tests/probes/gemm_trace.py 2>&1 | sed "s|^|$v |" | grep "k=8\|k=16 gemm1\|Error"
done
