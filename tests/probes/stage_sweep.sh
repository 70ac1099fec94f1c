#!/bin/bash
# GEMM ring-depth sensitivity (diagnostic): tensor-core GEMM time vs stages in use.
for ns in 2 3 4; do
  MOEPRISM_TC_STAGES=$ns python bench.py --steps 30 --warmup 5 --sweep 8 --no-cpu-baseline 2>/dev/null | \
    python -c "import json,sys; j=json.loads(sys.stdin.read()); s=j['stages_ms']; print('stages', $ns, 'gemm1', round(s['gemm1'],3), 'gemm2', round(s['gemm2'],3), 'step', round(j['ms_per_step'],3), 'clk', j['clocks']['sm_mhz'])"
done
