#!/bin/bash
# A/B: 128-row tiles (gemm_tc) vs 256-row two-accumulator tiles (gemm_tc2).
for t in 128 256; do
  MOEPRISM_TC_TILE=$t python bench.py --steps 40 --warmup 5 --sweep 2,4,8,16 --no-cpu-baseline 2>/dev/null | \
    python -c "
import json,sys; j=json.loads(sys.stdin.read())
print('tile', $t, 'clk', j['clocks']['sm_mhz'])
for s in j['sweep']: print('  k', s['k'], 'gemm1', round(s['stages_ms']['gemm1'],3), 'gemm2', round(s['stages_ms']['gemm2'],3), 'step', round(s['ms_per_step'],3))"
done
