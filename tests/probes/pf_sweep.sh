#!/bin/bash
# GEMM sensitivity to the L2 prefetch distance (k-blocks ahead of the TMA loads).
for pf in 0 4 8 16; do
  MOEPRISM_TC_PREFETCH=$pf python bench.py --steps 40 --warmup 5 --sweep 2,8,16 --no-cpu-baseline 2>/dev/null | \
    python -c "
import json,sys; j=json.loads(sys.stdin.read())
print('prefetch', $pf, 'clk', j['clocks']['sm_mhz'], ' '.join('k%s g1 %.3f g2 %.3f step %.3f' % (s['k'], s['stages_ms']['gemm1'], s['stages_ms']['gemm2'], s['ms_per_step']) for s in j['sweep'] if s['k'] != 'mixed'))"
done
