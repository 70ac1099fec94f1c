"""One-screen summary of a bench.py JSON line: python tests/probes/bench_summary.py file.json"""
import json, sys
j = json.load(open(sys.argv[1]))
print("headline", round(j['value'] / 1e6, 3), "M tok/s", round(j['ms_per_step'], 3), "ms; gemm1 frac",
      round(j['roofline']['frac'], 3), "layer frac", round(j['layer_roofline']['frac'], 3), j['clocks'],
      "e2e", round(j['e2e']['value'] / 1e6, 3), "steady", round(j.get('steady_state', {}).get('value', 0) / 1e6, 3))
for s in j['sweep']:
    kr = s.get('kernel_roofline', {})
    print(s['k'], round(s['tokens_per_s'] / 1e6, 3), round(s['ms_per_step'], 3), "layer", round(s['layer_roofline']['frac'], 3),
          "kern", round(kr.get('frac', 0), 3), {a: round(b, 3) for a, b in s['stages_ms'].items()})
oc = j.get('other_configs', {})
for s in oc.get('qwen', {}).get('sweep', []):
    gr = {a: round(b['frac'], 3) for a, b in s.get('routed_gemm_roofline', {}).items()}
    print('qwen', s['tokens'], s['k'], round(s['ms_per_step'], 4), round(s['roofline']['frac'], 3), gr)
for k in ('mixed_qos_32k',):
    if k in oc:
        v = oc[k]
        print(k, round(v['tokens_per_s'] / 1e6, 3), v.get('roofline', {}).get('frac'))
if 'stack32' in oc:
    for s in oc['stack32']['sweep']:
        print('stack32', s['k'], round(s['tokens_per_s'] / 1e3, 1), 'k tok/s', s.get('roofline', {}).get('frac'))
