"""Quick Mixtral-layer timing (T=4096, k=2/4/8/16) with the stage breakdown and
routing stats: python tests/probes/mixtral_quick.py [steps]"""
import json, sys
import torch
sys.path.insert(0, '.')
import bench
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
L, xs = bench.build_layer(0, 4096, 16)
y = torch.empty((4096, bench.D), dtype=torch.bfloat16, device='cuda')
for k in (2, 4, 8, 16):
    ms = bench.time_steps(lambda i: L.forward(xs[i % len(xs)], k=k, y=y), steps, 5, 1)
    st = bench.stage_profile([L], lambda x, kk, kpt, y=None: L.forward(x, k=kk, y=y), xs, k)
    print(json.dumps({"T": 4096, "k": k, "ms": round(ms, 4), "stages": {a: round(b, 4) for a, b in st.items()},
                      "routing": L.route_stats()}), flush=True)
