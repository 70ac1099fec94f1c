"""Quick Qwen-layer timing (decode T=64 and prefill T=8192, k=4/8/16) with the
stage breakdown: python tests/probes/qwen_quick.py [steps]"""
import json, sys
import torch
sys.path.insert(0, '.')
import bench
from paper_2510_19366_b200 import synth_fill
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
L = bench.build_qwen_layer(8192)
d = bench.QW["d"]
for T in [int(v) for v in __import__("os").environ.get("QWEN_T", "64,8192").split(",")]:
    xs = [synth_fill(torch.empty((T, d), dtype=torch.bfloat16, device='cuda'), 19 + i, 1.0) for i in range(4)]
    y = torch.empty((T, d), dtype=torch.bfloat16, device='cuda')
    for k in (4, 8, 16):
        ms = bench.time_steps(lambda i: L.forward(xs[i % 4], k=k, y=y), steps, 5, 1)
        st = bench.stage_profile([L], lambda x, kk, kpt, y=None: L.forward(x, k=kk, y=y), xs, k)
        print(json.dumps({"T": T, "k": k, "ms": round(ms, 4), "stages": {a: round(b, 4) for a, b in st.items()},
                          "routing": L.route_stats()}), flush=True)
