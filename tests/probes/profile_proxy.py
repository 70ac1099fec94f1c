"""Proxy-router routing at the Mixtral shape (T tokens, k) for ncu launch lists:
python tests/probes/profile_proxy.py [T] [k]"""
import math, sys
import numpy as np
import torch
sys.path.insert(0, '.')
import bench
from paper_2510_19366_b200 import MoeLayer, synth_fill
T = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
k = int(sys.argv[2]) if len(sys.argv) > 2 else 8
E, S, D, FF = bench.E, bench.S, bench.D, bench.FF
L = MoeLayer(E, S, D, FF, dtype="bf16", router="proxy", k_max=16, max_tokens=T)
buf = [torch.empty(D * FF, dtype=torch.float32, device="cuda") for _ in range(3)]
rng = np.random.default_rng(21)
for e in range(E):
    for m in range(3):
        synth_fill(buf[m], 100 + 3 * e + m, 1 / math.sqrt(D if m < 2 else FF))
    part = bench.balanced_partition(FF, S, 6000 + e)
    L.set_partition(e, part)
    L.load_expert(e, *buf)
    L.set_gates(e, 4, [sorted(rng.choice(np.flatnonzero(part == s), 4, replace=False).tolist()) for s in range(S)])
x = synth_fill(torch.empty((T, D), dtype=torch.bfloat16, device="cuda"), 11, 1.0)
for i in range(3):
    L.route(x, k=k)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
L.route(x, k=k)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("reselected, near ties:", L.route_stats())
