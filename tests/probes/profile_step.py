"""One warm layer forward at the bench workload (Mixtral shape, T=4096) for
ncu: python tests/probes/profile_step.py [k] [reps]"""
import sys
import torch
sys.path.insert(0, '.')
import bench
k = int(sys.argv[1]) if len(sys.argv) > 1 else 8
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
L, xs = bench.build_layer(0, 4096, 16)
y = torch.empty((4096, bench.D), dtype=torch.bfloat16, device='cuda')
for i in range(3):
    L.forward(xs[i], k=k, y=y)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for i in range(reps):
    L.forward(xs[3 + i % 4], k=k, y=y)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")
