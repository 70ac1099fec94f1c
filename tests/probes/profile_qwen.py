"""Qwen1.5-MoE-shape layer forward at a decode / prefill batch for ncu:
python tests/probes/profile_qwen.py T k reps"""
import sys
import torch
sys.path.insert(0, '.')
import bench
T = int(sys.argv[1]) if len(sys.argv) > 1 else 64
k = int(sys.argv[2]) if len(sys.argv) > 2 else 8
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
L = bench.build_qwen_layer(max(T, 64))
from paper_2510_19366_b200 import synth_fill
x = synth_fill(torch.empty((T, 2048), dtype=torch.bfloat16, device='cuda'), 19, 1.0)
y = torch.empty_like(x)
for i in range(3):
    L.forward(x, k=k, y=y)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for i in range(reps):
    L.forward(x, k=k, y=y)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done")
