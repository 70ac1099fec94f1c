"""Qwen decode (T=64) launch-path A/B: eager stream launches vs CUDA-graph
replay, plus the host cost of one forward call (no sync).  Run with
MOEPRISM_PDL=0/1 to compare programmatic dependent launch."""
import os, statistics, sys, time
import torch
sys.path.insert(0, '.')
import bench
from paper_2510_19366_b200 import synth_fill
T = int(os.environ.get("DEC_T", "64"))
L = bench.build_qwen_layer(8192)
d = bench.QW["d"]
xs = [synth_fill(torch.empty((T, d), dtype=torch.bfloat16, device='cuda'), 19 + i, 1.0) for i in range(8)]
y = torch.empty((T, d), dtype=torch.bfloat16, device='cuda')
for k in (4, 8):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(3):
            L.forward(xs[0], k=k, y=y)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(8):
                L.forward(xs[i], k=k, y=y)
    torch.cuda.synchronize()
    eager, graph, host = [], [], []
    for rep in range(5):
        eager.append(bench.time_steps(lambda i: L.forward(xs[i % 8], k=k, y=y), 40, 3, 1))
        graph.append(bench.time_steps(lambda i: g.replay(), 5, 1, 1) / 8)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(20):
            L.forward(xs[i % 8], k=k, y=y)
        host.append((time.perf_counter() - t0) / 20 * 1e3)
        torch.cuda.synchronize()
    print(f"PDL={os.environ.get('MOEPRISM_PDL', '1')} T={T} k={k}: eager {statistics.median(eager):.4f} ms | "
          f"graph {statistics.median(graph):.4f} ms | host/call {statistics.median(host):.4f} ms", flush=True)
