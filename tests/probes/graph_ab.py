"""Eager stream launches vs CUDA-graph replay of the same layer forward: the
difference is launch overhead / inter-kernel gaps."""
import statistics, sys
import torch
sys.path.insert(0, '.')
import bench
L, xs = bench.build_layer(0, 4096, 16)
y = torch.empty((4096, bench.D), dtype=torch.bfloat16, device='cuda')
for k in [int(a) for a in (sys.argv[1] if len(sys.argv) > 1 else "2,8").split(",")]:
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
    eager, graph = [], []
    for rep in range(5):
        eager.append(bench.time_steps(lambda i: L.forward(xs[i % 8], k=k, y=y), 40, 3, 1))
        graph.append(bench.time_steps(lambda i: g.replay(), 5, 1, 1) / 8)
    print(f"k={k}: eager {statistics.median(eager):.3f} ms/step | graph replay {statistics.median(graph):.3f} ms/step",
          flush=True)
