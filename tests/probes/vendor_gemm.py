"""Vendor comparator (not product): cuBLAS dense and torch._grouped_mm on the
Mixtral gemm1/gemm2 shapes, to calibrate the tcgen05 grouped GEMM."""
import torch, time
torch.manual_seed(0)
dev = "cuda"
def bench(fn, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(it): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / it
d, w, G = 4096, 1792, 64
for k in (2, 4, 8, 16):
    rows = 4096 * k
    A = torch.randn(rows, d, device=dev, dtype=torch.bfloat16)
    W1 = torch.randn(G, d, 2 * w, device=dev, dtype=torch.bfloat16)
    W1T = W1.transpose(1, 2).contiguous().transpose(1, 2)
    offs = torch.arange(1, G + 1, device=dev, dtype=torch.int32) * (rows // G)
    flops1 = 2.0 * rows * d * 2 * w
    dense = torch.randn(d, 2 * w, device=dev, dtype=torch.bfloat16)
    t_dense = bench(lambda: A @ dense)
    out = f"k={k} dense gemm1-shape {t_dense:.3f} ms {flops1/t_dense/1e9:.0f} TF/s"
    try:
        t_g = bench(lambda: torch._grouped_mm(A, W1T, offs=offs))
        out += f" | _grouped_mm {t_g:.3f} ms {flops1/t_g/1e9:.0f} TF/s"
    except Exception as ex:
        out += f" | _grouped_mm failed: {str(ex)[:80]}"
    print(out, flush=True)
    del A, W1, W1T
