"""Diagnostics for the tcgen05 grouped GEMMs (run on a GPU box):
compares the layer's internal h = SwiGLU(x_perm W1) and o = h W2 buffers with
torch fp32 math on the same bf16 operands and prints the error pattern."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))
from paper_2510_19366_b200 import MoeLayer, _lib  # noqa: E402


def bufs(L):
    lib = _lib.load()
    lib.mp_debug_buffers.argtypes = [C.c_void_p] + [C.POINTER(C.c_void_p)] * 5 + [C.c_void_p]
    ptrs = [C.c_void_p() for _ in range(5)]
    dims = (C.c_uint32 * 4)()
    _lib.check(lib.mp_debug_buffers(L.h, *[C.byref(p) for p in ptrs], dims))
    return [p.value for p in ptrs], list(dims)


def as_tensor(ptr, shape, dtype=torch.bfloat16):
    """Copy raw device memory at `ptr` into a new torch tensor."""
    import cuda.bindings.runtime as rt  # cuda-python
    n = int(np.prod(shape))
    t = torch.empty(shape, dtype=dtype, device="cuda")
    torch.cuda.synchronize()
    err, = rt.cudaMemcpy(t.data_ptr(), ptr, n * t.element_size(), rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice)
    assert int(err) == 0, err
    return t


def run(E, S, d, ff, T, k, seed=0):
    torch.manual_seed(seed)
    G = E * S
    L = MoeLayer(E, S, d, ff, dtype="bf16", weights="unit", k_max=k, max_tokens=T)
    for e in range(E):
        L.set_partition(e, (np.arange(ff) % S).astype(np.uint32))
        L.load_expert(e, *(torch.rand(d * ff, device="cuda") * 2 - 1 for _ in range(3)))
    x = (torch.rand(T, d, device="cuda") * 2 - 1).to(torch.bfloat16)
    rng = np.random.default_rng(seed)
    sel = np.stack([np.sort(rng.choice(G, k, replace=False)) for _ in range(T)]).astype(np.uint32)
    y, off = L.forward_selected(x, torch.from_numpy(sel.view(np.int32)), return_offsets=True)
    torch.cuda.synchronize()
    (xp, hp, op, w1p, w2p), (w_pad, d_pad, rows_cap, use_tc) = bufs(L)
    rows = T * k
    offs = off.cpu().numpy()
    Xp = as_tensor(xp, (rows, d_pad)).float()
    H = as_tensor(hp, (rows, w_pad)).float()
    O = as_tensor(op, (rows, d_pad)).float()
    W1 = as_tensor(w1p, (G, 2 * w_pad, d_pad)).float()
    W2 = as_tensor(w2p, (G, d_pad, w_pad)).float()
    worst_h = worst_o = 0.0
    for g in range(G):
        r0, r1 = int(offs[g]), int(offs[g + 1])
        if r1 == r0:
            continue
        acc = Xp[r0:r1] @ W1[g].T  # rows x 2w_pad
        acc = acc.view(r1 - r0, w_pad // 64, 2, 64)  # kIlv = 64 gate/up interleave
        gate, up = acc[:, :, 0, :].reshape(r1 - r0, w_pad), acc[:, :, 1, :].reshape(r1 - r0, w_pad)
        href = (torch.nn.functional.silu(gate) * up)
        eh = ((H[r0:r1] - href).abs() / (1 + href.abs()))
        oref = H[r0:r1] @ W2[g].T
        eo = ((O[r0:r1] - oref).abs() / (1 + oref.abs()))
        if eh.max() > 2e-2 or eo.max() > 2e-2:
            bad = (eh > 2e-2).nonzero()
            print(f"  g={g} rows {r0}:{r1} h max err {eh.max():.3g} ({bad.shape[0]} bad; rows {sorted(set(bad[:, 0].tolist()))[:10]} "
                  f"cols {sorted(set((bad[:, 1] // 32).tolist()))[:10]}x32) o max err {eo.max():.3g}")
        worst_h = max(worst_h, eh.max().item())
        worst_o = max(worst_o, eo.max().item())
    print(f"E={E} S={S} d={d} ff={ff} T={T} k={k} use_tc={use_tc}: worst h {worst_h:.3g} worst o {worst_o:.3g}")
    L.close()


if __name__ == "__main__":
    run(1, 1, 128, 128, 128, 1)
    run(1, 1, 256, 512, 300, 1)
    run(4, 4, 256, 512, 200, 4)
    run(8, 4, 512, 1024, 256, 4)
