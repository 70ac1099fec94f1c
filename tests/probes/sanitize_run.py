"""Small forwards over the kernel variants for compute-sanitizer
(memcheck / racecheck / synccheck): 1-SM GEMMs, CTA-pair GEMMs with swapped
remainder tiles (every remainder size: T = 1024 / 300 / 37 tokens) and with
plain remainders, the fused router with > 128 sub-experts (column split,
persistent grid-barrier bases), the shared expert, per-token k.
python tests/probes/sanitize_run.py"""
import ctypes as C, sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2510_19366_b200 import MoeLayer, synth_fill, _lib

lib = _lib.load()
lib.mp_debug_set_tile_mode.argtypes = [C.c_void_p, C.c_int]


def layer(E, S, d, ff, T, k_max, shared=0):
    L = MoeLayer(E, S, d, ff, dtype="bf16", k_max=k_max, max_tokens=T)
    for e in range(E):
        ws = [synth_fill(torch.empty(d * ff, dtype=torch.float32, device="cuda"), 100 + 3 * e + m, 0.05)
              for m in range(3)]
        L.set_partition(e, np.arange(ff, dtype=np.uint32) % S)
        L.load_expert(e, *ws)
    L.set_router(synth_fill(torch.empty(d * E * S, dtype=torch.float32, device="cuda"), 7, 0.05).cpu().numpy())
    if shared:
        sw = [synth_fill(torch.empty(d * shared, dtype=torch.float32, device="cuda"), 900 + m, 0.05).cpu().numpy()
              for m in range(3)]
        L.set_shared_expert(*sw, gate=np.full(d, 0.01, np.float32))
    return L


x = synth_fill(torch.empty((1024, 512), dtype=torch.bfloat16, device="cuda"), 11, 1.0)
L = layer(4, 4, 512, 1024, 1024, 16)
for mode in (0, 1, 2, 3):
    _lib.check(lib.mp_debug_set_tile_mode(L.h, mode))
    for T in (1024, 300, 37):
        for k in (4, 16):
            L.forward(x[:T], k=k)
kpt = torch.from_numpy(np.random.default_rng(1).choice([2, 4, 8, 16], size=1024).astype(np.int32)).cuda()
L.forward(x, k_per_token=kpt)
torch.cuda.synchronize()
L.close()
Lq = layer(36, 4, 256, 512, 512, 16, shared=512)  # 144 sub-experts: router column split
xq = synth_fill(torch.empty((512, 256), dtype=torch.bfloat16, device="cuda"), 12, 1.0)
for T in (3, 64, 512):
    Lq.forward(xq[:T], k=8)
torch.cuda.synchronize()
Lq.close()
print("sanitize run ok")
