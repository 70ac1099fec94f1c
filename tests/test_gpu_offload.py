"""Sub-expert offload cache: real host->device transfers under
the reference's LRU policy (cache_step, inc/offload.hpp:202-255).  Outputs
must equal the device-resident layer bit for bit; the per-forward miss counts
must equal the reference cache_step replayed on the same request sequence."""
import numpy as np
import pytest

from gpu_util import bf16_round, make_layer, toy_setup

pytestmark = pytest.mark.gpu
E, S, D, FF = 8, 4, 256, 512


@pytest.fixture(scope="module")
def torch_cuda(cuda_lib):
    import torch
    return torch


def _layers(oracle, T):
    experts, parts, wr, x = toy_setup(oracle, E, S, D, FF, T)
    res = make_layer(experts, parts, wr, S, "bf16", k_max=4, max_tokens=T)
    off = make_layer(experts, parts, wr, S, "bf16", k_max=4, max_tokens=T)
    return res, off


@pytest.mark.parametrize("monolithic,capacity", [(False, 12), (True, 6)])
def test_offload_bitwise_and_reference_lru(oracle, ref, torch_cuda, monolithic, capacity):
    torch = torch_cuda
    T = 6
    res, off = _layers(oracle, T)
    off.enable_offload(capacity, monolithic=monolithic)
    unit = S if monolithic else 1
    rng = np.random.default_rng(3 + monolithic)
    steps, misses = [], []
    last_bytes = 0
    for i in range(14):
        t = int(rng.integers(1, T + 1))
        k = int(rng.integers(1, 3))
        x = torch.from_numpy(bf16_round(oracle.uniform_pm1(100 + i, t * D))).reshape(t, D).cuda().to(torch.bfloat16)
        y0 = res.forward(x, k=k)
        try:
            y1 = off.forward(x, k=k)
        except Exception as exc:  # request larger than the cache: the reference's ValidationError
            assert "exceeds the cache capacity" in str(exc)
            continue
        assert torch.equal(y0, y1), f"step {i}: offloaded output differs"
        h, m, b, req, lm = off.offload_stats()
        steps.append(req.tolist())
        misses.append(lm)
        assert b - last_bytes == lm * unit * (2 * 128 * 256 + 256 * 128) * 2  # w_pad 128, d_pad 256, bf16
        last_bytes = b
    assert len(steps) >= 6
    want = ref.offload_replay((E * S) // unit, capacity, steps)
    assert want.tolist() == misses
    assert sum(misses) < sum(len(s) for s in steps)  # some hits
    res.close()
    off.close()


def test_offload_capacity_error_and_guards(oracle, torch_cuda):
    torch = torch_cuda
    from paper_2510_19366_b200 import ValidationError
    T = 32
    res, off = _layers(oracle, T)
    with pytest.raises(ValidationError, match="capacity"):
        off.enable_offload(0)
    off.enable_offload(4)
    x = torch.from_numpy(bf16_round(oracle.uniform_pm1(7, T * D))).reshape(T, D).cuda().to(torch.bfloat16)
    with pytest.raises(ValidationError, match="exceeds the cache capacity"):
        off.forward(x, k=4)
    with pytest.raises(ValidationError, match="already"):
        off.enable_offload(4)
    res.close()
    off.close()


@pytest.mark.parametrize("T", [200, 700])
def test_offload_with_cta_pairs(oracle, torch_cuda, T):
    """The offload cache under the CTA-pair GEMMs (full tiles and swapped
    remainder tiles read their weights through the group -> cache-slot map):
    bitwise equal to the resident layer on the same kernel."""
    import ctypes as C
    torch = torch_cuda
    from paper_2510_19366_b200 import _lib
    lib = _lib.load()
    lib.mp_debug_set_tile_mode.argtypes = [C.c_void_p, C.c_int]
    res, off = _layers(oracle, T)
    off.enable_offload(E * S)
    for L in (res, off):
        _lib.check(lib.mp_debug_set_tile_mode(L.h, 2))
    x = torch.from_numpy(bf16_round(oracle.uniform_pm1(77, T * D))).reshape(T, D).cuda().to(torch.bfloat16)
    for k in (1, 4):
        y0 = res.forward(x, k=k)
        y1 = off.forward(x, k=k)
        assert torch.equal(y0, y1)
    res.close()
    off.close()
