"""ctypes binding of the C-ABI in include/moeprism/moe_layer.h.

Loads the in-tree ``libmoeprism_b200.so`` (built by ``__graft_entry__.build()``
or ``make -C paper_2510_19366_b200/csrc``).  There is no fallback: if the
library is missing, ``load()`` raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libmoeprism_b200.so"
if os.environ.get("MOEPRISM_LIB"):  # alternative in-tree build (kernel A/B experiments)
    LIB_PATH = Path(os.environ["MOEPRISM_LIB"]).resolve()

MP_OK, MP_ERR_VALIDATION, MP_ERR_IO, MP_ERR_CUDA = 0, 1, 2, 3
MP_DTYPE_F32, MP_DTYPE_BF16 = 0, 1
MP_ROUTER_LINEAR, MP_ROUTER_PROXY = 0, 1
MP_WEIGHT_UNIT, MP_WEIGHT_SOFTMAX_RENORM = 0, 1
MP_SEL_NONE = 0xFFFFFFFF
MP_LAYER_ROUTER_ONLY, MP_LAYER_EXPERTS_ONLY, MP_LAYER_SHARED_SCRATCH = 1, 2, 4
MP_EP_NCCL_ID_BYTES, MP_EP_RESIDUAL = 128, 1

# The exported C-ABI (include/moeprism/moe_layer.h); tests check the .so
# exports every one of these.
EXPORTS = (
    "mp_version", "mp_last_error", "mp_device_check", "mp_layer_create", "mp_layer_destroy", "mp_layer_get_desc",
    "mp_layer_load_expert", "mp_layer_load_expert_file", "mp_layer_set_partition", "mp_layer_load_partition_map",
    "mp_layer_set_router", "mp_layer_set_gates", "mp_layer_set_shared_expert", "mp_layer_set_residual",
    "mp_layer_collect_activations", "mp_binarize_topk", "mp_coactivation", "mp_format_write_mpam", "mp_format_read_mpam",
    "mp_layer_enable_offload", "mp_layer_offload_stats", "mp_layer_forward_host_batches",
    "mp_select_gate_neurons", "mp_gating_fidelity",
    "mp_ep_p2p_setup", "mp_ep_p2p_open", "mp_ep_p2p_pack", "mp_ep_p2p_recv_buffers", "mp_ep_p2p_return",
    "mp_ep_p2p_combine", "mp_layer_forward", "mp_layer_forward_host",
    "mp_layer_forward_selected", "mp_layer_route", "mp_layer_check_errors", "mp_layer_set_profiling",
    "mp_layer_stage_times", "mp_layer_reset_stage_times", "mp_layer_launch_count", "mp_synth_fill",
    "mp_format_read_mpex", "mp_format_read_partition_doc", "mp_validate_partition", "mp_layer_forward_selected_host",
    "mp_ep_create", "mp_ep_create_subexpert", "mp_ep_destroy", "mp_ep_plan", "mp_ep_pack", "mp_ep_combine",
    "mp_layer_route_stats", "mp_ep_nccl_unique_id", "mp_ep_nccl_init", "mp_ep_forward", "mp_ep_last_counts",
)


class ValidationError(RuntimeError):
    """Status 1: the inputs violate a contract (inc/error.hpp:9-11)."""


class IoError(RuntimeError):
    """Status 2: filesystem / stream failure (inc/error.hpp:14-16)."""


class CudaError(RuntimeError):
    """Status 3: CUDA failure or no usable sm_100a device."""


class LayerDesc(C.Structure):
    _fields_ = [
        ("n_experts", C.c_uint32), ("n_subexperts", C.c_uint32), ("d_model", C.c_uint32), ("d_ff", C.c_uint32),
        ("dtype", C.c_uint32), ("router_mode", C.c_uint32), ("weight_mode", C.c_uint32), ("k_max", C.c_uint32),
        ("max_tokens", C.c_uint32), ("device", C.c_int32), ("flags", C.c_uint32),
    ]


_lib = None


def _sig(L):
    vp, u32, u64, sz, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_size_t, C.c_int32
    L.mp_version.restype = C.c_char_p
    L.mp_last_error.restype = C.c_char_p
    L.mp_device_check.argtypes = [i32]
    L.mp_layer_create.argtypes = [C.POINTER(LayerDesc), C.POINTER(vp)]
    L.mp_layer_destroy.argtypes = [vp]
    L.mp_layer_get_desc.argtypes = [vp, C.POINTER(LayerDesc)]
    L.mp_layer_load_expert.argtypes = [vp, u32, vp, vp, vp]
    L.mp_layer_load_expert_file.argtypes = [vp, u32, C.c_char_p]
    L.mp_layer_set_partition.argtypes = [vp, u32, u32, vp, sz]
    L.mp_layer_load_partition_map.argtypes = [vp, C.c_char_p]
    L.mp_layer_set_router.argtypes = [vp, vp]
    L.mp_layer_set_gates.argtypes = [vp, u32, u32, vp, vp]
    L.mp_layer_set_shared_expert.argtypes = [vp, u32, vp, vp, vp, vp]
    L.mp_layer_set_residual.argtypes = [vp, C.c_int]
    L.mp_layer_collect_activations.argtypes = [vp, u32, vp, u32, vp, vp]
    L.mp_binarize_topk.argtypes = [vp, u32, u32, u32, vp, vp]
    L.mp_coactivation.argtypes = [vp, u32, u32, vp, vp]
    L.mp_format_write_mpam.argtypes = [C.c_char_p, u32, u32, vp]
    L.mp_format_read_mpam.argtypes = [C.c_char_p, C.POINTER(u32), C.POINTER(u32), vp]
    L.mp_layer_enable_offload.argtypes = [vp, u32, u32]
    L.mp_layer_forward_host_batches.argtypes = [vp, u32, vp, vp, u32, vp, vp]
    L.mp_select_gate_neurons.argtypes = [vp, u32, u32, vp, u32, vp, vp, vp]
    L.mp_gating_fidelity.argtypes = [vp, u32, u32, u32, vp, vp, vp, u32, C.POINTER(C.c_double), vp]
    L.mp_layer_offload_stats.argtypes = [vp, vp, vp, vp, vp, u32, vp, vp]
    L.mp_layer_forward.argtypes = [vp, vp, u32, vp, u32, vp, vp, vp, vp, vp]
    L.mp_layer_forward_host.argtypes = [vp, vp, u32, vp, u32, vp, vp, vp, vp, vp]
    L.mp_layer_forward_selected.argtypes = [vp, vp, u32, vp, vp, vp, vp, vp]
    L.mp_layer_route.argtypes = [vp, vp, u32, vp, u32, vp, vp, vp]
    L.mp_layer_check_errors.argtypes = [vp, vp]
    L.mp_layer_route_stats.argtypes = [vp, C.POINTER(u32), C.POINTER(u32), vp]
    L.mp_layer_set_profiling.argtypes = [vp, C.c_int]
    L.mp_layer_stage_times.argtypes = [vp, C.c_char_p, sz, vp, vp, C.POINTER(u32), u32]
    L.mp_layer_reset_stage_times.argtypes = [vp]
    L.mp_layer_launch_count.argtypes = [vp]
    L.mp_layer_launch_count.restype = u64
    L.mp_synth_fill.argtypes = [vp, u32, sz, u64, u64, C.c_double, vp]
    L.mp_format_read_mpex.argtypes = [C.c_char_p, C.POINTER(u32), C.POINTER(u32), vp, vp, vp]
    L.mp_format_read_partition_doc.argtypes = [C.c_char_p, sz, C.POINTER(sz), C.POINTER(u64), C.POINTER(u32),
                                               C.POINTER(sz), vp, C.POINTER(u32), C.POINTER(sz), vp, vp]
    L.mp_validate_partition.argtypes = [u32, vp, sz]
    L.mp_layer_forward_selected_host.argtypes = [vp, vp, u32, vp, vp, vp, vp]
    L.mp_ep_create.argtypes = [u32, u32, u32, u32, u32, u32, u32, u32, i32, C.POINTER(vp)]
    L.mp_ep_create_subexpert.argtypes = [u32, u32, u32, u32, u32, u32, u32, u32, i32, C.POINTER(vp)]
    L.mp_ep_destroy.argtypes = [vp]
    L.mp_ep_p2p_setup.argtypes = [vp, u32, vp]
    L.mp_ep_p2p_open.argtypes = [vp, vp]
    L.mp_ep_p2p_pack.argtypes = [vp, vp, vp, vp, u32, vp, C.POINTER(u32), vp]
    L.mp_ep_p2p_recv_buffers.argtypes = [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)]
    L.mp_ep_p2p_return.argtypes = [vp, vp, u32, vp]
    L.mp_ep_p2p_combine.argtypes = [vp, u32, vp, vp]
    L.mp_ep_plan.argtypes = [vp, vp, u32, vp, vp]
    L.mp_ep_pack.argtypes = [vp, vp, vp, vp, u32, vp, vp, vp, vp]
    L.mp_ep_combine.argtypes = [vp, vp, u32, vp, vp]
    L.mp_ep_nccl_unique_id.argtypes = [vp]
    L.mp_ep_nccl_init.argtypes = [vp, vp]
    L.mp_ep_forward.argtypes = [vp, vp, vp, vp, u32, vp, u32, vp, u32, vp]
    L.mp_ep_last_counts.argtypes = [vp, vp, vp]


def load():
    """Load the product library (raises when it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise FileNotFoundError(
                f"{LIB_PATH} missing: build it with __graft_entry__.build() (no CPU fallback exists)")
        lib = C.CDLL(str(LIB_PATH))
        _sig(lib)
        _lib = lib
    return _lib


def check(rc: int):
    if rc == MP_OK:
        return
    msg = load().mp_last_error().decode(errors="replace")
    if rc == MP_ERR_VALIDATION:
        raise ValidationError(msg)
    if rc == MP_ERR_IO:
        raise IoError(msg)
    raise CudaError(msg)
