"""ctypes binding of libcocob200 (include/cocob200.h).

This is the only place the package touches the native library.  Loading fails
loudly when the .so is missing: there is no CPU fallback on the product path.
Status codes are mapped onto the reference's exception classes
(ops.py:24-46): CB_EINVAL -> OpError, CB_ENOMEM -> InfeasibleOpError,
CB_ENOREPLICA -> MissingReplicaError, everything else -> RuntimeError.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("COCOB200_LIB") or Path(__file__).resolve().parent / "libcocob200.so")  # override: A/B experiments

CB_OK = 0
CB_EINVAL = -1
CB_ENOMEM = -2
CB_ENOREPLICA = -3
CB_ECUDA = -4
CB_ESTATE = -5
CB_ENOTSUP = -6
CB_ECOMM = -7

PHASE_PREFILL = 0
PHASE_DECODE = 1

# ModuleKind ids in reference declaration order (domain.py:23-36)
KIND_IDS = {
    "attn_proj_q": 0,
    "attn_proj_k": 1,
    "attn_proj_v": 2,
    "attn_proj_o": 3,
    "self_attention": 4,
    "ffn_proj_gate": 5,
    "ffn_proj_up": 6,
    "ffn_proj_down": 7,
    "decoder_layer": 8,
    "kv_cache": 9,
    "attn_norm": 10,
    "ffn_norm": 11,
}


class ModelDesc(C.Structure):
    _fields_ = [
        ("n_layers", C.c_int32),
        ("d_model", C.c_int32),
        ("d_ff", C.c_int32),
        ("n_heads", C.c_int32),
        ("n_kv_heads", C.c_int32),
        ("vocab", C.c_int32),
        ("max_slots", C.c_int32),
        ("max_ctx", C.c_int32),
        ("max_tokens", C.c_int32),
        ("rope_theta", C.c_float),
        ("norm_eps", C.c_float),
    ]


class LayerWeights(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in (
        "attn_norm", "wq", "wk", "wv", "wo", "ffn_norm", "w_gate", "w_up", "w_down")]


class OpStats(C.Structure):
    _fields_ = [
        ("weight_bytes", C.c_uint64),
        ("kv_bytes", C.c_uint64),
        ("device_ms", C.c_float),
        ("shortfall_bytes", C.c_uint64),
        ("copy_ms", C.c_float),
        ("catchup_ms", C.c_float),
        ("catchup_bytes", C.c_uint64),
        ("done", C.c_int32),
        ("committed", C.c_int32),
    ]


class MemStats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "weight_bytes", "kv_bytes", "workspace_bytes", "reserved_bytes", "free_bytes", "total_bytes")]


class KStat(C.Structure):
    _fields_ = [("launches", C.c_uint32), ("ms", C.c_float), ("bytes", C.c_double), ("flops", C.c_double)]


KCLASSES = ("gemm", "attention", "elementwise", "copy")

_P = C.c_void_p
# cross-process transport callback of the SPMD runtime (cb_xfer_fn)
XFER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_uint64, C.c_void_p)
_I32P = C.POINTER(C.c_int32)
_I64P = C.POINTER(C.c_int64)
_F32P = C.POINTER(C.c_float)

_SIGS = {
    "cb_abi_version": (C.c_int, []),
    "cb_last_error": (C.c_char_p, []),
    "cb_split_batch": (C.c_int, [C.c_int32, C.c_int32, _I32P]),
    "cb_runtime_create": (C.c_int, [C.c_int32, _I32P, C.POINTER(_P)]),
    "cb_runtime_create_spmd": (C.c_int, [C.c_int32, _I32P, C.c_int32, C.c_int32, XFER_FN, _P, C.POINTER(_P)]),
    "cb_device_is_local": (C.c_int, [_P, C.c_int32, _I32P]),
    "cb_runtime_destroy": (C.c_int, [_P]),
    "cb_device_info": (C.c_int, [_P, C.c_int32, _I32P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "cb_model_create": (C.c_int, [_P, C.POINTER(ModelDesc), C.c_int32, C.POINTER(_P)]),
    "cb_model_destroy": (C.c_int, [_P]),
    "cb_module_bytes": (C.c_uint64, [_P, C.c_int32]),
    "cb_layer_load": (C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(LayerWeights)]),
    "cb_layer_init_random": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_uint64, C.c_float]),
    "cb_head_load": (C.c_int, [_P, _P, _P, _P]),
    "cb_head_init_random": (C.c_int, [_P, C.c_uint64, C.c_float]),
    "cb_module_read": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, _P, C.c_uint64]),
    "cb_kv_read": (C.c_int, [_P, C.c_int32, C.c_int32, _P, C.c_uint64, _I32P]),
    "cb_slot_len": (C.c_int, [_P, C.c_int32, _I32P]),
    "cb_get_placement": (C.c_int, [_P, _I64P, _I32P, C.c_int32, _I32P]),
    "cb_step": (C.c_int, [_P, C.c_int32, C.c_int32, _I32P, _I32P, _I32P, _I32P, _F32P, _F32P]),
    "cb_release_slots": (C.c_int, [_P, C.c_int32, _I32P]),
    "cb_last_routing": (C.c_int, [_P, C.c_int32, _I32P, _I32P, _I32P, C.c_int32, _I32P]),
    "cb_replicate_layer": (C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(OpStats)]),
    "cb_migrate_layer": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, C.POINTER(OpStats)]),
    "cb_migrate_submodule": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, C.POINTER(OpStats)]),
    "cb_evict_replica": (C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(OpStats)]),
    "cb_issue_replicate_layer": (C.c_int, [_P, C.c_int32, C.c_int32, _I64P, C.POINTER(C.c_uint64)]),
    "cb_issue_migrate_layer": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, _I64P, C.POINTER(C.c_uint64)]),
    "cb_issue_migrate_submodule": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, _I64P, C.POINTER(C.c_uint64)]),
    "cb_issue_evict_replica": (C.c_int, [_P, C.c_int32, C.c_int32, _I64P]),
    "cb_op_start": (C.c_int, [_P, C.c_int64]),
    "cb_op_poll": (C.c_int, [_P, C.c_int64, _I32P]),
    "cb_op_wait": (C.c_int, [_P, C.c_int64, C.POINTER(OpStats)]),
    "cb_commit": (C.c_int, [_P, C.c_int64, _I32P]),
    "cb_op_abort": (C.c_int, [_P, C.c_int64]),
    "cb_pending_ops": (C.c_int, [_P, _I32P]),
    "cb_mem_usage": (C.c_int, [_P, C.c_int32, C.POINTER(MemStats)]),
    "cb_set_copy_mode": (C.c_int, [_P, C.c_int32, C.c_uint64]),
    "cb_kv_offload": (C.c_int, [_P, C.c_int32, C.c_int32, C.POINTER(OpStats)]),
    "cb_kv_offloaded": (C.c_int, [_P, C.c_int32, _I32P]),
    "cb_profile": (C.c_int, [_P, C.c_int32]),
    "cb_profile_read": (C.c_int, [_P, C.c_int32, C.POINTER(KStat)]),
    # kernel-level test entry points (include/cocob200_testing.h)
    "cbt_gemm": (C.c_int, [_P, _P, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P, C.c_int64]),
    "cbt_gemm_plan": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P]),
    "cbt_gemm_bench": (C.c_int, [_P, _P, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P, C.c_int64,
                                 C.c_int32, C.c_int32, _F32P]),
    "cbt_rmsnorm": (C.c_int, [_P, _P, _P, C.c_int32, C.c_int32, C.c_float]),
    "cbt_rope_kv": (C.c_int, [_P, _P, _P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_float]),
    "cbt_attention": (C.c_int, [_P, _P, _P, _P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
    "cbt_attention_fused": (C.c_int, [_P, _P, _P, _P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                      C.c_float]),
    "cbt_attention_set_kv_slots": (C.c_int, [C.c_int32]),
    "cbt_attention_bench": (C.c_int, [_P, _P, _P, _P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                      C.c_int32, C.c_int32, _F32P]),
    "cbt_argmax": (C.c_int, [_P, _P, C.c_int32, C.c_int32]),
    "cbt_prefill_attention": (C.c_int, [_P, _P, _P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                        C.c_int32, C.c_int32]),
    "cbt_gemm_trace": (C.c_int, [_P, C.c_int32]),
    "cbt_mma_probe": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_double)]),
    "cbt_gemm_set_wcopies": (C.c_int, [C.c_int32, C.c_int64]),
    "cbt_last_enqueue_ms": (C.c_double, []),
    "cbt_gemm_set_norm": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_float]),
    "cbt_tma_probe": (C.c_int, [_P, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                C.c_int32, _F32P]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load():
    """Load libcocob200.so; raises (never falls back) if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2507_18006_b200._build` "
            "(there is no CPU fallback for the data path)")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    msg = load().cb_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str = "", shortfall_bytes: int = 0) -> None:
    """Raise the reference-compatible exception for a CB_E* status."""
    if status == CB_OK:
        return
    raise_status(status, f"{what}: {last_error()}" if what else last_error(), shortfall_bytes)


def raise_status(status: int, msg: str, shortfall_bytes: int = 0) -> None:
    """Raise the exception class of a CB_E* status with a given message."""
    from .ops import InfeasibleOpError, MissingReplicaError, OpError

    if status == CB_EINVAL:
        raise OpError(msg)
    if status == CB_ENOMEM:
        raise InfeasibleOpError(msg, shortfall_mb=shortfall_bytes / 1e6)
    if status == CB_ENOREPLICA:
        raise MissingReplicaError(msg)
    if status == CB_ENOTSUP:
        raise NotImplementedError(msg)
    raise RuntimeError(f"libcocob200 error {status}: {msg}")


def i32(arr):
    """ctypes int32 pointer to a contiguous numpy int32 array."""
    return arr.ctypes.data_as(_I32P)


def f32(arr):
    return arr.ctypes.data_as(_F32P)
