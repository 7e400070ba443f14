"""ctypes binding of the C-ABI library ``libleann_b200.so`` (include/leann_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).
There is no CPU fallback: importing an op without the library, or calling it
without a CUDA device, raises ``DeviceError``.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

from .errors import DeviceError, raise_for

LIB_PATH = Path(__file__).resolve().parent / "libleann_b200.so"

LV_METRIC = {"l2": 0, "ip": 1, "cosine": 2}
LV_MODE = {"exact_bestfirst": 0, "two_level": 1}
LV_SOURCE_MATRIX = 0
LV_SOURCE_ENCODER = 1
LV_SOURCE_CALLBACK = 2
LV_IO_DEVICE = 1
LV_NO_SHARED_RECOMPUTE = 2
LV_DRY_RECOMPUTE = 4
LV_SMEM_LUT = 8
LV_HASH_VISITED = 16


class IndexDesc(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("dim", C.c_int32), ("metric", C.c_int32),
        ("max_degree", C.c_int32), ("level_count", C.c_int32), ("entry_point", C.c_int64),
        ("level_offsets", C.POINTER(C.c_void_p)), ("level_neighbors", C.POINTER(C.c_void_p)),
        ("level_nnz", C.POINTER(C.c_uint64)), ("deleted", C.c_void_p),
        ("pq_m", C.c_int32), ("pq_padded_dim", C.c_int32),
        ("pq_codebooks", C.c_void_p), ("pq_codes", C.c_void_p),
    ]


class SearchParamsC(C.Structure):
    _fields_ = [
        ("k", C.c_int32), ("ef", C.c_int32), ("rerank_percent", C.c_double),
        ("batch_size", C.c_int32), ("mode", C.c_int32), ("source", C.c_int32),
        ("use_cache", C.c_int32), ("max_inflight", C.c_int32), ("flags", C.c_int32),
    ]


class SearchOutputs(C.Structure):
    _fields_ = [
        ("ids", C.c_void_p), ("dist", C.c_void_p), ("count", C.c_void_p),
        ("counters", C.c_void_p), ("status", C.c_void_p),
        ("visits", C.c_void_p), ("visits_cap", C.c_int32),
        ("batch_log", C.c_void_p), ("batch_log_cap", C.c_int32),
    ]


class SearchStats(C.Structure):
    _fields_ = [
        ("iterations", C.c_int64), ("logical_recomputes", C.c_int64),
        ("physical_encodes", C.c_int64), ("frontier_ms", C.c_double),
        ("encoder_ms", C.c_double), ("total_ms", C.c_double), ("adc_bytes", C.c_int64),
    ]


class EncoderConfigC(C.Structure):
    _fields_ = [
        ("arch", C.c_int32), ("layers", C.c_int32), ("hidden", C.c_int32),
        ("heads", C.c_int32), ("ffn", C.c_int32), ("vocab", C.c_int32),
        ("max_seq", C.c_int32), ("precision", C.c_int32), ("kv_heads", C.c_int32),
        ("head_dim", C.c_int32), ("rope_theta", C.c_float), ("norm_eps", C.c_float),
    ]


class EncoderStats(C.Structure):
    _fields_ = [
        ("passages", C.c_int64), ("gemm_launches", C.c_int64),
        ("gemm_ms", C.c_double), ("gemm_flops", C.c_double), ("gemm_bytes", C.c_double),
        ("attn_launches", C.c_int64), ("attn_ms", C.c_double), ("attn_flops", C.c_double),
        ("attn_bytes", C.c_double), ("fused_launches", C.c_int64), ("fused_ms", C.c_double),
        ("fused_flops", C.c_double), ("fused_bytes", C.c_double),
    ]


# int (*lv_fetch_fn)(void *user, const int64_t *ids, int32_t n, float *rows)
FETCH_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_int64), C.c_int32,
                       C.POINTER(C.c_float))

EXPORTS = {
    "lv_last_error": (C.c_char_p, []),
    "lv_version": (C.c_int, []),
    "lv_kernel_launches": (C.c_longlong, []),
    "lv_index_create": (C.c_int, [C.POINTER(IndexDesc), C.c_int, C.POINTER(C.c_void_p)]),
    "lv_index_destroy": (None, [C.c_void_p]),
    "lv_index_set_matrix": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    "lv_index_set_deleted": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    "lv_index_set_cache": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int]),
    "lv_index_attach_encoder": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                          C.c_int32, C.c_int]),
    "lv_index_set_fetch": (C.c_int, [C.c_void_p, FETCH_FN, C.c_void_p]),
    "lv_index_set_cache_rows": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    "lv_merge_pending": (C.c_int, [C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32,
                                   C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]),
    "lv_distance_gather": (C.c_int, [C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32,
                                     C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "lv_query_norms": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_int,
                                 C.c_void_p]),
    "lv_search_batch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                  C.POINTER(SearchParamsC), C.POINTER(SearchOutputs), C.c_void_p]),
    "lv_last_search_stats": (C.c_int, [C.c_void_p, C.POINTER(SearchStats)]),
    "lv_adc_tables": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p,
                                C.c_int, C.c_void_p]),
    "lv_adc_score": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                               C.c_int, C.c_void_p]),
    "lv_distance_many": (C.c_int, [C.c_int32, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p,
                                   C.c_float, C.c_void_p, C.c_int, C.c_void_p]),
    "lv_encoder_create": (C.c_int, [C.POINTER(EncoderConfigC), C.POINTER(C.c_void_p), C.c_int32,
                                    C.c_int, C.POINTER(C.c_void_p)]),
    "lv_encoder_destroy": (None, [C.c_void_p]),
    "lv_encoder_profile": (C.c_int, [C.c_void_p, C.c_int]),
    "lv_set_gemm_mode": (C.c_int, [C.c_int]),
    "lv_set_attention_mode": (C.c_int, [C.c_int]),
    "lv_set_fused_qkv_attention": (C.c_int, [C.c_int]),
    "lv_attention_gqa_bf16": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                        C.c_int32, C.c_int32, C.c_int32, C.c_void_p]),
    "lv_encoder_set_fused_ln": (C.c_int, [C.c_void_p, C.c_int]),
    "lv_encoder_set_split_residual": (C.c_int, [C.c_void_p, C.c_int]),
    "lv_attention_bf16": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                    C.c_int32, C.c_void_p]),
    "lv_encoder_stats": (C.c_int, [C.c_void_p, C.POINTER(EncoderStats)]),
    "lv_encoder_reset_stats": (C.c_int, [C.c_void_p]),
    "lv_gemm_bf16": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                               C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p]),
    "lv_encode": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_int32, C.c_void_p,
                            C.c_int, C.c_void_p]),
}

_lib = None


def lib():
    """Load (once) and return the library; raises DeviceError if it is missing."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise DeviceError(f"{LIB_PATH.name} not built; run __graft_entry__.build()")
        handle = C.CDLL(str(LIB_PATH))
        for name, (res, args) in EXPORTS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().lv_last_error().decode(errors="replace")
        raise_for(rc, msg)


def require_device() -> None:
    import torch
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the B200 search path has no CPU fallback")


def ptr(a) -> int | None:
    """Address of a numpy array / torch tensor (None passes through)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data
