"""ctypes binding of the C-ABI in include/ngram_b200.h (libngram_b200.so).

This is the Python side of the drop-in boundary: it binds exactly the extern "C"
surface a reference-side FFI would bind (INTEGRATION.md shows the C++ and ctypes
stubs).  The library is loaded from this package directory; if it is missing the
import fails loudly -- there is no CPU fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libngram_b200.so")

NGRAM_OK, NGRAM_EINVAL, NGRAM_ERANGE, NGRAM_EIO, NGRAM_EPARSE = 0, 1, 2, 3, 4
NGRAM_ECONFIG, NGRAM_ENUMERIC, NGRAM_ECUDA, NGRAM_ENCCL, NGRAM_ENOMEM = 5, 6, 7, 8, 9
NGRAM_F32, NGRAM_BF16 = 0, 1
NGRAM_BANK_HASH_ONLY = 1
NGRAM_BWD_SKIP_AMPLIFY = 1
NGRAM_GRAD_SPARSE_ROWS = 1
NGRAM_GRAD_TF32 = 2
NGRAM_GRAD_PEDANTIC = 4
NGRAM_GRAD_EXACT = 8
NGRAM_GRAD_SPARSE_BASE = 16
NGRAM_PLNE_FAST = 1
NGRAM_PLNE_PEDANTIC = 2
NGRAM_SHARD_HANDLE_BYTES = 128

# Exported symbols, in header order (tests check the .so exports every one).
SYMBOLS = [
    "ngram_last_error", "ngram_version", "ngram_kernel_launches", "ngram_config_validate",
    "ngram_make_default_config", "ngram_bank_create", "ngram_bank_create_ex", "ngram_bank_destroy", "ngram_bank_upload_f32",
    "ngram_bank_generate", "ngram_bank_load_file", "ngram_bank_reserve", "ngram_bank_get_info",
    "ngram_rolling_hash_batch", "ngram_hash_ids", "ngram_embed_forward", "ngram_prefill_path", "ngram_embed_from_ids",
    "ngram_sync_errors",
    "ngram_embed_sequence_host", "ngram_hash_ids_host", "ngram_rolling_hash_host", "ngram_embed_from_ids_host",
    "ngram_profile_enable", "ngram_profile_read", "ngram_decode_create", "ngram_decode_destroy", "ngram_decode_reset",
    "ngram_decode_step", "ngram_verify_block", "ngram_commit", "ngram_decode_reset_host", "ngram_decode_step_host",
    "ngram_verify_commit_host",
    "ngram_decode_get_state", "ngram_decode_set_state_host", "ngram_gemm_f32", "ngram_grad_sparse_base", "ngram_f64_forward",
    "ngram_f64_backward", "ngram_f64_amplify", "ngram_f64_amplify_backward", "ngram_f64_gated_ffn",
    "ngram_f64_gated_ffn_backward",
    "ngram_shard_rows", "ngram_shard_group_create", "ngram_shard_group_destroy", "ngram_shard_export", "ngram_shard_open",
    "ngram_shard_local_buffers", "ngram_shard_set_peer", "ngram_shard_scatter_rows", "ngram_shard_project",
    "ngram_shard_xchg_prepare", "ngram_shard_xchg_pack", "ngram_shard_xchg_unpack", "ngram_shard_pack_padded",
    "ngram_shard_home_x",
    "ngram_grad_create", "ngram_grad_destroy", "ngram_grad_zero", "ngram_embed_backward", "ngram_grad_tensor",
    "ngram_grad_download", "ngram_embed_backward_host",
    "ngram_plne_create", "ngram_plne_destroy", "ngram_plne_forward", "ngram_plne_backward",
    "ngram_plne_forward_host", "ngram_plne_backward_host",
    "ngram_grad_create_ex", "ngram_grad_sparse_rows", "ngram_grad_sparse_read", "ngram_amplify_host",
    "ngram_amplify_backward_host", "ngram_decode_ring", "ngram_decode_copy_ring",
    "ngram_analyzer_create", "ngram_analyzer_destroy", "ngram_analyzer_add", "ngram_analyzer_add_host",
    "ngram_analyzer_merge", "ngram_analyzer_sync_errors", "ngram_analyzer_stats", "ngram_analyzer_reserve",
    "ngram_plne_create_ex",
]


class NgramError(Exception):
    status = -1


class InvalidArgument(NgramError, ValueError):  # std::invalid_argument
    status = NGRAM_EINVAL


class OutOfRange(NgramError, IndexError):  # std::out_of_range
    status = NGRAM_ERANGE


class IoError(NgramError, OSError):  # ngram::io_error
    status = NGRAM_EIO


class ParseError(NgramError):  # ngram::parse_error
    status = NGRAM_EPARSE


class ConfigError(NgramError):  # ngram::config_error
    status = NGRAM_ECONFIG


class NumericError(NgramError):  # ngram::numeric_error
    status = NGRAM_ENUMERIC


class CudaError(NgramError, RuntimeError):
    status = NGRAM_ECUDA


_EXC = {NGRAM_EINVAL: InvalidArgument, NGRAM_ERANGE: OutOfRange, NGRAM_EIO: IoError, NGRAM_EPARSE: ParseError,
        NGRAM_ECONFIG: ConfigError, NGRAM_ENUMERIC: NumericError, NGRAM_ECUDA: CudaError, NGRAM_ENCCL: CudaError,
        NGRAM_ENOMEM: MemoryError}


class BankInfo(C.Structure):
    _fields_ = [("max_order", C.c_int), ("sub_tables", C.c_int), ("dim", C.c_int), ("branch_count", C.c_int),
                ("branch_dim", C.c_int), ("variant", C.c_int), ("amplification", C.c_int),
                ("merge_denominator", C.c_int), ("base_vocab", C.c_uint32), ("shard_rank", C.c_int),
                ("shard_count", C.c_int), ("tensor_core_path", C.c_int), ("device_bytes", C.c_uint64),
                ("sub_vocab", C.c_uint64 * 64), ("row_lo", C.c_int64 * 64), ("row_hi", C.c_int64 * 64),
                ("sub_ptr", C.c_void_p), ("e0_ptr", C.c_void_p), ("wcat_ptr", C.c_void_p)]


_LIB = None


def lib() -> C.CDLL:
    """Load libngram_b200.so (raises if it was not built -- no fallback)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2601_21204_b200.build` "
                          "(the CUDA path is the only implementation)")
    L = C.CDLL(LIB_PATH)
    vp, i64, i32, u32, u64 = C.c_void_p, C.c_int64, C.c_int, C.c_uint32, C.c_uint64
    sig = {
        "ngram_last_error": ([], C.c_char_p),
        "ngram_version": ([], C.c_char_p),
        "ngram_kernel_launches": ([], u64),
        "ngram_config_validate": ([C.c_char_p], i32),
        "ngram_make_default_config": ([u32, i32, i32, i32, C.c_char_p, C.c_size_t], i32),
        "ngram_bank_create": ([C.c_char_p, i32, i32, i32, C.POINTER(vp)], i32),
        "ngram_bank_create_ex": ([C.c_char_p, i32, i32, i32, i32, C.POINTER(vp)], i32),
        "ngram_bank_destroy": ([vp], i32),
        "ngram_bank_upload_f32": ([vp, vp, vp, vp, vp, vp], i32),
        "ngram_bank_generate": ([vp, u64, vp], i32),
        "ngram_bank_load_file": ([vp, C.c_char_p], i32),
        "ngram_bank_reserve": ([vp, i64], i32),
        "ngram_bank_get_info": ([vp, C.POINTER(BankInfo)], i32),
        "ngram_rolling_hash_batch": ([vp, i64, vp, vp, vp, vp, i64, vp, vp, vp], i32),
        "ngram_hash_ids": ([vp, vp, vp, i64, i64, vp, vp, i32, vp], i32),
        "ngram_embed_forward": ([vp, vp, vp, i64, i64, vp, vp, vp, i32, vp], i32),
        "ngram_prefill_path": ([vp, i64, vp], i32),
        "ngram_embed_from_ids": ([vp, vp, vp, i64, vp, i32, vp], i32),
        "ngram_sync_errors": ([vp, vp], i32),
        "ngram_embed_sequence_host": ([vp, vp, vp, i64, vp, vp, vp, i32], i32),
        "ngram_hash_ids_host": ([vp, vp, vp, i64, vp, vp], i32),
        "ngram_rolling_hash_host": ([vp, i64, vp, vp, vp, vp, i64, vp, vp], i32),
        "ngram_embed_from_ids_host": ([vp, vp, vp, i64, vp], i32),
        "ngram_profile_enable": ([vp, i32], i32),
        "ngram_profile_read": ([vp, C.POINTER(C.c_float), i32], i32),
        "ngram_decode_create": ([vp, i64, i32, C.POINTER(vp)], i32),
        "ngram_decode_destroy": ([vp], i32),
        "ngram_decode_reset": ([vp, vp, vp, vp], i32),
        "ngram_decode_step": ([vp, vp, vp, vp, i32, vp], i32),
        "ngram_verify_block": ([vp, vp, i32, vp, i32, vp], i32),
        "ngram_commit": ([vp, vp, i32, vp, vp], i32),
        "ngram_decode_reset_host": ([vp, vp, vp], i32),
        "ngram_decode_step_host": ([vp, vp, vp, vp], i32),
        "ngram_verify_commit_host": ([vp, vp, i32, vp, vp], i32),
        "ngram_decode_get_state": ([vp, vp, vp, vp], i32),
        "ngram_decode_set_state_host": ([vp, vp, vp, vp], i32),
        "ngram_grad_sparse_base": ([vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(i64)], i32),
        "ngram_gemm_f32": ([i32, i64, i64, i64, vp, i64, i32, vp, i64, i32, vp, i64, i32, i32, i32, vp], i32),
        "ngram_f64_forward": ([C.c_char_p, vp, vp, vp, vp, vp, vp, i64, vp, i64, vp, vp], i32),
        "ngram_f64_backward": ([C.c_char_p, vp, vp, vp, vp, vp, vp, i64, vp, i64, vp, vp, vp, vp, vp, vp, vp], i32),
        "ngram_f64_amplify": ([i32, i64, vp, vp, vp, vp], i32),
        "ngram_f64_amplify_backward": ([i32, i64, vp, vp, vp, vp, vp, vp], i32),
        "ngram_f64_gated_ffn": ([i32, i32, vp, vp, vp, vp, vp], i32),
        "ngram_f64_gated_ffn_backward": ([i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp], i32),
        "ngram_shard_rows": ([u64, i32, i32, C.POINTER(i64), C.POINTER(i64)], i32),
        "ngram_shard_group_create": ([vp, i64, C.POINTER(vp)], i32),
        "ngram_shard_group_destroy": ([vp], i32),
        "ngram_shard_export": ([vp, vp], i32),
        "ngram_shard_open": ([vp, i32, vp], i32),
        "ngram_shard_local_buffers": ([vp, C.POINTER(vp), C.POINTER(vp)], i32),
        "ngram_shard_set_peer": ([vp, i32, vp, vp], i32),
        "ngram_shard_scatter_rows": ([vp, vp, vp, i64, i64, vp, vp, vp], i32),
        "ngram_shard_project": ([vp, vp, i64, vp, vp, i32, vp], i32),
        "ngram_shard_xchg_prepare": ([vp, vp, vp, i64, i64, vp, vp, vp, vp, vp], i32),
        "ngram_shard_xchg_pack": ([vp, vp, vp], i32),
        "ngram_shard_xchg_unpack": ([vp, vp, vp], i32),
        "ngram_shard_pack_padded": ([vp, vp, vp, i64, i64, vp, vp, vp, vp], i32),
        "ngram_shard_home_x": ([vp, C.POINTER(vp)], i32),
        "ngram_grad_create": ([vp, C.POINTER(vp)], i32),
        "ngram_grad_destroy": ([vp], i32),
        "ngram_grad_zero": ([vp, vp], i32),
        "ngram_embed_backward": ([vp, vp, vp, i64, i64, vp, vp, vp, i32, vp], i32),
        "ngram_grad_tensor": ([vp, i32, C.POINTER(vp), C.POINTER(i64)], i32),
        "ngram_grad_download": ([vp, vp, vp, vp, vp, vp], i32),
        "ngram_embed_backward_host": ([vp, vp, vp, i64, vp, vp, vp, i32], i32),
        "ngram_plne_create": ([vp, i32, C.POINTER(vp)], i32),
        "ngram_plne_destroy": ([vp], i32),
        "ngram_plne_forward": ([vp, vp, vp, vp, vp, vp, i64, i64, vp, vp, vp], i32),
        "ngram_plne_backward": ([vp, vp, vp, vp, vp, vp, vp, i64, i64, vp, vp, vp, vp, vp, vp], i32),
        "ngram_plne_forward_host": ([vp, vp, vp, vp, vp, vp, i64, vp, vp], i32),
        "ngram_grad_create_ex": ([vp, i32, C.POINTER(vp)], i32),
        "ngram_grad_sparse_rows": ([vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(i64)], i32),
        "ngram_grad_sparse_read": ([vp, i64, i64, vp, vp, vp], i32),
        "ngram_amplify_host": ([i32, i32, i64, vp, vp, vp, vp], i32),
        "ngram_amplify_backward_host": ([vp, i64, vp, vp, vp, vp, vp], i32),
        "ngram_decode_ring": ([vp, C.POINTER(vp)], i32),
        "ngram_decode_copy_ring": ([vp, vp, vp], i32),
        "ngram_plne_backward_host": ([vp, vp, vp, vp, vp, vp, vp, i64, vp, vp, vp, vp, vp], i32),
        "ngram_analyzer_create": ([i32, u64, vp, i32, vp, i32, C.POINTER(vp)], i32),
        "ngram_analyzer_destroy": ([vp], None),
        "ngram_analyzer_add": ([vp, vp, vp, i64, i64, vp], i32),
        "ngram_analyzer_add_host": ([vp, vp, vp, i64], i32),
        "ngram_analyzer_merge": ([vp, vp, vp], i32),
        "ngram_analyzer_sync_errors": ([vp], i32),
        "ngram_analyzer_reserve": ([vp, u64], i32),
        "ngram_plne_create_ex": ([vp, i32, i32, C.POINTER(vp)], i32),
        "ngram_analyzer_stats": ([vp, vp, vp, vp, vp, vp], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _LIB = L
    return L


def check(rc: int) -> None:
    """Raise the Python mirror of the reference exception for a non-zero status."""
    if rc != NGRAM_OK:
        msg = lib().ngram_last_error().decode(errors="replace")
        raise _EXC.get(rc, NgramError)(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))
