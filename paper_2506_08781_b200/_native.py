"""ctypes binding of the C-ABI in include/poslo_gpu.h (libposlo_gpu.so).

The shared library is built in-tree by __graft_entry__.build() (or
`make -C paper_2506_08781_b200/csrc`). There is deliberately no fallback:
if the library is missing or no sm_100 device is present, every call raises.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libposlo_gpu.so")

OK, FORMAT_ERROR, STATE_ERROR, SEED_NOT_DISCLOSED, CUDA_ERROR, INVALID_ARGUMENT = range(6)


class PosloError(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("epoch", ctypes.c_uint32), ("message", ctypes.c_char * 240)]


class PosloBatch(ctypes.Structure):
    _fields_ = [
        ("suite", ctypes.c_uint8),
        ("n2", ctypes.c_uint32),
        ("payload", ctypes.c_void_p),
        ("payload_bytes", ctypes.c_uint64),
        ("offsets", ctypes.c_void_p),
        ("entry_len", ctypes.c_uint32),
        ("n_entries", ctypes.c_uint64),
        ("epochs", ctypes.c_void_p),
        ("epoch_starts", ctypes.c_void_p),
        ("n_epochs", ctypes.c_uint32),
        ("ds", ctypes.c_void_p),
        ("ds_len", ctypes.c_uint32),
        ("ds_capacity", ctypes.c_uint32),
        ("device_resident", ctypes.c_int32),
        ("ds_offsets", ctypes.c_void_p),
        ("record_header", ctypes.c_uint32),
        ("fill", ctypes.c_void_p),       # int (*)(void*, uint64_t, uint64_t, uint8_t*) or NULL
        ("fill_user", ctypes.c_void_p),
    ]


# poslo_batch.fill: int fill(void* user, uint64_t first, uint64_t count, uint8_t* dst)
FILL_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p)


class PosloFineBatch(ctypes.Structure):
    _fields_ = [
        ("suite", ctypes.c_uint8),
        ("payload", ctypes.c_void_p),
        ("payload_bytes", ctypes.c_uint64),
        ("offsets", ctypes.c_void_p),
        ("entry_len", ctypes.c_uint32),
        ("n_entries", ctypes.c_uint64),
        ("device_resident", ctypes.c_int32),
        ("seeds", ctypes.c_void_p),
        ("derive_slot", ctypes.c_void_p),
        ("j", ctypes.c_void_p),
        ("slot_epochs", ctypes.c_void_p),
        ("n_slots", ctypes.c_uint32),
        ("ds", ctypes.c_void_p),
        ("ds_len", ctypes.c_uint32),
        ("ds_capacity", ctypes.c_uint32),
        ("ds_offsets", ctypes.c_void_p),
    ]


EXPORTS = [
    "poslo_gpu_create", "poslo_gpu_destroy", "poslo_gpu_set_stream", "poslo_gpu_enable_timing",
    "poslo_gpu_last_timings", "poslo_gpu_last_launches", "poslo_gpu_version", "poslo_gpu_agg_ekeys",
    "poslo_gpu_paver", "poslo_gpu_epoch_verify", "poslo_gpu_sebver", "poslo_gpu_commit_check",
    "poslo_gpu_group_fold", "poslo_gpu_point_valid", "poslo_gpu_seed_retrieve",
    "poslo_gpu_entry_scalars", "poslo_gpu_group_check", "poslo_gpu_scalar_sum", "poslo_gpu_synth_log",
    "poslo_gpu_synth_varlog", "poslo_gpu_distill_coarse", "poslo_gpu_segfold", "poslo_gpu_fine_scalars",
    "poslo_gpu_fine_verify", "poslo_gpu_aver_f_batch", "poslo_log_scan", "poslo_gpu_kg_commitments",
    "poslo_gpu_sig_epochs", "poslo_gpu_log_scan", "poslo_gpu_create_multi", "poslo_gpu_member_count",
    "poslo_gpu_device_count", "poslo_gpu_agg_ekeys_partial", "poslo_gpu_combine_check",
    "poslo_gpu_group_op_counts", "poslo_gpu_reset_group_op_counts", "poslo_gpu_distill_coarse_ex",
    "poslo_gpu_distill_step", "poslo_gpu_combine_check_prepare",
]

_lib = None


def load():
    """Loads libposlo_gpu.so; raises (never falls back) when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
            "(the B200 verifier has no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    c = ctypes
    P = c.c_void_p
    E = c.POINTER(PosloError)
    B = c.POINTER(PosloBatch)
    F = c.POINTER(PosloFineBatch)
    sig = {
        "poslo_gpu_create": ([c.c_int, c.POINTER(c.c_void_p), E], c.c_int),
        "poslo_gpu_destroy": ([P], None),
        "poslo_gpu_set_stream": ([P, P], c.c_int),
        "poslo_gpu_enable_timing": ([P, c.c_int], c.c_int),
        "poslo_gpu_last_timings": ([P, c.POINTER(c.c_float)], c.c_int),
        "poslo_gpu_last_launches": ([P], c.c_uint32),
        "poslo_gpu_version": ([], c.c_char_p),
        "poslo_gpu_agg_ekeys": ([P, B, P, P, E], c.c_int),
        "poslo_gpu_paver": ([P, B, P, P, P, P, P, E], c.c_int),
        "poslo_gpu_epoch_verify": ([P, B, P, P, P, P, P, E], c.c_int),
        "poslo_gpu_sebver": ([P, B, P, c.c_uint32, c.c_uint32, P, P, P, c.c_uint32, P, P, P, P, P,
                              P, c.c_uint32, P, P, E], c.c_int),
        "poslo_gpu_commit_check": ([P, c.c_uint32, P, P, P, P, E], c.c_int),
        "poslo_gpu_group_fold": ([P, c.c_uint64, P, P, E], c.c_int),
        "poslo_gpu_point_valid": ([P, c.c_uint32, P, P, E], c.c_int),
        "poslo_gpu_seed_retrieve": ([P, c.c_uint8, P, c.c_uint32, c.c_uint32, P, c.c_uint32, P, E],
                                    c.c_int),
        "poslo_gpu_entry_scalars": ([P, B, P, E], c.c_int),
        "poslo_gpu_group_check": ([P, c.c_uint32, P, P, P, P, P, E], c.c_int),
        "poslo_gpu_scalar_sum": ([P, c.c_uint64, P, P, E], c.c_int),
        "poslo_gpu_synth_log": ([P, c.c_uint64, c.c_uint64, c.c_uint64, c.c_uint32, P, E], c.c_int),
        "poslo_gpu_synth_varlog": ([P, c.c_uint64, c.c_uint64, c.c_uint64, P, P, E], c.c_int),
        "poslo_gpu_distill_coarse": ([P, B, P, P, P, P, c.c_uint32, P, P, P, E], c.c_int),
        "poslo_gpu_segfold": ([P, c.c_uint32, P, P, P, P, c.c_uint32, P, P, E], c.c_int),
        "poslo_gpu_fine_scalars": ([P, F, P, P, E], c.c_int),
        "poslo_gpu_fine_verify": ([P, F, P, P, P, P, E], c.c_int),
        "poslo_gpu_aver_f_batch": ([P, F, P, P, P, P, E], c.c_int),
        "poslo_log_scan": ([P, c.c_uint64, P, c.c_uint64, c.POINTER(c.c_uint64), E], c.c_int),
        "poslo_gpu_kg_commitments": ([P, c.c_uint8, P, P, c.c_uint32, c.c_uint32, P, P, E], c.c_int),
        "poslo_gpu_sig_epochs": ([P, B, P, P, P, E], c.c_int),
        "poslo_gpu_log_scan": ([P, P, c.c_uint64, c.c_int32, P, c.c_uint64, c.POINTER(c.c_uint64), E], c.c_int),
        "poslo_gpu_create_multi": ([c.POINTER(c.c_int), c.c_int, c.POINTER(c.c_void_p), E], c.c_int),
        "poslo_gpu_member_count": ([P], c.c_int),
        "poslo_gpu_device_count": ([], c.c_int),
        "poslo_gpu_agg_ekeys_partial": ([P, B, P, E], c.c_int),
        "poslo_gpu_combine_check": ([P, c.c_uint32, P, c.c_int32, P, P, P, P, E], c.c_int),
        "poslo_gpu_group_op_counts": ([c.POINTER(c.c_uint64)], None),
        "poslo_gpu_reset_group_op_counts": ([], None),
        "poslo_gpu_distill_coarse_ex": ([P, B, P, P, P, P, c.c_uint32, P, P, P, P, E], c.c_int),
        "poslo_gpu_distill_step": ([P, B, P, P, P, P, P, P, P, P, E], c.c_int),
        "poslo_gpu_combine_check_prepare": ([P, P, P, P, E], c.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib
