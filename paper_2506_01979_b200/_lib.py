"""ctypes binding of libspecbranch.so (include/specbranch.h).  Argument marshalling only:
every step of the verify-and-branch path runs in the library's CUDA kernels.  There is
no CPU fallback — a missing or unloadable library raises."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.environ.get("SB_LIB_PATH") or os.path.join(HERE, "libspecbranch.so")  # override: A/B builds

SB_OK, SB_ERR_INVALID_ARG, SB_ERR_UNSUPPORTED, SB_ERR_CUDA, SB_ERR_NCCL, SB_ERR_WORKSPACE = range(6)
SB_BF16, SB_F32 = 0, 1
SB_SELECT_EQ9, SB_SELECT_ALG1 = 0, 1
SB_CONF_TOP1, SB_CONF_TOKEN, SB_CONF_ENTROPY = 0, 1, 2
SB_ST_GAMMA_CLAMPED, SB_ST_BRANCH_CLAMPED, SB_ST_BAD_TOKEN, SB_ST_NONFINITE, SB_ST_ZERO_RESID = 1, 2, 4, 8, 16
SB_ST_BAD_PARENT, SB_ST_RANGE = 32, 64

# every symbol include/specbranch.h declares
EXPORTS = ("sb_version", "sb_status_string", "sb_workspace_bytes", "sb_verify_branches",
           "sb_select_branch", "sb_verify_select", "sb_step_adaptive", "sb_verify_branches_reuse", "sb_draft_confidence", "sb_spawn_branches", "sb_kv_rollback", "sb_tree_workspace_bytes", "sb_tree_verify", "sb_hrad_workspace_bytes", "sb_hrad_predict", "sb_shard_partial_bytes", "sb_shard_verify_local",
           "sb_shard_verify_combine", "sb_shard_select_local", "sb_shard_select_sample",
           "sb_shard_select_commit", "sb_comm_unique_id_bytes", "sb_comm_unique_id", "sb_comm_create",
           "sb_comm_destroy", "sb_comm_check", "sb_comm_abort")


class sb_dims(ctypes.Structure):
    _fields_ = [
        ("B", ctypes.c_int32), ("K", ctypes.c_int32), ("G", ctypes.c_int32), ("V", ctypes.c_int32),
        ("v_offset", ctypes.c_int32), ("v_total", ctypes.c_int32),
        ("row_stride", ctypes.c_int64), ("seq_stride", ctypes.c_int64),
        ("dtype", ctypes.c_int32), ("reserved", ctypes.c_int32),
    ]


_P = ctypes.c_void_p
_I = ctypes.c_int
_F = ctypes.c_float
_S = ctypes.c_size_t
_D = ctypes.POINTER(sb_dims)

_SIGS = {
    "sb_version": ([], ctypes.c_char_p),
    "sb_status_string": ([_I], ctypes.c_char_p),
    "sb_workspace_bytes": ([_D], _S),
    "sb_verify_branches": ([_D] + [_P] * 18 + [_S, _P], _I),
    "sb_verify_branches_reuse": ([_D] + [_P] * 18 + [_S, _P], _I),
    "sb_select_branch": ([_D] + [_P] * 8 + [_I] + [_P] * 14 + [_S, _P], _I),
    "sb_draft_confidence": ([_D, _P, _P, _I, _F, _F, ctypes.c_int32] + [_P] * 10 + [_S, _P], _I),
    "sb_verify_select": ([_D] + [_P] * 7 + [_I] + [_P] * 22 + [_S, _P], _I),
    "sb_step_adaptive": ([_D] + [_P] * 6 + [_I, _F, ctypes.c_int32] + [_P] * 7 + [_P] * 21 + [_P, _S, _P, _S, _P], _I),
    "sb_spawn_branches": ([_D, _P, _P, _P, _I, ctypes.c_int32] + [_P] * 4 + [_P], _I),
    "sb_kv_rollback": ([_I, _I, _I, _P, ctypes.c_int64, ctypes.c_int64, _P, _P, _P], _I),
    "sb_tree_workspace_bytes": ([_D], _S),
    "sb_hrad_workspace_bytes": ([_I, _I], _S),
    "sb_hrad_predict": ([_I, _I, _I] + [_P] * 12 + [_P, _S, _P], _I),
    "sb_tree_verify": ([_D] + [_P] * 16 + [_S, _P], _I),
    "sb_shard_partial_bytes": ([_D], _S),
    "sb_shard_verify_local": ([_D] + [_P] * 8 + [_S, _P], _I),
    "sb_shard_verify_combine": ([_D, _P, _I] + [_P] * 13 + [_S, _P], _I),
    "sb_shard_select_local": ([_D] + [_P] * 5 + [_I, _P, _P, _S, _P], _I),
    "sb_shard_select_sample": ([_D, _P, _I, _I] + [_P] * 5 + [_S, _P], _I),
    "sb_shard_select_commit": ([_D] + [_P] * 15 + [_S, _P], _I),
    "sb_comm_unique_id_bytes": ([], _S),
    "sb_comm_unique_id": ([_P], _I),
    "sb_comm_create": ([_P, _I, _I, _D, ctypes.POINTER(ctypes.c_void_p)], _I),
    "sb_comm_destroy": ([_P], _I),
    "sb_comm_check": ([_P], _I),
    "sb_comm_abort": ([_P], _I),
}

_lib = None


def lib():
    """Load libspecbranch.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            raise RuntimeError(
                f"{SO} is missing: build it with `python -m paper_2506_01979_b200.build` "
                "(the verify-and-branch path has no CPU fallback)")
        L = ctypes.CDLL(SO)
        for name, (args, res) in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def check(rc: int, what: str):
    if rc != SB_OK:
        msg = lib().sb_status_string(rc).decode()
        raise RuntimeError(f"{what} failed: {msg} ({rc})")
