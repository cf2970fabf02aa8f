"""ctypes binding of libf2gpu.so (the C-ABI in include/f2gpu.h).

There is no fallback: if the shared library is missing or the device is not a
B200 (sm_100a), every entry point raises.  Status codes are translated into the
Python analogues of the reference's exceptions:
  F2GPU_EINVAL -> ValueError   (std::invalid_argument, e.g. m4rm.hpp:181)
  F2GPU_ERANGE -> IndexError   (std::out_of_range, e.g. m4rm.hpp:100,145)
  others       -> F2GpuError   (CUDA / NCCL / allocation failures)
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(os.environ["F2GPU_LIB"]) if os.environ.get("F2GPU_LIB") else Path(__file__).resolve().parent / "libf2gpu.so"  # F2GPU_LIB: A/B builds

OK, EINVAL, ERANGE, ECUDA, ENCCL, ENOMEM = range(6)
OWN_STREAM = (1 << 64) - 1  # F2GPU_OWN_STREAM (include/f2gpu.h)


class F2GpuError(RuntimeError):
    pass


# every exported symbol declared in include/f2gpu.h
SYMBOLS = [
    "f2gpu_last_error", "f2gpu_version", "f2gpu_options_describe",
    "f2gpu_ctx_create", "f2gpu_ctx_destroy", "f2gpu_ctx_set_stream", "f2gpu_ctx_sync",
    "f2gpu_ctx_launches", "f2gpu_ctx_set_strassen_cutover", "f2gpu_ctx_set_tc",
    "f2gpu_mat_alloc", "f2gpu_mat_free", "f2gpu_mat_shape", "f2gpu_mat_device_ptr",
    "f2gpu_mat_zero", "f2gpu_mat_upload", "f2gpu_mat_download", "f2gpu_mat_random_dense",
    "f2gpu_mat_copy", "f2gpu_mat_select_wcols", "f2gpu_mat_xor", "f2gpu_mat_transpose",
    "f2gpu_m4rm_mult", "f2gpu_m4rm_mult_acc", "f2gpu_mult_acc", "f2gpu_mult_acc_host", "f2gpu_strassen_mult",
    "f2gpu_gemm_tc",
    "f2gpu_update_tc", "f2gpu_panel_build_z", "f2gpu_trace_enable", "f2gpu_trace_read", "f2gpu_debug_panel_chain",
    "f2gpu_decompose_block", "f2gpu_decompose_recursive", "f2gpu_decompose_block_sharded",
    "f2gpu_rank",
    "f2gpu_m4rm_mult_host", "f2gpu_strassen_mult_host", "f2gpu_decompose_block_host",
    "f2gpu_decompose_recursive_host", "f2gpu_null_space", "f2gpu_solve",
    "f2gpu_rank_host",
    "f2gpu_nccl_unique_id", "f2gpu_ctx_init_comm", "f2gpu_decompose_block_dist",
    "f2gpu_decompose_recursive_dist", "f2gpu_decompose_recursive_sharded", "f2gpu_dist_schedule",
    "f2gpu_local_wcols", "f2gpu_mat_broadcast", "f2gpu_strassen_mult_dist",
]

sz = C.c_size_t
vp = C.c_void_p
u64p = C.POINTER(C.c_uint64)
u32p = C.POINTER(C.c_uint32)

_SIG = {
    "f2gpu_last_error": ([], C.c_char_p),
    "f2gpu_version": ([], C.c_char_p),
    "f2gpu_options_describe": ([C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)], C.c_int),
    "f2gpu_ctx_create": ([C.c_int, C.POINTER(vp)], C.c_int),
    "f2gpu_ctx_destroy": ([vp], C.c_int),
    "f2gpu_ctx_set_stream": ([vp, vp], C.c_int),
    "f2gpu_ctx_sync": ([vp], C.c_int),
    "f2gpu_ctx_launches": ([vp], C.c_uint64),
    "f2gpu_ctx_set_strassen_cutover": ([vp, sz], C.c_int),
    "f2gpu_ctx_set_tc": ([vp, C.c_int, sz], C.c_int),
    "f2gpu_mat_alloc": ([vp, sz, sz, C.POINTER(vp)], C.c_int),
    "f2gpu_mat_free": ([vp], C.c_int),
    "f2gpu_mat_shape": ([vp, C.POINTER(sz), C.POINTER(sz), C.POINTER(sz)], C.c_int),
    "f2gpu_mat_device_ptr": ([vp, C.POINTER(vp)], C.c_int),
    "f2gpu_mat_zero": ([vp, vp], C.c_int),
    "f2gpu_mat_upload": ([vp, vp, vp, sz], C.c_int),
    "f2gpu_mat_download": ([vp, vp, vp, sz], C.c_int),
    "f2gpu_mat_random_dense": ([vp, vp, C.c_double, C.c_uint64], C.c_int),
    "f2gpu_mat_copy": ([vp, vp, vp], C.c_int),
    "f2gpu_mat_select_wcols": ([vp, vp, vp, sz, sz, C.c_int], C.c_int),
    "f2gpu_mat_xor": ([vp, vp, vp], C.c_int),
    "f2gpu_mat_transpose": ([vp, vp, vp], C.c_int),
    "f2gpu_m4rm_mult": ([vp, vp, vp, vp, C.c_uint], C.c_int),
    "f2gpu_m4rm_mult_acc": ([vp, vp, vp, vp], C.c_int),
    "f2gpu_mult_acc": ([vp, vp, sz, sz, sz, vp, sz, sz, vp, sz, sz], C.c_int),
    "f2gpu_mult_acc_host": ([vp, vp, sz, sz, sz, sz, sz, vp, sz, vp, sz, sz, sz, sz, sz, sz, sz], C.c_int),
    "f2gpu_strassen_mult": ([vp, vp, vp, vp, sz], C.c_int),
    "f2gpu_gemm_tc": ([vp, vp, vp, vp, C.c_int], C.c_int),
    "f2gpu_update_tc": ([vp, vp, sz, sz, sz, sz, vp, sz, sz, vp], C.c_int),
    "f2gpu_decompose_block": ([vp, vp, vp, vp, C.POINTER(sz)], C.c_int),
    "f2gpu_decompose_block_sharded": ([vp, vp, C.c_int, vp, vp, C.POINTER(sz)], C.c_int),
    "f2gpu_decompose_recursive": ([vp, vp, sz, vp, vp, C.POINTER(sz)], C.c_int),
    "f2gpu_rank": ([vp, vp, C.POINTER(sz)], C.c_int),
    "f2gpu_m4rm_mult_host": ([vp, vp, sz, sz, sz, vp, sz, sz, vp, sz, C.c_uint], C.c_int),
    "f2gpu_strassen_mult_host": ([vp, vp, sz, sz, sz, vp, sz, sz, vp, sz, sz], C.c_int),
    "f2gpu_decompose_block_host": ([vp, vp, sz, sz, sz, vp, vp, vp, C.POINTER(sz)], C.c_int),
    "f2gpu_decompose_recursive_host": ([vp, vp, sz, sz, sz, sz, vp, vp, vp, C.POINTER(sz)], C.c_int),
    "f2gpu_rank_host": ([vp, vp, sz, sz, sz, C.POINTER(sz)], C.c_int),
    "f2gpu_null_space": ([vp, vp, C.POINTER(vp), C.POINTER(sz)], C.c_int),
    "f2gpu_trace_enable": ([vp, sz], C.c_int),
    "f2gpu_debug_panel_chain": ([vp, vp, sz], C.c_int),
    "f2gpu_trace_read": ([vp, vp, sz, C.POINTER(sz)], C.c_int),
    "f2gpu_panel_build_z": ([vp, vp, sz, vp, vp, C.POINTER(C.c_uint32), vp, C.POINTER(C.c_uint32)], C.c_int),
    "f2gpu_solve": ([vp, vp, vp, vp, C.POINTER(C.c_int)], C.c_int),
    "f2gpu_nccl_unique_id": ([vp], C.c_int),
    "f2gpu_ctx_init_comm": ([vp, C.c_int, C.c_int, vp], C.c_int),
    "f2gpu_decompose_block_dist": ([vp, vp, sz, vp, vp, C.POINTER(sz)], C.c_int),
    "f2gpu_local_wcols": ([sz, C.c_int, C.c_int], sz),
    "f2gpu_decompose_recursive_dist": ([vp, vp, sz, sz, vp, vp, C.POINTER(sz)], C.c_int),
    "f2gpu_decompose_recursive_sharded": ([vp, vp, C.c_int, sz, vp, vp, C.POINTER(sz)], C.c_int),
    "f2gpu_mat_broadcast": ([vp, vp, C.c_int], C.c_int),
    "f2gpu_strassen_mult_dist": ([vp, vp, vp, vp, sz], C.c_int),
}

# f2gpu_dist_ops (include/f2gpu.h): the distributed recursion's callbacks
PANEL_FN = C.CFUNCTYPE(C.c_int, vp, sz, C.c_int, sz)
APPLY_FN = C.CFUNCTYPE(C.c_int, vp, sz, C.c_int, sz, sz)
STATE_FN = C.CFUNCTYPE(C.c_int, vp, sz, C.POINTER(sz), C.POINTER(sz))
GATHER_FN = C.CFUNCTYPE(C.c_int, vp, sz, sz, sz)
SOLVE_FN = C.CFUNCTYPE(C.c_int, vp, sz, sz, sz, sz, sz)
PRODUCT_FN = C.CFUNCTYPE(C.c_int, vp, sz, sz, sz, sz, sz, sz)
RANKUPD_FN = C.CFUNCTYPE(C.c_int, vp, sz, sz, sz, sz)
LEAF_FN = C.CFUNCTYPE(C.c_int, vp, sz, sz, sz)


class DistOps(C.Structure):
    _fields_ = [("user", vp), ("panel", PANEL_FN), ("apply", APPLY_FN), ("state", STATE_FN),
                ("gather", GATHER_FN), ("solve", SOLVE_FN), ("product", PRODUCT_FN),
                ("rank_update", RANKUPD_FN), ("leaf", LEAF_FN)]


_SIG["f2gpu_dist_schedule"] = ([sz, sz, C.c_int, sz, sz, sz, C.POINTER(DistOps)], C.c_int)

_lib = None


def load(build_if_missing: bool = True) -> C.CDLL:
    """Load libf2gpu.so (building it in place with nvcc when absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        if not build_if_missing:
            raise F2GpuError(f"{LIB_PATH} is missing; run paper_1209_5198_b200.build.build()")
        from . import build as _build

        _build.build()
    lib = C.CDLL(str(LIB_PATH))
    for name, (args, res) in _SIG.items():
        if os.environ.get("F2GPU_LIB") and not hasattr(lib, name):
            continue  # an older build selected for an A/B run
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def check(rc: int, what: str = "") -> None:
    if rc == OK:
        return
    msg = load().f2gpu_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == EINVAL:
        raise ValueError(text)
    if rc == ERANGE:
        raise IndexError(text)
    raise F2GpuError(f"[code {rc}] {text}")
