"""ctypes view of the CPU oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module, and only as the checker (or the timed
CPU baseline).  The product package `paper_1209_5198_b200` never imports it.

Matrices are numpy uint64 arrays of shape (mu, stride) in the reference's
word-column-major layout (proj/include/f2la/bit_matrix.hpp:74-81): word (i, q)
is ``arr[q, i]``; bit k of it is entry (i, 64*q + k).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
REF_LIB = HERE / "_ref" / "libf2la_ref.so"

u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
sz = C.c_size_t


def build(ref: bool = False) -> None:
    """Compile the oracle (and, when /root/reference exists, oracle/_ref)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    if ref and Path("/root/reference/proj/include/f2la").is_dir():
        subprocess.run(["make", "-s", "-C", str(HERE), "ref"], check=True)


def _load() -> C.CDLL:
    if not LIB.exists():
        build()
    lib = C.CDLL(str(LIB))
    lib.f2o_random_dense.argtypes = [u64p, sz, sz, sz, C.c_double, C.c_uint64]
    lib.f2o_mul_naive.argtypes = [u64p, sz, sz, sz, u64p, sz, sz, u64p, sz]
    lib.f2o_m4rm_mult.argtypes = [u64p, sz, sz, sz, u64p, sz, sz, u64p, sz, C.c_uint]
    lib.f2o_build_z.argtypes = [u64p, sz, i64p, u64p, u64p]
    lib.f2o_build_z.restype = C.c_int
    lib.f2o_decompose_block.argtypes = [u64p, sz, sz, sz, u32p, u32p, C.c_uint, sz]
    lib.f2o_decompose_block.restype = sz
    lib.f2o_rank_ge.argtypes = [u64p, sz, sz, sz]
    lib.f2o_rank_ge.restype = sz
    lib.f2o_transpose.argtypes = [u64p, sz, sz, sz, u64p, sz]
    lib.f2o_digest.argtypes = [u64p, sz, sz, sz]
    lib.f2o_digest.restype = C.c_uint64
    lib.f2o_digest_u32.argtypes = [u32p, sz]
    lib.f2o_digest_u32.restype = C.c_uint64
    lib.f2o_extract_lu.argtypes = [u64p, sz, sz, sz, u32p, sz, u64p, sz, u64p, sz]
    lib.f2o_check_plu.argtypes = [u64p, u64p, sz, sz, sz, u32p, u32p, C.c_uint64]
    lib.f2o_check_plu.restype = C.c_int
    lib.f2o_m4rm_cost.argtypes = [C.c_uint, C.c_uint, C.c_double]
    lib.f2o_m4rm_cost.restype = C.c_double
    lib.f2o_optimal_table_size.argtypes = [C.c_uint, C.c_double]
    lib.f2o_optimal_table_size.restype = C.c_uint
    lib.f2o_strassen_threshold.argtypes = [C.c_uint]
    lib.f2o_strassen_threshold.restype = sz
    lib.f2o_rng_next.argtypes = [C.POINTER(C.c_uint64)]
    lib.f2o_rng_next.restype = C.c_uint64
    lib.f2o_rng_seed.argtypes = [C.c_uint64]
    lib.f2o_rng_seed.restype = C.c_uint64
    lib.f2o_bernoulli_threshold.argtypes = [C.c_double]
    lib.f2o_bernoulli_threshold.restype = C.c_uint64
    lib.f2o_num_threads.restype = C.c_int
    return lib


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        _lib = _load()
    return _lib


def ref_available() -> bool:
    return REF_LIB.exists()


_ref = None


def ref() -> C.CDLL:
    """The reference headers compiled in place (oracle/_ref)."""
    global _ref
    if _ref is None:
        if not REF_LIB.exists():
            build(ref=True)
        r = C.CDLL(str(REF_LIB))
        r.ref_rng_outputs.argtypes = [C.c_uint64, u64p, sz]
        r.ref_col_stride.argtypes = [sz]
        r.ref_col_stride.restype = sz
        r.ref_random_dense.argtypes = [u64p, sz, sz, sz, C.c_double, C.c_uint64]
        r.ref_m4rm_mult.argtypes = [u64p, sz, sz, sz, u64p, sz, sz, u64p, sz, sz]
        r.ref_m4rm_mult.restype = C.c_int
        r.ref_transpose.argtypes = [u64p, sz, sz, sz, u64p, sz]
        r.ref_matrix_new.argtypes = [u64p, sz, sz, sz]
        r.ref_matrix_new.restype = C.c_void_p
        r.ref_matrix_random.argtypes = [sz, sz, C.c_double, C.c_uint64]
        r.ref_matrix_random.restype = C.c_void_p
        r.ref_matrix_free.argtypes = [C.c_void_p]
        r.ref_matrix_read.argtypes = [C.c_void_p, u64p, sz]
        r.ref_matrix_mult.argtypes = [C.c_void_p, C.c_void_p, sz]
        r.ref_matrix_mult.restype = C.c_void_p
        r.ref_decompose_block.argtypes = [C.c_void_p, u32p, u32p, sz, sz]
        r.ref_decompose_block.restype = sz
        _ref = r
    return _ref


# ---------------------------------------------------------------------------
# numpy helpers
# ---------------------------------------------------------------------------
def wcols(m: int) -> int:
    return (m + 63) // 64


def stride_for(n: int) -> int:
    """Reference col_stride: rows rounded up to a 64-byte line (bit_matrix.hpp:330-333)."""
    return (n + 7) // 8 * 8


def zeros(n: int, m: int, stride: int | None = None) -> np.ndarray:
    s = stride_for(n) if stride is None else stride
    return np.zeros((max(wcols(m), 0), max(s, 1)), dtype=np.uint64)


def random_dense(n: int, m: int, density: float, seed: int, stride: int | None = None) -> np.ndarray:
    a = zeros(n, m, stride)
    if a.size and n and m:
        lib().f2o_random_dense(a, n, m, a.shape[1], float(density), seed & (2**64 - 1))
    return a


def mul_naive(a, n, k, b, m) -> np.ndarray:
    c = zeros(n, m)
    if n and m:
        lib().f2o_mul_naive(_nz(a), n, k, a.shape[1], _nz(b), m, b.shape[1], c, c.shape[1])
    return c


def m4rm_mult(a, n, k, b, m, tc: int = 8) -> np.ndarray:
    c = zeros(n, m)
    if n and m:
        lib().f2o_m4rm_mult(_nz(a), n, k, a.shape[1], _nz(b), m, b.shape[1], c, c.shape[1], tc)
    return c


def _nz(a: np.ndarray) -> np.ndarray:
    return a if a.size else np.zeros((1, 1), dtype=np.uint64)


def build_z(panel: np.ndarray):
    """Procedure buildZ on a copy of `panel` (1-D uint64 words)."""
    A = np.ascontiguousarray(panel, dtype=np.uint64).copy()
    P = np.zeros(64, dtype=np.int64)
    Z = np.zeros(64, dtype=np.uint64)
    sb = np.zeros(64, dtype=np.uint64)
    r = lib().f2o_build_z(_nz(A) if A.size else np.zeros(1, np.uint64), A.size, P, Z, sb)
    return r, A, P, Z, sb[:r].copy()


def decompose_block(a: np.ndarray, n: int, m: int, tc: int = 8, max_panels: int | None = None):
    """Returns (W, perm, rj, rank) — the canonical parity artifact."""
    w = np.ascontiguousarray(a.copy())
    perm = np.zeros(max(n, 1), dtype=np.uint32)
    rj = np.zeros(max(wcols(m), 1), dtype=np.uint32)
    mp = (2**63) if max_panels is None else max_panels
    rank = 0
    if n and m:
        rank = lib().f2o_decompose_block(w, n, m, w.shape[1], perm, rj, tc, mp)
    return w, perm[:n], rj[: wcols(m)], int(rank)


def rank_ge(a: np.ndarray, n: int, m: int) -> int:
    if not (n and m):
        return 0
    return int(lib().f2o_rank_ge(a, n, m, a.shape[1]))


def transpose(a: np.ndarray, n: int, m: int) -> np.ndarray:
    out = zeros(m, n)
    if n and m:
        lib().f2o_transpose(a, n, m, a.shape[1], out, out.shape[1])
    return out


def digest(a: np.ndarray, n: int, m: int) -> int:
    return int(lib().f2o_digest(_nz(a), n, m, a.shape[1] if a.size else 1))


def digest_u32(v: np.ndarray) -> int:
    v = np.ascontiguousarray(v, dtype=np.uint32)
    return int(lib().f2o_digest_u32(v if v.size else np.zeros(1, np.uint32), v.size))


def extract_lu(w, n, m, rj):
    rank = int(np.sum(rj, dtype=np.int64))
    L = zeros(n, rank)
    U = zeros(rank, m)
    Lc = L if L.size else np.zeros((1, 1), np.uint64)
    Uc = U if U.size else np.zeros((1, 1), np.uint64)
    lib().f2o_extract_lu(w, n, m, w.shape[1], np.ascontiguousarray(rj, dtype=np.uint32), rank,
                         Lc, Lc.shape[1], Uc, Uc.shape[1])
    return L, U, rank


def check_plu(a, w, n, m, perm, rj, seed: int = 12345) -> bool:
    return bool(lib().f2o_check_plu(a, w, n, m, a.shape[1],
                                    np.ascontiguousarray(perm, dtype=np.uint32),
                                    np.ascontiguousarray(rj, dtype=np.uint32), seed))


# ---- dense <-> packed conversions for small cases ----
def to_dense(a: np.ndarray, n: int, m: int) -> np.ndarray:
    out = np.zeros((n, m), dtype=np.uint8)
    for j in range(m):
        out[:, j] = (a[j // 64, :n] >> np.uint64(j % 64)) & np.uint64(1)
    return out


def from_dense(d: np.ndarray, stride: int | None = None) -> np.ndarray:
    n, m = d.shape
    a = zeros(n, m, stride)
    for j in range(m):
        a[j // 64, :n] |= d[:, j].astype(np.uint64) << np.uint64(j % 64)
    return a


# ---- reference (oracle/_ref) wrappers ----
def ref_random_dense(n, m, density, seed, stride=None):
    a = zeros(n, m, stride)
    if a.size and n and m:
        ref().ref_random_dense(a, n, m, a.shape[1], float(density), seed)
    return a


def ref_m4rm_mult(a, n, k, b, m, tc=8):
    c = zeros(n, m)
    rc = ref().ref_m4rm_mult(_nz(a), n, k, a.shape[1], _nz(b), m, b.shape[1], _nz(c),
                             c.shape[1] if c.size else 1, tc)
    if rc:
        raise ValueError("m4rm_mult: shape mismatch")
    return c


def ref_decompose_block(a, n, m, tc=8, max_panels=None):
    r = ref()
    h = r.ref_matrix_new(a, n, m, a.shape[1])
    perm = np.zeros(max(n, 1), dtype=np.uint32)
    rj = np.zeros(max(wcols(m), 1), dtype=np.uint32)
    try:
        rank = r.ref_decompose_block(h, perm, rj, tc, (2**63) if max_panels is None else max_panels)
        w = zeros(n, m, a.shape[1])
        r.ref_matrix_read(h, w, w.shape[1])
    finally:
        r.ref_matrix_free(h)
    return w, perm[:n], rj[: wcols(m)], int(rank)


def num_threads() -> int:
    return int(lib().f2o_num_threads())


os.environ.setdefault("OMP_PROC_BIND", "false")
