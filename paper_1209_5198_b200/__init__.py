"""paper_1209_5198_b200 — B200-native GF(2) block decomposition (arXiv 1209.5198).

Python mirror of the reference's f2la API (/root/reference/proj/include/f2la/)
over the C-ABI of libf2gpu.so (include/f2gpu.h).  Every compute call runs the
hand-written sm_100a kernels; there is no CPU fallback — without the shared
library or a B200 the calls raise.

Reference surface mirrored here (names and argument meaning kept):
  BitMatrix            PackedMatrix<uint64_t>          bit_matrix.hpp:82-348
  RowPermutation       RowPermutation                  bit_matrix.hpp:351-371
  m4rm_mult            m4rm_mult(A, B, c)              m4rm.hpp:177-196
  build_tables/mult_acc (fused on device)              m4rm.hpp:93-172
  strassen_mult        strassen_mult(A, B, thr, c)
  decompose_block      decompose_block(A) -> LUFactors SPEC.md:319-327
  rank                 rank(A)
  tuning.*             tuning::*                       tuning.hpp:11-41
"""
from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _lib, tuning
from ._lib import F2GpuError

__all__ = [
    "BitMatrix", "RowPermutation", "LUFactors", "Context", "DeviceMatrix", "M4rmTables",
    "m4rm_mult", "strassen_mult", "build_tables", "mult_acc", "decompose_block",
    "decompose_recursive", "rank",
    "make_splits", "tuning", "F2GpuError", "default_context", "null_space", "solve"]


def _ptr(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


# ---------------------------------------------------------------------------
# host matrix (layout contract of the reference)
# ---------------------------------------------------------------------------
class BitMatrix:
    """Dense n x m matrix over F2, word-column-major (bit_matrix.hpp:74-81).

    ``words`` is a numpy uint64 array of shape (word_cols, col_stride): word
    (i, q) is ``words[q, i]``; bit k is entry (i, 64q+k).  col_stride is the
    reference's ceil(n/8)*8 (bit_matrix.hpp:330-333).  Padding bits are zero.
    """

    word_bits = 64

    def __init__(self, n_rows: int = 0, n_cols: int = 0, words: np.ndarray | None = None):
        self._n, self._m = int(n_rows), int(n_cols)
        mu = (self._m + 63) // 64
        stride = (self._n + 7) // 8 * 8
        if words is None:
            words = np.zeros((mu, stride), dtype=np.uint64)
        words = np.ascontiguousarray(words, dtype=np.uint64)
        if words.shape[0] != mu or words.shape[1] < self._n:
            raise ValueError("BitMatrix: words array has the wrong shape")
        self.words = words

    # --- constructors (bit_matrix.hpp:91-162) ---
    @classmethod
    def identity(cls, n: int) -> "BitMatrix":
        a = cls(n, n)
        for i in range(n):
            a.words[i // 64, i] |= np.uint64(1) << np.uint64(i % 64)
        return a

    @classmethod
    def from_rows(cls, rows: list[str]) -> "BitMatrix":
        n = len(rows)
        m = len(rows[0]) if n else 0
        a = cls(n, m)
        for i, r in enumerate(rows):
            if len(r) != m:
                raise ValueError("from_rows: ragged rows")
            for j, ch in enumerate(r):
                if ch not in "01":
                    raise ValueError("from_rows: entry not in {0,1}")
                if ch == "1":
                    a.words[j // 64, i] |= np.uint64(1) << np.uint64(j % 64)
        return a

    @classmethod
    def random_dense(cls, n: int, m: int, density: float, seed: int,
                     ctx: "Context | None" = None) -> "BitMatrix":
        """Bit-exact PackedMatrix::random_dense (bit_matrix.hpp:125-142), generated
        on the GPU by the jump-ahead kernel."""
        ctx = ctx or default_context()
        d = DeviceMatrix(n, m, ctx)
        d.random_dense(density, seed)
        return d.download()

    # --- accessors (bit_matrix.hpp:164-200) ---
    def rows(self) -> int: return self._n
    def cols(self) -> int: return self._m
    def word_cols(self) -> int: return self.words.shape[0]
    def col_stride(self) -> int: return self.words.shape[1]
    def empty(self) -> bool: return self._n == 0 or self._m == 0
    def col_block(self, q: int) -> np.ndarray: return self.words[q]
    def word(self, i: int, q: int) -> int: return int(self.words[q, i])

    def get(self, i: int, j: int) -> bool:
        if not (0 <= i < self._n and 0 <= j < self._m):
            raise IndexError("matrix index")
        return bool((int(self.words[j // 64, i]) >> (j % 64)) & 1)

    def set(self, i: int, j: int, v: bool) -> None:
        if not (0 <= i < self._n and 0 <= j < self._m):
            raise IndexError("matrix index")
        bit = np.uint64(1) << np.uint64(j % 64)
        if v:
            self.words[j // 64, i] |= bit
        else:
            self.words[j // 64, i] &= ~bit

    def row_swap(self, i: int, k: int) -> None:
        if not (0 <= i < self._n and 0 <= k < self._n):
            raise IndexError("row index")
        self.words[:, [i, k]] = self.words[:, [k, i]]

    def __eq__(self, other) -> bool:
        return (isinstance(other, BitMatrix) and self._n == other._n and self._m == other._m
                and bool(np.array_equal(self.words[:, : self._n], other.words[:, : other._n])))

    def padding_is_zero(self) -> bool:
        rem = self._m % 64
        if rem == 0 or self.word_cols() == 0:
            return True
        mask = np.uint64((1 << rem) - 1)
        return not bool(np.any(self.words[-1, : self._n] & ~mask))

    def copy(self) -> "BitMatrix":
        return BitMatrix(self._n, self._m, self.words.copy())

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self._n, self._m), dtype=np.uint8)
        for j in range(self._m):
            out[:, j] = (self.words[j // 64, : self._n] >> np.uint64(j % 64)) & np.uint64(1)
        return out

    def __repr__(self) -> str:
        return f"BitMatrix({self._n}x{self._m})"


@dataclass
class RowPermutation:
    """(P A) row i = A row perm[i]  (bit_matrix.hpp:350-371)."""
    perm: np.ndarray

    @classmethod
    def identity(cls, n: int) -> "RowPermutation":
        return cls(np.arange(n, dtype=np.uint32))

    def size(self) -> int:
        return int(self.perm.size)

    def is_bijection(self) -> bool:
        return bool(np.array_equal(np.sort(self.perm), np.arange(self.perm.size)))


@dataclass
class LUFactors:
    """P*A = L*U.  ``overlay`` is the in-place overlay W the
    device produces (L left/below the block staircase, U on the pivot rows)."""
    P: RowPermutation
    overlay: BitMatrix
    rank: int
    block_ranks: np.ndarray
    _L: BitMatrix | None = field(default=None, repr=False)
    _U: BitMatrix | None = field(default=None, repr=False)

    def _extract(self) -> None:
        n, m = self.overlay.rows(), self.overlay.cols()
        r = self.rank
        L = BitMatrix(n, r)
        U = BitMatrix(r, m)
        W = self.overlay.words
        R = 0
        for j, rj in enumerate(self.block_ranks.tolist()):
            if rj == 0:
                continue
            # L block column at bit offset R: I on pivot rows, Y^(j) below
            col = W[j, :n].copy()
            col[R:R + rj] = np.left_shift(np.uint64(1), np.arange(rj, dtype=np.uint64))
            col[:R] = 0
            q, s = divmod(R, 64)
            L.words[q, :n] ^= col << np.uint64(s)
            if s:
                hi = col >> np.uint64(64 - s)
                if q + 1 < L.word_cols():
                    L.words[q + 1, :n] ^= hi
            U.words[j:, R:R + rj] = W[j:, R:R + rj]
            R += rj
        self._L, self._U = L, U

    @property
    def L(self) -> BitMatrix:
        if self._L is None:
            self._extract()
        return self._L

    @property
    def U(self) -> BitMatrix:
        if self._U is None:
            self._extract()
        return self._U


# ---------------------------------------------------------------------------
# device context / matrices
# ---------------------------------------------------------------------------
class Context:
    """One CUDA device + stream (+ NCCL communicator for multi-GPU)."""

    def __init__(self, device: int = 0):
        lib = _lib.load()
        h = C.c_void_p()
        _lib.check(lib.f2gpu_ctx_create(int(device), C.byref(h)), "ctx_create")
        self._h = h
        self.device = device
        self._mats = weakref.WeakSet()  # live matrices: freed before the context is destroyed
        self.stream = None  # None: the context's own stream
        self.rank, self.world = 0, 1

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def set_stream(self, cuda_stream: int | None) -> None:
        """Run on an external CUDA stream handle (e.g. ``torch.cuda.current_stream().cuda_stream``;
        0 is the legacy default stream, i.e. torch's default stream); None returns to the
        context's own stream."""
        h = _lib.OWN_STREAM if cuda_stream is None else int(cuda_stream)
        _lib.check(_lib.load().f2gpu_ctx_set_stream(self._h, C.c_void_p(h)))
        self.stream = cuda_stream

    def sync(self) -> None:
        _lib.check(_lib.load().f2gpu_ctx_sync(self._h), "sync")

    def launches(self) -> int:
        return int(_lib.load().f2gpu_ctx_launches(self._h))

    def set_strassen_cutover(self, bits: int) -> None:
        _lib.check(_lib.load().f2gpu_ctx_set_strassen_cutover(self._h, int(bits)))

    def set_tc(self, on: bool, min_leaf_bits: int = 0) -> None:
        """Allow the fp4 tensor-core product leaf (bit-identical results)."""
        _lib.check(_lib.load().f2gpu_ctx_set_tc(self._h, 1 if on else 0, int(min_leaf_bits)))

    def init_comm(self, rank: int, world: int, uid: bytes) -> None:
        buf = C.create_string_buffer(bytes(uid), 128)
        _lib.check(_lib.load().f2gpu_ctx_init_comm(self._h, rank, world, buf), "init_comm")
        self.rank, self.world = rank, world

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _lib.check(_lib.load().f2gpu_nccl_unique_id(buf), "nccl_unique_id")
        return buf.raw

    def close(self) -> None:
        """Destroy the context; matrices still alive on it are freed first (a device
        matrix must not outlive its context, include/f2gpu.h)."""
        if getattr(self, "_h", None):
            for m in list(getattr(self, "_mats", ())):
                m.free()
            _lib.load().f2gpu_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default: Context | None = None


def options() -> str:
    """Every switch of the library (csrc/options.h) with the value in effect: one line per
    environment variable, "NAME value[*] (default D) meaning" (* = set in the environment)."""
    lib = _lib.load()
    n = C.c_size_t()
    _lib.check(lib.f2gpu_options_describe(None, 0, C.byref(n)), "options_describe")
    buf = C.create_string_buffer(n.value + 1)
    _lib.check(lib.f2gpu_options_describe(buf, n.value + 1, None), "options_describe")
    return buf.value.decode()


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context(0)
    return _default


class DeviceMatrix:
    """Device-resident packed matrix (stride: rows rounded up to 128 words), owned by the library."""

    def __init__(self, n_rows: int, n_cols: int, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        lib = _lib.load()
        h = C.c_void_p()
        _lib.check(lib.f2gpu_mat_alloc(self.ctx.handle, int(n_rows), int(n_cols), C.byref(h)),
                   "mat_alloc")
        self._h = h
        self.ctx._mats.add(self)
        self.n, self.m = int(n_rows), int(n_cols)
        r, c, s = C.c_size_t(), C.c_size_t(), C.c_size_t()
        lib.f2gpu_mat_shape(h, C.byref(r), C.byref(c), C.byref(s))
        self.stride = s.value

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    @classmethod
    def _adopt(cls, h: C.c_void_p, ctx: Context) -> "DeviceMatrix":
        """Wrap a matrix handle the library allocated (e.g. f2gpu_null_space's basis)."""
        d = cls.__new__(cls)
        d.ctx, d._h = ctx, h
        ctx._mats.add(d)
        r, c, st = C.c_size_t(), C.c_size_t(), C.c_size_t()
        _lib.load().f2gpu_mat_shape(h, C.byref(r), C.byref(c), C.byref(st))
        d.n, d.m, d.stride = int(r.value), int(c.value), int(st.value)
        return d

    @classmethod
    def from_host(cls, a: BitMatrix, ctx: Context | None = None) -> "DeviceMatrix":
        d = cls(a.rows(), a.cols(), ctx)
        d.upload(a)
        return d

    def upload(self, a: BitMatrix) -> None:
        if (a.rows(), a.cols()) != (self.n, self.m):
            raise ValueError("upload: shape mismatch")
        _lib.check(_lib.load().f2gpu_mat_upload(self.ctx.handle, self._h, _ptr(a.words),
                                                a.col_stride()), "upload")

    def upload_words(self, words: np.ndarray, host_stride: int) -> None:
        _lib.check(_lib.load().f2gpu_mat_upload(self.ctx.handle, self._h, _ptr(words),
                                                host_stride), "upload")

    def download(self, out: BitMatrix | None = None) -> BitMatrix:
        out = out or BitMatrix(self.n, self.m)
        _lib.check(_lib.load().f2gpu_mat_download(self.ctx.handle, self._h, _ptr(out.words),
                                                  out.col_stride()), "download")
        return out

    def random_dense(self, density: float, seed: int) -> None:
        _lib.check(_lib.load().f2gpu_mat_random_dense(self.ctx.handle, self._h, float(density),
                                                      int(seed) & (2**64 - 1)), "random_dense")

    def zero(self) -> None:
        _lib.check(_lib.load().f2gpu_mat_zero(self.ctx.handle, self._h))

    def device_ptr(self) -> int:
        p = C.c_void_p()
        _lib.check(_lib.load().f2gpu_mat_device_ptr(self._h, C.byref(p)))
        return int(p.value or 0)

    def free(self) -> None:
        if getattr(self, "_h", None):
            _lib.load().f2gpu_mat_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# M4RM / Strassen (m4rm.hpp:39-196)
# ---------------------------------------------------------------------------
def make_splits(k_bits: int, c: int) -> list[int]:
    """m4rm.hpp:39-48 (kept for API parity; the device uses a fixed 7x8+8 split)."""
    if c == 0:
        raise ValueError("make_splits: c must be positive")
    out, done = [], 0
    while done < k_bits:
        l_ = min(c, k_bits - done)
        out.append(l_)
        done += l_
    return out


def _shape(x) -> tuple[int, int]:
    return (x.rows(), x.cols()) if isinstance(x, BitMatrix) else (x.n, x.m)


def _as_dev(x, ctx):
    return x if isinstance(x, DeviceMatrix) else DeviceMatrix.from_host(x, ctx)


def m4rm_mult(a, b, c: int = 0, ctx: Context | None = None):
    """Exact A*B over F2 (m4rm.hpp:177-196) on the GPU.  Accepts BitMatrix (returns
    BitMatrix) or DeviceMatrix (returns DeviceMatrix)."""
    ctx = ctx or (a.ctx if isinstance(a, DeviceMatrix) else default_context())
    if _shape(a)[1] != _shape(b)[0]:
        raise ValueError("m4rm_mult: shape mismatch")  # m4rm.hpp:181
    da, db = _as_dev(a, ctx), _as_dev(b, ctx)
    dc = DeviceMatrix(da.n, db.m, ctx)
    _lib.check(_lib.load().f2gpu_m4rm_mult(ctx.handle, da.handle, db.handle, dc.handle, int(c)),
               "m4rm_mult")
    return dc.download() if isinstance(a, BitMatrix) else dc


def strassen_mult(a, b, threshold: int = 0, c: int = 0, ctx: Context | None = None):
    """Strassen-Winograd product with M4RM leaves."""
    ctx = ctx or (a.ctx if isinstance(a, DeviceMatrix) else default_context())
    da, db = _as_dev(a, ctx), _as_dev(b, ctx)
    if da.m != db.n:
        raise ValueError("strassen_mult: shape mismatch")
    dc = DeviceMatrix(da.n, db.m, ctx)
    _lib.check(_lib.load().f2gpu_strassen_mult(ctx.handle, da.handle, db.handle, dc.handle,
                                               int(threshold)), "strassen_mult")
    return dc.download() if isinstance(a, BitMatrix) else dc


@dataclass
class M4rmTables:
    """Lazy table spec (m4rm.hpp:21-35): the device builds the tables in shared
    memory inside the fused mult_acc kernel, so this only records the B block."""
    b: DeviceMatrix
    row0: int
    k_bits: int
    wcol0: int
    n_wcols: int


def build_tables(b, row0: int, k_bits: int, wcol0: int, n_wcols: int,
                 ctx: Context | None = None) -> M4rmTables:
    """build_tables(B, row0, k, wcol0, n) (m4rm.hpp:93-113)."""
    if k_bits > 64:
        raise ValueError("build_tables: block taller than a word")
    nb, mb = (b.rows(), b.cols()) if isinstance(b, BitMatrix) else (b.n, b.m)
    if row0 + k_bits > nb or wcol0 + n_wcols > (mb + 63) // 64:
        raise IndexError("build_tables: block outside B")
    return M4rmTables(_as_dev(b, ctx or default_context()), row0, k_bits, wcol0, n_wcols)


def mult_acc(c_mat: DeviceMatrix, c_row0: int, c_wcol0: int, a_words, tables: M4rmTables) -> None:
    """C[c_row0+i, c_wcol0..+w) ^= a_words[i] * B (m4rm.hpp:140-172), fused table
    build + XOR sweep on the device.  a_words: numpy uint64 array or a torch
    CUDA tensor of dtype int64/uint64."""
    ctx = c_mat.ctx
    lib = _lib.load()
    if hasattr(a_words, "data_ptr"):  # a torch tensor: validated, then ordered after its producer
        import torch

        if not a_words.is_cuda or a_words.device.index != ctx.device:
            raise ValueError(f"mult_acc: a_words must be a CUDA tensor on device {ctx.device}")
        if a_words.element_size() != 8 or a_words.is_floating_point() or a_words.is_complex():
            raise ValueError("mult_acc: a_words must be a 64-bit integer tensor")
        if not a_words.is_contiguous() or a_words.dim() != 1:
            raise ValueError("mult_acc: a_words must be a contiguous 1-D tensor")
        producer = torch.cuda.current_stream(a_words.device)
        if ctx.stream is None or int(ctx.stream) != producer.cuda_stream:
            # the library runs on another stream: finish the torch work that writes a_words
            producer.synchronize()
        ptr, n_rows, keep = a_words.data_ptr(), a_words.numel(), None
    else:
        host = np.ascontiguousarray(a_words, dtype=np.uint64)
        n_rows = host.size
        keep = DeviceMatrix(max(n_rows, 1), 64, ctx)
        keep.upload_words(host.reshape(1, -1) if n_rows else np.zeros((1, 1), np.uint64),
                          max(n_rows, 1))
        ptr = keep.device_ptr()
    _lib.check(lib.f2gpu_mult_acc(ctx.handle, c_mat.handle, c_row0, c_wcol0, tables.n_wcols,
                                  C.c_void_p(ptr), n_rows, tables.k_bits, tables.b.handle,
                                  tables.row0, tables.wcol0), "mult_acc")
    ctx.sync()
    del keep


# ---------------------------------------------------------------------------
# decomposition
# ---------------------------------------------------------------------------
def decompose_block(a, ctx: Context | None = None, shards: int = 1) -> LUFactors:
    """Column-swap-free block decomposition P*A = L*U on the GPU.
    The input is never modified."""
    ctx = ctx or (a.ctx if isinstance(a, DeviceMatrix) else default_context())
    lib = _lib.load()
    if isinstance(a, DeviceMatrix):
        host = a.download()
    else:
        host = a
    n, m = host.rows(), host.cols()
    w = DeviceMatrix.from_host(host, ctx)
    perm = np.zeros(max(n, 1), dtype=np.uint32)
    rj = np.zeros(max((m + 63) // 64, 1), dtype=np.uint32)
    rank_ = C.c_size_t()
    if shards == 1:
        rc = lib.f2gpu_decompose_block(ctx.handle, w.handle, _ptr(perm), _ptr(rj), C.byref(rank_))
    else:
        rc = lib.f2gpu_decompose_block_sharded(ctx.handle, w.handle, int(shards), _ptr(perm),
                                               _ptr(rj), C.byref(rank_))
    _lib.check(rc, "decompose_block")
    W = w.download()
    return LUFactors(RowPermutation(perm[:n].copy()), W, int(rank_.value),
                     rj[: (m + 63) // 64].copy())


def decompose_recursive(a, min_cols: int = 0, ctx: Context | None = None) -> LUFactors:
    """Recursive column-split variant: left
    half recursively, right half brought up to date by a block TRSM and one
    Strassen-Winograd GEMM (A' = D + L21 L11^-1 C), then recursion.  Exact
    arithmetic with 64-aligned splits: the factors equal decompose_block's
    bit-for-bit.  min_cols = 0 picks the device default (leaves of at most 256 panels =
    16384 columns; 64 panels once a leaf has >= 30000 rows below it; csrc/options.h)."""
    ctx = ctx or (a.ctx if isinstance(a, DeviceMatrix) else default_context())
    host = a.download() if isinstance(a, DeviceMatrix) else a
    n, m = host.rows(), host.cols()
    w = DeviceMatrix.from_host(host, ctx)
    perm = np.zeros(max(n, 1), dtype=np.uint32)
    rj = np.zeros(max((m + 63) // 64, 1), dtype=np.uint32)
    rank_ = C.c_size_t()
    _lib.check(_lib.load().f2gpu_decompose_recursive(ctx.handle, w.handle, int(min_cols),
                                                     _ptr(perm), _ptr(rj), C.byref(rank_)),
               "decompose_recursive")
    W = w.download()
    return LUFactors(RowPermutation(perm[:n].copy()), W, int(rank_.value),
                     rj[: (m + 63) // 64].copy())


def _pack_bits(bits, n: int) -> np.ndarray:
    v = np.zeros(max(1, (n + 63) // 64), np.uint64)
    b = np.asarray(bits, dtype=np.uint8).reshape(-1)[:n]
    for i in np.nonzero(b)[0]:
        v[i // 64] |= np.uint64(1) << np.uint64(i % 64)
    return v


def _unpack_bits(words: np.ndarray, n: int) -> np.ndarray:
    idx = np.arange(n)
    return ((words[idx // 64] >> (idx % 64).astype(np.uint64)) & np.uint64(1)).astype(np.uint8)


def null_space(a, ctx: Context | None = None) -> BitMatrix:
    """m x (m - rank) basis N with A*N = 0, computed on the device by a
    partial block decomposition of [A^T | I]."""
    ctx = ctx or (a.ctx if isinstance(a, DeviceMatrix) else default_context())
    d = _as_dev(a, ctx)
    h, nul = C.c_void_p(), C.c_size_t()
    _lib.check(_lib.load().f2gpu_null_space(ctx.handle, d.handle, C.byref(h), C.byref(nul)), "null_space")
    N = DeviceMatrix._adopt(h, ctx)
    try:
        return N.download()
    finally:
        N.free()


def solve(a, rhs, ctx: Context | None = None) -> np.ndarray | None:
    """x (m bits, uint8) with A x = rhs over F2, or None when the system is inconsistent
    (signalled, not an error)."""
    ctx = ctx or (a.ctx if isinstance(a, DeviceMatrix) else default_context())
    d = _as_dev(a, ctx)
    n, m = d.n, d.m
    if len(np.asarray(rhs).reshape(-1)) != n:
        raise ValueError("solve: rhs length must equal the number of rows")
    b = _pack_bits(rhs, n)
    x = np.zeros(max(1, (m + 63) // 64), np.uint64)
    ok = C.c_int()
    _lib.check(_lib.load().f2gpu_solve(ctx.handle, d.handle, _ptr(b), _ptr(x), C.byref(ok)), "solve")
    return _unpack_bits(x, m) if ok.value else None


def rank(a, ctx: Context | None = None) -> int:
    """rank(A) = sum r_j, transposing wide inputs."""
    ctx = ctx or (a.ctx if isinstance(a, DeviceMatrix) else default_context())
    d = _as_dev(a, ctx)
    r = C.c_size_t()
    _lib.check(_lib.load().f2gpu_rank(ctx.handle, d.handle, C.byref(r)), "rank")
    return int(r.value)
