"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle, bit-exact.

All integer/bitwise work, so the bar is bit-exact equality (no tolerance).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def experimental() -> bool:
    """libf2gpu built with F2GPU_BUILD_EXPERIMENTAL=1 (the evaluated-and-rejected variants)."""
    from paper_1209_5198_b200 import _lib

    return b"experimental" in _lib.load().f2gpu_version()


needs_experimental = pytest.mark.skipif("not experimental()",
                                        reason="variant built only with F2GPU_BUILD_EXPERIMENTAL=1")


def bm(f2, arr, n, m):
    return f2.BitMatrix(n, m, arr)


def same(a, b, n):
    return np.array_equal(a[:, :n], b[:, :n])


# ---------------------------------------------------------------------------
# K0 random_dense
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n,m", [(1, 1), (4, 5), (100, 130), (65, 64), (333, 777), (1000, 4096),
                                 (4097, 1000), (31, 4160)])
@pytest.mark.parametrize("p", [0.5, 0.05, 0.3])
def test_random_dense(f2, ctx, po, n, m, p):
    seed = n * 7 + m
    want = po.random_dense(n, m, p, seed)
    got = f2.BitMatrix.random_dense(n, m, p, seed, ctx=ctx)
    assert same(got.words, want, n)
    assert got.padding_is_zero()


@pytest.mark.parametrize("p", [0.0, 1.0, -1.0, 2.0])
def test_random_dense_degenerate(f2, ctx, po, p):
    want = po.random_dense(70, 130, p, 3)
    got = f2.BitMatrix.random_dense(70, 130, p, 3, ctx=ctx)
    assert same(got.words, want, 70)


def test_random_dense_seed_zero(f2, ctx, po):
    assert same(f2.BitMatrix.random_dense(50, 200, 0.5, 0, ctx=ctx).words,
                po.random_dense(50, 200, 0.5, 0), 50)


# ---------------------------------------------------------------------------
# K1+K2 M4RM products
# ---------------------------------------------------------------------------
SHAPES = [(1, 1, 1), (5, 64, 7), (64, 64, 64), (100, 129, 200), (300, 129, 200), (1025, 63, 17),
          (2047, 130, 1030), (1000, 1000, 1000), (4096, 4096, 4096), (33, 5000, 1024),
          (3000, 64, 1500), (1024, 1, 2048)]


@pytest.mark.parametrize("n,k,m", SHAPES)
def test_m4rm_mult(f2, ctx, po, n, k, m):
    a = po.random_dense(n, k, 0.5, n + 1)
    b = po.random_dense(k, m, 0.5, m + 2)
    want = po.m4rm_mult(a, n, k, b, m)
    got = f2.m4rm_mult(bm(f2, a, n, k), bm(f2, b, k, m), ctx=ctx)
    assert same(got.words, want, n)


def test_m4rm_mult_random_shapes(f2, ctx, po):
    rng = np.random.default_rng(7)
    for t in range(60):
        n, k, m = (int(x) for x in rng.integers(1, 1100, 3))
        a = po.random_dense(n, k, [0.5, 0.1, 0.01][t % 3], 100 + t)
        b = po.random_dense(k, m, 0.5, 200 + t)
        want = po.mul_naive(a, n, k, b, m) if n * k * m < 2e8 else po.m4rm_mult(a, n, k, b, m)
        got = f2.m4rm_mult(bm(f2, a, n, k), bm(f2, b, k, m), ctx=ctx)
        assert same(got.words, want, n), (n, k, m)


def test_m4rm_mult_shape_mismatch(f2, ctx):
    with pytest.raises(ValueError):
        f2.m4rm_mult(f2.BitMatrix(4, 5), f2.BitMatrix(6, 7), ctx=ctx)


def test_m4rm_mult_cfg2(f2, ctx, po):
    """BASELINE config 2: 16384^2 x 16384^2, seeds A=2, B=3."""
    n = 16384
    a = po.random_dense(n, n, 0.5, 2)
    b = po.random_dense(n, n, 0.5, 3)
    want = po.m4rm_mult(a, n, n, b, n)
    got = f2.m4rm_mult(bm(f2, a, n, n), bm(f2, b, n, n), ctx=ctx)
    assert same(got.words, want, n)


@pytest.mark.parametrize("n,k,m,cut", [(256, 256, 256, 128), (1024, 512, 768, 256),
                                       (512, 1024, 2048, 256), (2048, 2048, 2048, 512),
                                       (1000, 1000, 1000, 128)])
def test_strassen(f2, ctx, po, n, k, m, cut):
    a = po.random_dense(n, k, 0.5, 11)
    b = po.random_dense(k, m, 0.5, 12)
    want = po.m4rm_mult(a, n, k, b, m)
    got = f2.strassen_mult(bm(f2, a, n, k), bm(f2, b, k, m), threshold=cut, ctx=ctx)
    assert same(got.words, want, n)


def test_strassen_cfg2(f2, ctx, po):
    n = 16384
    a = po.random_dense(n, n, 0.5, 2)
    b = po.random_dense(n, n, 0.5, 3)
    want = po.m4rm_mult(a, n, n, b, n)
    got = f2.strassen_mult(bm(f2, a, n, n), bm(f2, b, n, n), threshold=4096, ctx=ctx)
    assert same(got.words, want, n)


# tensor-core leaf (evaluated alternative, tc_leaf.cu): 256x256 tiles on a
# pre-transposed B when m % 256 == 0, else the 128-column v1 kernel
TC_SHAPES = [(256, 64, 128), (256, 128, 256), (512, 64, 256), (256, 640, 384), (512, 192, 512),
             (1024, 1024, 1024), (2048, 4096, 1536), (768, 4160, 512),
             # block-scaled fp4 leaf: ragged n (240-row tiles) and ragged k
             (240, 64, 256), (1, 1, 256), (7, 100, 512), (1000, 777, 768), (4097, 130, 256),
             (3000, 5000, 1024)]


def _tc(f2, ctx, lib, a, b, n, k, m, acc, c0=None):
    A = f2.DeviceMatrix.from_host(f2.BitMatrix(n, k, a), ctx)
    B = f2.DeviceMatrix.from_host(f2.BitMatrix(k, m, b), ctx)
    C = f2.DeviceMatrix.from_host(f2.BitMatrix(n, m, c0), ctx) if c0 is not None else f2.DeviceMatrix(n, m, ctx)
    f2._lib.check(lib.f2gpu_gemm_tc(ctx.handle, A.handle, B.handle, C.handle, acc))
    return C.download().words


@pytest.mark.parametrize("n,k,m", TC_SHAPES)
def test_gemm_tc(f2, ctx, po, n, k, m):
    lib = f2._lib.load()
    if m % 256 and not experimental():  # the int8 leaf: only in experimental builds
        with pytest.raises(ValueError):
            _tc(f2, ctx, lib, po.zeros(n, k), po.zeros(k, m), n, k, m, 0)
        return
    a = po.random_dense(n, k, 0.5, n + 3 * k)
    b = po.random_dense(k, m, 0.5, k + 5 * m)
    assert same(_tc(f2, ctx, lib, a, b, n, k, m, 0), po.m4rm_mult(a, n, k, b, m), n)


def test_gemm_tc_accumulate(f2, ctx, po):
    lib = f2._lib.load()
    n, k, m = 512, 384, 512
    a, b, c = po.random_dense(n, k, 0.5, 1), po.random_dense(k, m, 0.5, 2), po.random_dense(n, m, 0.5, 3)
    want = po.m4rm_mult(a, n, k, b, m) ^ c
    assert same(_tc(f2, ctx, lib, a, b, n, k, m, 1, c0=c), want, n)


def test_gemm_tc_multiwave(f2, ctx, po):
    """4096^3: 256 CTAs over 148 SMs, 64 k-blocks (the raw/expanded rings wrap many
    times) -- the configuration that exposed a release-before-consume race."""
    lib = f2._lib.load()
    n = 4096
    A, B, Ct = (f2.DeviceMatrix(n, n, ctx) for _ in range(3))
    A.random_dense(0.5, 11)
    B.random_dense(0.5, 12)
    want = po.m4rm_mult(po.random_dense(n, n, 0.5, 11), n, n, po.random_dense(n, n, 0.5, 12), n)
    for _ in range(3):
        f2._lib.check(lib.f2gpu_gemm_tc(ctx.handle, A.handle, B.handle, Ct.handle, 0))
        assert np.array_equal(Ct.download().words[:, :n], want[:, :n])


def test_gemm_tc_rejects_shapes(f2, ctx):
    lib = f2._lib.load()
    A, B, C = f2.DeviceMatrix(200, 60, ctx), f2.DeviceMatrix(60, 128, ctx), f2.DeviceMatrix(200, 128, ctx)
    with pytest.raises(ValueError):
        f2._lib.check(lib.f2gpu_gemm_tc(ctx.handle, A.handle, B.handle, C.handle, 0))


# tensor-core trailing update (csrc/experimental/tc_update.cu): C[lo, hi) x [q0, q0+nwc) ^= A * BT^T
UPD_TC_CASES = [  # n, m, lo, hi, q0, nwc, kwords
    (300, 640, 5, 290, 1, 7, 2), (1000, 192, 0, 1000, 0, 3, 1), (4096, 1280, 1000, 4096, 3, 17, 2),
    (129, 256, 128, 129, 0, 4, 2), (20000, 3200, 777, 19999, 2, 47, 2), (640, 128, 0, 640, 0, 1, 2),
    (5000, 4096, 4999, 5000, 10, 54, 1)]


@needs_experimental
@pytest.mark.parametrize("n,m,lo,hi,q0,nwc,kw", UPD_TC_CASES)
def test_update_tc(f2, ctx, po, n, m, lo, hi, q0, nwc, kw):
    lib = f2._lib.load()
    seed = n + m + lo
    c = po.random_dense(n, m, 0.5, seed)
    a = po.random_dense(n, kw * 64, 0.5, seed + 1)
    bt = po.random_dense(nwc * 64, kw * 64, 0.5, seed + 2)
    am = a.copy()
    am[:, :lo] = 0
    am[:, hi:] = 0
    prod = po.m4rm_mult(am, n, kw * 64, po.transpose(bt, nwc * 64, kw * 64), nwc * 64)
    want = c.copy()
    want[q0:q0 + nwc, :n] ^= prod[:, :n]
    C = f2.DeviceMatrix.from_host(f2.BitMatrix(n, m, c), ctx)
    A = f2.DeviceMatrix.from_host(f2.BitMatrix(n, kw * 64, a), ctx)
    BT = f2.DeviceMatrix.from_host(f2.BitMatrix(nwc * 64, kw * 64, bt), ctx)
    f2._lib.check(lib.f2gpu_update_tc(ctx.handle, C.handle, lo, hi, q0, nwc, A.handle, 0, kw, BT.handle))
    assert same(C.download().words, want, n)


@pytest.mark.parametrize("k", [1, 7, 13, 56, 57, 64])
def test_mult_acc(f2, ctx, po, k):
    """C[r0.., w0..w0+nw) ^= a * B[b0..b0+k, bw0..] (m4rm.hpp:93-172 semantics)."""
    n, m = 3000, 64 * 40
    c = po.random_dense(n, m, 0.5, 5)
    b = po.random_dense(200, m, 0.5, 6)
    r0, nr, w0, nw, b0, bw0 = 37, 2500, 3, 21, 11, 5
    rng = np.random.default_rng(k)
    aw = rng.integers(0, 2**63, nr, dtype=np.uint64) & np.uint64((1 << k) - 1 if k < 64 else 2**64 - 1)
    want = c.copy()
    for q in range(nw):
        brow = b[bw0 + q, b0:b0 + k]
        for i in range(nr):
            x = int(aw[i])
            acc = 0
            while x:
                t = (x & -x).bit_length() - 1
                acc ^= int(brow[t])
                x &= x - 1
            want[w0 + q, r0 + i] ^= np.uint64(acc)
    dc = f2.DeviceMatrix.from_host(bm(f2, c, n, m), ctx)
    tables = f2.build_tables(bm(f2, b, 200, m), b0, k, bw0, nw, ctx=ctx)
    f2.mult_acc(dc, r0, w0, aw, tables)
    assert same(dc.download().words, want, n)


def test_mult_acc_errors(f2, ctx):
    with pytest.raises(ValueError):
        f2.build_tables(f2.BitMatrix(100, 64), 0, 65, 0, 1, ctx=ctx)
    with pytest.raises(IndexError):
        f2.build_tables(f2.BitMatrix(100, 64), 50, 64, 0, 1, ctx=ctx)


# ---------------------------------------------------------------------------
# decomposition
# ---------------------------------------------------------------------------
def check_decomp(f2, ctx, po, a, n, m, shards=1):
    w, perm, rj, rank = po.decompose_block(a, n, m)
    got = f2.decompose_block(bm(f2, a, n, m), ctx=ctx, shards=shards)
    assert got.rank == rank
    assert np.array_equal(got.block_ranks, rj)
    assert np.array_equal(got.P.perm, perm)
    assert same(got.overlay.words, w, n)
    return got


def _ymap(z, d):
    """Y_i = D_i * Z for a vector of 64-bit rows (bit b of D selects Z[b])."""
    y = np.zeros(d.shape, np.uint64)
    for b in range(64):
        y ^= np.where((d >> np.uint64(b)) & np.uint64(1), z[b], np.uint64(0)).astype(np.uint64)
    return y


def _panel_gpu(f2, ctx, col):
    import ctypes as C
    from paper_1209_5198_b200 import _lib
    col = np.ascontiguousarray(col, dtype=np.uint64)
    out = np.zeros(max(col.size, 1), np.uint64)
    z = np.zeros(64, np.uint64)
    r = C.c_uint32()
    pairs = np.zeros(256, np.uint32)
    npairs = C.c_uint32()
    _lib.check(_lib.load().f2gpu_panel_build_z(ctx.handle, col.ctypes.data, col.size, out.ctypes.data,
                                               z.ctypes.data, C.byref(r), pairs.ctypes.data, C.byref(npairs)))
    # the pair list must reproduce the swapped column from the input
    np_ = npairs.value
    assert np_ <= 128
    moved = col.copy()
    moved[pairs[:np_].astype(np.int64)] = col[pairs[128:128 + np_].astype(np.int64)]
    assert np.array_equal(moved, out[:col.size]), "pair list disagrees with the swapped column"
    return r.value, out[:col.size], z


def _panel_cases():
    rng = np.random.default_rng(7)
    cases = []
    for rows in (1, 5, 63, 64, 65, 96, 97, 100, 130, 300, 2047, 2048, 2049, 5000):
        for p in (0.5, 0.1, 0.01, 0.002):
            bits = rng.random((rows, 64)) < p
            col = np.zeros(rows, np.uint64)
            for b in range(64):
                col |= bits[:, b].astype(np.uint64) << np.uint64(b)
            cases.append(col)
    # pivots only beyond the 2048-row window (ext rows), duplicates, zeros
    far = np.zeros(4000, np.uint64)
    far[2500:2600] = rng.integers(0, 2**63, 100, dtype=np.uint64)
    cases.append(far)
    dup = rng.integers(0, 2**63, 200, dtype=np.uint64)
    dup[1::2] = dup[0::2]
    cases.append(dup)
    cases.append(np.zeros(300, np.uint64))
    return cases


def test_panel_build_z(f2, ctx, po):
    """The panel kernel against Procedure buildZ: block rank,
    the swapped column and Y = D*Z for every row below the pivots."""
    for col in _panel_cases():
        r, a, _, zo, _ = po.build_z(col)
        rg, ag, zg = _panel_gpu(f2, ctx, col)
        assert rg == r, (col.size, rg, r)
        assert np.array_equal(ag, a[:col.size]), col.size
        assert np.array_equal(_ymap(zg, ag[r:]), _ymap(zo, a[r:col.size])), col.size


DECOMP_SHAPES = [(1, 1), (4, 5), (64, 64), (100, 100), (200, 130), (130, 200), (513, 257),
                 (1000, 640), (640, 1000), (2048, 2048), (100, 3000), (3000, 100)]


@pytest.mark.parametrize("n,m", DECOMP_SHAPES)
@pytest.mark.parametrize("p", [0.5, 0.1, 0.01])
def test_decompose(f2, ctx, po, n, m, p):
    a = po.random_dense(n, m, p, n * 31 + m)
    check_decomp(f2, ctx, po, a, n, m)


def test_decompose_paper_example(f2, ctx, po):
    """PAPER.md section 3 example: rank 4."""
    A = f2.BitMatrix.from_rows(["10111", "10001", "11010", "00111"])
    got = check_decomp(f2, ctx, po, A.words, 4, 5)
    assert got.rank == 4


def test_decompose_adversarial(f2, ctx, po):
    n, m = 700, 500
    cases = [np.zeros((8, 704), np.uint64)]
    ident = f2.BitMatrix.identity(500)
    cases_nm = [(cases[0], n, m), (ident.words, 500, 500)]
    # rank-1 outer product u v^T
    rng = np.random.default_rng(1)
    u = rng.integers(0, 2, n).astype(np.uint8)
    v = rng.integers(0, 2, m).astype(np.uint8)
    cases_nm.append((po.from_dense(np.outer(u, v).astype(np.uint8)), n, m))
    # duplicate rows
    d = rng.integers(0, 2, (n, m)).astype(np.uint8)
    d[1::2] = d[0::2]
    cases_nm.append((po.from_dense(d), n, m))
    for a, nn, mm in cases_nm:
        got = check_decomp(f2, ctx, po, a, nn, mm)
        assert got.rank == po.rank_ge(a, nn, mm)


def test_decompose_rank_deficient_xy(f2, ctx, po):
    """cfg3 in miniature: A = X*Y with X 2048x1500, Y 1500x8192 (rank <= 1500)."""
    x = po.random_dense(2048, 1500, 0.5, 4)
    y = po.random_dense(1500, 8192, 0.5, 5)
    a = po.m4rm_mult(x, 2048, 1500, y, 8192)
    got = check_decomp(f2, ctx, po, a, 2048, 8192)
    assert got.rank == 1500


@pytest.mark.parametrize("shards", [2, 3, 4, 8])
def test_decompose_sharded(f2, ctx, po, shards):
    for (n, m, p) in [(1000, 1000, 0.5), (700, 1300, 0.1), (1500, 640, 0.5)]:
        a = po.random_dense(n, m, p, 17 + shards)
        check_decomp(f2, ctx, po, a, n, m, shards=shards)


def test_decompose_recomposes(f2, ctx, po):
    n, m = 1000, 900
    a = po.random_dense(n, m, 0.5, 9)
    got = f2.decompose_block(bm(f2, a, n, m), ctx=ctx)
    L, U = got.L, got.U
    lu = po.mul_naive(L.words, n, got.rank, U.words, m)
    pa = a[:, got.P.perm]
    assert np.array_equal(lu[:, :n], pa[:, :n])


def test_decompose_cfg1(f2, ctx, po):
    """BASELINE config 1: 4096^2, p=0.5, seed 1 — full bit-exact compare."""
    a = po.random_dense(4096, 4096, 0.5, 1)
    check_decomp(f2, ctx, po, a, 4096, 4096)


@pytest.mark.parametrize("n,m", [(300, 700), (700, 300), (64, 4096), (1000, 1000), (5, 3000)])
def test_rank(f2, ctx, po, n, m):
    a = po.random_dense(n, m, 0.5, 21)
    assert f2.rank(bm(f2, a, n, m), ctx=ctx) == po.rank_ge(a, n, m)


def test_rank_low(f2, ctx, po):
    x = po.random_dense(900, 37, 0.5, 1)
    y = po.random_dense(37, 1200, 0.5, 2)
    a = po.m4rm_mult(x, 900, 37, y, 1200)
    assert f2.rank(bm(f2, a, 900, 1200), ctx=ctx) == po.rank_ge(a, 900, 1200) <= 37


@pytest.mark.parametrize("n,m", [(64, 64), (100, 37), (37, 100), (1000, 4097), (130, 1)])
def test_transpose(f2, ctx, po, n, m):
    import ctypes as C
    from paper_1209_5198_b200 import _lib

    a = po.random_dense(n, m, 0.5, 3)
    want = po.transpose(a, n, m)
    da = f2.DeviceMatrix.from_host(bm(f2, a, n, m), ctx)
    dt = f2.DeviceMatrix(m, n, ctx)
    _lib.check(_lib.load().f2gpu_mat_transpose(ctx.handle, da.handle, dt.handle))
    assert same(dt.download().words, want, m)


def test_decompose_graph_replay(f2, ctx, po):
    """Same matrix/shape three times: eager run, graph capture, graph replay —
    all bit-identical to the oracle (the replay must not reuse stale state)."""
    import ctypes as C

    from paper_1209_5198_b200 import _lib

    lib = _lib.load()
    n, m = 3000, 2500
    for seed in (1, 2):  # second seed: same shape, new content through the replayed graph
        a = po.random_dense(n, m, 0.5, seed)
        w, perm, rj, rank = po.decompose_block(a, n, m)
        A = f2.DeviceMatrix.from_host(f2.BitMatrix(n, m, a), ctx)
        W = f2.DeviceMatrix(n, m, ctx)
        for it in range(3):
            _lib.check(lib.f2gpu_mat_copy(ctx.handle, W.handle, A.handle))
            p = np.zeros(n, np.uint32)
            r = np.zeros((m + 63) // 64, np.uint32)
            rk = C.c_size_t()
            _lib.check(lib.f2gpu_decompose_block(ctx.handle, W.handle, p.ctypes.data,
                                                 r.ctypes.data, C.byref(rk)))
            got = W.download()
            assert rk.value == rank and np.array_equal(p, perm) and np.array_equal(r, rj)
            assert np.array_equal(got.words[:, :n], w[:, :n]), (seed, it)


# ---------------------------------------------------------------------------
# decompose_recursive: bit-identical to the block algorithm (oracle)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n,m,p,min_cols", [(1000, 1000, 0.5, 64), (2048, 2048, 0.5, 128),
                                            (3000, 2500, 0.5, 64), (700, 1300, 0.1, 64),
                                            (1300, 700, 0.5, 128), (4096, 4096, 0.5, 256),
                                            (2000, 2000, 0.01, 64), (640, 1000, 0.5, 64)])
def test_decompose_recursive(f2, ctx, po, n, m, p, min_cols):
    a = po.random_dense(n, m, p, n + 3 * m)
    w, perm, rj, rank = po.decompose_block(a, n, m)
    got = f2.decompose_recursive(bm(f2, a, n, m), min_cols=min_cols, ctx=ctx)
    assert got.rank == rank
    assert np.array_equal(got.block_ranks, rj)
    assert np.array_equal(got.P.perm, perm)
    assert same(got.overlay.words, w, n)


def test_decompose_recursive_rank_deficient(f2, ctx, po):
    """Left halves below full rank take the exact rank-r_j fallback."""
    x = po.random_dense(3000, 900, 0.5, 4)
    y = po.random_dense(900, 4000, 0.5, 5)
    a = po.m4rm_mult(x, 3000, 900, y, 4000)
    w, perm, rj, rank = po.decompose_block(a, 3000, 4000)
    got = f2.decompose_recursive(bm(f2, a, 3000, 4000), min_cols=128, ctx=ctx)
    assert got.rank == rank == 900
    assert np.array_equal(got.P.perm, perm) and np.array_equal(got.block_ranks, rj)
    assert same(got.overlay.words, w, 3000)


def _wcols(po, n, parts, seed):
    """Word-column concatenation of blocks: ("rand", cols) | ("zero", cols) | ("xy", cols, rank)."""
    out = []
    for i, part in enumerate(parts):
        kind, cols = part[0], part[1]
        assert cols % 64 == 0
        if kind == "rand":
            blk = po.random_dense(n, cols, 0.5, seed + 10 * i)
        elif kind == "zero":
            blk = np.zeros_like(po.random_dense(n, cols, 0.5, 1))
        else:
            blk = po.m4rm_mult(po.random_dense(n, part[2], 0.5, seed + 10 * i), n, part[2],
                               po.random_dense(part[2], cols, 0.5, seed + 10 * i + 1), cols)
        out.append(blk[:cols // 64])
    return np.ascontiguousarray(np.concatenate(out, axis=0))


@pytest.mark.parametrize("n,parts,min_cols", [
    # left half = 5 full-rank panels, 2 zero panels, 1 full panel; the rest is dense
    (2048, [("rand", 320), ("zero", 128), ("rand", 1600)], 512),
    # a full-rank prefix, then rank 100 spread over two panels, then nothing (all-zero remainder)
    (2048, [("rand", 640), ("xy", 3456, 100)], 1024),
    # no rows left after the left half (n < m): every later panel has rank 0
    (512, [("rand", 2048)], 512),
    # rank runs out inside a left half whose pivot rows are not 64-aligned
    (1500, [("xy", 1024, 70), ("rand", 1024)], 256),
    # all zero
    (700, [("zero", 1024)], 256),
])
def test_decompose_recursive_deficient_splits(f2, ctx, po, n, parts, min_cols):
    """Rank-deficient left halves: the full-rank prefix goes through TRSM + product,
    the panels after it through rank-r_j updates (zero-rank ones skipped), and an
    all-zero remainder skips its panel chain (k_any_nonzero / k_fill_zero_states)."""
    m = sum(p[1] for p in parts)
    a = _wcols(po, n, parts, 31)
    w, perm, rj, rank = po.decompose_block(a, n, m)
    for _ in range(3):  # eager, capture, replay of the leaves
        got = f2.decompose_recursive(bm(f2, a, n, m), min_cols=min_cols, ctx=ctx)
        assert got.rank == rank
        assert np.array_equal(got.P.perm, perm) and np.array_equal(got.block_ranks, rj)
        assert same(got.overlay.words, w, n)


# ---------------------------------------------------------------------------
# product leaf selection: the fp4 tensor-core Strassen plan (B transposed once,
# batched leaves) against M4RM and the oracle, 0-2 Strassen levels
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n,k,m,leaf", [(2048, 2048, 2048, 512), (1024, 1536, 2048, 512), (2048, 1024, 1024, 256),
                                        (1000, 700, 1300, 256), (4096, 4096, 4096, 1024)])
def test_strassen_tc_plan(f2, ctx, po, n, k, m, leaf):
    lib = f2._lib.load()
    a = po.random_dense(n, k, 0.5, n + 1)
    b = po.random_dense(k, m, 0.5, m + 2)
    A = f2.DeviceMatrix.from_host(f2.BitMatrix(n, k, a), ctx)
    B = f2.DeviceMatrix.from_host(f2.BitMatrix(k, m, b), ctx)
    C1, C2 = f2.DeviceMatrix(n, m, ctx), f2.DeviceMatrix(n, m, ctx)
    try:
        ctx.set_tc(True, leaf)
        f2._lib.check(lib.f2gpu_strassen_mult(ctx.handle, A.handle, B.handle, C1.handle, 0))
        ctx.set_tc(False)
        f2._lib.check(lib.f2gpu_strassen_mult(ctx.handle, A.handle, B.handle, C2.handle, 0))
    finally:
        ctx.set_tc(True)
    want = po.m4rm_mult(a, n, k, b, m)
    assert same(C1.download().words, want, n)
    assert same(C2.download().words, want, n)


@pytest.mark.parametrize("n,m,kind,mc", [(1500, 2300, "dense", 256), (4096, 8192, "dense", 1024),
                                         (3000, 5000, "xy", 512), (777, 4160, "dense", 64)])
def test_decompose_recursive_host(f2, ctx, po, n, m, kind, mc):
    """Host entry with the overlapped chunked upload (chunks of mc columns are
    materialised under the running row permutation when first needed)."""
    import ctypes as C
    lib = f2._lib.load()
    a = po.random_dense(n, m, 0.5, 77) if kind == "dense" else _xy(po, n, 1000, m, 5)
    w, perm, rj, rank = po.decompose_block(a, n, m)
    stride = a.shape[1]
    wout = np.zeros_like(a)
    p = np.zeros(n, np.uint32)
    r = np.zeros((m + 63) // 64, np.uint32)
    rk = C.c_size_t()
    f2._lib.check(lib.f2gpu_decompose_recursive_host(ctx.handle, a.ctypes.data, n, m, stride, mc,
                                                     wout.ctypes.data, p.ctypes.data, r.ctypes.data,
                                                     C.byref(rk)))
    assert rk.value == rank
    assert np.array_equal(p, perm) and np.array_equal(r, rj)
    assert same(wout, w, n)


@needs_experimental
def test_gemm_tc_pair_kernel(f2, po):
    """The cta_group::2 leaf (opt-in via F2GPU_TC_PAIR=1) in a fresh process."""
    import os
    import subprocess
    import sys
    code = ("import numpy as np, paper_1209_5198_b200 as f2; from oracle import pyoracle as po; "
            "ctx=f2.Context(0); lib=f2._lib.load()\n"
            "for (n,k,m) in [(7,100,512),(2048,4096,1536),(3000,5000,1024),(481,64,512)]:\n"
            "    a=po.random_dense(n,k,0.5,n+k); b=po.random_dense(k,m,0.5,k+m)\n"
            "    A=f2.DeviceMatrix.from_host(f2.BitMatrix(n,k,a),ctx); B=f2.DeviceMatrix.from_host(f2.BitMatrix(k,m,b),ctx)\n"
            "    Cm=f2.DeviceMatrix(n,m,ctx); f2._lib.check(lib.f2gpu_gemm_tc(ctx.handle,A.handle,B.handle,Cm.handle,0))\n"
            "    assert np.array_equal(Cm.download().words[:, :n], po.m4rm_mult(a,n,k,b,m)[:, :n]), (n,k,m)\n"
            "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, F2GPU_TC_PAIR="1", PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@needs_experimental
def test_gemm_tc_persistent_kernel(f2, po):
    """The persistent fp4 leaf k_gemm_tc5 (opt-in via F2GPU_TC_PERSIST=1), in a fresh
    process: single products across tile counts below / above one wave, and the
    batched Strassen-Winograd path (problems of one launch share the tile loop)."""
    import os
    import subprocess
    import sys
    code = ("import numpy as np, paper_1209_5198_b200 as f2; from oracle import pyoracle as po; "
            "ctx=f2.Context(0); lib=f2._lib.load()\n"
            "for (n,k,m) in [(7,100,512),(2048,4096,1536),(3000,5000,1024),(481,64,512),(4800,1024,9728)]:\n"
            "    a=po.random_dense(n,k,0.5,n+k); b=po.random_dense(k,m,0.5,k+m)\n"
            "    A=f2.DeviceMatrix.from_host(f2.BitMatrix(n,k,a),ctx); B=f2.DeviceMatrix.from_host(f2.BitMatrix(k,m,b),ctx)\n"
            "    Cm=f2.DeviceMatrix(n,m,ctx); f2._lib.check(lib.f2gpu_gemm_tc(ctx.handle,A.handle,B.handle,Cm.handle,0))\n"
            "    assert np.array_equal(Cm.download().words[:, :n], po.m4rm_mult(a,n,k,b,m)[:, :n]), (n,k,m)\n"
            "n=1024; a=po.random_dense(n,n,0.5,5); b=po.random_dense(n,n,0.5,6); ctx.set_tc(True, 256)\n"
            "got=f2.strassen_mult(f2.BitMatrix(n,n,a), f2.BitMatrix(n,n,b), ctx=ctx)\n"
            "assert np.array_equal(got.words[:, :n], po.m4rm_mult(a,n,n,b,n)[:, :n])\n"
            "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, F2GPU_TC_PERSIST="1", F2GPU_TC5_MAXK="100000", PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@needs_experimental
def test_gemm_tc_double_buffered_kernel(f2, po):
    """The double-buffered short-k fp4 leaf k_gemm_tc6 (opt-in via F2GPU_TC6_MAXK) in a
    fresh process, on every product and on the batched Strassen-Winograd leaves."""
    import os
    import subprocess
    import sys
    code = ("import numpy as np, paper_1209_5198_b200 as f2; from oracle import pyoracle as po; "
            "ctx=f2.Context(0); lib=f2._lib.load()\n"
            "for (n,k,m) in [(7,100,512),(2048,4096,1536),(3000,5000,1024),(481,64,512),(4800,1024,9728),(240,64,256)]:\n"
            "    a=po.random_dense(n,k,0.5,n+k); b=po.random_dense(k,m,0.5,k+m)\n"
            "    A=f2.DeviceMatrix.from_host(f2.BitMatrix(n,k,a),ctx); B=f2.DeviceMatrix.from_host(f2.BitMatrix(k,m,b),ctx)\n"
            "    Cm=f2.DeviceMatrix(n,m,ctx); f2._lib.check(lib.f2gpu_gemm_tc(ctx.handle,A.handle,B.handle,Cm.handle,0))\n"
            "    assert np.array_equal(Cm.download().words[:, :n], po.m4rm_mult(a,n,k,b,m)[:, :n]), (n,k,m)\n"
            "n=1024; a=po.random_dense(n,n,0.5,5); b=po.random_dense(n,n,0.5,6); ctx.set_tc(True, 256)\n"
            "got=f2.strassen_mult(f2.BitMatrix(n,n,a), f2.BitMatrix(n,n,b), ctx=ctx)\n"
            "assert np.array_equal(got.words[:, :n], po.m4rm_mult(a,n,n,b,n)[:, :n])\n"
            "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, F2GPU_TC6_MAXK="100000", PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def _fresh_process(code, **env_extra):
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PYTHONPATH=root, **env_extra)
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def test_scratch_growth_one_context():
    """Growing shapes in ONE fresh context: every growth reallocates the panel
    scratch (states, perm, counters, hand-off words) and drops the captured graphs;
    the first decomposition after each growth must still match the oracle."""
    _fresh_process(
        "import numpy as np, paper_1209_5198_b200 as f2; from oracle import pyoracle as po\n"
        "ctx=f2.Context(0)\n"
        "for n in (300, 1024, 1024, 2048, 4096):\n"
        "  for fn in (f2.decompose_block, f2.decompose_recursive):\n"
        "    a=po.random_dense(n,n,0.5,n); w,perm,rj,rank=po.decompose_block(a,n,n)\n"
        "    got=fn(f2.BitMatrix(n,n,a), ctx=ctx)\n"
        "    assert got.rank==rank and np.array_equal(got.P.perm, perm), (n, fn)\n"
        "    assert np.array_equal(got.overlay.words[:, :n], w[:, :n]), (n, fn)\n"
        "print('ok')\n")


def test_panel_hand_off():
    """The opt-in panel hand-off (F2GPU_PANEL_HAND=1: P(j+1) starts on P(j)'s done
    counter and applies panel j to its own first rows) on ragged and rank-deficient
    shapes, block and recursive."""
    _fresh_process(
        "import numpy as np, paper_1209_5198_b200 as f2; from oracle import pyoracle as po\n"
        "ctx=f2.Context(0)\n"
        "for (n,m,d,seed) in [(300,257,0.5,1),(1000,257,0.5,2),(513,257,0.5,3),(2000,700,0.5,4),"
        "(700,2000,0.5,5),(3000,3000,0.02,6),(4096,4096,0.5,7)]:\n"
        "  a=po.random_dense(n,m,d,seed); w,perm,rj,rank=po.decompose_block(a,n,m)\n"
        "  for fn in (f2.decompose_block, f2.decompose_recursive):\n"
        "    got=fn(f2.BitMatrix(n,m,a), ctx=ctx)\n"
        "    assert got.rank==rank and np.array_equal(got.P.perm, perm), (n, m, fn)\n"
        "    assert np.array_equal(got.overlay.words[:, :n], w[:, :n]), (n, m, fn)\n"
        "print('ok')\n", F2GPU_PANEL_HAND="1")


_CHAIN_CASES = (
    "import numpy as np, paper_1209_5198_b200 as f2; from oracle import pyoracle as po\n"
    "ctx=f2.Context(0)\n"
    # dense, ragged, wide (no rows left), sparse (pivots beyond the register block and the
    # 2048-row window: the slow path through slot/orig), rank-deficient, all-zero
    "cases=[(300,257,0.5,1),(1000,257,0.5,2),(513,257,0.5,3),(2000,700,0.5,4),(700,2000,0.5,5),"
    "(3000,3000,0.02,6),(6000,1024,0.003,8),(4096,4096,0.5,7),(5000,640,0.0,9)]\n"
    "for (n,m,d,seed) in cases:\n"
    "  a=po.random_dense(n,m,d,seed); w,perm,rj,rank=po.decompose_block(a,n,m)\n"
    "  for fn in (f2.decompose_block, f2.decompose_recursive):\n"
    "    for rep in range(3):\n"  # eager, capture (chain kernel outside the graph), replay
    "      got=fn(f2.BitMatrix(n,m,a), ctx=ctx)\n"
    "      assert got.rank==rank and np.array_equal(got.P.perm, perm), (n, m, fn, rep)\n"
    "      assert np.array_equal(got.block_ranks, rj), (n, m, fn, rep)\n"
    "      assert np.array_equal(got.overlay.words[:, :n], w[:, :n]), (n, m, fn, rep)\n"
    "x=po.random_dense(3000,900,0.5,4); y=po.random_dense(900,4000,0.5,5); a=po.m4rm_mult(x,3000,900,y,4000)\n"
    "w,perm,rj,rank=po.decompose_block(a,3000,4000)\n"
    "for fn in (f2.decompose_block, f2.decompose_recursive):\n"
    "  got=fn(f2.BitMatrix(3000,4000,a), ctx=ctx)\n"
    "  assert got.rank==rank==900 and np.array_equal(got.P.perm, perm) and np.array_equal(got.block_ranks, rj)\n"
    "  assert np.array_equal(got.overlay.words[:, :3000], w[:, :3000])\n"
    "print('ok')\n")


def test_panel_chain_fresh_process():
    """k_panel_chain (default): the very first decomposition of a process -- the chain
    CTA spins on counters of kernels launched after it, so every kernel of the fused
    schedule must already be loaded (CUDA loads lazily) -- then dense, ragged, wide,
    sparse (slow path), rank-deficient and zero inputs, eager / captured / replayed."""
    _fresh_process(_CHAIN_CASES, F2GPU_PANEL_CHAIN="1")


def test_panel_per_kernel_schedule():
    """F2GPU_PANEL_CHAIN=0: one k_panel_gj launch per panel on alternating side streams
    (the round-1/2 schedule, still used when a caller captures the library's launches)."""
    _fresh_process(_CHAIN_CASES, F2GPU_PANEL_CHAIN="0")


def test_panel_chain_one_sm_left():
    """F2GPU_CHAIN_SMS=1: the updates take every SM but the chain's."""
    _fresh_process(_CHAIN_CASES, F2GPU_PANEL_CHAIN="1", F2GPU_CHAIN_SMS="1")


@pytest.mark.parametrize("G", [2, 3, 8])
def test_strassen_mult_dist_shards(f2, ctx, po, G):
    """The column-sharded multiply at world 1 (broadcast = no-op), G shards emulated
    with f2gpu_mat_select_wcols: every shard's C columns equal the global product."""
    lib = f2._lib.load()
    n, k, m = 1500, 1200, 64 * 40
    a = po.random_dense(n, k, 0.5, 31)
    b = po.random_dense(k, m, 0.5, 32)
    want = po.m4rm_mult(a, n, k, b, m)
    A = f2.DeviceMatrix.from_host(f2.BitMatrix(n, k, a), ctx)
    B = f2.DeviceMatrix.from_host(f2.BitMatrix(k, m, b), ctx)
    C = f2.DeviceMatrix(n, m, ctx)
    mu = m // 64
    for g in range(G):
        lw = int(lib.f2gpu_local_wcols(mu, g, G))
        Bl, Cl = f2.DeviceMatrix(k, 64 * lw, ctx), f2.DeviceMatrix(n, 64 * lw, ctx)
        f2._lib.check(lib.f2gpu_mat_select_wcols(ctx.handle, Bl.handle, B.handle, g, G, 0))
        f2._lib.check(lib.f2gpu_strassen_mult_dist(ctx.handle, A.handle, Bl.handle, Cl.handle, 0))
        f2._lib.check(lib.f2gpu_mat_select_wcols(ctx.handle, C.handle, Cl.handle, g, G, 1))
    assert same(C.download().words, want, n)


# ---------------------------------------------------------------------------
# null space / solve: properties against the oracle
# ---------------------------------------------------------------------------
def _xy(po, n, k, m, seed):
    x, y = po.random_dense(n, k, 0.5, seed), po.random_dense(k, m, 0.5, seed + 1)
    return po.m4rm_mult(x, n, k, y, m)


NS_CASES = [("dense", 300, 300), ("dense", 100, 700), ("dense", 700, 100), ("xy", 500, 640), ("xy", 640, 500),
            ("zero", 70, 130), ("ident", 128, 128), ("dense", 1, 1), ("dense", 1, 65), ("xy", 2000, 3000)]


@pytest.mark.parametrize("kind,n,m", NS_CASES)
def test_null_space(f2, ctx, po, kind, n, m):
    if kind == "dense":
        a = po.random_dense(n, m, 0.5, n + 3 * m)
    elif kind == "xy":
        a = _xy(po, n, min(n, m) // 3, m, n + m)
    elif kind == "zero":
        a = po.zeros(n, m)
    else:
        a = po.from_dense(np.eye(n, dtype=np.uint8))
    r = po.rank_ge(a, n, m)
    N = f2.null_space(f2.BitMatrix(n, m, a), ctx=ctx)
    assert N.rows() == m and N.cols() == m - r
    if N.cols():
        assert not po.m4rm_mult(a, n, m, N.words, N.cols())[:, :n].any()   # A * N = 0
        assert po.rank_ge(N.words, m, N.cols()) == N.cols()                 # independent columns


def _matvec(po, a, n, m, x):
    xm = po.zeros(m, 1)
    xm[0, :m] = x.astype(np.uint64)
    return (po.m4rm_mult(a, n, m, xm, 1)[0, :n] & np.uint64(1)).astype(np.uint8)


@pytest.mark.parametrize("kind,n,m", [("dense", 300, 300), ("dense", 200, 500), ("xy", 400, 300),
                                      ("xy", 300, 700), ("dense", 700, 100)])
def test_solve(f2, ctx, po, kind, n, m):
    a = po.random_dense(n, m, 0.5, 5 * n + m) if kind == "dense" else _xy(po, n, min(n, m) // 4, m, n)
    A = f2.BitMatrix(n, m, a)
    rng = np.random.default_rng(n * m)
    # consistent: b = A x0
    x0 = rng.integers(0, 2, m, dtype=np.uint8)
    b = _matvec(po, a, n, m, x0)
    x = f2.solve(A, b, ctx=ctx)
    assert x is not None and np.array_equal(_matvec(po, a, n, m, x), b)
    # random rhs: solvable exactly when rank([A | b]) == rank(A)
    b2 = rng.integers(0, 2, n, dtype=np.uint8)
    ab = po.zeros(n, m + 1)
    ab[: (m + 63) // 64, : a.shape[1]] = a
    ab[m // 64, :n] |= b2.astype(np.uint64) << np.uint64(m % 64)
    consistent = po.rank_ge(ab, n, m + 1) == po.rank_ge(a, n, m)
    x2 = f2.solve(A, b2, ctx=ctx)
    assert (x2 is not None) == consistent
    if x2 is not None:
        assert np.array_equal(_matvec(po, a, n, m, x2), b2)
