"""Exactness of the fp4 tensor-core leaf at large k with dense operands.

The leaf maps bits to E2M1 1.0 / 0.0 and reads the parity of the f32
accumulator (LSB of v + 2^23), so it is exact only if the tensor cores sum up
to k ones without rounding.  Bernoulli(0.5) operands keep the sums near k/4;
these tests drive the sums to k itself (all-ones, where C = k mod 2 in every
entry -- an analytic oracle) and to ~0.9 k (density 0.95, against the CPU
oracle), for k up to 65536, through f2gpu_gemm_tc (direct leaf, accumulating
and not) and strassen_mult (the leaf under Strassen-Winograd).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ones(po, n, m):
    a = po.zeros(n, m)
    full, rem = divmod(m, 64)
    a[:full, :n] = np.uint64(0xFFFFFFFFFFFFFFFF)
    if rem:
        a[full, :n] = np.uint64((1 << rem) - 1)
    return a


def _gemm_tc(f2, ctx, a, b, n, k, m, acc=0, c0=None):
    lib = f2._lib.load()
    A = f2.DeviceMatrix.from_host(f2.BitMatrix(n, k, a), ctx)
    B = f2.DeviceMatrix.from_host(f2.BitMatrix(k, m, b), ctx)
    Cm = f2.DeviceMatrix.from_host(f2.BitMatrix(n, m, c0), ctx) if c0 is not None else f2.DeviceMatrix(n, m, ctx)
    f2._lib.check(lib.f2gpu_gemm_tc(ctx.handle, A.handle, B.handle, Cm.handle, acc))
    out = Cm.download().words
    A.free(); B.free(); Cm.free()
    return out


@pytest.mark.parametrize("k", [16384, 16383, 32768, 32767, 65536, 65535])
def test_tc_leaf_all_ones(f2, ctx, po, k):
    n, m = 496, 512
    got = _gemm_tc(f2, ctx, _ones(po, n, k), _ones(po, k, m), n, k, m)
    want = _ones(po, n, m) if k % 2 else po.zeros(n, m)
    assert np.array_equal(got[:, :n], want[:, :n])


@pytest.mark.parametrize("k", [16384, 32768, 65536, 65535])
def test_tc_leaf_dense_095(f2, ctx, po, k):
    n, m = 480, 256
    a = po.random_dense(n, k, 0.95, k + 1)
    b = po.random_dense(k, m, 0.95, k + 2)
    c0 = po.random_dense(n, m, 0.5, k + 3)
    want = po.m4rm_mult(a, n, k, b, m)
    assert np.array_equal(_gemm_tc(f2, ctx, a, b, n, k, m)[:, :n], want[:, :n])
    assert np.array_equal(_gemm_tc(f2, ctx, a, b, n, k, m, acc=1, c0=c0)[:, :n], (want ^ c0)[:, :n])


@pytest.mark.parametrize("n,k,m,leaf", [(16384, 16384, 16384, 8192), (4096, 32768, 4096, 2048),
                                        (2048, 65536, 1024, 0)])
def test_tc_strassen_dense_095(f2, ctx, po, n, k, m, leaf):
    """strassen_mult on the fp4 leaf with density-0.95 operands (Strassen sums of
    dense quadrants are ~half dense, the unsplit products stay at 0.9 k)."""
    a = po.random_dense(n, k, 0.95, 11)
    b = po.random_dense(k, m, 0.95, 12)
    try:
        ctx.set_tc(True, leaf)
        got = f2.strassen_mult(f2.BitMatrix(n, k, a), f2.BitMatrix(k, m, b), threshold=0, ctx=ctx)
    finally:
        ctx.set_tc(True)
    assert np.array_equal(got.words[:, :n], po.m4rm_mult(a, n, k, b, m)[:, :n])
