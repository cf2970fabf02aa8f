"""GPU edge cases: empty shapes, structured matrices (zero, identity, all-ones,
one nonzero column) — bit-exact against the CPU oracle where it defines the
answer, else against the reference's documented result (SPEC.md:319-353:
an empty or all-zero matrix has rank 0, every r_j = 0, perm = identity).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

EMPTY = [(0, 0), (0, 5), (0, 130), (5, 0), (70, 0)]


def _check(f2, po, lu, a, n, m):
    w, perm, rj, rank = po.decompose_block(a, n, m)
    assert lu.rank == rank
    assert np.array_equal(lu.P.perm, perm[:n])
    assert np.array_equal(lu.block_ranks, rj[: (m + 63) // 64])
    assert np.array_equal(lu.overlay.words[:, :n], w[:, :n])


@pytest.mark.parametrize("n,m", EMPTY)
def test_decompose_empty(f2, ctx, po, n, m):
    a = f2.BitMatrix(n, m)
    for fn in (f2.decompose_block, f2.decompose_recursive):
        lu = fn(a, ctx=ctx)
        assert lu.rank == 0
        assert lu.P.perm.tolist() == list(range(n))
        assert lu.block_ranks.tolist() == [0] * ((m + 63) // 64)
    assert f2.rank(a, ctx=ctx) == 0


@pytest.mark.parametrize("n,k,m", [(0, 5, 7), (4, 0, 7), (4, 5, 0), (0, 0, 0), (130, 0, 70)])
def test_products_empty(f2, ctx, n, k, m):
    a, b = f2.BitMatrix(n, k), f2.BitMatrix(k, m)
    for c in (f2.m4rm_mult(a, b, ctx=ctx), f2.strassen_mult(a, b, ctx=ctx)):
        assert (c.rows(), c.cols()) == (n, m)
        assert not c.words.any()


@pytest.mark.parametrize("n,m", [(300, 200), (200, 300), (4096, 4096), (1000, 129)])
@pytest.mark.parametrize("kind", ["zero", "identity", "ones", "one_col"])
def test_decompose_structured(f2, ctx, po, n, m, kind):
    d = np.zeros((n, m), np.uint8)
    if kind == "identity":
        np.fill_diagonal(d, 1)
    elif kind == "ones":
        d[:] = 1
    elif kind == "one_col":
        d[n // 3:, m - 1] = 1  # only the last (ragged) column is nonzero
    a = f2.BitMatrix(n, m)
    for i, j in zip(*np.nonzero(d)):
        a.set(int(i), int(j), True)
    want_rank = {"zero": 0, "identity": min(n, m), "ones": 1, "one_col": 1}[kind]
    for fn in (f2.decompose_block, f2.decompose_recursive):
        lu = fn(a, ctx=ctx)
        assert lu.rank == want_rank, (fn.__name__, lu.rank)
        _check(f2, po, lu, a.words, n, m)
    assert f2.rank(a, ctx=ctx) == want_rank
