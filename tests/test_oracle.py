"""CPU: the oracle pinned against the reference (compiled in place) and the
committed golden fixtures, plus the SPEC known-answer tests and properties.

Runs without a GPU (-m "not gpu").
"""
import json
from pathlib import Path

import numpy as np
import pytest

GOLD = Path(__file__).resolve().parent / "golden"


# ---------------------------------------------------------------------------
# SPEC known-answer tests (SPEC.md section "packed_matrix", "tuning", "pivoting")
# ---------------------------------------------------------------------------
def test_paper_example_packing(po):
    """PAPER.md section 3: [10111;10001;11010;00111] -> at b=64 words 29,17,11,28
    (b=3 grid [[5,3],[1,2],[3,1],[4,3]])."""
    d = np.array([[1, 0, 1, 1, 1], [1, 0, 0, 0, 1], [1, 1, 0, 1, 0], [0, 0, 1, 1, 1]], np.uint8)
    a = po.from_dense(d)
    assert a[0, :4].tolist() == [29, 17, 11, 28]
    # b = 3 emulated packing: word (i,q) = sum_k d[i,3q+k] 2^k
    grid = [[sum(int(d[i, 3 * q + k]) << k for k in range(3) if 3 * q + k < 5) for q in range(2)]
            for i in range(4)]
    assert grid == [[5, 3], [1, 2], [3, 1], [4, 3]]
    assert d[0, 2] == 1 and d[3, 0] == 0  # get(0,2)=1, get(3,0)=0
    # row-XOR of r1 into r0 over both word-columns -> (4, 1) at b=3
    assert [grid[0][q] ^ grid[1][q] for q in range(2)] == [4, 1]


def test_paper_example_rank(po):
    d = np.array([[1, 0, 1, 1, 1], [1, 0, 0, 0, 1], [1, 1, 0, 1, 0], [0, 0, 1, 1, 1]], np.uint8)
    a = po.from_dense(d)
    w, perm, rj, rank = po.decompose_block(a, 4, 5)
    assert rank == 4 == po.rank_ge(a, 4, 5)


def test_tuning_kats(po):
    """SPEC.md:409,425-427,528."""
    from paper_1209_5198_b200 import tuning

    assert po.lib().f2o_m4rm_cost(64, 5, 64) == pytest.approx(1216.0)
    assert tuning.m4rm_cost(64, 5, 64) == pytest.approx(1216.0)
    for c, v in [(5, 406), (2, 106), (8, 1882)]:
        assert po.lib().f2o_strassen_threshold(c) == v == tuning.strassen_threshold(c)
    # integer argmin over c in 2..10 of C(64,c,64) = 5; of C(32,c,32) = 4
    assert min(range(2, 11), key=lambda c: tuning.m4rm_cost(64, c, 64)) == 5
    assert min(range(2, 11), key=lambda c: tuning.m4rm_cost(32, c, 32)) == 4
    assert tuning.optimal_table_size(64, 64) == 5 == po.lib().f2o_optimal_table_size(64, 64.0)
    assert tuning.optimal_table_size(32, 32) == 4
    for n, c in [(1024, 8), (4096, 9), (16384, 11), (65536, 13)]:
        assert tuning.optimal_table_size(64, n) == c == po.lib().f2o_optimal_table_size(64, float(n))
    assert tuning.optimal_table_size(64, 1e6) >= tuning.optimal_table_size(64, 10)
    assert tuning.predicted_decomposition_cost(64.0, 64, 1, "one") / \
        tuning.predicted_decomposition_cost(64.0, 64, 1, "full") == pytest.approx(1.5)


def test_build_z_identity_and_zero(po):
    ident = np.array([1 << i for i in range(64)], dtype=np.uint64)
    r, A, P, Z, sb = po.build_z(ident)
    assert r == 64 and P.tolist() == list(range(64)) and Z.tolist() == ident.tolist()
    r, A, P, Z, sb = po.build_z(np.zeros(100, np.uint64))
    assert r == 0 and (P == -1).all()


def _mul_word(y, rows):
    acc = 0
    y = int(y)
    while y:
        t = (y & -y).bit_length() - 1
        acc ^= int(rows[t])
        y &= y - 1
    return acc


@pytest.mark.parametrize("rank_target", [0, 1, 5, 17, 40, 63, 64])
def test_build_z_properties(po, rank_target):
    """B'Z = I_r and every rejected row lies in span(B')."""
    rng = np.random.default_rng(rank_target)
    for trial in range(30):
        basis = rng.integers(0, 2**63, rank_target, dtype=np.uint64) * np.uint64(2) + \
            rng.integers(0, 2, rank_target, dtype=np.uint64)
        rows = int(rng.integers(rank_target, 300)) if rank_target else int(rng.integers(1, 300))
        coef = rng.integers(0, 2**63, rows, dtype=np.uint64)
        panel = np.array([_mul_word(int(coef[i]) & ((1 << rank_target) - 1), basis)
                          for i in range(rows)], dtype=np.uint64)
        r, A, P, Z, sb = po.build_z(panel)
        assert r <= rank_target
        B = A[:r]
        for t in range(r):  # row t of B'Z = e_t
            assert _mul_word(B[t], Z) == (1 << t)
        for i in range(r, rows):  # D = (D Z) B'
            y = _mul_word(A[i], Z)
            assert _mul_word(y, B) == int(A[i])
        assert sorted(A.tolist()) == sorted(panel.tolist())  # a permutation of the rows


# ---------------------------------------------------------------------------
# oracle vs the reference compiled in place (oracle/_ref) and golden fixtures
# ---------------------------------------------------------------------------
def test_prng_golden(po):
    g = json.loads((GOLD / "prng.json").read_text())
    for seed, outs in g["xorshift64star"].items():
        import ctypes as C

        st = C.c_uint64(po.lib().f2o_rng_seed(int(seed)))
        got = [po.lib().f2o_rng_next(C.byref(st)) for _ in range(len(outs))]
        assert got == outs
    assert po.lib().f2o_bernoulli_threshold(0.05) == 0x0CCCCCCCCCCCCD00
    assert po.lib().f2o_bernoulli_threshold(0.5) == 1 << 63


def test_random_dense_golden(po):
    data = np.load(GOLD / "random_dense.npz")
    meta = json.loads((GOLD / "random_dense.json").read_text())
    for key, (n, m, p, seed) in meta.items():
        want = data[key]
        got = po.random_dense(n, m, p, seed)
        assert np.array_equal(got[:, :n], want[:, :n]), key


def test_m4rm_golden(po):
    data = np.load(GOLD / "m4rm.npz")
    meta = json.loads((GOLD / "m4rm.json").read_text())
    for key, (n, k, m, sa, sb) in meta.items():
        a = po.random_dense(n, k, 0.5, sa)
        b = po.random_dense(k, m, 0.5, sb)
        assert np.array_equal(po.m4rm_mult(a, n, k, b, m)[:, :n], data[key][:, :n]), key
        assert np.array_equal(po.mul_naive(a, n, k, b, m)[:, :n], data[key][:, :n]), key


def test_transpose_golden(po):
    data = np.load(GOLD / "transpose.npz")
    for key in data.files:
        n, m = (int(x) for x in key.split("x"))
        a = po.random_dense(n, m, 0.5, n + m)
        assert np.array_equal(po.transpose(a, n, m)[:, :m], data[key][:, :m]), key


def test_decompose_golden(po):
    """Decomposition fixtures from oracle/_ref (reference build_tables/mult_acc +
    restated buildZ): overlay, perm, r_j, rank bit-exact."""
    data = np.load(GOLD / "decompose.npz")
    meta = json.loads((GOLD / "decompose.json").read_text())
    for key, (n, m, p, seed) in meta.items():
        a = po.random_dense(n, m, p, seed)
        w, perm, rj, rank = po.decompose_block(a, n, m)
        assert rank == int(data[key + "_rank"])
        assert np.array_equal(perm, data[key + "_perm"])
        assert np.array_equal(rj, data[key + "_rj"])
        assert np.array_equal(w[:, :n], data[key + "_w"][:, :n])


def test_digests_golden(po):
    """Full-size digests computed once with the oracle (tests/golden/make_golden.py)."""
    g = json.loads((GOLD / "digests.json").read_text())
    c = g["cfg1"]
    a = po.random_dense(c["n"], c["m"], c["p"], c["seed"])
    assert po.digest(a, c["n"], c["m"]) == c["input_digest"]
    w, perm, rj, rank = po.decompose_block(a, c["n"], c["m"])
    assert rank == c["rank"]
    assert po.digest(w, c["n"], c["m"]) == c["w_digest"]
    assert po.digest_u32(perm) == c["perm_digest"]


# ---------------------------------------------------------------------------
# properties (SPEC.md acceptance criteria 1-4, scaled to the CPU budget)
# ---------------------------------------------------------------------------
def test_mult_exact_random_shapes(po):
    """m4rm equals the naive triple loop on random shapes <= 1024."""
    rng = np.random.default_rng(0)
    for t in range(500):
        n, k, m = (int(x) for x in rng.integers(1, 1025 if t < 40 else 200, 3))
        a = po.random_dense(n, k, 0.5, t + 1)
        b = po.random_dense(k, m, 0.5, t + 1000)
        assert np.array_equal(po.m4rm_mult(a, n, k, b, m, int(rng.integers(2, 12)))[:, :n],
                              po.mul_naive(a, n, k, b, m)[:, :n]), (n, k, m)


def test_decompose_properties(po):
    """P A = L U, rank = Gaussian elimination, L/U structure."""
    rng = np.random.default_rng(1)
    for t in range(300):
        n, m = (int(x) for x in rng.integers(1, 300, 2))
        p = [0.01, 0.1, 0.5][t % 3]
        a = po.random_dense(n, m, p, t)
        w, perm, rj, rank = po.decompose_block(a, n, m)
        assert rank == po.rank_ge(a, n, m)
        assert sorted(perm.tolist()) == list(range(n))
        L, U, r = po.extract_lu(w, n, m, rj)
        lu = po.mul_naive(L, n, r, U, m) if r else po.zeros(n, m)
        assert np.array_equal(lu[:, :n], a[:, perm][:, :n])
        Ld = po.to_dense(L, n, r)
        for i in range(r):  # unit diagonal, zero above
            assert Ld[i, i] == 1 and not Ld[i, i + 1:].any()
        # U block staircase: block row j zero in word-columns < j
        R = 0
        for j, x in enumerate(rj.tolist()):
            if x:
                assert not U[:j, R:R + x].any()
            R += x


def test_decompose_adversarial(po):
    rng = np.random.default_rng(2)
    n, m = 200, 150
    cases = [np.zeros((n, m), np.uint8), np.eye(n, m, dtype=np.uint8)]
    u, v = rng.integers(0, 2, n), rng.integers(0, 2, m)
    cases.append(np.outer(u, v).astype(np.uint8))
    d = rng.integers(0, 2, (n, m)).astype(np.uint8)
    d[1::2] = d[0::2]
    cases.append(d)
    for dd in cases:
        a = po.from_dense(dd)
        w, perm, rj, rank = po.decompose_block(a, n, m)
        assert rank == po.rank_ge(a, n, m)
        assert po.check_plu(a, w, n, m, perm, rj, 3)


def test_check_plu_detects_corruption(po):
    """cmd_verify with an injected bit flip must fail."""
    n, m = 300, 300
    a = po.random_dense(n, m, 0.5, 5)
    w, perm, rj, rank = po.decompose_block(a, n, m)
    assert po.check_plu(a, w, n, m, perm, rj, 1)
    w2 = w.copy()
    w2[2, 100] ^= np.uint64(1 << 7)
    assert not (po.check_plu(a, w2, n, m, perm, rj, 1) and po.check_plu(a, w2, n, m, perm, rj, 2))


def test_ref_agrees_when_available(po):
    if not po.ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    rng = np.random.default_rng(3)
    for t in range(40):
        n, m = (int(x) for x in rng.integers(1, 500, 2))
        a = po.random_dense(n, m, [0.5, 0.05][t % 2], t)
        assert np.array_equal(po.ref_random_dense(n, m, [0.5, 0.05][t % 2], t)[:, :n], a[:, :n])
        r1 = po.decompose_block(a, n, m)
        r2 = po.ref_decompose_block(a, n, m)
        for x, y in zip(r1[:3], r2[:3]):
            assert np.array_equal(x, y)
        assert r1[3] == r2[3]
