"""CPU: serialization round trips (acceptance criterion 8)."""
import numpy as np
import pytest


def test_roundtrip_binary_and_text(po, tmp_path):
    from paper_1209_5198_b200 import BitMatrix
    from paper_1209_5198_b200.io import read_matrix, write_matrix

    rng = np.random.default_rng(0)
    for t in range(100):
        n, m = int(rng.integers(0, 140)), int(rng.integers(0, 200))
        a = BitMatrix(n, m, po.random_dense(n, m, 0.5, t)) if n and m else BitMatrix(n, m)
        for fmt in ("binary", "text"):
            p = tmp_path / f"m{t}.{fmt}"
            write_matrix(a, p, fmt)
            b = read_matrix(p)
            assert b.rows() == n and b.cols() == m and b == a


def test_paper_example_text(tmp_path):
    from paper_1209_5198_b200 import BitMatrix
    from paper_1209_5198_b200.io import read_matrix, write_matrix

    a = BitMatrix.from_rows(["10111", "10001", "11010", "00111"])
    p = tmp_path / "ex.txt"
    write_matrix(a, p, "text")
    text = p.read_text().splitlines()
    assert text[0] == "4 5" and text[1] == "10111"
    assert [read_matrix(p).word(i, 0) for i in range(4)] == [29, 17, 11, 28]
    q = tmp_path / "ex.bin"
    write_matrix(a, q, "binary")
    raw = q.read_bytes()
    assert raw[:4] == b"F2MX" and len(raw) == 4 + 24 + 4 * 8


def test_malformed(tmp_path):
    from paper_1209_5198_b200.io import read_matrix

    p = tmp_path / "bad.bin"
    p.write_bytes(b"F2MX" + (3).to_bytes(8, "little") + (3).to_bytes(8, "little") + (64).to_bytes(8, "little"))
    with pytest.raises(ValueError):
        read_matrix(p)
    q = tmp_path / "bad.txt"
    q.write_text("2 3\n101\n")
    with pytest.raises(ValueError):
        read_matrix(q)
