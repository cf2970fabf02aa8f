"""Matrix serialization (External Interfaces of `packed_matrix`).

Text:   line 1 "n m", then n lines of m characters from {0,1}; leftmost = column 0.
Binary: magic "F2MX", u64 LE n, m, b (= 64), then mu*n words of b bits, little-endian,
        in storage order (word-column-major, rows within a column, no padding rows).
"""
from __future__ import annotations

import io as _io
import struct
from pathlib import Path

import numpy as np

from . import BitMatrix

MAGIC = b"F2MX"


def write_matrix(a: BitMatrix, path, fmt: str = "binary") -> None:
    n, m = a.rows(), a.cols()
    if fmt == "binary":
        with open(path, "wb") as f:
            f.write(MAGIC + struct.pack("<QQQ", n, m, 64))
            f.write(np.ascontiguousarray(a.words[:, :n]).astype("<u8").tobytes())
    elif fmt == "text":
        d = a.to_dense()
        with open(path, "w") as f:
            f.write(f"{n} {m}\n")
            for i in range(n):
                f.write("".join("1" if x else "0" for x in d[i]) + "\n")
    else:
        raise ValueError(f"unknown format {fmt!r}")


def read_matrix(path, fmt: str | None = None) -> BitMatrix:
    raw = Path(path).read_bytes()
    if fmt is None:
        fmt = "binary" if raw[:4] == MAGIC else "text"
    if fmt == "binary":
        if raw[:4] != MAGIC or len(raw) < 28:
            raise ValueError("read_matrix: malformed header")
        n, m, b = struct.unpack("<QQQ", raw[4:28])
        if b != 64:
            raise ValueError(f"read_matrix: word size {b} not supported (64 only)")
        mu = (m + 63) // 64
        need = 28 + mu * n * 8
        if len(raw) < need:
            raise ValueError("read_matrix: truncated payload")
        a = BitMatrix(n, m)
        if n and mu:
            a.words[:, :n] = np.frombuffer(raw, dtype="<u8", count=mu * n, offset=28).reshape(mu, n)
        if not a.padding_is_zero():
            raise ValueError("read_matrix: nonzero padding bits")
        return a
    if fmt == "text":
        lines = _io.StringIO(raw.decode()).read().split("\n")
        try:
            n, m = (int(x) for x in lines[0].split())
        except Exception as e:
            raise ValueError("read_matrix: malformed header") from e
        rows = [ln.strip() for ln in lines[1:1 + n]]
        if len(rows) < n or any(len(r) != m for r in rows):
            raise ValueError("read_matrix: truncated or ragged payload")
        return BitMatrix.from_rows(rows) if n else BitMatrix(0, m)
    raise ValueError(f"unknown format {fmt!r}")
