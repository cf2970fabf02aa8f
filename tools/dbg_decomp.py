"""Decompose one shape on the device and diff it against the oracle: ranks,
permutation and the first differing word-columns."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_1209_5198_b200 as f2  # noqa: E402
from oracle import pyoracle as po  # noqa: E402

n, m, p, seed = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4]) if len(sys.argv) > 4 else 0
ctx = f2.Context(0)
a = po.random_dense(n, m, p, seed if seed else n + m)
w, perm, rj, rank = po.decompose_block(a, n, m)
got = f2.decompose_block(f2.BitMatrix(n, m, a), ctx=ctx)
print("rank", got.rank, rank, "rj equal", np.array_equal(got.block_ranks, rj))
print("perm equal", np.array_equal(got.P.perm, perm))
d = np.nonzero(got.P.perm != perm)[0]
print("perm diffs at", d[:20])
gw = got.overlay.words
bad = [q for q in range(w.shape[0]) if not np.array_equal(gw[q, :n], w[q, :n])]
print("bad word-columns", bad[:20])
for q in bad[:3]:
    rows = np.nonzero(gw[q, :n] != w[q, :n])[0]
    print(" col", q, "rows", rows[:20], "count", len(rows))
print("R per panel", np.cumsum(rj)[:20])
