"""Repeat device decompositions of several shapes in one context and count oracle mismatches."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_1209_5198_b200 as f2  # noqa: E402
from oracle import pyoracle as po  # noqa: E402

ctx = f2.Context(0)
shapes = [(1, 1), (4, 5), (64, 64), (100, 100), (200, 130), (130, 200), (513, 257), (1000, 640), (640, 1000),
          (2048, 2048), (100, 3000), (3000, 100)]
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
bad = 0
for rep in range(reps):
    for (n, m) in shapes:
        for p in (0.5, 0.1, 0.01):
            a = po.random_dense(n, m, p, n * 31 + m)
            w, perm, rj, rank = po.decompose_block(a, n, m)
            try:
                got = f2.decompose_block(f2.BitMatrix(n, m, a), ctx=ctx)
            except Exception as e:  # noqa: BLE001
                print("ERROR rep", rep, n, m, p, e, flush=True)
                raise
            ok = (got.rank == rank and np.array_equal(got.block_ranks, rj) and np.array_equal(got.P.perm, perm)
                  and np.array_equal(got.overlay.words[:, :n], w[:, :n]))
            if not ok:
                bad += 1
                print("MISMATCH rep", rep, n, m, p, "rank", got.rank, rank, "perm",
                      np.array_equal(got.P.perm, perm), flush=True)
print("bad", bad)
