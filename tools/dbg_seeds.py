"""Device decomposition vs the oracle over seeds for one shape: which seeds fail."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import paper_1209_5198_b200 as f2  # noqa: E402
from oracle import pyoracle as po  # noqa: E402
ctx = f2.Context(0)
n, m = int(sys.argv[1]), int(sys.argv[2])
bad = []
for seed in range(1, 13):
    a = po.random_dense(n, m, 0.5, seed)
    w, perm, rj, rank = po.decompose_block(a, n, m)
    got = f2.decompose_block(f2.BitMatrix(n, m, a), ctx=ctx)
    if not (np.array_equal(got.P.perm, perm) and np.array_equal(got.overlay.words[:, :n], w[:, :n])):
        bad.append(seed)
print(n, m, "failing seeds", bad)
