import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import paper_1209_5198_b200 as f2  # noqa: E402
from oracle import pyoracle as po  # noqa: E402
ctx = f2.Context(0)
n, m, p = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
a = po.random_dense(n, m, p, n * 31 + m)
w, perm, rj, rank = po.decompose_block(a, n, m)
for it in range(int(sys.argv[4])):
    got = f2.decompose_block(f2.BitMatrix(n, m, a), ctx=ctx)
    gp = got.P.perm
    if not np.array_equal(gp, perm):
        d = np.nonzero(gp != perm)[0]
        ow = [q for q in range(w.shape[0]) if not np.array_equal(got.overlay.words[q, :n], w[q, :n])]
        print("it", it, "perm diffs", len(d), d[:8], "got", gp[d[:8]], "want", perm[d[:8]], "bad wcols", ow,
              "rj", list(got.block_ranks), flush=True)
print("done")
