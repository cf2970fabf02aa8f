"""Stress the panel kernel alone: many random columns (sizes across the window
edge, sparse densities so the slow path and ext rows run) vs Procedure buildZ."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np  # noqa: E402
import paper_1209_5198_b200 as f2  # noqa: E402
from oracle import pyoracle as po  # noqa: E402
from test_gpu_parity import _panel_gpu, _ymap  # noqa: E402
ctx = f2.Context(0)
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
N = int(sys.argv[1]) if len(sys.argv) > 1 else 500
bad = 0
for it in range(N):
    rows = int(rng.choice([50, 97, 200, 700, 2000, 2100, 3000, 5000]))
    p = float(rng.choice([0.5, 0.1, 0.03, 0.01, 0.003, 0.001]))
    bits = rng.random((rows, 64)) < p
    col = np.zeros(rows, np.uint64)
    for b in range(64):
        col |= bits[:, b].astype(np.uint64) << np.uint64(b)
    r, a, _, zo, _ = po.build_z(col)
    rg, ag, zg = _panel_gpu(f2, ctx, col)
    ok = rg == r and np.array_equal(ag, a[:rows]) and np.array_equal(_ymap(zg, ag[r:]), _ymap(zo, a[r:rows]))
    if not ok:
        bad += 1
        if bad <= 5:
            d = np.nonzero(ag != a[:rows])[0]
            print("it", it, "rows", rows, "p", p, "r", rg, r, "diff rows", d[:10], flush=True)
print("bad", bad, "of", N)
