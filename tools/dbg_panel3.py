import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np  # noqa: E402
import paper_1209_5198_b200 as f2  # noqa: E402
from oracle import pyoracle as po  # noqa: E402
from test_gpu_parity import _panel_gpu, _ymap  # noqa: E402
ctx = f2.Context(0)
n, m, p = 3000, 100, 0.5
a = po.random_dense(n, m, p, n * 31 + m)
w1, perm1, rj1, rank1 = po.decompose_block(a, n, m, max_panels=1)
R = int(rj1[0])
col = np.ascontiguousarray(w1[1, R:n])
r, ao, _, zo, _ = po.build_z(col)
bad = 0
for it in range(int(sys.argv[1])):
    rg, ag, zg = _panel_gpu(f2, ctx, col)
    ok = rg == r and np.array_equal(ag, ao[:col.size]) and np.array_equal(_ymap(zg, ag[r:]), _ymap(zo, ao[r:col.size]))
    if not ok:
        bad += 1
        d = np.nonzero(ag != ao[:col.size])[0]
        if bad < 4: print("it", it, "r", rg, r, "diff", d[:10], flush=True)
print("R", R, "r", r, "bad", bad)
