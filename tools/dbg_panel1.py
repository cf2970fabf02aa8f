import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np  # noqa: E402
import paper_1209_5198_b200 as f2  # noqa: E402
from oracle import pyoracle as po  # noqa: E402
from test_gpu_parity import _panel_gpu, _ymap  # noqa: E402
ctx = f2.Context(0)
rng = np.random.default_rng(3)
col = rng.integers(0, 2**63, 70, dtype=np.uint64)
r, a, zo, P, sb = po.build_z(col)
rg, ag, zg = _panel_gpu(f2, ctx, col)
print("r", r, rg, "rows equal", np.array_equal(ag, a[:70]))
print("zo", [hex(int(v)) for v in zo[:4]])
print("zg", [hex(int(v)) for v in zg[:4]])
print("Yo", [hex(int(v)) for v in _ymap(zo, a[r:70])])
print("Yg", [hex(int(v)) for v in _ymap(zg, ag[r:70])])
