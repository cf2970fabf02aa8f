import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np  # noqa: E402
import paper_1209_5198_b200 as f2  # noqa: E402
from oracle import pyoracle as po  # noqa: E402
from test_gpu_parity import _panel_cases, _panel_gpu  # noqa: E402
ctx = f2.Context(0)
col = _panel_cases()[56]
r, a, _, zo, _ = po.build_z(col)
rg, ag, zg = _panel_gpu(f2, ctx, col)
idx = {int(v): i for i, v in enumerate(col) if v}
for i in range(16):
    print(i, hex(int(a[i])), idx.get(int(a[i])), hex(int(ag[i])), idx.get(int(ag[i])))
