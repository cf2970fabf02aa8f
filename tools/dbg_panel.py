"""Panel kernel vs Procedure buildZ on the cases of test_panel_build_z, with details."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_1209_5198_b200 as f2  # noqa: E402
from oracle import pyoracle as po  # noqa: E402
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
from test_gpu_parity import _panel_cases, _panel_gpu, _ymap  # noqa: E402

ctx = f2.Context(0)
for ci, col in enumerate(_panel_cases()):
    r, a, _, zo, _ = po.build_z(col)
    rg, ag, zg = _panel_gpu(f2, ctx, col)
    a = a[:col.size]
    ok_a = np.array_equal(ag, a)
    ok_y = np.array_equal(_ymap(zg, ag[r:]), _ymap(zo, a[r:])) if ok_a else False
    if rg != r or not ok_a or not ok_y:
        d = np.nonzero(ag != a)[0]
        dens = np.mean([bin(int(v)).count('1') for v in col]) / 64
        print(f"case {ci} rows {col.size} dens {dens:.3f} r {rg} vs {r} rows_ok {ok_a} y_ok {ok_y} "
              f"diff_rows {d[:12]}")
print("done")
