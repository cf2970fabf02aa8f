"""Debug dump of the fp4 leaf's raw f32 accumulators (F2GPU_TC_MODE=3) for tile (0,0)
against popcount dot products (diagnostic tool)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_1209_5198_b200 as f2  # noqa: E402
from oracle import pyoracle as po  # noqa: E402
from paper_1209_5198_b200 import _lib  # noqa: E402

os.environ["F2GPU_TC_MODE"] = "3"
lib = _lib.load()
ctx = f2.Context(0)
n, k, m = 8192, int(sys.argv[1]) if len(sys.argv) > 1 else 64, 256
a = po.random_dense(n, k, 0.5, 5)
b = po.random_dense(k, m, 0.5, 6)
A = f2.DeviceMatrix.from_host(f2.BitMatrix(n, k, a), ctx)
B = f2.DeviceMatrix.from_host(f2.BitMatrix(k, m, b), ctx)
Cm = f2.DeviceMatrix(n, m, ctx)
_lib.check(lib.f2gpu_gemm_tc(ctx.handle, A.handle, B.handle, Cm.handle, 0))
raw = Cm.download().words.reshape(-1).view(np.float32)[: 256 * 240].reshape(256, 240)  # [col][row]
ad = f2.BitMatrix(n, k, a).to_dense()[:240].astype(np.int64)
bd = f2.BitMatrix(k, m, b).to_dense().astype(np.int64)
want = (ad @ bd).T  # [col][row]
print("want[0,:8]", want[0, :8].tolist())
print("got [0,:8]", raw[0, :8].tolist())
print("want[1,:8]", want[1, :8].tolist())
print("got [1,:8]", raw[1, :8].tolist())
print("got [130,:8]", raw[130, :8].tolist(), "want", want[130, :8].tolist())
ratio = raw / np.maximum(want, 1)
print("ratio stats", float(np.median(ratio)), float(ratio.min()), float(ratio.max()))
print("exact", int((raw == want).sum()), "of", raw.size)
# does got match a different pairing? check correlation with transposed roles / permuted cols
for name, w in (("want", want),):
    c = np.corrcoef(raw.reshape(-1), w.reshape(-1))[0, 1]
    print("corr", name, c)
