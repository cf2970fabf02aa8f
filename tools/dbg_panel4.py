import sys, ctypes as C
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import paper_1209_5198_b200 as f2  # noqa: E402
from paper_1209_5198_b200 import _lib  # noqa: E402
from oracle import pyoracle as po  # noqa: E402
ctx = f2.Context(0)
n, m, p = 3000, 100, 0.5
a = po.random_dense(n, m, p, n * 31 + m)
w1, perm1, rj1, rank1 = po.decompose_block(a, n, m, max_panels=1)
R = int(rj1[0])
col = np.ascontiguousarray(w1[1, R:n])
lib = _lib.load()
for it in range(300):
    out = np.zeros(col.size, np.uint64); z = np.zeros(64, np.uint64); r = C.c_uint32()
    pairs = np.zeros(256, np.uint32); npr = C.c_uint32()
    _lib.check(lib.f2gpu_panel_build_z(ctx.handle, col.ctypes.data, col.size, out.ctypes.data, z.ctypes.data,
                                       C.byref(r), pairs.ctypes.data, C.byref(npr)))
    k = npr.value
    moved = col.copy()
    moved[pairs[:k].astype(np.int64)] = col[pairs[128:128 + k].astype(np.int64)]
    if not np.array_equal(moved, out):
        d = np.nonzero(moved != out)[0]
        print("it", it, "np", k, "r", r.value, "bad positions", d[:20])
        print(" dst", pairs[:k].tolist())
        print(" src", pairs[128:128 + k].tolist())
        srcset = set(pairs[128:128+k].tolist()); dstset = set(pairs[:k].tolist())
        print(" src-dst", sorted(srcset - dstset), "dst-src", sorted(dstset - srcset))
        break
else:
    print("no failure")
