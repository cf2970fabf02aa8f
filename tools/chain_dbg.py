"""Debug: block decomposition n x w once (eager), print rank + digest of W/perm; env switches apply."""
import ctypes as C, sys, zlib
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_1209_5198_b200 as f2
from paper_1209_5198_b200 import _lib
lib = _lib.load()
ctx = f2.Context(0)
n, w = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
A = f2.DeviceMatrix(n, w, ctx); A.random_dense(0.5, 6)
W = f2.DeviceMatrix(n, w, ctx)
perm = np.zeros(n, np.uint32); rj = np.zeros(w // 64, np.uint32); rk = C.c_size_t()
for i in range(reps):
    _lib.check(lib.f2gpu_mat_copy(ctx.handle, W.handle, A.handle))
    _lib.check(lib.f2gpu_decompose_block(ctx.handle, W.handle, perm.ctypes.data, rj.ctypes.data, C.byref(rk)))
    h = W.download().words
    print(n, w, "rep", i, "rank", rk.value, "W", zlib.crc32(np.ascontiguousarray(h[:, :n]).tobytes()), "perm", zlib.crc32(perm.tobytes()), flush=True)
