"""Where the host entry's time goes at 65536^2: full e2e, without the downloads
(w_out = NULL), and the device-resident decomposition of the same input."""
import ctypes as C
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_1209_5198_b200 as f2  # noqa: E402
from paper_1209_5198_b200 import _lib  # noqa: E402

lib = _lib.load()
ctx = f2.Context(0)
n = 65536
A = f2.DeviceMatrix(n, n, ctx); A.random_dense(0.5, 6)
words = A.download().words
stride = words.shape[1]
a = torch.from_numpy(np.ascontiguousarray(words).view(np.int64)).pin_memory()
w = torch.empty_like(a).pin_memory()
perm = np.zeros(n, np.uint32); rj = np.zeros(n // 64, np.uint32); rk = C.c_size_t()
W = f2.DeviceMatrix(n, n, ctx)


def host(wout):
    _lib.check(lib.f2gpu_decompose_recursive_host(ctx.handle, C.c_void_p(a.data_ptr()), n, n, stride, 0,
                                                  C.c_void_p(wout), perm.ctypes.data, rj.ctypes.data,
                                                  C.byref(rk)))


def dev():
    _lib.check(lib.f2gpu_mat_copy(ctx.handle, W.handle, A.handle))
    _lib.check(lib.f2gpu_decompose_recursive(ctx.handle, W.handle, 0, perm.ctypes.data, rj.ctypes.data,
                                             C.byref(rk)))
    torch.cuda.synchronize()


for name, fn in [("device", dev), ("host e2e", lambda: host(w.data_ptr())), ("host no download", lambda: host(0)),
                 ("device", dev), ("host e2e", lambda: host(w.data_ptr())), ("host no download", lambda: host(0))]:
    for _ in range(3):
        fn()
    ts = []
    for _ in range(5):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{name:18s} wall ms: min {min(ts):7.2f} median {sorted(ts)[2]:7.2f}", flush=True)
