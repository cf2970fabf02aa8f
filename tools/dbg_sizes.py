"""Run device decompose_recursive on growing square sizes (time + rank), stop at the first error."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1209_5198_b200 as f2  # noqa: E402
from paper_1209_5198_b200 import _lib  # noqa: E402
import ctypes as C  # noqa: E402

ctx = f2.Context(0)
lib = _lib.load()
sizes = [int(x) for x in sys.argv[1:]] or [8192, 16384, 24576, 32768, 49152, 65536]
for n in sizes:
    W = f2.DeviceMatrix(n, n, ctx)
    lib.f2gpu_mat_random_dense(ctx.handle, W.handle, C.c_double(0.5), C.c_uint64(6))
    rank = C.c_size_t(0)
    for it in range(3):
        lib.f2gpu_mat_random_dense(ctx.handle, W.handle, C.c_double(0.5), C.c_uint64(6))
        ctx.sync()
        t = time.time()
        rc = lib.f2gpu_decompose_recursive(ctx.handle, W.handle, 0, None, None, C.byref(rank))
        dt = time.time() - t
        print(n, it, "rc", rc, "rank", rank.value, f"{dt*1e3:.1f} ms", lib.f2gpu_last_error().decode() if rc else "", flush=True)
        if rc:
            sys.exit(1)
