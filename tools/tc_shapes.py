"""fp4 tensor-core product (f2gpu_gemm_tc) throughput across TRSM-like shapes (n x k x m)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1209_5198_b200 as f2  # noqa: E402
from paper_1209_5198_b200 import _lib  # noqa: E402

lib = _lib.load()
ctx = f2.Context(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
shapes = [(1024, 1024, 32768), (2048, 2048, 32768), (4096, 4096, 32768), (8192, 8192, 32768),
          (16384, 16384, 16384), (32768, 1024, 32768), (1024, 1024, 8192), (16384, 4096, 16384)]
for (n, k, m) in shapes:
    A, B, C = f2.DeviceMatrix(n, k, ctx), f2.DeviceMatrix(k, m, ctx), f2.DeviceMatrix(n, m, ctx)
    A.random_dense(0.5, 1)
    B.random_dense(0.5, 2)
    fn = lambda: _lib.check(lib.f2gpu_gemm_tc(ctx.handle, A.handle, B.handle, C.handle, 0))  # noqa: E731
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(10):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10
    print(f"{n:6d} x {k:6d} x {m:6d}: {t * 1000:9.1f} us  {n * k * m / (t * 1e-3) / 1e12:8.1f} Tbitop/s", flush=True)
    A.free(); B.free(); C.free()
