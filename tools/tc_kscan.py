import sys
sys.path.insert(0, '/root/repo')
import torch
import paper_1209_5198_b200 as f2
from paper_1209_5198_b200 import _lib
lib = _lib.load()
ctx = f2.Context(0)
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream); ctx.set_stream(stream.cuda_stream)
n, m = 2400, 37888  # 10 x 148 tiles: exactly 10 waves... (n/240=10 row tiles, m/256=148 col tiles)
for k in (64, 128, 256, 512, 1024, 2048):
    A, B, C = f2.DeviceMatrix(n, k, ctx), f2.DeviceMatrix(k, m, ctx), f2.DeviceMatrix(n, m, ctx)
    A.random_dense(0.5, 1); B.random_dense(0.5, 2)
    fn = lambda: _lib.check(lib.f2gpu_gemm_tc(ctx.handle, A.handle, B.handle, C.handle, 0))
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(10): fn()
    e1.record(stream); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10
    print(f"k={k:5d}: {t*1000:8.1f} us total, {t*1000/10:6.2f} us per wave (1480 tiles = 10 waves)", flush=True)
    A.free(); B.free(); C.free()
