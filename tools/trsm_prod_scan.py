"""TRSM-shaped products C(n x m) ^= A(n x k) B(k x m), n = k: fp4 TC leaf vs M4RM."""
import sys
sys.path.insert(0, '/root/repo')
import torch
import paper_1209_5198_b200 as f2
from paper_1209_5198_b200 import _lib
lib = _lib.load()
ctx = f2.Context(0)
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream); ctx.set_stream(stream.cuda_stream)


def tm(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps): fn()
    e1.record(stream); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1000


for k in (512, 1024, 2048, 4096):
    for m in (8192, 32768, 57344):
        n = k
        A, B, C = f2.DeviceMatrix(n, k, ctx), f2.DeviceMatrix(k, m, ctx), f2.DeviceMatrix(n, m, ctx)
        A.random_dense(0.5, 1); B.random_dense(0.5, 2)
        t_tc = tm(lambda: _lib.check(lib.f2gpu_gemm_tc(ctx.handle, A.handle, B.handle, C.handle, 1)))
        t_m4 = tm(lambda: _lib.check(lib.f2gpu_m4rm_mult_acc(ctx.handle, A.handle, B.handle, C.handle)))
        print(f"n=k={k:5d} m={m:6d}  tc {t_tc:8.1f} us   m4rm {t_m4:8.1f} us   ratio {t_m4 / t_tc:5.2f}", flush=True)
