import sys
sys.path.insert(0, '/root/repo')
import torch
import paper_1209_5198_b200 as f2
from paper_1209_5198_b200 import _lib
lib = _lib.load(); ctx = f2.Context(0)
n = 16384
A, B, C = (f2.DeviceMatrix(n, n, ctx) for _ in range(3))
A.random_dense(0.5, 1); B.random_dense(0.5, 2)
for _ in range(3):
    _lib.check(lib.f2gpu_gemm_tc(ctx.handle, A.handle, B.handle, C.handle, 0))
torch.cuda.synchronize()
