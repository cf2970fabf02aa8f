import sys; sys.path.insert(0,'/root/repo')
import paper_1209_5198_b200 as f2
from paper_1209_5198_b200 import _lib
lib=_lib.load(); ctx=f2.Context(0)
n=16384
A,B,Cm=(f2.DeviceMatrix(n,n,ctx) for _ in range(3)); A.random_dense(0.5,2); B.random_dense(0.5,3)
for _ in range(2): _lib.check(lib.f2gpu_gemm_tc(ctx.handle,A.handle,B.handle,Cm.handle,0))
ctx.sync(); print("ok")
