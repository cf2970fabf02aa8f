"""The NCCL exchange path of the distributed driver on one GPU: a 1-rank
communicator (F2GPU_FORCE_NCCL=1) drives f2gpu_decompose_block_dist through
ncclBroadcast; results must equal the oracle bit-for-bit."""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_dist_decompose_through_nccl_one_rank(f2, po, monkeypatch):
    import torch  # noqa: F401  (loads torch's libnccl.so.2 first, as in bench.py)

    from paper_1209_5198_b200 import _lib

    monkeypatch.setenv("F2GPU_FORCE_NCCL", "1")
    lib = _lib.load()
    ctx = f2.Context(0)
    uid = f2.Context.nccl_unique_id()
    ctx.init_comm(0, 1, uid)
    n, m = 2000, 1500
    a = po.random_dense(n, m, 0.5, 31)
    W = f2.DeviceMatrix.from_host(f2.BitMatrix(n, m, a), ctx)
    perm = np.zeros(n, np.uint32)
    rj = np.zeros((m + 63) // 64, np.uint32)
    rk = C.c_size_t()
    _lib.check(lib.f2gpu_decompose_block_dist(ctx.handle, W.handle, m, perm.ctypes.data,
                                              rj.ctypes.data, C.byref(rk)))
    w, p0, r0, rank = po.decompose_block(a, n, m)
    assert rk.value == rank and np.array_equal(perm, p0) and np.array_equal(rj, r0)
    assert np.array_equal(W.download().words[:, :n], w[:, :n])
    W.free()
    ctx.close()
