"""CPU, world_size 2 (gloo): the sharded decomposition protocol.

Restates, in numpy over torch.distributed(gloo), the exchange that
libf2gpu's decompose_sharded / f2gpu_decompose_block_dist performs with NCCL:
word-columns round-robin over ranks; per panel j the owner (j mod G) runs
buildZ on its local column, forms the composite row permutation and Y = D*Z,
and broadcasts {R, r, permutation pairs, panel column}; every rank mirrors the
permutation on its local columns and applies the Schur update to its local
columns right of j.  The gathered result must equal the single-process oracle
bit-for-bit (W, perm, r_j).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def composite_pairs(sb, r):
    """Transpositions (k, sb[k]) applied in order -> pairs new[dst] = old[src]."""
    orig = {}

    def get(x):
        return orig.get(x, x)

    for k in range(r):
        a, b = k, int(sb[k])
        oa, ob = get(a), get(b)
        orig[a], orig[b] = ob, oa
    return [(x, o) for x, o in sorted(orig.items()) if x != o]


def first_local_after(j, g, G):
    return 0 if j < g else (j - g) // G + 1


def worker(rank, world, port, n, m, p, seed, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import pyoracle as po

    a = po.random_dense(n, m, p, seed)
    mu = (m + 63) // 64
    mine = list(range(rank, mu, world))
    W = a[mine].copy() if mine else np.zeros((0, a.shape[1]), np.uint64)  # local columns
    perm = np.arange(n, dtype=np.uint32)
    rj = np.zeros(mu, np.uint32)
    R = 0
    for j in range(mu):
        owner, lj = j % world, j // world
        hdr = torch.zeros(4 + 256, dtype=torch.int64)
        col = torch.zeros(n, dtype=torch.int64)
        if rank == owner:
            panel = W[lj, R:n].copy()
            r, A, P, Z, sb = po.build_z(panel) if n - R > 0 else (0, panel, None, np.zeros(64, np.uint64), [])
            pairs = composite_pairs(sb, r)
            # Y = D*Z over D
            D = A[r:]
            Y = np.zeros_like(D)
            for t in range(64):
                sel = ((D >> np.uint64(t)) & np.uint64(1)).astype(bool)
                Y[sel] ^= Z[t]
            A[r:] = Y
            W[lj, R:n] = A
            hdr[0], hdr[1], hdr[2] = R, r, len(pairs)
            for e, (d_, s_) in enumerate(pairs):
                hdr[4 + e], hdr[4 + 128 + e] = d_, s_
            col[:] = torch.from_numpy(W[lj, :n].view(np.int64).copy())
        dist.broadcast(hdr, src=owner)
        dist.broadcast(col, src=owner)
        R0, r, npairs = int(hdr[0]), int(hdr[1]), int(hdr[2])
        assert R0 == R
        pairs = [(int(hdr[4 + e]), int(hdr[4 + 128 + e])) for e in range(npairs)]
        colv = col.numpy().view(np.uint64)
        # mirror the permutation on every local column except the owner's panel
        for l in range(W.shape[0]):
            if rank == owner and l == lj:
                continue
            old = W[l, R:n].copy()
            for d_, s_ in pairs:
                W[l, R + d_] = old[s_]
        oldp = perm[R:n].copy()
        for d_, s_ in pairs:
            perm[R + d_] = oldp[s_]
        # Schur update of local columns right of j
        l0 = first_local_after(j, rank, world)
        Y = colv[R + r:n]
        for l in range(l0, W.shape[0]):
            for t in range(r):
                sel = ((Y >> np.uint64(t)) & np.uint64(1)).astype(bool)
                W[l, R + r:n][sel] ^= W[l, R + t]
        rj[j] = r
        R += r
    out_q.put((rank, mine, W, perm, rj))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n,m,p", [(300, 500, 0.5), (500, 300, 0.1), (257, 640, 0.5),
                                   (200, 200, 0.01)])
def test_sharded_protocol_matches_oracle(po, n, m, p):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, n, m, p, 11, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    w, perm, rj, rank = po.decompose_block(po.random_dense(n, m, p, 11), n, m)
    for r_, mine, W, prm, rjj in res:
        assert np.array_equal(prm, perm)
        assert np.array_equal(rjj, rj)
        for l, qcol in enumerate(mine):
            assert np.array_equal(W[l, :n], w[qcol, :n]), (r_, qcol)


def test_local_column_bookkeeping():
    """first_local_after + f2gpu_local_wcols agree with the round-robin ownership."""
    from paper_1209_5198_b200 import _lib

    lib = _lib.load()
    for G in (1, 2, 3, 8):
        for mu in (1, 5, 64):
            for g in range(G):
                owned = list(range(g, mu, G))
                assert lib.f2gpu_local_wcols(mu, g, G) == len(owned)
                for j in range(mu):
                    l0 = first_local_after(j, g, G)
                    assert [q for q in owned if q > j] == owned[l0:]


def mult_worker(rank, world, port, n, k, m, q):
    """Rank r owns word-columns q = r, r+G, ... of B and C; A comes from rank 0 by
    one broadcast (f2gpu_strassen_mult_dist's exchange), then C_local = A * B_local."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import pyoracle as po
    a = po.random_dense(n, k, 0.5, 21) if rank == 0 else np.zeros((po.wcols(k), po.stride_for(n)), np.uint64)
    t = torch.from_numpy(a.view(np.int64))
    dist.broadcast(t, src=0)
    a = t.numpy().view(np.uint64)
    b = po.random_dense(k, m, 0.5, 22)          # every rank can generate B; it keeps its columns only
    mine = list(range(rank, po.wcols(m), world))
    b_local = np.ascontiguousarray(b[mine])
    c_local = po.m4rm_mult(a, n, k, b_local, 64 * len(mine)) if mine else np.zeros((0, 1), np.uint64)
    q.put((rank, mine, c_local))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n,k,m", [(300, 200, 640), (130, 700, 130)])
def test_sharded_multiply_protocol(po, n, k, m):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=mult_worker, args=(r, world, port, n, k, m, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    want = po.m4rm_mult(po.random_dense(n, k, 0.5, 21), n, k, po.random_dense(k, m, 0.5, 22), m)
    seen = set()
    for _, mine, c_local in res:
        for l, qcol in enumerate(mine):
            # the last word-column's padding bits past m are zero in both
            assert np.array_equal(c_local[l, :n], want[qcol, :n]), qcol
            seen.add(qcol)
    assert seen == set(range(po.wcols(m)))
