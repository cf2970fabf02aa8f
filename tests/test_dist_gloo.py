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


# ---------------------------------------------------------------------------
# decompose_recursive over column shards: the library's OWN schedule
# (f2gpu_dist_schedule, the host code the GPU drivers run) executed on two
# gloo ranks with numpy/oracle callbacks for the device work.
# ---------------------------------------------------------------------------
def rec_worker(rank, world, port, n, m, kind, leaf, whole_leaf, out_q):
    import ctypes as C
    import traceback

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import pyoracle as po
    from paper_1209_5198_b200 import _lib

    lib = _lib.load()
    ol = po.lib()
    u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
    ol.f2o_m4rm_update.argtypes = [u64p, C.c_size_t, C.c_size_t, u64p, C.c_size_t, C.c_size_t, u64p,
                                   C.c_size_t, C.c_size_t, C.c_size_t, C.c_uint]
    a = make_input(po, n, m, kind)
    mu = (m + 63) // 64
    mine = list(range(rank, mu, world))
    S = a.shape[1]
    W = a[mine].copy() if mine else np.zeros((0, S), np.uint64)
    perm = np.arange(n, dtype=np.uint32)
    Rj = np.zeros(mu + 1, np.int64)          # R_j (replicated); R_{j+1} = R_j + r_j
    rj = np.zeros(mu, np.int64)
    pairs_of = {}
    land = np.zeros(S, np.uint64)
    Lg = {}

    def local_of(q):
        return q // world if q % world == rank else None

    def own_cols(lo, hi):
        return [(l, q) for l, q in enumerate(mine) if lo <= q < hi]

    def permute(col, R, pairs):
        old = col[R:n].copy()
        for d_, s_ in pairs:
            col[R + d_] = old[s_]

    def update(l, a_col, R, r):
        """W[l] rows [R+r, n) ^= a_col rows (low r bits) * W[l] rows [R, R+r)."""
        if r == 0 or R + r >= n:
            return
        aw = np.ascontiguousarray(a_col[R + r:n])
        colv = np.ascontiguousarray(W[l:l + 1])
        ol.f2o_m4rm_update(colv, S, R + r, aw, n - R - r, r, colv, S, R, 1, 8)
        W[l] = colv[0]

    def guard(fn):
        def inner(*args):
            try:
                fn(*args)
                return 0
            except Exception:
                traceback.print_exc()
                return 3
        return inner

    @guard
    def panel(_, j, owner, row_lo):
        R = int(Rj[j])
        hdr = torch.zeros(2 + 256, dtype=torch.int64)
        col = torch.zeros(n - row_lo, dtype=torch.int64)
        if rank == owner:
            lj = local_of(j)
            pnl = W[lj, R:n].copy()
            r, A, P, Z, sb = po.build_z(pnl) if n - R > 0 else (0, pnl, None, np.zeros(64, np.uint64), [])
            pairs = composite_pairs(sb, r)
            D = A[r:]
            Y = np.zeros_like(D)
            for t in range(64):
                sel = ((D >> np.uint64(t)) & np.uint64(1)).astype(bool)
                Y[sel] ^= Z[t]
            A[r:] = Y
            W[lj, R:n] = A
            for l in range(W.shape[0]):      # the post: swaps on the owner's other columns
                if l != lj:
                    permute(W[l], R, pairs)
            permute(perm, R, pairs)
            hdr[0], hdr[1] = r, len(pairs)
            for e, (d_, s_) in enumerate(pairs):
                hdr[2 + e], hdr[2 + 128 + e] = d_, s_
            col[:] = torch.from_numpy(W[lj, row_lo:n].view(np.int64).copy())
        dist.broadcast(hdr, src=owner)
        dist.broadcast(col, src=owner)
        r, npairs = int(hdr[0]), int(hdr[1])
        rj[j] = r
        Rj[j + 1] = R + r
        pairs_of[j] = [(int(hdr[2 + e]), int(hdr[2 + 128 + e])) for e in range(npairs)]
        land[:] = 0
        land[row_lo:n] = col.numpy().view(np.uint64)

    @guard
    def apply(_, j, owner, lo, hi):
        R, r = int(Rj[j]), int(rj[j])
        if rank != owner:
            for l in range(W.shape[0]):
                permute(W[l], R, pairs_of[j])
            permute(perm, R, pairs_of[j])
        a_col = W[local_of(j)].copy() if rank == owner else land.copy()
        for l, _q in own_cols(lo, hi):
            update(l, a_col, R, r)

    @guard
    def state(_, j, Rp, rp):
        Rp[0], rp[0] = int(Rj[j]), int(rj[j])

    @guard
    def gather(_, c0, cm, row_lo):
        Lg.clear()
        for q in range(c0, cm):
            t = torch.zeros(n - row_lo, dtype=torch.int64)
            if q % world == rank:
                t[:] = torch.from_numpy(W[local_of(q), row_lo:n].view(np.int64).copy())
            dist.broadcast(t, src=q % world)
            full = np.zeros(S, np.uint64)
            full[row_lo:n] = t.numpy().view(np.uint64)
            Lg[q] = full

    @guard
    def solve(_, c0, cm, R0, lo, hi):
        R1 = R0 + 64 * (cm - c0)
        for l, _q in own_cols(lo, hi):
            for t in range(c0, cm):        # forward substitution inside the pivot block
                Rt = R0 + 64 * (t - c0)
                rows = np.ascontiguousarray(Lg[t][Rt + 64:R1])
                if rows.size:
                    colv = np.ascontiguousarray(W[l:l + 1])
                    ol.f2o_m4rm_update(colv, S, Rt + 64, rows, R1 - Rt - 64, 64, colv, S, Rt, 1, 8)
                    W[l] = colv[0]

    @guard
    def product(_, c0, cm, R0, R1, lo, hi):
        for l, _q in own_cols(lo, hi):
            for t in range(c0, cm):        # A' = D ^ L21 X, one 64-column block of L21 at a time
                Rt = R0 + 64 * (t - c0)
                rows = np.ascontiguousarray(Lg[t][R1:n])
                colv = np.ascontiguousarray(W[l:l + 1])
                ol.f2o_m4rm_update(colv, S, R1, rows, n - R1, 64, colv, S, Rt, 1, 8)
                W[l] = colv[0]

    @guard
    def rank_update(_, c0, cm, lo, hi):
        for j in range(c0, cm):
            for l, _q in own_cols(lo, hi):
                update(l, Lg[j], int(Rj[j]), int(rj[j]))

    @guard
    def leaf_op(_, c0, c1, row_lo):
        """Whole-leaf mode: replicate the leaf's columns once, factor the leaf on every
        rank's copy (no further exchange), keep the own columns, swap the others."""
        L = {}
        for q in range(c0, c1):
            t = torch.zeros(n - row_lo, dtype=torch.int64)
            if q % world == rank:
                t[:] = torch.from_numpy(W[local_of(q), row_lo:n].view(np.int64).copy())
            dist.broadcast(t, src=q % world)
            full = np.zeros(S, np.uint64)
            full[row_lo:n] = t.numpy().view(np.uint64)
            L[q] = full
        for j in range(c0, c1):
            R = int(Rj[j])
            pnl = L[j][R:n].copy()
            r, A, P, Z, sb = po.build_z(pnl) if n - R > 0 else (0, pnl, None, np.zeros(64, np.uint64), [])
            pairs = composite_pairs(sb, r)
            D = A[r:]
            Y = np.zeros_like(D)
            for t in range(64):
                sel = ((D >> np.uint64(t)) & np.uint64(1)).astype(bool)
                Y[sel] ^= Z[t]
            A[r:] = Y
            L[j][R:n] = A
            for q in range(c0, c1):
                if q != j:
                    permute(L[q], R, pairs)
            permute(perm, R, pairs)
            rj[j] = r
            Rj[j + 1] = R + r
            pairs_of[j] = pairs
            if r and R + r < n:
                aw = np.ascontiguousarray(L[j][R + r:n])
                for q in range(j + 1, c1):
                    colv = np.ascontiguousarray(L[q][None, :])
                    ol.f2o_m4rm_update(colv, S, R + r, aw, n - R - r, r, colv, S, R, 1, 8)
                    L[q] = colv[0]
        for l, q in enumerate(mine):
            if c0 <= q < c1:
                W[l, row_lo:n] = L[q][row_lo:n]
            else:
                for j in range(c0, c1):
                    permute(W[l], int(Rj[j]), pairs_of[j])
        Lg.clear()
        Lg.update(L)  # a split whose left half is this leaf reuses the copy (DistGpu::gather)

    ops = _lib.DistOps(None, _lib.PANEL_FN(panel), _lib.APPLY_FN(apply), _lib.STATE_FN(state),
                       _lib.GATHER_FN(gather), _lib.SOLVE_FN(solve), _lib.PRODUCT_FN(product),
                       _lib.RANKUPD_FN(rank_update))
    if whole_leaf:
        ops.leaf = _lib.LEAF_FN(leaf_op)
    rc = lib.f2gpu_dist_schedule(n, mu, world, leaf, 0, leaf, C.byref(ops))
    out_q.put((rank, rc, mine, W, perm, rj.astype(np.uint32)))
    dist.barrier()
    dist.destroy_process_group()


def make_input(po, n, m, kind):
    if kind == "xy":  # rank-deficient: the splits take the rank-r_j path
        k = 70
        return po.m4rm_mult(po.random_dense(n, k, 0.5, 31), n, k, po.random_dense(k, m, 0.5, 32), m)
    return po.random_dense(n, m, 0.5 if kind == "dense" else 0.05, 33)


@pytest.mark.parametrize("whole_leaf", [False, True], ids=["per_panel", "whole_leaf"])
@pytest.mark.parametrize("n,m,kind,leaf", [(700, 640, "dense", 2), (400, 1000, "dense", 1), (900, 512, "xy", 2),
                                           (300, 577, "sparse", 3)])
def test_recursive_schedule_matches_oracle(po, n, m, kind, leaf, whole_leaf):
    """The distributed recursion (leaves, splits with gather + solve + product, and
    the rank-deficient fallback) driven by libf2gpu's f2gpu_dist_schedule on two
    gloo ranks gives the single-process oracle's W, perm and r_j bit-for-bit, with
    per-panel replication and with whole leaves factored on a replicated copy (the
    GPU drivers' default, f2gpu_dist_ops.leaf)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=rec_worker, args=(r, world, port, n, m, kind, leaf, whole_leaf, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    w, perm, rj, rank = po.decompose_block(make_input(po, n, m, kind), n, m)
    for r_, rc, mine, W, prm, rjj in res:
        assert rc == 0
        assert np.array_equal(prm, perm), r_
        assert np.array_equal(rjj, rj), r_
        for l, qcol in enumerate(mine):
            assert np.array_equal(W[l, :n], w[qcol, :n]), (r_, qcol)
