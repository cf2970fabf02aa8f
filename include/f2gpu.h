/*
 * f2gpu.h — C-ABI of the B200-native GF(2) block decomposition library
 * (libf2gpu.so, built from paper_1209_5198_b200/csrc/).
 *
 * This is the drop-in boundary for the reference's free-function API on
 * f2la::BitMatrix (= PackedMatrix<uint64_t>, /root/reference/proj/include/f2la/
 * bit_matrix.hpp:348).  The reference has no FFI of its own: it is a header-only
 * C++20 library.  Each entry point below names the reference interface it
 * replaces (file:line); include/f2la_gpu.hpp is the C++ forwarding shim with
 * the reference's own signatures, and INTEGRATION.md shows the bindings.
 *
 * Layout contract (bit_matrix.hpp:74-81): a matrix is n_rows x n_cols bits, as
 * mu = ceil(n_cols/64) word-columns; word (i, q) is at base[q*col_stride + i];
 * bit k of word (i,q) is entry (i, 64q+k) (LSB = leftmost column); padding bits
 * are zero.  Host buffers carry their own col_stride (the reference uses
 * ceil(n/8)*8, bit_matrix.hpp:330-333); device matrices use a stride of rows
 * rounded up to 128 words (1 KiB column segments for the bulk-copy kernels;
 * f2gpu_mat_shape reports it).
 *
 * Errors: every function returns an int status.  The codes mirror the
 * reference's exceptions: F2GPU_EINVAL <-> std::invalid_argument (shape
 * mismatch, m4rm.hpp:181), F2GPU_ERANGE <-> std::out_of_range (m4rm.hpp:100,145).
 * f2gpu_last_error() returns a thread-local message for the last failure.
 *
 * Threading: a context owns one CUDA device + stream; it is not shared between
 * host threads (the reference contract is single-threaded per call).
 * Distinct contexts may be used concurrently.
 *
 * Device use: the decompositions' lookahead schedule runs kernels on two
 * streams (the posts and updates of a leaf, and its one persistent panel-chain
 * CTA) that wait on each other through device counters, so they must be
 * co-resident: run them with the GPU to themselves (no concurrent kernels from
 * other streams or MPS clients).  Every such wait is bounded (20 s); a wait that
 * expires traps and the call returns F2GPU_ECUDA instead of hanging.  The chain
 * launch is never captured: inside a caller's own stream capture the library
 * uses one panel kernel per panel instead.
 */
#ifndef F2GPU_H
#define F2GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define F2GPU_OK 0
#define F2GPU_EINVAL 1 /* std::invalid_argument */
#define F2GPU_ERANGE 2 /* std::out_of_range */
#define F2GPU_ECUDA 3  /* CUDA runtime failure */
#define F2GPU_ENCCL 4  /* NCCL failure / NCCL not loadable */
#define F2GPU_ENOMEM 5 /* device allocation failed */

typedef struct f2gpu_ctx f2gpu_ctx; /* device, stream, workspaces, NCCL comm */
typedef struct f2gpu_mat f2gpu_mat; /* device-resident packed matrix (owning) */

const char *f2gpu_last_error(void);
const char *f2gpu_version(void);

/* Every switch of the library (environment variables, read once; all of them select
 * among bit-identical paths, tune a size, or turn on a diagnostic) as a text table:
 * one line per switch, "NAME value[*] (default D) meaning", * = set in the
 * environment.  Writes at most cap-1 bytes + NUL into buf (buf may be NULL);
 * *len (if non-NULL) = the full length. */
int f2gpu_options_describe(char *buf, size_t cap, size_t *len);

/* ---- context -------------------------------------------------------------- */
int f2gpu_ctx_create(int device, f2gpu_ctx **out);
int f2gpu_ctx_destroy(f2gpu_ctx *ctx);
/* Run subsequent work on an external CUDA stream (e.g. torch's current stream);
 * F2GPU_OWN_STREAM returns to the context's own stream.  Handle 0 is the legacy
 * default stream (torch's default stream), not "own": work is ordered with it,
 * and CUDA-graph replay is off while it (or cudaStreamPerThread) is selected,
 * because stream capture is illegal there. */
#define F2GPU_OWN_STREAM ((void *)(~(uintptr_t)0))
int f2gpu_ctx_set_stream(f2gpu_ctx *ctx, void *cuda_stream);
int f2gpu_ctx_sync(f2gpu_ctx *ctx);
/* Kernel launches issued through this context since creation (evidence for
 * bench.py's gpu_launches). */
uint64_t f2gpu_ctx_launches(const f2gpu_ctx *ctx);
/* Tuning knobs: table-group layout is fixed (9 tables, 7x8+8 bits); the
 * Strassen cutover (minimum dimension in bits below which the M4RM leaf runs;
 * 0 = default) replaces tuning::strassen_threshold (tuning.hpp:30). */
int f2gpu_ctx_set_strassen_cutover(f2gpu_ctx *ctx, size_t min_dim_bits);
/* Product leaf: on != 0 (default) lets strassen_mult and the recursive
 * decomposition use the fp4 tensor-core leaf where the shape allows (n, k, m
 * >= 256); tc_min_leaf_bits = minimum Strassen leaf size over that leaf
 * (0 = default 16384).  Results are bit-identical either way. */
int f2gpu_ctx_set_tc(f2gpu_ctx *ctx, int on, size_t tc_min_leaf_bits);

/* Device trace (diagnostics, no reference counterpart): with cap > 0 the panel,
 * fused-post and update kernels append globaltimer stamps
 * (ns << 16) | (event << 12) | panel_index to a device buffer of cap entries;
 * trace_read synchronizes, copies up to cap entries out and restarts the trace.
 * cap = 0 turns it off.  One trace per process (a device symbol). */
int f2gpu_trace_enable(f2gpu_ctx *ctx, size_t cap);
int f2gpu_trace_read(f2gpu_ctx *ctx, uint64_t *out, size_t cap, size_t *n);

/* Profiling hook (diagnostics, no reference counterpart): k_panel_chain ALONE on
 * the word-columns [1, ncols) of a device matrix, every counter it would wait on
 * pre-satisfied, so the chain free-runs (no posts, no updates: each panel is
 * factored on the column as it stands, and the matrix is NOT a decomposition
 * afterwards).  In the pipeline the chain spins on kernels launched after it and
 * cannot run under ncu, which serialises kernels; this entry can.  It also gives
 * the chain's intrinsic per-panel cycle (selection + in-CTA hand-off). */
int f2gpu_debug_panel_chain(f2gpu_ctx *ctx, f2gpu_mat *a, size_t ncols);

/* One panel kernel (Procedure buildZ) on a host column of
 * n words: col_out receives the column with the panel's row swaps applied,
 * z_out the 64 words of the pseudo-inverse Z and r_out the block rank;
 * pairs_out (optional, 256 words: dst[128] then src[128]) and npairs_out the
 * composite row permutation new[dst[e]] = old[src[e]] that the other word-
 * columns receive.  Z is only defined on the span of the selected rows, which
 * holds every row below the pivots: parity is on r, col_out, the pairs and
 * Y_i = col_out[i] * Z for i >= r.  (Kernel-level check of the path's first
 * step; replaces no reference call.) */
int f2gpu_panel_build_z(f2gpu_ctx *ctx, const uint64_t *col, size_t n, uint64_t *col_out, uint64_t *z_out,
                        uint32_t *r_out, uint32_t *pairs_out, uint32_t *npairs_out);

/* ---- device matrix store (replaces PackedMatrix<uint64_t> storage,
 *      bit_matrix.hpp:82-346) ------------------------------------------------- */
int f2gpu_mat_alloc(f2gpu_ctx *ctx, size_t n_rows, size_t n_cols, f2gpu_mat **out);
/* a matrix must be freed before the context it was allocated on is destroyed */
int f2gpu_mat_free(f2gpu_mat *m);
int f2gpu_mat_shape(const f2gpu_mat *m, size_t *n_rows, size_t *n_cols, size_t *col_stride);
/* raw device pointer to word (0,0) (for interop, e.g. torch.from_blob) */
int f2gpu_mat_device_ptr(const f2gpu_mat *m, uint64_t **dptr);
int f2gpu_mat_zero(f2gpu_ctx *ctx, f2gpu_mat *m);
/* host <-> device; host_stride in words (>= n_rows) */
int f2gpu_mat_upload(f2gpu_ctx *ctx, f2gpu_mat *m, const uint64_t *host, size_t host_stride);
int f2gpu_mat_download(f2gpu_ctx *ctx, const f2gpu_mat *m, uint64_t *host, size_t host_stride);
/* Bit-exact device twin of PackedMatrix::random_dense (bit_matrix.hpp:125-142,
 * Rng prng.hpp:18-47): entry (i,j) uses xorshift64* draw #(i*m+j). */
int f2gpu_mat_random_dense(f2gpu_ctx *ctx, f2gpu_mat *m, double density, uint64_t seed);
/* dst = src (same shape) */
int f2gpu_mat_copy(f2gpu_ctx *ctx, f2gpu_mat *dst, const f2gpu_mat *src);
/* dst word-column l = src word-column first + l*step (round-robin column
 * sharding; scatter=0) or the reverse (scatter=1: src col l -> dst col first+l*step) */
int f2gpu_mat_select_wcols(f2gpu_ctx *ctx, f2gpu_mat *dst, const f2gpu_mat *src, size_t first,
                           size_t step, int scatter);
/* entrywise dst ^= src (xor_with, bit_matrix.hpp:241-250) */
int f2gpu_mat_xor(f2gpu_ctx *ctx, f2gpu_mat *dst, const f2gpu_mat *src);
/* out = transpose(a) (transposed, bit_matrix.hpp:220-238); out must be m x n */
int f2gpu_mat_transpose(f2gpu_ctx *ctx, const f2gpu_mat *a, f2gpu_mat *out);

/* ---- M4RM products (m4rm.hpp:93-196) -------------------------------------- */
/* C = A*B (m4rm_mult, m4rm.hpp:177-196). C must be a.rows x b.cols.
 * `c` is the reference's table-size argument; the device kernel uses a fixed
 * 9-table split (7x8+8 bits) sized for shared memory, so any c is accepted and
 * results are identical (SPEC.md: "Result independent of the chosen splits"). */
int f2gpu_m4rm_mult(f2gpu_ctx *ctx, const f2gpu_mat *a, const f2gpu_mat *b, f2gpu_mat *c,
                    unsigned table_size);
/* C ^= A*B */
int f2gpu_m4rm_mult_acc(f2gpu_ctx *ctx, const f2gpu_mat *a, const f2gpu_mat *b, f2gpu_mat *c);
/* C rows [c_row0, c_row0+n_rows) x word-cols [c_wcol0, c_wcol0+n_wcols)
 *   ^= a_words * B[b_row0 .. b_row0+k_bits) x word-cols [b_wcol0, +n_wcols)
 * with a_words a DEVICE array of n_rows words (bits >= k_bits must be zero).
 * This is mult_acc over build_tables(B, row0, k, wcol0, n) (m4rm.hpp:93-113,
 * 140-172) as one fused kernel (table build in shared memory + XOR sweep). */
int f2gpu_mult_acc(f2gpu_ctx *ctx, f2gpu_mat *c, size_t c_row0, size_t c_wcol0,
                   size_t n_wcols, const uint64_t *d_a_words, size_t n_rows, size_t k_bits,
                   const f2gpu_mat *b, size_t b_row0, size_t b_wcol0);
/* The same on HOST matrices in the reference layout (what f2la::gpu::mult_acc
 * over f2la::gpu::build_tables calls): C (c_rows x c_cols, c_stride) rows
 * [c_row0, c_row0+n_rows) x word-cols [c_wcol0, c_wcol0+n_wcols) ^= a_words[i] *
 * B[b_row0, b_row0+k_bits) x word-cols [b_wcol0, b_wcol0+n_wcols), B being
 * b_rows x b_cols with b_stride.  Replaces build_tables(B, row0, k, wcol0, n,
 * splits) (m4rm.hpp:93-113) + mult_acc(C, c_row0, c_wcol0, a_words, tables)
 * (m4rm.hpp:140-172); the result does not depend on the splits, bits
 * of a_words at or above k_bits are ignored.  Errors: k_bits > 64 ->
 * F2GPU_EINVAL (m4rm.hpp:97-98); block outside B / destination outside C ->
 * F2GPU_ERANGE (m4rm.hpp:99-100, 144-145).  C is updated when the call returns. */
int f2gpu_mult_acc_host(f2gpu_ctx *ctx, uint64_t *c, size_t c_rows, size_t c_cols, size_t c_stride,
                        size_t c_row0, size_t c_wcol0, const uint64_t *a_words, size_t n_rows,
                        const uint64_t *b, size_t b_rows, size_t b_cols, size_t b_stride, size_t b_row0,
                        size_t k_bits, size_t b_wcol0, size_t n_wcols);
/* The evaluated alternative leaf (north_star): C = A*B (acc=0) or C ^= A*B on the
 * tensor cores.  Default: tcgen05.mma kind::mxf4 (bits as E2M1 1.0/0.0, unit
 * E8M0 scales, exact f32 sums, parity), any n and k, m % 256 == 0.  With
 * F2GPU_TC_KIND=i8 (or m % 256 != 0): kind::i8 on 0/1 bytes, n % 256 == 0,
 * m % 128 == 0, k % 64 == 0. */
int f2gpu_gemm_tc(f2gpu_ctx *ctx, const f2gpu_mat *a, const f2gpu_mat *b, f2gpu_mat *c, int acc);
/* Tensor-core trailing update (the blocked decomposition's GEMM step):
 *   C[row_lo, row_hi) x word-cols [c_wcol0, c_wcol0 + n_wcols)
 *     ^= A[same rows] x word-cols [a_wcol0, a_wcol0 + kwords)  *  BT^T
 * with BT an (n_wcols*64) x (kwords*64) matrix holding B transposed, kwords <= 2
 * (rank <= 128).  Rows of A outside [row_lo, row_hi) do not contribute. */
int f2gpu_update_tc(f2gpu_ctx *ctx, f2gpu_mat *c, size_t row_lo, size_t row_hi, size_t c_wcol0,
                    size_t n_wcols, const f2gpu_mat *a, size_t a_wcol0, size_t kwords,
                    const f2gpu_mat *bt);
/* Strassen-Winograd over device sub-blocks, M4RM leaves
 * below the cutover. threshold = 0 -> context cutover. C = A*B. */
int f2gpu_strassen_mult(f2gpu_ctx *ctx, const f2gpu_mat *a, const f2gpu_mat *b, f2gpu_mat *c,
                        size_t threshold);

/* ---- decomposition ------------------- */
/* decompose_block in place: on return `w` holds the overlay W (L below/left of
 * the block staircase, U on the pivot rows), perm[n_rows]
 * ((PA)_i = A_{perm[i]}, bit_matrix.hpp:350) and rj[mu] (block ranks) are
 * written to HOST arrays (either may be NULL), *rank = sum rj. */
int f2gpu_decompose_block(f2gpu_ctx *ctx, f2gpu_mat *w, uint32_t *perm, uint32_t *rj,
                          size_t *rank);
/* decompose_recursive: split the columns,
 * factor the left half, update the right half with a block TRSM + one
 * Strassen-Winograd GEMM (A' = D ^ L21 L11^-1 C), recurse.  Exact arithmetic and
 * 64-aligned splits make the result bit-identical to decompose_block.
 * min_cols = 0 -> leaves of at most 256 panels (16384 columns), 64 panels once
 * a leaf has >= 30000 rows below its first panel (csrc/options.h). */
int f2gpu_decompose_recursive(f2gpu_ctx *ctx, f2gpu_mat *w, size_t min_cols, uint32_t *perm,
                              uint32_t *rj, size_t *rank);
/* Same algorithm, column blocks distributed round-robin over `shards` logical
 * shards that live on this device (testing the sharded driver on one GPU). */
int f2gpu_decompose_block_sharded(f2gpu_ctx *ctx, f2gpu_mat *w, int shards, uint32_t *perm,
                                  uint32_t *rj, size_t *rank);
/* rank(A): transposes when n_rows < n_cols; a is not modified */
int f2gpu_rank(f2gpu_ctx *ctx, const f2gpu_mat *a, size_t *rank);

/* ---- host-buffer entry points (what the reference-side shim calls) ---------- */
int f2gpu_m4rm_mult_host(f2gpu_ctx *ctx, const uint64_t *a, size_t n, size_t k, size_t sa,
                         const uint64_t *b, size_t m, size_t sb, uint64_t *c, size_t sc,
                         unsigned table_size);
int f2gpu_strassen_mult_host(f2gpu_ctx *ctx, const uint64_t *a, size_t n, size_t k, size_t sa,
                             const uint64_t *b, size_t m, size_t sb, uint64_t *c, size_t sc,
                             size_t threshold);
/* decompose a host matrix: w_out receives the overlay (same stride as input) */
int f2gpu_decompose_block_host(f2gpu_ctx *ctx, const uint64_t *a, size_t n, size_t m,
                               size_t stride, uint64_t *w_out, uint32_t *perm, uint32_t *rj,
                               size_t *rank);
/* the same through decompose_recursive (min_cols = 0: default leaf width) */
int f2gpu_decompose_recursive_host(f2gpu_ctx *ctx, const uint64_t *a, size_t n, size_t m,
                                   size_t stride, size_t min_cols, uint64_t *w_out, uint32_t *perm,
                                   uint32_t *rj, size_t *rank);
int f2gpu_rank_host(f2gpu_ctx *ctx, const uint64_t *a, size_t n, size_t m, size_t stride,
                    size_t *rank);

/* ---- null space and linear systems ------
 * Partial block decomposition of [A^T | I]: the A^T panels are eliminated exactly
 * as decompose_block does, the identity part records the row operations.
 * null_space: *basis = new m x (m - rank) matrix, A * N = 0, columns independent
 *             (free with f2gpu_mat_free); *nullity = m - rank.
 * solve:      rhs = ceil(n/64) host words (bit i = b_i); on *solvable = 1, x =
 *             ceil(m/64) host words with A x = b; *solvable = 0 signals an
 *             inconsistent system (not an error). */
int f2gpu_null_space(f2gpu_ctx *ctx, const f2gpu_mat *a, f2gpu_mat **basis, size_t *nullity);
int f2gpu_solve(f2gpu_ctx *ctx, const f2gpu_mat *a, const uint64_t *rhs, uint64_t *x, int *solvable);

/* ---- multi-GPU (one process per GPU, NCCL over NVLink) ---------------------- */
/* 128-byte ncclUniqueId, produced on rank 0 and shared by the caller (e.g. via
 * torch.distributed); NCCL is loaded at run time (dlopen libnccl.so.2). */
int f2gpu_nccl_unique_id(void *out128);
int f2gpu_ctx_init_comm(f2gpu_ctx *ctx, int rank, int world, const void *id128);
/* Distributed decomposition: this rank holds word-columns q = rank, rank+world,
 * ... of the global n x m matrix as a LOCAL matrix `w_local` (n rows, its local
 * word-columns packed densely).  Per panel the owner factors and broadcasts
 * {r_j, transpositions, Y}; every rank updates its own trailing columns.
 * perm/rj are replicated on every rank. */
int f2gpu_decompose_block_dist(f2gpu_ctx *ctx, f2gpu_mat *w_local, size_t n_cols_global,
                               uint32_t *perm, uint32_t *rj, size_t *rank);
/* number of local word-columns rank `rank` owns out of mu */
size_t f2gpu_local_wcols(size_t mu, int rank, int world);
/* decompose_recursive over word-column shards: the same
 * factors as f2gpu_decompose_recursive.  Per leaf panel the owner factors and
 * replicates {state, column rows [R_lb, n)} (R_lb = the leaf's first R); per
 * split the left columns (rows [R0, n)) are replicated once and every rank
 * solves X = L11^-1 C and forms A' = D ^ L21 X on its OWN right-half columns.
 * _dist: one rank per GPU over NCCL (w_local as for f2gpu_decompose_block_dist;
 * world 1 without a communicator = f2gpu_decompose_recursive).  _sharded: the
 * same schedule over `shards` logical shards on this device (testing). */
int f2gpu_decompose_recursive_dist(f2gpu_ctx *ctx, f2gpu_mat *w_local, size_t n_cols_global, size_t min_cols,
                                   uint32_t *perm, uint32_t *rj, size_t *rank);
int f2gpu_decompose_recursive_sharded(f2gpu_ctx *ctx, f2gpu_mat *w, int shards, size_t min_cols, uint32_t *perm,
                                      uint32_t *rj, size_t *rank);
/* The recursion's schedule alone (host code, no device work): calls `ops` in the
 * order the distributed drivers execute them, for rank-agnostic callbacks
 * (each callback acts for the calling rank).  Used by the CPU protocol test
 * (tests/test_dist_gloo.py) to run the library's own plan over gloo.
 *   panel(j, owner, row_lo):  owner factors panel j; state j and the panel
 *                             column rows [row_lo, n) become replicated
 *   apply(j, owner, lo, hi):  non-owners apply panel j's row swaps to all their
 *                             columns; every rank updates its columns in [lo, hi)
 *   state(j, *R, *r):         replicated R_j, r_j
 *   gather(c0, cm, row_lo):   replicate columns [c0, cm), rows [row_lo, n)
 *   solve(c0, cm, R0, lo, hi): X = L11^-1 C on own columns in [lo, hi)
 *   product(c0, cm, R0, R1, lo, hi): rows [R1, n) of own columns ^= L21 X
 *   rank_update(c0, cm, lo, hi): panels [c0, cm) as rank-r_j updates (not full rank)
 *   leaf(c0, c1, row_lo):     OPTIONAL (may be NULL).  When set it replaces the
 *                             per-panel panel/apply calls of a leaf: columns
 *                             [c0, c1), rows [row_lo, n), are replicated once, every
 *                             rank factors the leaf on its copy (deterministic, so
 *                             states and perm agree without a further exchange),
 *                             keeps its own columns and applies the leaf's row swaps
 *                             to its other columns.  The GPU drivers use it unless
 *                             F2GPU_DIST_LEAF=0.
 * A non-zero callback return aborts the schedule with that code. */
typedef struct f2gpu_dist_ops {
    void *user;
    int (*panel)(void *user, size_t j, int owner, size_t row_lo);
    int (*apply)(void *user, size_t j, int owner, size_t col_lo, size_t col_hi);
    int (*state)(void *user, size_t j, size_t *R, size_t *r);
    int (*gather)(void *user, size_t c0, size_t cm, size_t row_lo);
    int (*solve)(void *user, size_t c0, size_t cm, size_t R0, size_t col_lo, size_t col_hi);
    int (*product)(void *user, size_t c0, size_t cm, size_t R0, size_t R1, size_t col_lo, size_t col_hi);
    int (*rank_update)(void *user, size_t c0, size_t cm, size_t col_lo, size_t col_hi);
    int (*leaf)(void *user, size_t c0, size_t c1, size_t row_lo);
} f2gpu_dist_ops;
int f2gpu_dist_schedule(size_t n_rows, size_t mu, int world, size_t leaf_panels, size_t tall_rows,
                        size_t tall_leaf_panels, const f2gpu_dist_ops *ops);
/* NCCL broadcast of a whole device matrix from `root` (no-op at world 1). */
int f2gpu_mat_broadcast(f2gpu_ctx *ctx, f2gpu_mat *m, int root);
/* Multiply sharded by column blocks (BASELINE configs[1] on G GPUs):
 * rank r holds word-columns q = r, r+G, ... of B and C (f2gpu_mat_select_wcols);
 * A is broadcast from rank 0 into every rank's `a`, then c_local = a * b_local
 * (strassen_mult semantics; threshold 0 = default).  No per-step exchange. */
int f2gpu_strassen_mult_dist(f2gpu_ctx *ctx, f2gpu_mat *a, const f2gpu_mat *b_local, f2gpu_mat *c_local,
                             size_t threshold);

#ifdef __cplusplus
}
#endif
#endif
