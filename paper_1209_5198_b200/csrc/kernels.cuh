// kernels.cuh — sm_100a kernels of the GF(2) block decomposition hot path.
//
// Layout (reference bit_matrix.hpp:74-81): word (i,q) at p[q*stride + i],
// bit k = entry (i, 64q+k).  Device strides are multiples of 128 words (api.cu dev_stride), so every
// 16-row unit is 128-byte aligned (LDG/STG.256 friendly).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace f2 {

// ---- M4RM table geometry (shared by the update and GEMM kernels) ----------
// A 64-bit driving word is split into 9 groups: 8 x 7 bits + 1 x 8 bits
// (make_splits analogue, m4rm.hpp:39-48, with mixed sizes — SPEC.md allows
// any l_1..l_K summing to b).  Entries per column: 8*128 + 256 = 1280.
// A CTA owns 16 word-columns: 1280 * 16 * 8 B = 160 KiB of shared memory, and
// a half-warp reading 16 consecutive columns of one entry is one 128-byte
// wavefront (bank-conflict free regardless of the data-dependent index).
constexpr int kTabCols = 16;
constexpr int kNumTab = 9;
constexpr int kTabEntries = 1280;
constexpr size_t kTabBytes = size_t(kTabEntries) * kTabCols * 8;  // 163840

// Per-panel record, written by the panel kernel on the owner and broadcast to
// every shard.  All row indices are relative to R.
struct PanelState {
    uint32_t R;       // rows eliminated before this panel (sum of earlier r_j)
    uint32_t r;       // block rank r_j
    uint32_t npairs;  // entries of the composite row permutation below
    uint32_t flags;
    uint64_t Z[64];   // compressed pseudo-inverse rows (bit t < r)
    uint32_t dst[128];  // new[dst[e]] = old[src[e]]  (rows R + .)
    uint32_t src[128];
};
static_assert(sizeof(PanelState) == 16 + 512 + 1024, "PanelState layout");

struct UpdateArgs {
    uint64_t* C; size_t sc; size_t c_wcol0; int ncols;   // destination word-columns
    size_t row_lo, row_hi;                               // C rows to update
    const uint64_t* a;                                   // a[i] = driving word of C row i
    int k_bits;
    const uint64_t* B; size_t sb; size_t b_row0; size_t b_wcol0;
    const PanelState* st;  // non-null: R,r from state -> row_lo=R+r, k=r, b_row0=R
    // Early release (lookahead): when non-null, column group 0 (the next panel's
    // column) is split over ALL CTAs and done first; each CTA then increments
    // *release once its group-0 updates are complete in memory (exactly once per
    // CTA, also when it has no work).  The next panel kernel waits for the count.
    uint32_t* release;
    // with release: the first column (the one the next panel kernel waits for)
    // alone first, split by rows over every CTA with a 4-bit table, then the
    // release, then the remaining columns in 16-column groups
    bool first_col = false;
    // first_col: only the last fc_ctas CTAs do the first column (the others signal
    // the release at once and start their tiles); their share of the bulk tiles is
    // fc_weight / 4 of a full one.  0: every CTA does a slice of it
    int fc_ctas = 0;
    int fc_weight = 3;
    int tag = -1;  // panel index for the device trace; >= 0 only while it is on
    // launched as a programmatic dependent of the preceding kernel (k_post_col):
    // the CTAs start as its blocks retire and wait (griddepcontrol.wait) before
    // reading any data
    bool pdl = false;
};

// Device trace (diagnostics): when enabled, the panel / fused-post / update
// kernels append globaltimer stamps  (ns << 16) | (event << 12) | panel.
enum TraceEvent : uint32_t {
    kTrPanelBegin = 1, kTrPanelChainEnd = 2, kTrPanelEnd = 3,
    kTrPostBegin = 4, kTrPostHead = 5, kTrPostEnd = 6,
    kTrUpdBegin = 7, kTrUpdRelease = 8, kTrUpdEnd = 9,
};
cudaError_t trace_set(unsigned long long* buf, uint32_t cap);  // buf = nullptr: off
cudaError_t spin_diag_set(unsigned long long* mapped);            // device view of host-mapped memory
cudaError_t trace_count(uint32_t* n);

struct GemmArgs {
    const uint64_t* A; size_t sa; size_t n;   // A: n rows, k bits
    const uint64_t* B; size_t sb; size_t k;   // B: k rows
    uint64_t* C; size_t sc; int mcols;        // C: n rows, mcols word-columns (XOR-accumulated)
    // addressable rows from A / B base within a column (>= n / k); bulk loads of
    // 1024-row A segments and 64-row B blocks are clamped to these
    size_t a_cap = 0, b_cap = 0;
};

struct XorJob {  // dst = (acc ? dst : 0) ^ src[0..3] over rows x wcols (rows % 4 == 0, 32-B aligned)
    uint64_t* dst; size_t sd;
    const uint64_t* src[4]; size_t ss[4];
    size_t rows, wcols;
    int acc;
};

// launchers (return cudaError_t of the launch)
cudaError_t launch_random_dense(uint64_t* w, size_t n, size_t m, size_t stride, double density,
                                uint64_t seed, const uint64_t* d_jump, cudaStream_t s);
cudaError_t launch_update(const UpdateArgs& a, int num_sms, cudaStream_t s);
cudaError_t launch_gemm(const GemmArgs& g, int num_sms, cudaStream_t s);
cudaError_t launch_panel(uint64_t* col, size_t n, PanelState* st_all, int j, cudaStream_t s,
                         const uint32_t* wait_flag = nullptr, uint32_t wait_count = 0);
// can launch_update take the bulk-reduction path (required for early release)?
bool update_fast_ok(const UpdateArgs& a);
cudaError_t launch_panel_y(uint64_t* col, size_t n, const PanelState* st, int num_sms,
                           cudaStream_t s);
cudaError_t launch_swaps(uint64_t* w, size_t stride, int ncols, int skip_col, uint32_t* perm,
                         const PanelState* st, cudaStream_t s);
// the row swaps of panels [j0, j1) in order, on word-columns outside [skip_lo, skip_hi)
// and on perm (may be null); st = the state array (distributed leaves)
cudaError_t launch_swaps_range(uint64_t* w, size_t stride, int ncols, int skip_lo, int skip_hi, uint32_t* perm,
                               const PanelState* st, int j0, int j1, cudaStream_t s);
// rank-deficient inputs: *flag |= 1 unless rows [row0, n) of nwc word-columns at w are all zero
cudaError_t launch_any_nonzero(const uint64_t* w, size_t stride, size_t row0, size_t n, size_t nwc, uint32_t* flag,
                               int num_sms, cudaStream_t s);
// states of panels [j0, j1) as the panel kernel leaves them on all-zero columns (R, r = 0, no swaps)
cudaError_t launch_fill_zero_states(PanelState* st, int j0, int j1, uint32_t R, cudaStream_t s);
// swaps on all columns but panel_col (+perm) and Y on panel_col, one launch
cudaError_t launch_post(uint64_t* w, size_t stride, int ncols, int panel_col, uint32_t* perm,
                        size_t n, const PanelState* st, cudaStream_t s);
// dst = (acc ? dst : 0) ^ a ^ b ^ c ^ d over a rows x wcols block (any input may be null)
cudaError_t launch_xor(uint64_t* dst, size_t sd, const uint64_t* a, size_t sa,
                       const uint64_t* b, size_t sb, const uint64_t* c, size_t scc,
                       const uint64_t* d, size_t sdd, size_t rows, size_t wcols, bool acc,
                       cudaStream_t s);
cudaError_t launch_transpose(const uint64_t* a, size_t n, size_t m, size_t sa, uint64_t* out,
                             size_t so, cudaStream_t s);
// Fused lookahead link of one panel kernel (k_panel_gj):
//   head/win/all: counters of the previous k_post_col (block 0's first rows,
//   the first 8 blocks = the 2048-row window, every row block) that the
//   selection warp, the window load and the beyond-window scan wait for;
//   next: column j+1, which receives this panel's row swaps at the end once
//   *next_ready >= next_count (the update of column j+1 by the previous panel).
struct PanelLink {
    const uint32_t* head; uint32_t head_count;
    const uint32_t* win; uint32_t win_count;
    const uint32_t* all; uint32_t all_count;
    uint64_t* next;
    const uint32_t* next_ready; uint32_t next_count;
    uint32_t poll_ns = 0;  // sleep between polls of the consumer warps
    bool trace = false;    // device trace stamps (diagnostics)
    // head_out != nullptr (needs next): the panel kernel itself writes Y and the
    // next column's update for the first kPanelHeadRows rows below its pivots,
    // then increments *head_out (the next panel kernel's head counter); the
    // fused post skips those rows
    uint32_t* head_out = nullptr;
    // done_out: incremented once every write of this panel kernel (state, pair
    // list, swapped window, next-column swaps) is in memory; a fused post queued
    // ahead of time waits on it instead of a cross-stream event
    uint32_t* done_out = nullptr;
    // hand-off (fused schedule): hand_out != nullptr -> at its end this panel kernel
    // writes kHandWords words: the next column's pivot rows (64), the next column's
    // next kGjPos rows, and its own column's kGjPos rows below the pivots (D), all
    // swapped, before incrementing done_out.  hand_in != nullptr -> this kernel
    // starts on the previous panel's done counter (link.head) and applies the
    // previous panel's update to its first kGjPos rows itself (Y = D*Z, x ^= Y*B)
    // instead of waiting for the fused post's first rows.
    uint64_t* hand_out = nullptr;
    const uint64_t* hand_in = nullptr;
    const PanelState* prev = nullptr;  // the previous panel's state (Z, r) for hand_in
    // the leaf's first panel kernel under the chain schedule: it does not exit before
    // *chain_up != 0, i.e. before k_panel_chain is resident.  The posts that follow in
    // stream order spin with blocks on every SM, and the chain CTA needs a whole one.
    const uint32_t* chain_up = nullptr;
};
constexpr int kHandWords = 256;
constexpr int kPanelHeadRows = 256;
cudaError_t launch_panel_link(uint64_t* col, size_t n, PanelState* st_all, int j, const PanelLink& link,
                              cudaStream_t s);
bool panel_link_ok();  // false when F2GPU_PANEL=0 selects the older panel kernel
// The panel chain of a whole leaf [c0, c1) in one persistent CTA (k_panel_chain): the
// same inputs, waits and outputs as launch_panel_link per panel under the fused
// schedule with counter-driven posts (done counter = flags[j * flags_per_panel + 4]),
// but panel j+1 starts on an in-CTA hand-off from panel j.
struct ChainArgs {
    uint64_t* w;        // the matrix the leaf runs on; its word-column 0 is global column coff
    size_t stride, n;
    PanelState* st;     // global panel index
    uint32_t* flags;    // kFlagsPerPanel counters per panel (global panel index)
    int flags_per_panel;
    int leaf0;          // the leaf's first panel (panels > leaf0 wait on the previous post / update)
    int c0, c1, coff;   // the chain's panels [c0, c1), c0 >= leaf0
    uint32_t yblocks;   // post_col_yblocks(n)
    uint32_t upd_grid;  // CTAs of the update (first-column release count)
    uint32_t poll_ns;
    bool trace;
};
cudaError_t launch_panel_chain(const ChainArgs& a, cudaStream_t s);
// POST + the next column's update in one launch: swaps on every word-column
// except panel_col and next_col, Y = D*Z on the panel column, and (next_col >=
// 0) next[i] ^= Y_i * B for i >= R + r.  flags[0] += 1 by row block 0 after
// its first 256 rows, flags[1] += 1 by row blocks < 8 likewise, flags[2] += 1
// by every row block at its end.
int post_col_yblocks(size_t n);
cudaError_t launch_post_col(uint64_t* w, size_t stride, int ncols, int panel_col, int next_col, uint32_t* perm,
                            size_t n, const PanelState* st, uint32_t* flags, cudaStream_t s,
                            bool trace = false, int skip = 0, const uint32_t* wait_panel = nullptr,
                            bool pdl = false);
// lookahead: panel j's update of word-column j+1 only; increments *done per CTA
int update_col_grid(size_t n, int num_sms);
cudaError_t launch_update_col(uint64_t* next, const uint64_t* ycol, size_t n, const PanelState* st, uint32_t* done,
                              int grid, cudaStream_t s);
cudaError_t launch_iota(uint32_t* p, size_t n, cudaStream_t s);
cudaError_t launch_set_diag(uint64_t* w, size_t stride, size_t rows, size_t wcol0, cudaStream_t s);
cudaError_t launch_gather_rows(uint64_t* dst, size_t sd, const uint64_t* src, size_t ss, const uint32_t* perm,
                               size_t n, size_t nq, cudaStream_t s);
cudaError_t launch_mask_cols(uint64_t* w, size_t stride, size_t n, size_t m, cudaStream_t s);

// batched products / XORs (device arrays of descriptors)
cudaError_t launch_gemm_batched(const GemmArgs* d_probs, const size_t* d_offs, int nprob,
                                size_t total_units, int num_sms, cudaStream_t s);
cudaError_t launch_xor_batched(const XorJob* d_jobs, int njobs, size_t max_rows, size_t max_wcols,
                               cudaStream_t s);
size_t gemm_units_host(const GemmArgs& p);
bool gemm_fast_ok(const GemmArgs& g);

// evaluated tensor-core leaf (tc_leaf.cu): int8 tcgen05 GF(2) product,
// n % 256 == 0, m % 128 == 0, k % 64 == 0
bool gemm_tc_ok(size_t n, size_t k, size_t m);
cudaError_t launch_gemm_tc(const uint64_t* A, size_t sa, const uint64_t* B, size_t sb, uint64_t* C,
                           size_t sc, size_t n, size_t k, size_t m, bool acc, cudaStream_t s);
// 256x256-tile variant on a pre-transposed B (BT = B^T, m x k):
// n % 256 == 0, m % 256 == 0, k % 64 == 0
bool gemm_tc2_ok(size_t n, size_t k, size_t m);
cudaError_t launch_gemm_tc2(const uint64_t* A, size_t sa, const uint64_t* BT, size_t sbt, uint64_t* C,
                            size_t sc, size_t n, size_t k, size_t m, bool acc, cudaStream_t s);
// block-scaled FP4 variant: n, k arbitrary (B^T bits past k zero), m % 256 == 0
struct TcGemmArgs {
    const uint64_t* A; size_t sa, n;     // A: n x k, word (i, q) at A[q*sa + i]
    const uint64_t* BT; size_t sbt;      // B^T: m x k
    uint64_t* C; size_t sc;              // C: n x m
    size_t k, m;
    int acc;                             // C ^= A*B (else C = A*B)
};
cudaError_t launch_gemm_tc3_batched(const TcGemmArgs* h_probs, const TcGemmArgs* d_probs, int nprob,
                                    cudaStream_t s);
bool gemm_tc3_ok(size_t n, size_t k, size_t m);
// k_gemm_tc7 (tc_pair.cu): the same product on CTA pairs, persistent, M-side operand
// in TMEM; m % 256 == 0.  F2GPU_TC7=0 disables it (A/B checks).
bool gemm_tc7_enabled();
cudaError_t launch_gemm_tc7(const TcGemmArgs& p, cudaStream_t s);
cudaError_t launch_gemm_tc7_batched(const TcGemmArgs* h_probs, const TcGemmArgs* d_probs, int nprob,
                                    cudaStream_t s);
cudaError_t launch_gemm_tc3(const uint64_t* A, size_t sa, size_t n, const uint64_t* BT, size_t sbt,
                            uint64_t* C, size_t sc, size_t k, size_t m, bool acc, cudaStream_t s);

// tensor-core trailing update (tc_update.cu): C[lo..hi) x [q0, q0+ncols) ^= A * B,
// A = kwords (<= 2) word-columns at a (stride sa), B^T = ncols*64 rows x kwords
// words at bt (stride sbt >= update_tc_bt_rows(ncols)); lo = st->R + st->r when
// st is set.  release: lookahead counter, update_tc_release_count() increments
// once column tile 0 (the next block's panel columns) is complete in memory.
struct TcUpdateArgs {
    uint64_t* C; size_t sc; size_t q0; int ncols;
    size_t row_lo, row_hi;
    const uint64_t* a; size_t sa; int kwords;
    const uint64_t* bt; size_t sbt;
    const PanelState* st;
    uint32_t* release;
};
bool update_tc_ok(const TcUpdateArgs& a);
int update_tc_segments(const TcUpdateArgs& a, int grid);
int update_tc_release_count(const TcUpdateArgs& a, int grid);
size_t update_tc_bt_rows(int ncols);
cudaError_t launch_update_tc(const TcUpdateArgs& a, int grid, cudaStream_t s);

// block TRSM base (decompose_recursive, full rank): P <= 16 panels a.., pivot
// rows Ra .. Ra+64P, in place on word-columns [col0, col0+ncols)
int trsm_max_panels();  // largest P one k_trsm_block launch solves
cudaError_t launch_trsm_block(uint64_t* W, size_t stride, int a, int P, size_t Ra, size_t col0, int ncols,
                              cudaStream_t s);
// the same with L and C in separate matrices: L = panel a's column at row Ra
// (panel a+t at L + t*ls), C = the first target word-column at row Ra
cudaError_t launch_trsm_block_l(const uint64_t* L, size_t ls, uint64_t* C, size_t sc, int P, int ncols,
                                cudaStream_t s);

// per-device one-time setup (dynamic shared memory opt-in)
cudaError_t init_kernel_attrs();

// host helper: the 64 jump matrices T^(2^s) of the xorshift64* state map
void host_jump_tables(uint64_t out[64 * 64]);

}  // namespace f2
