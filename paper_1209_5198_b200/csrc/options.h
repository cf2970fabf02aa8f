// options.h — every switch of libf2gpu in one table: field, environment variable,
// default, meaning.  f2::options() reads the environment once (first call) and the
// library reads its switches only from there (contexts copy the schedule fields at
// creation); f2gpu_options_describe() prints the table with the values in effect.
// Every switch only selects among bit-identical paths, tunes a size, or turns on a
// diagnostic.  INTEGRATION.md lists the ones a caller may want.
#pragma once
#include <cstddef>

// X(field, "ENV", default, "meaning")
#define F2_OPTIONS(X)                                                                                          \
    /* ---- decomposition schedule (per context, copied at f2gpu_ctx_create) ---- */                         \
    X(graphs, "F2GPU_GRAPHS", 1, "capture the panel loops as CUDA graphs and replay them (0: direct launches)") \
    X(profile, "F2GPU_PROFILE", 0, "per-kernel CUDA-event timeline of each decomposition on stderr")           \
    X(lookahead, "F2GPU_LOOKAHEAD", 1, "depth-1 lookahead: P(j+1) on side streams overlaps update j")          \
    X(lookahead_col, "F2GPU_LOOKAHEAD_COL", 1, "unfused schedule: the next column updated by its own kernel")  \
    X(postcol, "F2GPU_POSTCOL", 1, "fused k_post_col (swaps + Y + next column) (0: k_post + k_update_col)")      \
    X(panel_early, "F2GPU_PANEL_EARLY", 1, "queue P(j+1) ahead on alternating side streams (0: after post j)")  \
    X(poll_ns, "F2GPU_POLL_NS", 0, "sleep (ns) between polls of the panel kernel's consumer warps")            \
    X(u_firstcol, "F2GPU_U_FIRSTCOL", 1, "the update releases the next panel's column first (0: group 0)")     \
    X(u_fc_ctas, "F2GPU_U_FC_CTAS", 24, "update CTAs doing that first column (0: all; unset: 40 in chain-schedule leaves)")                       \
    X(u_fc_w, "F2GPU_U_FC_W", 3, "their share of the bulk tiles, in quarters (1..4; unset: 2 in chain-schedule leaves)")                        \
    X(panel_head, "F2GPU_PANEL_HEAD", 0, "the panel kernel computes the first 256 rows below its pivots")      \
    X(post_spin, "F2GPU_POST_SPIN", 1, "k_post_col waits for its panel kernel on a counter (0: by event)")     \
    X(pdl, "F2GPU_PDL", 1, "the update is a programmatic dependent launch of k_post_col")                    \
    X(post_pdl, "F2GPU_POST_PDL", 0, "k_post_col as a programmatic dependent of the previous update (unset: on in the chain schedule, off with per-panel launches, where it can starve P)") \
    X(panel_hand, "F2GPU_PANEL_HAND", 0, "P(j+1) starts on P(j)'s done counter with a hand-off block")         \
    X(panel_chain, "F2GPU_PANEL_CHAIN", 1, "one persistent k_panel_chain CTA per leaf: panel j+1 starts on an in-CTA hand-off") \
    X(chain_sms, "F2GPU_CHAIN_SMS", 2, "SMs the updates leave free under F2GPU_PANEL_CHAIN (the chain CTA needs one)") \
    X(tc, "F2GPU_TC", 1, "products on the fp4 tensor-core leaf (0: M4RM only)")                              \
    X(tc_cut, "F2GPU_TC_CUT", 16384, "Strassen-Winograd leaf of the tensor-core products (strassen_mult)")    \
    X(spin_diag, "F2GPU_SPIN_DIAG", 0, "record a timed-out cross-kernel wait in host-mapped memory")          \
    X(force_nccl, "F2GPU_FORCE_NCCL", 0, "build a 1-rank NCCL communicator at world size 1 (read per call)")  \
    /* ---- decompose_recursive ---- */                                                                      \
    X(rec_cut, "F2GPU_REC_CUT", 16384, "Strassen cutover of the recursion's M4RM products")                   \
    X(rec_base, "F2GPU_REC_BASE", 256, "leaf width in panels (when set: overrides min_cols)")                \
    X(rec_tbase, "F2GPU_REC_TBASE", 32, "TRSM base in panels (one k_trsm_block launch; <= 64)")              \
    X(rec_trsm, "F2GPU_REC_TRSM", 1, "TRSM base by k_trsm_block (0: rank-64 updates)")                        \
    X(rec_tall, "F2GPU_REC_TALL", 30000, "leaves with at least this many rows below them are narrower")      \
    X(rec_tall_base, "F2GPU_REC_TALL_BASE", 64, "their width in panels")                                      \
    X(rec_tc_cut, "F2GPU_REC_TC_CUT", 8192, "Strassen-Winograd leaf of the recursion's tensor-core products") \
    X(rec_final, "F2GPU_REC_FINAL", 32, "host entry: right-spine leaf width (panels) for early downloads")    \
    X(rec_first, "F2GPU_REC_FIRST", 64, "host entry: first leaf / upload chunk width (panels)")              \
    X(trsm_m4rm_k, "F2GPU_TRSM_M4RM_K", 1024, "TRSM products with k <= this run on M4RM")                     \
    X(trsm_kernel, "F2GPU_TRSM_KERNEL", 0, "1: k_trsm_block prefetching two panels ahead (512 threads at P > 32)") \
    X(dist_leaf, "F2GPU_DIST_LEAF", 1, "distributed recursion: leaves factored whole on a replicated copy (0: per-panel broadcasts)") \
    X(rec_times, "F2GPU_REC_TIMES", 0, "per-phase CUDA-event times of the recursion on stderr")               \
    X(no_upload_overlap, "F2GPU_NO_UPLOAD_OVERLAP", 0, "host entry: upload everything before factoring")     \
    /* ---- kernel selection ---- */                                                                          \
    X(update, "F2GPU_UPDATE", 4, "Schur update kernel: 4 = k_update_v4 (8-column groups, 8-bit tables, 24 consumer warps), 3 = k_update_v3 (16-column groups, 7-bit tables)") \
    X(panel, "F2GPU_PANEL", 1, "panel kernel k_panel_gj (0: the older transposed-M k_panel)")                 \
    X(panel_smem, "F2GPU_PANEL_SMEM", 1, "the panel kernel reserves a whole SM's shared memory")              \
    X(tc7, "F2GPU_TC7", 1, "fp4 pair leaf k_gemm_tc7 geometry 1..7 (0: single-CTA k_gemm_tc3)")               \
    X(tc7_mode, "F2GPU_TC7_MODE", 0, "k_gemm_tc7 diagnostics (1 no MMA, 7 cycle accounting, 8 trace, ...)")   \
    X(tc_mode, "F2GPU_TC_MODE", 0, "k_gemm_tc3 diagnostics / variants")                                        \
    X(tc_persist, "F2GPU_TC_PERSIST", 0, "experimental builds: persistent k_gemm_tc5")                         \
    X(tc5_maxk, "F2GPU_TC5_MAXK", 2048, "experimental builds: k_gemm_tc5 up to this k")                        \
    X(tc6_maxk, "F2GPU_TC6_MAXK", 0, "experimental builds: k_gemm_tc6 up to this k")                           \
    X(tc_pair, "F2GPU_TC_PAIR", 0, "experimental builds: single-CTA pair leaf k_gemm_tc4")                     \
    X(tc_kind, "F2GPU_TC_KIND", 4, "experimental builds: 8 (or i8) = the int8 leaf for f2gpu_gemm_tc")        \
    X(ut_mode, "F2GPU_UT_MODE", 0, "experimental builds: tensor-core update variant")

namespace f2 {

struct Options {
#define F2_OPT_FIELD(field, env, def, doc) \
    long long field = def;                 \
    bool field##_set = false;
    F2_OPTIONS(F2_OPT_FIELD)
#undef F2_OPT_FIELD
};

const Options& options();  // the environment, read once
// one variable, read now (for the few switches read per call: F2GPU_FORCE_NCCL)
bool env_value(const char* env, long long* v);

}  // namespace f2
