// api.cu — C-ABI (include/f2gpu.h) and the native host drivers:
//   * device matrix store (PackedMatrix<uint64_t> analogue, bit_matrix.hpp:82-346)
//   * decompose_block driver: per panel  buildZ -> swaps -> Y -> Schur,
//     all enqueued without host synchronisation (R and r_j stay on the device)
//   * sharded / distributed driver: word-columns round-robin over shards, the
//     panel owner broadcasts {PanelState, panel column} (NCCL over NVLink)
//   * Strassen-Winograd recursion over device sub-blocks
#include <dlfcn.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <array>
#include <string>
#include <vector>

#include "../../include/f2gpu.h"
#include "kernels.cuh"
#include "options.h"

#define F2GPU_VERSION "0.2.0"

namespace f2 {
// options.h: the environment read once.  A value is parsed after any leading
// non-digits ("i8" -> 8); an unparsable one keeps the default.
// One environment variable: true (and *v set) when present and parsable.
bool env_value(const char* env, long long* v) {
    const char* e = getenv(env);
    if (!e) return false;
    const char* q = e;
    while (*q && !(*q >= '0' && *q <= '9') && *q != '-') ++q;
    char* end = nullptr;
    const long long x = strtoll(q, &end, 10);
    if (end == q) return false;
    *v = x;
    return true;
}

const Options& options() {
    static const Options o = [] {
        Options r;
        auto rd = [](const char* env, long long& v, bool& set) {
            if (env_value(env, &v)) set = true;
        };
#define F2_OPT_READ(field, env, def, doc) rd(env, r.field, r.field##_set);
        F2_OPTIONS(F2_OPT_READ)
#undef F2_OPT_READ
        return r;
    }();
    return o;
}
}  // namespace f2

namespace {

thread_local std::string g_err;
// F2GPU_SPIN_DIAG=1: host-mapped record of a timed-out cross-kernel wait (kernels.cu
// SpinGuard), appended to the next CUDA error message; g_diag_flags = the counter base
unsigned long long* g_diag = nullptr;
const void* g_diag_flags = nullptr;

int set_err(int code, const std::string& msg) {
    g_err = msg;
    if (code == F2GPU_ECUDA && g_diag && (g_diag[0] & 1)) {
        const long long off = static_cast<long long>(g_diag[2]) - reinterpret_cast<long long>(g_diag_flags);
        char b[256];
        snprintf(b, sizeof b, " [spin timeout: site %llu block %llu counter +%lld B (panel %lld idx %lld) value %llu target %llu]",
                 g_diag[0] >> 8, g_diag[1], off, off / 32, (off % 32) / 4, g_diag[3] >> 32, g_diag[3] & 0xffffffffull);
        g_err += b;
        if (g_diag[6]) {  // k_panel_chain's progress: panel << 8 | stage per team
            snprintf(b, sizeof b, " [chain %llu..%llu: team 0 panel %llu stage %llu, team 1 panel %llu stage %llu]",
                     g_diag[6] >> 32, g_diag[6] & 0xffffffffull, g_diag[4] >> 8, g_diag[4] & 255, g_diag[5] >> 8,
                     g_diag[5] & 255);
            g_err += b;
        }
    }
    return code;
}

#define CUDA_TRY(expr)                                                                    \
    do {                                                                                  \
        cudaError_t _e = (expr);                                                          \
        if (_e != cudaSuccess)                                                            \
            return set_err(_e == cudaErrorMemoryAllocation ? F2GPU_ENOMEM : F2GPU_ECUDA, \
                           std::string(#expr) + ": " + cudaGetErrorString(_e));           \
    } while (0)

#define F2_TRY(expr)                   \
    do {                               \
        int _rc = (expr);              \
        if (_rc != F2GPU_OK) return _rc; \
    } while (0)

size_t ceil64(size_t x) { return (x + 63) / 64; }
// 128-row (1 KiB) granularity: the bulk-copy update kernel moves 128-row column segments
size_t dev_stride(size_t rows) { return std::max<size_t>(128, (rows + 127) / 128 * 128); }

// ---- NCCL, loaded at run time --------------------------------------------
struct Id128 { char b[128]; };  // ncclUniqueId (NCCL_UNIQUE_ID_BYTES = 128), passed by value
typedef int (*CommInitRankFn)(void**, int, Id128, int);

struct NcclApi {
    void* h = nullptr;
    int (*getUniqueId)(void*) = nullptr;
    void* commInitRankSym = nullptr;
    int (*broadcast)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*commDestroy)(void*) = nullptr;
    int (*groupStart)() = nullptr;
    int (*groupEnd)() = nullptr;
    const char* (*getErrorString)(int) = nullptr;
    bool ok = false;
    std::string why;
};

NcclApi& nccl() {
    static NcclApi api;
    static bool tried = false;
    if (!tried) {
        tried = true;
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* nm : names) {
            api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
            if (api.h) break;
        }
        if (!api.h) {
            api.why = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
            return api;
        }
        api.getUniqueId = (int (*)(void*))dlsym(api.h, "ncclGetUniqueId");
        api.commInitRankSym = dlsym(api.h, "ncclCommInitRank");
        api.broadcast = (int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t))dlsym(
            api.h, "ncclBroadcast");
        api.commDestroy = (int (*)(void*))dlsym(api.h, "ncclCommDestroy");
        api.groupStart = (int (*)())dlsym(api.h, "ncclGroupStart");
        api.groupEnd = (int (*)())dlsym(api.h, "ncclGroupEnd");
        api.getErrorString = (const char* (*)(int))dlsym(api.h, "ncclGetErrorString");
        api.ok = api.getUniqueId && api.commInitRankSym && api.broadcast && api.commDestroy && api.groupStart &&
                 api.groupEnd;
        if (!api.ok) api.why = "libnccl.so.2 lacks required symbols";
    }
    return api;
}

constexpr int kNcclUint8 = 1;  // ncclDataType_t ncclUint8 (nccl.h)

}  // namespace

// ---------------------------------------------------------------------------
// Opt-in timeline (F2GPU_PROFILE=1): an event after every launch; per-kernel
// device time = sum of the gaps ending at that kernel's event (so it includes
// the launch gap in front of it).  Printed to stderr after each decomposition.
struct Timeline {
    bool on = false;
    std::vector<cudaEvent_t> pool;
    std::vector<std::pair<cudaEvent_t, const char*>> marks;
    void mark(cudaStream_t s, const char* what) {
        if (!on) return;
        if (marks.size() == pool.size()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            pool.push_back(e);
        }
        cudaEvent_t e = pool[marks.size()];
        cudaEventRecord(e, s);
        marks.emplace_back(e, what);
    }
    void report(const char* title) {
        if (!on || marks.size() < 2) { marks.clear(); return; }
        cudaEventSynchronize(marks.back().first);
        std::vector<std::pair<std::string, std::pair<double, int>>> acc;
        for (size_t i = 1; i < marks.size(); ++i) {
            float ms = 0;
            cudaEventElapsedTime(&ms, marks[i - 1].first, marks[i].first);
            auto it = std::find_if(acc.begin(), acc.end(),
                                   [&](const auto& x) { return x.first == marks[i].second; });
            if (it == acc.end()) acc.push_back({marks[i].second, {ms, 1}});
            else { it->second.first += ms; it->second.second += 1; }
        }
        float tot = 0;
        cudaEventElapsedTime(&tot, marks.front().first, marks.back().first);
        fprintf(stderr, "{\"f2gpu_profile\": \"%s\", \"total_ms\": %.3f", title, tot);
        for (auto& x : acc)
            fprintf(stderr, ", \"%s\": [%.3f, %d]", x.first.c_str(), x.second.first, x.second.second);
        fprintf(stderr, "}\n");
        marks.clear();
    }
    ~Timeline() { for (auto e : pool) cudaEventDestroy(e); }
};

// Replayable decomposition: the panel loop never synchronises with the host
// (R and r_j live in device PanelStates), so for a repeated (matrix, shape) the
// whole launch sequence is captured once into a CUDA graph and replayed.
struct GraphCache {
    uint64_t* w = nullptr;
    size_t stride = 0, n = 0, mu = 0;
    void* st = nullptr;
    int seen = 0;                 // eager runs with this key
    cudaGraphExec_t exec = nullptr;
    uint64_t nodes = 0;
    bool has_chain = false;       // k_panel_chain is launched outside the graph (see LeafGraph)
    f2::ChainArgs chain{};
    void reset() {
        if (exec) cudaGraphExecDestroy(exec);
        exec = nullptr;
        seen = 0;
        nodes = 0;
        w = nullptr;
        has_chain = false;
    }
    bool match(uint64_t* w_, size_t s_, size_t n_, size_t mu_, void* st_) const {
        return w == w_ && stride == s_ && n == n_ && mu == mu_ && st == st_;
    }
};

// decompose_recursive: one captured graph per leaf (matrix, shape, column range)
struct LeafGraph {
    int seen = 0;
    cudaGraphExec_t exec = nullptr;
    uint64_t nodes = 0;
    // the leaf's k_panel_chain launch stays OUTSIDE the graph (launched on the side
    // stream just before the graph): the kernels in the graph spin on its counters, and
    // a graph gives no guarantee that an independent root node is submitted before
    // ~770 dependent nodes of the other branch have been (seen: it was not, at 256 panels)
    bool has_chain = false;
    f2::ChainArgs chain{};
};
struct LeafGraphs {
    std::map<std::array<uintptr_t, 8>, LeafGraph> m;
    void clear() {
        for (auto& kv : m)
            if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
        m.clear();
    }
};

struct f2gpu_mat;
struct f2gpu_ctx {
    Timeline tl;
    f2gpu_mat* stage = nullptr;           // reusable device matrix for host-buffer calls
    GraphCache graph;
    LeafGraphs leaf_graphs;
    bool use_graphs = true;
    bool graphs_stream_ok = true;  // false on the legacy / per-thread default stream (no capture)
    bool lookahead = true;
    bool lookahead_col = true;  // F2GPU_LOOKAHEAD_COL=0: release from the update's column group 0 instead
    bool fuse_post = true;      // F2GPU_POSTCOL=0: separate POST and next-column kernels
    bool panel_early = true;    // F2GPU_PANEL_EARLY=0: launch P(j+1) after k_post_col(j) completes
    uint32_t poll_ns = 0;       // F2GPU_POLL_NS: panel consumer warps' poll sleep
    bool u_first_col = true;    // F2GPU_U_FIRSTCOL=0: release after column group 0 instead
    int u_fc_ctas = 24;         // F2GPU_U_FC_CTAS: CTAs doing that first column (0: all; 65536^2:
                                // 16: 63.18, 20: 63.21, 24: 63.00, 28: 63.30, 32: 63.28 ms)
    int u_fc_weight = 3;        // F2GPU_U_FC_W: their bulk share in quarters
    bool u_fc_ctas_set = false, u_fc_w_set = false;  // given in the environment (else 40, 2/4 in chain leaves)
    bool panel_head = false;    // F2GPU_PANEL_HEAD=1: the panel kernel does the first rows itself (measured slower)
    bool post_spin = true;      // F2GPU_POST_SPIN=0: k_post_col(j) waits for P(j) by event, not by counter
    bool pdl = true;            // F2GPU_PDL=0: the update after k_post_col is a plain stream-ordered launch
    // F2GPU_PANEL_HAND=1: P(j+1) starts on P(j)'s done counter with P(j)'s hand-off block.
    // Off: measured no faster at 65536^2 (64.12 vs 64.17 ms); kept opt-in
    // (tests/test_gpu_parity.py::test_panel_hand_off)
    bool panel_hand = false;
    // the panel chain of a leaf in one persistent CTA (k_panel_chain): panel j+1 starts
    // on an in-CTA hand-off instead of k_post_col(j)'s first rows
    bool panel_chain = false;
    int chain_sms = 2;
    cudaEvent_t ev_panel2 = nullptr;
    cudaStream_t side = nullptr;          // lookahead: panel kernels run here
    cudaStream_t side2 = nullptr;         // fused schedule: alternate panels (the next one is resident early)
    cudaStream_t copy = nullptr;          // decompose_recursive_host: chunked uploads
    std::vector<cudaEvent_t> chunk_ev;    // one per uploaded column chunk
    void* pend = nullptr;                 // uploaded, not yet materialised columns
    size_t pend_bytes = 0;
    cudaEvent_t ev_post = nullptr, ev_panel = nullptr;
    unsigned long long* trace_buf = nullptr;  // device trace (diagnostics)
    size_t trace_cap = 0;
    uint32_t* scr_flags = nullptr;        // per-panel counters (kFlagsPerPanel each)
    // device copies of batched-launch descriptors (Strassen XOR jobs, M4RM / fp4 problem
    // lists), cached by content: a repeated call (same operands and shapes) launches
    // without an in-stream H2D copy (desc_copy)
    struct DescEntry {
        std::string key;
        void* d = nullptr;
        cudaStream_t origin = nullptr;
        cudaEvent_t ready = nullptr;
        uint64_t used = 0;
    };
    std::vector<DescEntry> desc_cache;
    uint64_t desc_tick = 0;
    size_t scr_flags_cap = 0;
    uint64_t* scr_hand = nullptr;         // per-panel hand-off blocks (f2::kHandWords each)
    uint32_t* zero_flag = nullptr;        // rank-deficient splits: "trailing block is not all zero"
    uint64_t* leafbuf = nullptr;          // distributed leaves: the gathered leaf columns (persistent: graph keys)
    size_t leafbuf_words = 0;
    void* scr_st = nullptr;   // persistent PanelState[mu]
    size_t scr_st_cap = 0;
    uint32_t* scr_perm = nullptr;
    size_t scr_perm_cap = 0;
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    uint64_t* d_jump = nullptr;
    uint64_t launches = 0;
    size_t strassen_cutover = 4096;  // measured: 16384^3 -> 3 levels, 2.77 ms vs 3.15 ms plain M4RM
    // fp4 tensor-core leaf (F2GPU_TC=0 disables): products with n, k, m >= 256
    bool use_tc = true;
    size_t tc_cutover = 16384;  // minimum TC Strassen leaf size (F2GPU_TC_CUT)
    bool use_tc_cut_default = true;  // false once tc_cutover is set explicitly
    void* comm = nullptr;
    int rank = 0, world = 1;
};

struct f2gpu_mat {
    f2gpu_ctx* ctx = nullptr;
    uint64_t* d = nullptr;
    size_t rows = 0, cols = 0, stride = 0;
};

namespace {

struct View {  // non-owning device sub-block: rows x cols bits, word (i,q) at p[q*stride+i]
    uint64_t* p;
    size_t rows, cols, stride;
    size_t cap;   // addressable rows from p within a column (stride - row offset)
    size_t wcols() const { return ceil64(cols); }
    View sub(size_t r0, size_t nr, size_t wc0, size_t nwc) const {
        return View{p + wc0 * stride + r0, nr, nwc * 64, stride, cap - r0};
    }
};

View view_of(const f2gpu_mat* m) { return View{m->d, m->rows, m->cols, m->stride, m->stride}; }

int count(f2gpu_ctx* c, int n = 1) {
    c->launches += uint64_t(n);
    return F2GPU_OK;
}

int check_launch(f2gpu_ctx* c, cudaError_t e, const char* what) {
    if (e != cudaSuccess) return set_err(F2GPU_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    c->tl.mark(c->stream, what);
    return count(c);
}

int dev_alloc(f2gpu_ctx* c, void** p, size_t bytes) {
    if (bytes == 0) bytes = 8;
    cudaError_t e = cudaMallocAsync(p, bytes, c->stream);
    if (e != cudaSuccess) return set_err(F2GPU_ENOMEM, std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
    return F2GPU_OK;
}
void dev_free(f2gpu_ctx* c, void* p) {
    if (p) cudaFreeAsync(p, c->stream);
}

struct DevBuf {  // RAII stream-ordered allocation
    f2gpu_ctx* c;
    void* p = nullptr;
    explicit DevBuf(f2gpu_ctx* cc) : c(cc) {}
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { dev_free(c, p); }
    int alloc(size_t bytes) { return dev_alloc(c, &p, bytes); }
    template <class T> T* as() const { return static_cast<T*>(p); }
};

// A batched launch's descriptor array on the device.  Outside a stream capture it comes
// from the context's content-keyed cache (a hit on another stream waits for the copy);
// inside one it is a stream-ordered allocation that `tmp` frees after the launch.
int desc_copy(f2gpu_ctx* c, const void* host, size_t bytes, DevBuf& tmp, const void** out) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    CUDA_TRY(cudaStreamIsCapturing(c->stream, &cap));
    if (cap != cudaStreamCaptureStatusNone) {
        F2_TRY(tmp.alloc(bytes));
        CUDA_TRY(cudaMemcpyAsync(tmp.p, host, bytes, cudaMemcpyHostToDevice, c->stream));
        *out = tmp.p;
        return F2GPU_OK;
    }
    const std::string key(static_cast<const char*>(host), bytes);
    for (auto& e : c->desc_cache) {
        if (e.key == key) {
            if (e.origin != c->stream) CUDA_TRY(cudaStreamWaitEvent(c->stream, e.ready, 0));
            e.used = ++c->desc_tick;
            *out = e.d;
            return F2GPU_OK;
        }
    }
    if (c->desc_cache.size() >= 1024) {  // evict the least recently used
        size_t v = 0;
        for (size_t i = 1; i < c->desc_cache.size(); ++i)
            if (c->desc_cache[i].used < c->desc_cache[v].used) v = i;
        CUDA_TRY(cudaFree(c->desc_cache[v].d));  // synchronising: no launch still reads it
        cudaEventDestroy(c->desc_cache[v].ready);
        c->desc_cache.erase(c->desc_cache.begin() + long(v));
    }
    f2gpu_ctx::DescEntry e;
    e.key = key;
    e.origin = c->stream;
    e.used = ++c->desc_tick;
    CUDA_TRY(cudaMalloc(&e.d, bytes));
    CUDA_TRY(cudaMemcpyAsync(e.d, host, bytes, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(cudaEventCreateWithFlags(&e.ready, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(e.ready, c->stream));
    *out = e.d;
    c->desc_cache.push_back(std::move(e));
    return F2GPU_OK;
}

// C ^= A*B on views (stream-K M4RM kernel)
int gemm_acc(f2gpu_ctx* c, View C, View A, View B) {
    if (A.rows == 0 || A.cols == 0 || B.cols == 0) return F2GPU_OK;
    f2::GemmArgs g{A.p, A.stride, A.rows, B.p, B.stride, A.cols, C.p, C.stride, int(C.wcols()),
                   A.cap, B.cap};
    return check_launch(c, f2::launch_gemm(g, c->num_sms, c->stream), "k_gemm");
}

int xor_views(f2gpu_ctx* c, View dst, bool acc, const View* a, const View* b = nullptr,
              const View* cc = nullptr, const View* d = nullptr) {
    return check_launch(
        c,
        f2::launch_xor(dst.p, dst.stride, a ? a->p : nullptr, a ? a->stride : 0, b ? b->p : nullptr,
                       b ? b->stride : 0, cc ? cc->p : nullptr, cc ? cc->stride : 0,
                       d ? d->p : nullptr, d ? d->stride : 0, dst.rows, dst.wcols(), acc,
                       c->stream),
        "k_xor");
}

int zero_view(f2gpu_ctx* c, View v) {
    if (v.rows == 0 || v.wcols() == 0) return F2GPU_OK;
    CUDA_TRY(cudaMemset2DAsync(v.p, v.stride * 8, 0, v.rows * 8, v.wcols(), c->stream));
    c->tl.mark(c->stream, "memset2d");
    return F2GPU_OK;
}

// Strassen-Winograd, C ^= A*B, over F2 where
// every +/- is XOR.  Winograd's 7 products with all operand sums taken directly
// from quadrants (so a level's 8 pre-additions are independent):
//   S1=A21+A22  S2=A11+A21+A22  S3=A11+A21  S4=A11+A12+A21+A22
//   T1=B11+B12  T2=B11+B12+B22  T3=B12+B22  T4=B11+B12+B21+B22
//   P1=A11B11 P2=A12B21 P3=S4B22 P4=A22T4 P5=S1T1 P6=S2T2 P7=S3T3
//   C11+=P1+P2  C12+=P1+P6+P5+P3  C21+=P1+P6+P7+P4  C22+=P1+P6+P7+P5
// Executed level by level: one batched XOR launch per level for the pre-adds,
// ONE batched M4RM launch for all 7^L leaf products (zeroed P temps), then one
// batched XOR launch per level for the post-adds, bottom-up.  Recursion while
// every dimension is >= the cutover and halves stay 64-aligned.
int strassen_levels(size_t n, size_t k, size_t m, size_t cutover) {
    int L = 0;
    while (cutover >= 128 && n >= cutover && k >= cutover && m >= cutover && n % 128 == 0 &&
           k % 128 == 0 && m % 128 == 0 && L < 4) {
        n /= 2; k /= 2; m /= 2; ++L;
    }
    return L;
}

struct StrNode { View C, A, B; };

f2::XorJob xjob(View dst, bool acc, std::initializer_list<View> srcs) {
    f2::XorJob j{};
    j.dst = dst.p; j.sd = dst.stride; j.rows = dst.rows; j.wcols = dst.wcols(); j.acc = acc ? 1 : 0;
    int t = 0;
    for (const View& v : srcs) { j.src[t] = v.p; j.ss[t] = v.stride; ++t; }
    return j;
}

int launch_xor_jobs(f2gpu_ctx* c, const std::vector<f2::XorJob>& jobs) {
    if (jobs.empty()) return F2GPU_OK;
    DevBuf tmp(c);
    const void* d = nullptr;
    F2_TRY(desc_copy(c, jobs.data(), jobs.size() * sizeof(f2::XorJob), tmp, &d));
    size_t mr = 0, mw = 0;
    for (auto& j : jobs) { mr = std::max(mr, j.rows); mw = std::max(mw, j.wcols); }
    return check_launch(c, f2::launch_xor_batched(static_cast<const f2::XorJob*>(d), int(jobs.size()), mr, mw,
                                                  c->stream),
                        "k_xor_batched");
}

int strassen_acc(f2gpu_ctx* c, View C, View A, View B, size_t cutover) {
    const int L = strassen_levels(A.rows, A.cols, B.cols, cutover);
    if (L == 0) return gemm_acc(c, C, A, B);
    // temps: per node, S1..S4 (n2 x k2), T1..T4 (k2 x m2), P1..P7 (n2 x m2)
    size_t bytes = 0, pbytes = 0;
    {
        size_t n = A.rows, k = A.cols, m = B.cols, nodes = 1;
        for (int l = 0; l < L; ++l) {
            n /= 2; k /= 2; m /= 2;
            bytes += nodes * (4 * dev_stride(n) * (k / 64) + 4 * dev_stride(k) * (m / 64)) * 8;
            pbytes += nodes * 7 * dev_stride(n) * (m / 64) * 8;
            nodes *= 7;
        }
    }
    DevBuf arena(c);
    F2_TRY(arena.alloc(bytes + pbytes));
    unsigned char* st_ptr = arena.as<unsigned char>();
    unsigned char* p_ptr = st_ptr + bytes;
    CUDA_TRY(cudaMemsetAsync(p_ptr, 0, pbytes, c->stream));  // P temps accumulate by XOR
    auto take = [&](unsigned char*& cur, size_t rows, size_t cols) {
        const size_t s = dev_stride(rows);
        View v{reinterpret_cast<uint64_t*>(cur), rows, cols, s, s};
        cur += s * (cols / 64) * 8;
        return v;
    };
    std::vector<StrNode> level{{C, A, B}};
    std::vector<std::vector<f2::XorJob>> post(L);
    for (int l = 0; l < L; ++l) {
        std::vector<f2::XorJob> pre;
        std::vector<StrNode> next;
        for (const StrNode& nd : level) {
            const size_t n2 = nd.A.rows / 2, k2 = nd.A.cols / 2, m2 = nd.B.cols / 2;
            const size_t kw = k2 / 64, mw = m2 / 64;
            View A11 = nd.A.sub(0, n2, 0, kw), A12 = nd.A.sub(0, n2, kw, kw);
            View A21 = nd.A.sub(n2, n2, 0, kw), A22 = nd.A.sub(n2, n2, kw, kw);
            View B11 = nd.B.sub(0, k2, 0, mw), B12 = nd.B.sub(0, k2, mw, mw);
            View B21 = nd.B.sub(k2, k2, 0, mw), B22 = nd.B.sub(k2, k2, mw, mw);
            View C11 = nd.C.sub(0, n2, 0, mw), C12 = nd.C.sub(0, n2, mw, mw);
            View C21 = nd.C.sub(n2, n2, 0, mw), C22 = nd.C.sub(n2, n2, mw, mw);
            View S1 = take(st_ptr, n2, k2), S2 = take(st_ptr, n2, k2), S3 = take(st_ptr, n2, k2),
                 S4 = take(st_ptr, n2, k2);
            View T1 = take(st_ptr, k2, m2), T2 = take(st_ptr, k2, m2), T3 = take(st_ptr, k2, m2),
                 T4 = take(st_ptr, k2, m2);
            View P[7];
            for (auto& v : P) v = take(p_ptr, n2, m2);
            pre.push_back(xjob(S1, false, {A21, A22}));
            pre.push_back(xjob(S2, false, {A11, A21, A22}));
            pre.push_back(xjob(S3, false, {A11, A21}));
            pre.push_back(xjob(S4, false, {A11, A12, A21, A22}));
            pre.push_back(xjob(T1, false, {B11, B12}));
            pre.push_back(xjob(T2, false, {B11, B12, B22}));
            pre.push_back(xjob(T3, false, {B12, B22}));
            pre.push_back(xjob(T4, false, {B11, B12, B21, B22}));
            next.push_back({P[0], A11, B11});
            next.push_back({P[1], A12, B21});
            next.push_back({P[2], S4, B22});
            next.push_back({P[3], A22, T4});
            next.push_back({P[4], S1, T1});
            next.push_back({P[5], S2, T2});
            next.push_back({P[6], S3, T3});
            post[l].push_back(xjob(C11, true, {P[0], P[1]}));
            post[l].push_back(xjob(C12, true, {P[0], P[5], P[4], P[2]}));
            post[l].push_back(xjob(C21, true, {P[0], P[5], P[6], P[3]}));
            post[l].push_back(xjob(C22, true, {P[0], P[5], P[6], P[4]}));
        }
        F2_TRY(launch_xor_jobs(c, pre));
        level.swap(next);
    }
    // all 7^L leaf products in one launch
    std::vector<f2::GemmArgs> probs;
    std::vector<size_t> offs{0};
    for (const StrNode& nd : level) {
        f2::GemmArgs g{nd.A.p, nd.A.stride, nd.A.rows, nd.B.p, nd.B.stride, nd.A.cols,
                       nd.C.p, nd.C.stride, int(nd.C.wcols()), nd.A.cap, nd.B.cap};
        if (!f2::gemm_fast_ok(g)) return set_err(F2GPU_ECUDA, "strassen: leaf operands not aligned");
        probs.push_back(g);
        offs.push_back(offs.back() + f2::gemm_units_host(g));
    }
    DevBuf tp(c), toff(c);
    const void *dp = nullptr, *doff = nullptr;
    F2_TRY(desc_copy(c, probs.data(), probs.size() * sizeof(f2::GemmArgs), tp, &dp));
    F2_TRY(desc_copy(c, offs.data(), offs.size() * sizeof(size_t), toff, &doff));
    F2_TRY(check_launch(c, f2::launch_gemm_batched(static_cast<const f2::GemmArgs*>(dp), static_cast<const size_t*>(doff),
                                                   int(probs.size()), offs.back(), c->num_sms,
                                                   c->stream),
                        "k_gemm_batched"));
    for (int l = L - 1; l >= 0; --l) F2_TRY(launch_xor_jobs(c, post[l]));
    return F2GPU_OK;
}

// ---- tensor-core products (fp4 leaf, tc_leaf.cu) ---------------------------
// Strassen-Winograd over (A, B^T): B is transposed once up front, so every leaf
// product gets its B^T operand as a plain view.  The B-side sums are formed on
// the transposed quadrants (B_ij^T is quadrant (j, i) of B^T); P temps are
// written by the leaves (acc = 0), the top level accumulates.
int strassen_tc(f2gpu_ctx* c, View C, View A, View BT, int L) {
    const size_t n0 = A.rows, k0 = A.cols, m0 = BT.rows;
    if (L == 0) {
        f2::TcGemmArgs g{A.p, A.stride, n0, BT.p, BT.stride, C.p, C.stride, k0, m0, 1};
        return check_launch(c, f2::launch_gemm_tc3(g.A, g.sa, g.n, g.BT, g.sbt, g.C, g.sc, g.k, g.m, true,
                                                   c->stream),
                            "k_gemm_tc3");
    }
    size_t bytes = 0;
    {
        size_t n = n0, k = k0, m = m0, nodes = 1;
        for (int l = 0; l < L; ++l) {
            n /= 2; k /= 2; m /= 2;
            bytes += nodes * (4 * dev_stride(n) * (k / 64) + 4 * dev_stride(m) * (k / 64) +
                              7 * dev_stride(n) * (m / 64)) * 8;
            nodes *= 7;
        }
    }
    DevBuf arena(c);
    F2_TRY(arena.alloc(bytes));
    unsigned char* cur = arena.as<unsigned char>();
    auto take = [&](size_t rows, size_t cols) {
        const size_t s = dev_stride(rows);
        View v{reinterpret_cast<uint64_t*>(cur), rows, cols, s, s};
        cur += s * (cols / 64) * 8;
        return v;
    };
    struct Node { View C, A, BT; };
    std::vector<Node> level{{C, A, BT}};
    std::vector<std::vector<f2::XorJob>> post(L);
    for (int l = 0; l < L; ++l) {
        std::vector<f2::XorJob> pre;
        std::vector<Node> next;
        for (const Node& nd : level) {
            const size_t n2 = nd.A.rows / 2, k2 = nd.A.cols / 2, m2 = nd.BT.rows / 2;
            const size_t kw = k2 / 64, mw = m2 / 64;
            View A11 = nd.A.sub(0, n2, 0, kw), A12 = nd.A.sub(0, n2, kw, kw);
            View A21 = nd.A.sub(n2, n2, 0, kw), A22 = nd.A.sub(n2, n2, kw, kw);
            // B_ij^T: rows = the j-th half of m, word-columns = the i-th half of k
            View B11 = nd.BT.sub(0, m2, 0, kw), B12 = nd.BT.sub(m2, m2, 0, kw);
            View B21 = nd.BT.sub(0, m2, kw, kw), B22 = nd.BT.sub(m2, m2, kw, kw);
            View C11 = nd.C.sub(0, n2, 0, mw), C12 = nd.C.sub(0, n2, mw, mw);
            View C21 = nd.C.sub(n2, n2, 0, mw), C22 = nd.C.sub(n2, n2, mw, mw);
            View S1 = take(n2, k2), S2 = take(n2, k2), S3 = take(n2, k2), S4 = take(n2, k2);
            View T1 = take(m2, k2), T2 = take(m2, k2), T3 = take(m2, k2), T4 = take(m2, k2);
            View P[7];
            for (auto& v : P) v = take(n2, m2);
            pre.push_back(xjob(S1, false, {A21, A22}));
            pre.push_back(xjob(S2, false, {A11, A21, A22}));
            pre.push_back(xjob(S3, false, {A11, A21}));
            pre.push_back(xjob(S4, false, {A11, A12, A21, A22}));
            pre.push_back(xjob(T1, false, {B11, B12}));
            pre.push_back(xjob(T2, false, {B11, B12, B22}));
            pre.push_back(xjob(T3, false, {B12, B22}));
            pre.push_back(xjob(T4, false, {B11, B12, B21, B22}));
            next.push_back({P[0], A11, B11});
            next.push_back({P[1], A12, B21});
            next.push_back({P[2], S4, B22});
            next.push_back({P[3], A22, T4});
            next.push_back({P[4], S1, T1});
            next.push_back({P[5], S2, T2});
            next.push_back({P[6], S3, T3});
            // level 0 accumulates into C; deeper levels fill fresh P temps of the
            // level above, each quadrant by exactly one job
            const bool acc = l == 0;
            post[l].push_back(xjob(C11, acc, {P[0], P[1]}));
            post[l].push_back(xjob(C12, acc, {P[0], P[5], P[4], P[2]}));
            post[l].push_back(xjob(C21, acc, {P[0], P[5], P[6], P[3]}));
            post[l].push_back(xjob(C22, acc, {P[0], P[5], P[6], P[4]}));
        }
        F2_TRY(launch_xor_jobs(c, pre));
        level.swap(next);
    }
    std::vector<f2::TcGemmArgs> probs;
    for (const Node& nd : level)
        probs.push_back({nd.A.p, nd.A.stride, nd.A.rows, nd.BT.p, nd.BT.stride, nd.C.p, nd.C.stride, nd.A.cols,
                         nd.BT.rows, 0});
    // the pair leaf (default) takes the host list (its own descriptor cache); the
    // single-CTA leaves read a device copy
    DevBuf tp(c);
    const void* dp = nullptr;
    if (!f2::gemm_tc7_enabled()) F2_TRY(desc_copy(c, probs.data(), probs.size() * sizeof(f2::TcGemmArgs), tp, &dp));
    F2_TRY(check_launch(c, f2::launch_gemm_tc3_batched(probs.data(), static_cast<const f2::TcGemmArgs*>(dp),
                                                       int(probs.size()), c->stream),
                        "k_gemm_tc3_batched"));
    for (int l = L - 1; l >= 0; --l) F2_TRY(launch_xor_jobs(c, post[l]));
    return F2GPU_OK;
}

// levels of the tensor-core Strassen plan: halve while every leaf dimension stays
// at or above the cutover (the minimum leaf size) and leaves keep 256-column,
// 128-row granularity.  Measured (B200, fp4 leaf): 16384^3 direct 1.97 ms vs
// 2.12 ms with one level; 32768^3 one level (16384 leaves) 13.0 ms vs 15.3 ms
// direct -> default cutover 16384.
int strassen_tc_levels(size_t n, size_t k, size_t m, size_t cutover) {
    int L = 0;
    while (cutover >= 256 && n / 2 >= cutover && k / 2 >= cutover && m / 2 >= cutover && n % 256 == 0 &&
           k % 128 == 0 && m % 512 == 0 && L < 4) {
        n /= 2; k /= 2; m /= 2; ++L;
    }
    return L;
}

bool tc_product_ok(f2gpu_ctx* c, size_t n, size_t k, size_t m) {
    return c->use_tc && n >= 256 && k >= 256 && m >= 256;
}

// C ^= A*B with the fp4 tensor-core leaf on the first floor(m/256)*256 columns
// (Strassen-Winograd over tc_cutover) and M4RM on the rest
int tc_product(f2gpu_ctx* c, View C, View A, View B, size_t tc_cut) {
    const size_t n = A.rows, k = A.cols, m = B.cols, m256 = m / 256 * 256;
    if (m256 < m) {
        const size_t w0 = m256 / 64, nw = B.wcols() - w0;
        F2_TRY(strassen_acc(c, C.sub(0, n, w0, nw), A, B.sub(0, k, w0, nw), c->strassen_cutover));
    }
    if (m256 == 0) return F2GPU_OK;
    const size_t sbt = dev_stride(m256);
    DevBuf bt(c);
    F2_TRY(bt.alloc(sbt * ceil64(k) * 8));
    F2_TRY(check_launch(c, f2::launch_transpose(B.p, k, m256, B.stride, bt.as<uint64_t>(), sbt, c->stream),
                        "k_transpose"));
    View BT{bt.as<uint64_t>(), m256, k, sbt, sbt};
    View Cl{C.p, n, m256, C.stride, C.cap};
    return strassen_tc(c, Cl, A, BT, strassen_tc_levels(n, k, m256, tc_cut));
}

// the product used by the Strassen API and the recursive decomposition
int best_product(f2gpu_ctx* c, View C, View A, View B, size_t m4rm_cutover, size_t tc_cutover) {
    if (tc_product_ok(c, A.rows, A.cols, B.cols)) return tc_product(c, C, A, B, tc_cutover);
    return strassen_acc(c, C, A, B, m4rm_cutover);
}

// ---- decomposition drivers -------------------------------------------------

// One logical shard: a local packed matrix of the word-columns it owns.
struct Shard {
    View w;                      // n rows x (local wcols * 64)
    size_t lw = 0;               // local word-columns
    f2::PanelState* st = nullptr;  // mu states (device)
    uint32_t* perm = nullptr;    // device perm (replicated)
    uint64_t* bcast = nullptr;   // [PanelState | n words] broadcast landing buffer
    uint64_t* land = nullptr;    // recursive variant: landing column (stride rows; rows >= row_lo filled)
};

constexpr size_t kStateBytes = sizeof(f2::PanelState);
constexpr size_t kBcastHdr = 2048;  // state padded

// first local column whose global index is > j, for shard g of G
size_t first_local_after(size_t j, int g, int G) {
    if (j + 1 <= size_t(g)) return 0;
    return (j - size_t(g)) / size_t(G) + 1;
}

// Enqueue one panel step of the single-shard (G=1) decomposition.
int step_single(f2gpu_ctx* c, Shard& s, size_t n, size_t mu, size_t j) {
    uint64_t* colj = s.w.p + j * s.w.stride;
    F2_TRY(check_launch(c, f2::launch_panel(colj, n, s.st, int(j), c->stream), "k_panel"));
    F2_TRY(check_launch(c, f2::launch_post(s.w.p, s.w.stride, int(mu), int(j), s.perm, n,
                                           s.st + j, c->stream),
                        "k_post"));
    if (j + 1 < mu) {
        f2::UpdateArgs u{};
        u.C = s.w.p; u.sc = s.w.stride; u.c_wcol0 = j + 1; u.ncols = int(mu - j - 1);
        u.row_lo = 0; u.row_hi = n; u.a = colj; u.k_bits = 0;
        u.B = s.w.p; u.sb = s.w.stride; u.b_row0 = 0; u.b_wcol0 = j + 1;
        u.st = s.st + j;
        F2_TRY(check_launch(c, f2::launch_update(u, c->num_sms, c->stream), "k_update"));
    }
    return F2GPU_OK;
}

int read_results(f2gpu_ctx* c, const Shard& s, size_t n, size_t mu, uint32_t* perm,
                 uint32_t* rj, size_t* rank) {
    std::vector<f2::PanelState> hs(mu);
    if (mu)
        CUDA_TRY(cudaMemcpyAsync(hs.data(), s.st, mu * kStateBytes, cudaMemcpyDeviceToHost,
                                 c->stream));
    if (perm && n)
        CUDA_TRY(cudaMemcpyAsync(perm, s.perm, n * 4, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    size_t tot = 0;
    for (size_t j = 0; j < mu; ++j) {
        if (rj) rj[j] = hs[j].r;
        tot += hs[j].r;
    }
    if (rank) *rank = tot;
    return F2GPU_OK;
}

// per panel j: [0] head, [1] window, [2] all row blocks of k_post_col(j);
// [3] the release of update j's first column (group); [4] panel kernel j done;
// [5] (a leaf's first panel) k_panel_chain is resident
// (plain lookahead: [0] only)
constexpr size_t kFlagsPerPanel = 8;

int ensure_scratch(f2gpu_ctx* c, size_t n, size_t mu) {
    if (c->scr_st_cap < mu || c->scr_perm_cap < n || c->scr_flags_cap < mu) {
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        c->graph.reset();  // graphs hold the old pointers
        c->leaf_graphs.clear();
        if (c->scr_st_cap < mu) {
            cudaFree(c->scr_st);
            c->scr_st = nullptr;
            CUDA_TRY(cudaMalloc(&c->scr_st, mu * kStateBytes));
            c->scr_st_cap = mu;
        }
        if (c->scr_perm_cap < n) {
            cudaFree(c->scr_perm);
            c->scr_perm = nullptr;
            CUDA_TRY(cudaMalloc(&c->scr_perm, n * 4));
            c->scr_perm_cap = n;
        }
        if (c->scr_flags_cap < mu) {
            cudaFree(c->scr_hand);
            c->scr_hand = nullptr;
            CUDA_TRY(cudaMalloc(&c->scr_hand, mu * 8 * f2::kHandWords));
            cudaFree(c->scr_flags);
            c->scr_flags = nullptr;
            CUDA_TRY(cudaMalloc(&c->scr_flags, mu * 4 * kFlagsPerPanel));
            g_diag_flags = c->scr_flags;
            c->scr_flags_cap = mu;
        }
    }
    return F2GPU_OK;
}

// Lookahead schedule (two streams, capture-able):
//   main: POST(j) -> U(j) [SMs-1 CTAs, column j+1 first, then release flag j]
//   side: P(j+1) waits POST(j) (event) and then spins on flag j on the spare SM,
//         so the panel factorisation of j+1 overlaps the bulk of update j.
//   main waits P(j+1) (event) before POST(j+1).
// Panels [c0, c1) with their Schur updates restricted to word-columns < c1
// (c1 = mu for the block algorithm; a leaf range for the recursive one).  The
// swaps of every panel are applied to all mu word-columns.
// swap_cols: word-columns [0, swap_cols) receive the row swaps (default: all);
// the recursive driver's upload overlap keeps not-yet-materialised columns out
// chain_defer: when the stream is being captured, the k_panel_chain launch (and its
// fork / join) is left to the caller, who gets its arguments here (has = true) and must
// launch it on c->side before the graph (chain_fork / chain_join); a capturing caller
// without chain_defer gets the per-panel launches instead
struct ChainDefer {
    bool has = false;
    f2::ChainArgs args{};
};
int chain_fork(f2gpu_ctx* c, const f2::ChainArgs& a);
int chain_join(f2gpu_ctx* c);

int enqueue_panels(f2gpu_ctx* c, Shard& s, size_t n, size_t mu, size_t c0, size_t c1, bool la,
                   size_t swap_cols = size_t(-1), size_t coff = 0, ChainDefer* chain_defer = nullptr) {
    // coff: s.w's word-column 0 is global word-column coff (a distributed leaf runs on
    // a gathered copy of its own columns); states, flags and c0/c1/j stay global
    if (swap_cols > mu) swap_cols = mu;
    auto colp = [&](size_t j) { return s.w.p + (j - coff) * s.w.stride; };
    const bool fused = la && c->fuse_post && f2::panel_link_ok();
    // chain: the leaf's panel kernels are one persistent CTA (needs counter-driven posts)
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    CUDA_TRY(cudaStreamIsCapturing(c->stream, &cap));
    const bool capturing = cap != cudaStreamCaptureStatusNone;
    const bool chain = fused && c->panel_chain && c->post_spin && c->panel_early && !c->panel_head &&
                       !c->panel_hand && c->num_sms > 2 && (!capturing || chain_defer != nullptr);
    // fused schedule: two panel kernels can be resident (the running one and the
    // next one waiting for its head), each on its own SM
    const int grid = !la ? c->num_sms
                         : (chain ? c->num_sms - std::max(1, std::min(c->chain_sms, c->num_sms - 1))
                                  : (fused && c->num_sms > 2 ? c->num_sms - 2 : c->num_sms - 1));
    auto upd = [&](size_t j, uint32_t* release, size_t skip = 0, bool pdl = false) {
        f2::UpdateArgs u{};
        u.C = s.w.p; u.sc = s.w.stride; u.c_wcol0 = j + 1 + skip - coff; u.ncols = int(c1 - j - 1 - skip);
        if (u.ncols <= 0) return F2GPU_OK;
        u.row_lo = 0; u.row_hi = n; u.a = colp(j); u.k_bits = 0;
        u.B = s.w.p; u.sb = s.w.stride; u.b_row0 = 0; u.b_wcol0 = j + 1 + skip - coff;
        u.st = s.st + j;
        u.release = release;
        u.first_col = release != nullptr && c->u_first_col;
        // chain schedule, leaves of the recursion (<= 256 panels): the update's END is on the
        // critical path (the next post waits for it) and its first-column CTAs finish last,
        // while the release has ~2 us of slack: more of them with a smaller bulk share
        // (40 CTAs, 2/4: 48.25 -> 47.93 ms at 65536^2; wider block-variant runs keep 24, 3/4)
        const bool narrow = chain && c1 - c0 <= 256;
        u.fc_ctas = narrow && !c->u_fc_ctas_set ? 40 : c->u_fc_ctas;
        u.fc_weight = narrow && !c->u_fc_w_set ? 2 : c->u_fc_weight;
        u.tag = c->trace_buf ? int(j) : -1;
        u.pdl = pdl;
        return check_launch(c, f2::launch_update(u, grid, c->stream), "k_update");
    };
    const bool colfirst = c->lookahead_col;
    if (!la) {
        for (size_t j = c0; j < c1; ++j) {
            F2_TRY(check_launch(c, f2::launch_panel(colp(j), n, s.st, int(j),
                                                    c->stream),
                                "k_panel"));
            F2_TRY(check_launch(c, f2::launch_post(s.w.p, s.w.stride, int(swap_cols), int(j - coff), s.perm, n,
                                                   s.st + j, c->stream),
                                "k_post"));
            if (j + 1 < c1) F2_TRY(upd(j, nullptr));
        }
        return F2GPU_OK;
    }
    if (fused) {
        // Fused schedule:
        //   side: P(j+1) [waits k_post_col(j)'s counters: first rows / window / all;
        //         at its end applies its swaps to column j+2 once update j released it]
        //   main: k_post_col(j) [swaps except j, j+1; Y_j; column j+1 updated] ->
        //         U(j) on columns j+2.. [release after column group 0]
        // k_post_col(j) queued ahead on the main stream waits on P(j)'s done counter
        // (needs P(j+1) queued early on the alternating side streams)
        const bool spin = c->post_spin && c->panel_early;
        // hand-off: P(j+1) starts on P(j)'s done counter with P(j)'s hand-off block
        // (not on k_post_col(j)'s first rows); needs P(j+1) queued early
        const bool hand = c->panel_hand && c->panel_early && !c->panel_head;
        auto link_for = [&](size_t j) {  // P(j)'s link
            f2::PanelLink l{};
            if (j > c0) {
                uint32_t* f = c->scr_flags + (j - 1) * kFlagsPerPanel;
                l.head = f; l.head_count = 1;  // P(j-1)'s head chunk (or k_post_col's block 0)
                if (hand) {
                    l.head = f + 4;  // P(j-1) done
                    l.hand_in = c->scr_hand + (j - 1) * f2::kHandWords;
                    l.prev = s.st + (j - 1);
                }
                l.win = f + 1; l.win_count = c->panel_head ? 8 - f2::kPanelHeadRows / 256 : 8;
                l.all = f + 2; l.all_count = uint32_t(f2::post_col_yblocks(n));
                if (j + 1 < c1) { l.next_ready = f + 3; l.next_count = uint32_t(grid); }
            }
            if (j + 1 < c1) {
                l.next = colp(j + 1);
                if (c->panel_head) l.head_out = c->scr_flags + j * kFlagsPerPanel;  // this panel's head counter
            }
            l.poll_ns = c->poll_ns;
            l.trace = c->trace_buf != nullptr;
            if (spin || hand) l.done_out = c->scr_flags + j * kFlagsPerPanel + 4;
            if (hand && j + 1 < c1) l.hand_out = c->scr_hand + j * f2::kHandWords;
            return l;
        };
        if (chain) {
            // P(c0) in stream order, then one k_panel_chain launch on the side stream for
            // panels (c0, c1), forked BEFORE P(c0) so that the chain CTA is resident while
            // P(c0) runs; the posts on the main stream wait on the done counters, the
            // updates are unchanged
            const bool has_chain = c0 + 1 < c1;
            // k_post_col as a programmatic dependent of the previous update: its blocks are
            // placed as soon as the update's CTAs have left (47.98 -> 47.80 ms).  On by default
            // HERE only: with per-panel launches an early-placed post could take the SM its own
            // panel kernel still needed; the chain CTA is resident for the whole leaf.
            const bool chain_post_pdl = f2::options().post_pdl_set ? f2::options().post_pdl != 0 : true;
            f2::ChainArgs a{};
            a.w = s.w.p; a.stride = s.w.stride; a.n = n; a.st = s.st; a.flags = c->scr_flags;
            a.flags_per_panel = int(kFlagsPerPanel);
            a.leaf0 = int(c0); a.c0 = int(c0 + 1); a.c1 = int(c1); a.coff = int(coff);
            a.yblocks = uint32_t(f2::post_col_yblocks(n));
            a.upd_grid = uint32_t(grid);
            a.poll_ns = uint32_t(c->poll_ns);
            a.trace = c->trace_buf != nullptr;
            if (has_chain) {
                if (capturing) {
                    chain_defer->has = true;
                    chain_defer->args = a;
                } else {
                    F2_TRY(chain_fork(c, a));
                }
            }
            f2::PanelLink l0 = link_for(c0);
            if (has_chain) l0.chain_up = c->scr_flags + c0 * kFlagsPerPanel + 5;
            F2_TRY(check_launch(c, f2::launch_panel_link(colp(c0), n, s.st, int(c0), l0, c->stream), "k_panel"));
            for (size_t j = c0; j < c1; ++j) {
                uint32_t* f = c->scr_flags + j * kFlagsPerPanel;
                F2_TRY(check_launch(c, f2::launch_post_col(s.w.p, s.w.stride, int(swap_cols), int(j - coff),
                                                           j + 1 < c1 ? int(j + 1 - coff) : -1, s.perm, n, s.st + j,
                                                           f, c->stream, c->trace_buf != nullptr, 0,
                                                           j > c0 ? f + 4 : nullptr, j > c0 && chain_post_pdl),
                                    "k_post_col"));
                if (j + 1 >= c1) break;
                F2_TRY(upd(j, f + 3, 1, c->pdl));
            }
            if (has_chain && !capturing) F2_TRY(chain_join(c));
            return F2GPU_OK;
        }
        F2_TRY(check_launch(c, f2::launch_panel_link(colp(c0), n, s.st, int(c0), link_for(c0),
                                                     c->stream),
                            "k_panel"));
        // the side stream forks once after P(c0); every later panel kernel is queued
        // right behind its predecessor and spins on k_post_col's counters, so it is
        // resident (on the SM the update leaves free) before its column is ready
        cudaStream_t sides[2] = {c->side, c->side2};
        if (c0 + 1 < c1 && c->panel_early) {
            CUDA_TRY(cudaEventRecord(c->ev_post, c->stream));
            CUDA_TRY(cudaStreamWaitEvent(c->side, c->ev_post, 0));
            CUDA_TRY(cudaStreamWaitEvent(c->side2, c->ev_post, 0));
        }
        for (size_t j = c0; j < c1; ++j) {
            if (j > c0 && !spin) CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_panel, 0));
            uint32_t* f = c->scr_flags + j * kFlagsPerPanel;
            F2_TRY(check_launch(c, f2::launch_post_col(s.w.p, s.w.stride, int(swap_cols), int(j - coff),
                                                       j + 1 < c1 ? int(j + 1 - coff) : -1, s.perm, n, s.st + j, f,
                                                       c->stream, c->trace_buf != nullptr,
                                                       j + 1 < c1 && c->panel_head ? f2::kPanelHeadRows : 0,
                                                       j > c0 && spin ? f + 4 : nullptr,
                                                       j > c0 && spin && f2::options().post_pdl),
                                "k_post_col"));
            if (j + 1 >= c1) break;
            if (!c->panel_early) CUDA_TRY(cudaEventRecord(c->ev_post, c->stream));
            F2_TRY(upd(j, f + 3, 1, spin && c->pdl));
            // P(j+1) alternates between the two side streams: queued behind P(j-1),
            // it is resident while P(j) runs and starts on P(j)'s head counter
            cudaStream_t ps = c->panel_early ? sides[(j - c0) & 1] : c->side;
            if (!c->panel_early) CUDA_TRY(cudaStreamWaitEvent(ps, c->ev_post, 0));
            F2_TRY(check_launch(c, f2::launch_panel_link(colp(j + 1), n, s.st, int(j + 1),
                                                         link_for(j + 1), ps),
                                "k_panel"));
            CUDA_TRY(cudaEventRecord(c->ev_panel, ps));
        }
        if (spin && c0 + 1 < c1) {  // join both side streams (the posts only waited on counters)
            CUDA_TRY(cudaEventRecord(c->ev_panel, c->side));
            CUDA_TRY(cudaEventRecord(c->ev_panel2, c->side2));
            CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_panel, 0));
            CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_panel2, 0));
        }
        return F2GPU_OK;
    }
    F2_TRY(check_launch(c, f2::launch_panel(colp(c0), n, s.st, int(c0), c->stream),
                        "k_panel"));
    for (size_t j = c0; j < c1; ++j) {
        if (j > c0) CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_panel, 0));
        F2_TRY(check_launch(c, f2::launch_post(s.w.p, s.w.stride, int(swap_cols), int(j - coff), s.perm, n,
                                               s.st + j, c->stream),
                            "k_post"));
        if (j + 1 >= c1) break;
        CUDA_TRY(cudaEventRecord(c->ev_post, c->stream));
        uint32_t wait_count = uint32_t(grid);
        if (colfirst) {
            // the next panel's column alone first (small CTAs, counter), then the
            // persistent update from column j+2 with no early release
            const int g1 = f2::update_col_grid(n, c->num_sms);
            F2_TRY(check_launch(c, f2::launch_update_col(colp(j + 1), colp(j), n,
                                                         s.st + j, c->scr_flags + j * kFlagsPerPanel, g1,
                                                         c->stream),
                                "k_update_col"));
            F2_TRY(upd(j, nullptr, 1));
            wait_count = uint32_t(g1);
        } else {
            F2_TRY(upd(j, c->scr_flags + j * kFlagsPerPanel));
        }
        CUDA_TRY(cudaStreamWaitEvent(c->side, c->ev_post, 0));
        F2_TRY(check_launch(c, f2::launch_panel(colp(j + 1), n, s.st, int(j + 1),
                                                c->side, c->scr_flags + j * kFlagsPerPanel, wait_count),
                            "k_panel"));
        CUDA_TRY(cudaEventRecord(c->ev_panel, c->side));
    }
    return F2GPU_OK;
}

// the k_panel_chain launch of a leaf on the side stream, ordered after the main stream's
// earlier work, and the join after the leaf's main-stream launches (or graph)
int chain_fork(f2gpu_ctx* c, const f2::ChainArgs& a) {
    CUDA_TRY(cudaEventRecord(c->ev_post, c->stream));
    CUDA_TRY(cudaStreamWaitEvent(c->side, c->ev_post, 0));
    return check_launch(c, f2::launch_panel_chain(a, c->side), "k_panel_chain");
}
int chain_join(f2gpu_ctx* c) {
    CUDA_TRY(cudaEventRecord(c->ev_panel, c->side));
    CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_panel, 0));
    return F2GPU_OK;
}

// Lookahead schedule (two streams, capture-able):
//   main: POST(j) -> U(j) [SMs-1 CTAs, column j+1 first, then release flag j]
//   side: P(j+1) waits POST(j) (event) and then spins on flag j on the spare SM,
//         so the panel factorisation of j+1 overlaps the bulk of update j.
//   main waits P(j+1) (event) before POST(j+1).
// cd != nullptr (captured by decompose_single): the caller zeroes the counters itself,
// before it forks the chain kernel -- a memset inside the graph could wipe the chain's
// "resident" counter
int enqueue_lookahead(f2gpu_ctx* c, Shard& s, size_t n, size_t mu, ChainDefer* cd = nullptr) {
    if (!cd) CUDA_TRY(cudaMemsetAsync(c->scr_flags, 0, mu * 4 * kFlagsPerPanel, c->stream));
    F2_TRY(check_launch(c, f2::launch_iota(s.perm, n, c->stream), "k_iota"));
    return enqueue_panels(c, s, n, mu, 0, mu, true, size_t(-1), 0, cd);
}

bool lookahead_ok(f2gpu_ctx* c, const Shard& s, size_t n) {
    if (!c->lookahead || c->num_sms < 2 || !c->side) return false;
    f2::UpdateArgs u{};
    u.C = s.w.p; u.sc = s.w.stride; u.a = s.w.p; u.row_hi = n;
    return f2::update_fast_ok(u);
}

int enqueue_single(f2gpu_ctx* c, Shard& s, size_t n, size_t mu, ChainDefer* cd = nullptr) {
    if (lookahead_ok(c, s, n)) return enqueue_lookahead(c, s, n, mu, cd);
    F2_TRY(check_launch(c, f2::launch_iota(s.perm, n, c->stream), "k_iota"));
    for (size_t j = 0; j < mu; ++j) F2_TRY(step_single(c, s, n, mu, j));
    return F2GPU_OK;
}

// ---- decompose_recursive -------------
// Column split at cm: factor the left half recursively, then bring the right
// half up to date with the left panels in two big steps instead of one rank-64
// update per panel:
//   X  = L11^-1 C   (in place on the left pivot rows of the right half; L11 has
//                    identity 64x64 diagonal blocks, so a recursive block TRSM of
//                    rank-64 updates + GEMMs)
//   A' = D ^ L21 X  (one Strassen-Winograd/M4RM GEMM)
// then recurse on the right half.  Deferred updates commute with the later row
// swaps (SURVEY Probe P5), so W, perm and r_j are bit-identical to
// decompose_block.  The fast path needs the left half at full rank (R_j = R0 +
// 64(j-c0), 64-aligned); otherwise the left panels' updates are applied to the
// right half as rank-r_j updates (always exact).
struct RecRun {
    f2gpu_ctx* c;
    Shard* s;
    size_t n, mu, base;
    bool la;
    size_t cut;    // Strassen cutover inside the recursion (XOR traffic vs multiply)
    size_t tbase;  // TRSM base (panels solved in one k_trsm_block launch)
    size_t tall_rows = 0, tall_base = 0;  // leaves with >= tall_rows rows: at most tall_base panels
    // TRSM products with k <= this go to M4RM: at k = 1024 it beats the fp4 leaf's
    // per-tile fixed cost (n = k = 1024, m = 8192 / 32768 / 57344: 23 / 54 / 72 us vs
    // 26 / 60 / 95 us; ties at k = 2048, loses at 4096 -- tools/trsm_prod_scan.py)
    size_t trsm_m4rm_k = 1024;            // F2GPU_TRSM_M4RM_K
    size_t first_base = 0;                // left-spine leaves when uploads overlap (= the upload chunk)
    size_t final_base = 32;               // right-spine leaves when downloads overlap (F2GPU_REC_FINAL;
                                          // e2e at 65536^2: 32: 68.1-68.5 ms, 64: 68.6, off: 69.8)
    // F2GPU_REC_TIMES=1: CUDA events around every leaf / TRSM / product on the main
    // stream, summed per phase and printed (diagnostics; the side stream is untouched)
    struct Phase { std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev; };
    std::map<std::string, Phase>* phases = nullptr;
    size_t tc_cut = 8192;  // Strassen-Winograd leaf of the TC products (F2GPU_REC_TC_CUT; 65536^2:
                           // 8192 -> 66.9 ms, 16384 -> 67.3, 4096 -> 69.4, 32768 -> 69.7)
    bool trsm_kernel = true;  // F2GPU_REC_TRSM=0: rank-64 updates instead (A/B check)
    // upload overlap (f2gpu_decompose_recursive_host): word-columns >= frontier are
    // still in `pend` (original row order, column q at pend + (q - frontier0) * ps),
    // chunk i of `chunk` word-columns complete at event chunk_ev[i]
    size_t frontier = size_t(-1), frontier0 = 0, chunk = 0, ps = 0;
    const uint64_t* pend = nullptr;
    // download overlap: called (stream-ordered) when rows [0, R) are final in
    // every word-column -- after a split's TRSM/update on the recursion's right
    // spine: rows above R_J are never swapped or updated by a later panel
    std::function<int(size_t)> on_final;
};

// materialise word-columns up to c1: wait for their upload, gather them under the
// current composite permutation (swaps of every panel factored so far)
int ensure_cols(RecRun& r, size_t c1) {
    f2gpu_ctx* c = r.c;
    while (r.frontier < c1 && r.frontier < r.mu) {
        const size_t idx = (r.frontier - r.frontier0) / r.chunk;
        CUDA_TRY(cudaStreamWaitEvent(c->stream, c->chunk_ev[idx], 0));
        const size_t nq = std::min(r.chunk, r.mu - r.frontier);
        Shard& s = *r.s;
        F2_TRY(check_launch(c, f2::launch_gather_rows(s.w.p + r.frontier * s.w.stride, s.w.stride,
                                                      r.pend + (r.frontier - r.frontier0) * r.ps, r.ps, s.perm,
                                                      r.n, nq, c->stream),
                            "k_gather_rows"));
        r.frontier += nq;
    }
    return F2GPU_OK;
}

int rec_state(RecRun& r, size_t j, size_t* R, size_t* rr) {
    f2::PanelState h;
    CUDA_TRY(cudaStreamSynchronize(r.c->stream));
    CUDA_TRY(cudaMemcpy(&h, r.s->st + j, 16, cudaMemcpyDeviceToHost));
    *R = h.R;
    *rr = h.r;
    return F2GPU_OK;
}

// panels [a, b) applied to word-cols [col0, col1), rows (R_j + r_j) .. row_hi
int rank_updates(RecRun& r, size_t a, size_t b, size_t col0, size_t col1, size_t row_hi,
                 const char* what = "k_update") {
    Shard& s = *r.s;
    for (size_t j = a; j < b; ++j) {
        f2::UpdateArgs u{};
        u.C = s.w.p; u.sc = s.w.stride; u.c_wcol0 = col0; u.ncols = int(col1 - col0);
        u.row_lo = 0; u.row_hi = row_hi; u.a = s.w.p + j * s.w.stride; u.k_bits = 0;
        u.B = s.w.p; u.sb = s.w.stride; u.b_row0 = 0; u.b_wcol0 = col0;
        u.st = s.st + j;
        F2_TRY(check_launch(r.c, f2::launch_update(u, r.c->num_sms, r.c->stream), what));
    }
    return F2GPU_OK;
}

View wview(const Shard& s, size_t r0, size_t nr, size_t wc0, size_t nwc) {
    return View{s.w.p + wc0 * s.w.stride + r0, nr, nwc * 64, s.w.stride, s.w.stride - r0};
}

// full-rank block TRSM: panels [a, b) own pivot rows [Ra, Ra + 64(b-a)); solve in
// place on word-cols [col0, col1) of those rows.
template <typename F>
int timed(RecRun& r, const char* what, F&& f);

int rec_trsm(RecRun& r, size_t a, size_t b, size_t Ra, size_t col0, size_t col1) {
    const size_t Rb = Ra + 64 * (b - a);
    if (b - a <= r.tbase) {
        if (b - a <= size_t(f2::trsm_max_panels()) && r.trsm_kernel)
            return timed(r, "trsm.base", [&] {
                return check_launch(r.c, f2::launch_trsm_block(r.s->w.p, r.s->w.stride, int(a), int(b - a), Ra,
                                                               col0, int(col1 - col0), r.c->stream),
                                    "k_trsm_block");
            });
        return rank_updates(r, a, b, col0, col1, Rb, "k_update(trsm)");
    }
    const size_t m = a + (b - a) / 2, Rm = Ra + 64 * (m - a);
    F2_TRY(rec_trsm(r, a, m, Ra, col0, col1));
    F2_TRY(timed(r, (m - a) * 64 >= 8192 ? "trsm.prod.big" : "trsm.prod.small", [&] {
        const View C = wview(*r.s, Rm, Rb - Rm, col0, col1 - col0), A = wview(*r.s, Rm, Rb - Rm, a, m - a),
                   B = wview(*r.s, Ra, Rm - Ra, col0, col1 - col0);
        if ((m - a) * 64 <= r.trsm_m4rm_k) return strassen_acc(r.c, C, A, B, r.cut);
        return best_product(r.c, C, A, B, r.cut, r.tc_cut);
    }));
    return rec_trsm(r, m, b, Rm, col0, col1);
}

// Run `enqueue` (a leaf's launch sequence) through the per-context leaf-graph cache:
// eager on the first call with this key, captured + instantiated + launched on the
// second, replayed from the third.
template <typename F>
int leaf_graph_run(f2gpu_ctx* c, const std::array<uintptr_t, 8>& key, F&& enqueue) {
    if (!c->use_graphs || !c->graphs_stream_ok || c->tl.on) return enqueue(nullptr);
    LeafGraph& g = c->leaf_graphs.m[key];
    auto launch = [&]() {
        if (g.has_chain) F2_TRY(chain_fork(c, g.chain));
        CUDA_TRY(cudaGraphLaunch(g.exec, c->stream));
        if (g.has_chain) F2_TRY(chain_join(c));
        return int(F2GPU_OK);
    };
    if (g.exec) {
        F2_TRY(launch());
        c->launches += g.nodes;
        return F2GPU_OK;
    }
    if (g.seen < 1) {
        g.seen += 1;
        return enqueue(nullptr);
    }
    cudaGraph_t graph = nullptr;
    const uint64_t l0 = c->launches;
    ChainDefer cd;
    CUDA_TRY(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    int rc = enqueue(&cd);
    cudaError_t ec = cudaStreamEndCapture(c->stream, &graph);
    if (rc != F2GPU_OK) { if (graph) cudaGraphDestroy(graph); return rc; }
    if (ec != cudaSuccess) return set_err(F2GPU_ECUDA, std::string("leaf graph capture: ") + cudaGetErrorString(ec));
    cudaError_t ei = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ei != cudaSuccess) {
        g.exec = nullptr;
        return set_err(F2GPU_ECUDA, std::string("leaf graph instantiate: ") + cudaGetErrorString(ei));
    }
    g.nodes = c->launches - l0;
    g.has_chain = cd.has;
    g.chain = cd.args;
    return launch();
}

// a leaf: the block algorithm (with lookahead) on panels [c0, c1), replayed from
// a CUDA graph from the second call with the same matrix, shape and range
int rec_leaf(RecRun& r, size_t c0, size_t c1) {
    f2gpu_ctx* c = r.c;
    Shard& s = *r.s;
    F2_TRY(ensure_cols(r, c1));
    const size_t sw = std::min(r.frontier, r.mu);
    const std::array<uintptr_t, 8> key{uintptr_t(s.w.p), s.w.stride, r.n, r.mu, c0, c1,
                                       uintptr_t(s.st) ^ (r.la ? 1u : 0u), sw};
    return leaf_graph_run(c, key, [&](ChainDefer* cd) {
        return enqueue_panels(c, s, r.n, r.mu, c0, c1, r.la, sw, 0, cd);
    });
}

template <typename F>
int timed(RecRun& r, const char* what, F&& f) {
    if (!r.phases) return f();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, r.c->stream);
    const int rc = f();
    cudaEventRecord(b, r.c->stream);
    (*r.phases)[what].ev.push_back({a, b});
    return rc;
}

int rec_decompose(RecRun& r, size_t c0, size_t c1) {
    // tall leaves are update-bound (the trailing update streams rows x remaining
    // leaf columns per panel), so they are narrower than short, chain-bound ones
    const size_t rows0 = r.n - std::min(r.n, 64 * c0);  // rows below the leaf's first panel at full rank
    size_t leaf = (r.tall_rows && rows0 >= r.tall_rows) ? std::min(r.base, r.tall_base) : r.base;
    // with a download hook (the host entry), leaves on the right spine are narrow so
    // the final row blocks go back to the host while the last panels are factored
    if (r.on_final && c1 == r.mu && r.final_base) leaf = std::min(leaf, r.final_base);
    // and on the left spine the first leaf is one upload chunk, so the factorisation
    // starts after that chunk's copy instead of a whole tall leaf's
    if (r.on_final && c0 == 0 && r.first_base) leaf = std::min(leaf, r.first_base);
    if (c1 - c0 <= leaf) return timed(r, "leaf", [&] { return rec_leaf(r, c0, c1); });
    const size_t cm = c0 + (c1 - c0) / 2;
    F2_TRY(rec_decompose(r, c0, cm));
    // (R_j, r_j) of the left half in one read-back (one stream sync per split)
    std::vector<uint32_t> Rr(2 * (cm - c0));
    CUDA_TRY(cudaStreamSynchronize(r.c->stream));
    CUDA_TRY(cudaMemcpy2D(Rr.data(), 8, r.s->st + c0, kStateBytes, 8, cm - c0, cudaMemcpyDeviceToHost));
    const size_t R0 = Rr[0], R1 = size_t(Rr[2 * (cm - c0 - 1)]) + Rr[2 * (cm - c0 - 1) + 1];
    // cf: the left half's full-rank prefix [c0, cf) (r_j = 64, pivot rows 64-aligned):
    // its panels reach the right half as X = L11^-1 C and A' = D ^ L21 X; the panels
    // after it (rank-deficient inputs only) as rank-r_j updates, zero-rank ones skipped
    size_t cf = c0;
    if (R0 % 64 == 0)
        while (cf < cm && Rr[2 * (cf - c0) + 1] == 64) ++cf;
    const bool full = cf == cm;
    const size_t Rf = R0 + 64 * (cf - c0);
    F2_TRY(ensure_cols(r, c1));
    if (cf > c0) {
        F2_TRY(timed(r, "trsm", [&] { return rec_trsm(r, c0, cf, R0, cm, c1); }));
        // rows [0, R1) are final once the TRSM is done (the product writes rows >= R1
        // only), so their download overlaps the product too
        if (full && c1 == r.mu && r.on_final) F2_TRY(r.on_final(R1));
        if (Rf < r.n)
            F2_TRY(timed(r, "product", [&] {
                return best_product(r.c, wview(*r.s, Rf, r.n - Rf, cm, c1 - cm),
                                    wview(*r.s, Rf, r.n - Rf, c0, cf - c0),
                                    wview(*r.s, R0, Rf - R0, cm, c1 - cm), r.cut, r.tc_cut);
            }));
    }
    if (!full) {
        for (size_t j = cf; j < cm; ++j)
            if (Rr[2 * (j - c0) + 1] != 0) F2_TRY(rank_updates(r, j, j + 1, cm, c1, r.n));
        if (c1 == r.mu && r.on_final) F2_TRY(r.on_final(R1));
        // a rank-deficient left half: when what is left of the right half is all zero
        // (or no rows are left), its panels have rank 0 and no swaps -- skip the chain
        bool zero = R1 >= r.n;
        if (!zero) {
            f2gpu_ctx* c = r.c;
            if (!c->zero_flag) CUDA_TRY(cudaMalloc(&c->zero_flag, 4));
            CUDA_TRY(cudaMemsetAsync(c->zero_flag, 0, 4, c->stream));
            F2_TRY(check_launch(c, f2::launch_any_nonzero(r.s->w.p + cm * r.s->w.stride, r.s->w.stride, R1, r.n,
                                                          c1 - cm, c->zero_flag, c->num_sms, c->stream),
                                "k_any_nonzero"));
            uint32_t nz = 1;
            CUDA_TRY(cudaMemcpyAsync(&nz, c->zero_flag, 4, cudaMemcpyDeviceToHost, c->stream));
            CUDA_TRY(cudaStreamSynchronize(c->stream));
            zero = nz == 0;
        }
        if (zero)
            return check_launch(r.c, f2::launch_fill_zero_states(r.s->st, int(cm), int(c1), uint32_t(std::min(R1, r.n)),
                                                                 r.c->stream),
                                "k_fill_zero_states");
    }
    return rec_decompose(r, cm, c1);
}

int decompose_recursive(f2gpu_ctx* c, View w, size_t min_cols, uint32_t* perm, uint32_t* rj,
                        size_t* rank, size_t frontier = size_t(-1), const uint64_t* pend = nullptr,
                        size_t ps = 0, size_t chunk = 0, std::function<int(size_t)> on_final = {}) {
    const size_t n = w.rows, mu = w.wcols();
    if (n == 0 || mu == 0) {
        if (rank) *rank = 0;
        if (rj) std::fill(rj, rj + mu, 0u);
        if (perm) for (size_t i = 0; i < n; ++i) perm[i] = uint32_t(i);
        return F2GPU_OK;
    }
    F2_TRY(ensure_scratch(c, n, mu));
    Shard s;
    s.w = w; s.lw = mu; s.st = static_cast<f2::PanelState*>(c->scr_st); s.perm = c->scr_perm;
    // defaults from a sweep at 65536^2 with the fp4 tensor-core products (leaves
    // 2048..32768 columns x TRSM base 4..64 panels): 16384-column leaves, base 16
    // -> 87.6 ms (8192: 93.4, 32768: 88.9), see DESIGN.md
    RecRun r{c, &s, n, mu, std::max<size_t>(1, (min_cols ? min_cols : 256 * 64) / 64),
             lookahead_ok(c, s, n), 16384, 16};
    const f2::Options& o = f2::options();
    r.cut = size_t(o.rec_cut);
    if (o.rec_base_set) r.base = std::max<size_t>(1, size_t(o.rec_base));
    r.tbase = std::max<size_t>(1, size_t(o.rec_tbase));  // > trsm_max_panels(): rank-64 updates below
    r.trsm_kernel = o.rec_trsm != 0;
    // tall leaves: 128 panels once a leaf has >= 20000 rows below its first panel
    // (65536^2 sweeps over 12000..56000 rows x 32..128 panels; first 70.5 -> 67.5 ms
    // with 64 panels, re-swept after the panel-chain work: 128 panels 64.3 ms,
    // 64: 64.6, 32: 66.3)
    r.tall_rows = size_t(o.rec_tall);
    r.tall_base = std::max<size_t>(1, size_t(o.rec_tall_base));
    if (!r.c->use_tc_cut_default) r.tc_cut = r.c->tc_cutover;  // set explicitly (F2GPU_TC_CUT / ctx_set_tc)
    if (o.rec_tc_cut_set || r.c->use_tc_cut_default) r.tc_cut = size_t(o.rec_tc_cut);
    r.final_base = size_t(o.rec_final);
    r.trsm_m4rm_k = size_t(o.trsm_m4rm_k);
    r.on_final = std::move(on_final);
    if (pend && frontier < mu) {
        r.frontier = r.frontier0 = frontier;
        r.pend = pend;
        r.ps = ps;
        r.chunk = chunk;
        if (r.on_final) r.first_base = chunk;
    }
    CUDA_TRY(cudaMemsetAsync(c->scr_flags, 0, mu * 4 * kFlagsPerPanel, c->stream));
    c->tl.mark(c->stream, "start");
    F2_TRY(check_launch(c, f2::launch_iota(s.perm, n, c->stream), "k_iota"));
    std::map<std::string, RecRun::Phase> phases;
    if (f2::options().rec_times) r.phases = &phases;
    F2_TRY(rec_decompose(r, 0, mu));
    if (r.phases) {
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        float tot = 0;
        for (auto& [name, ph] : phases) {
            float sum = 0;
            for (auto& [a, b] : ph.ev) {
                float ms = 0;
                cudaEventElapsedTime(&ms, a, b);
                sum += ms;
                cudaEventDestroy(a);
                cudaEventDestroy(b);
            }
            tot += sum;
            fprintf(stderr, "[rec] %-8s %4zu x  %8.3f ms\n", name.c_str(), ph.ev.size(), sum);
        }
        fprintf(stderr, "[rec] total    %8.3f ms (phases on the main stream)\n", tot);
    }
    c->tl.report("decompose_recursive");
    return read_results(c, s, n, mu, perm, rj, rank);
}

int decompose_single(f2gpu_ctx* c, View w, uint32_t* perm, uint32_t* rj, size_t* rank) {
    const size_t n = w.rows, mu = w.wcols();
    if (n == 0 || mu == 0) {
        if (rank) *rank = 0;
        if (rj) std::fill(rj, rj + mu, 0u);
        if (perm) for (size_t i = 0; i < n; ++i) perm[i] = uint32_t(i);
        return F2GPU_OK;
    }
    F2_TRY(ensure_scratch(c, n, mu));
    Shard s;
    s.w = w; s.lw = mu; s.st = static_cast<f2::PanelState*>(c->scr_st); s.perm = c->scr_perm;
    GraphCache& g = c->graph;
    const bool graphs = c->use_graphs && c->graphs_stream_ok && !c->tl.on;
    auto launch = [&]() {
        // the counters are zeroed here, not in the graph (enqueue_lookahead)
        CUDA_TRY(cudaMemsetAsync(c->scr_flags, 0, mu * 4 * kFlagsPerPanel, c->stream));
        if (g.has_chain) F2_TRY(chain_fork(c, g.chain));
        CUDA_TRY(cudaGraphLaunch(g.exec, c->stream));
        if (g.has_chain) F2_TRY(chain_join(c));
        return int(F2GPU_OK);
    };
    if (graphs && g.match(w.p, w.stride, n, mu, s.st) && g.exec) {
        F2_TRY(launch());
        c->launches += g.nodes;
    } else if (graphs && g.match(w.p, w.stride, n, mu, s.st) && g.seen >= 1) {
        // second run with this key: capture the launch sequence once, then replay
        cudaGraph_t graph = nullptr;
        const uint64_t l0 = c->launches;
        ChainDefer cd;
        CUDA_TRY(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        int rc = enqueue_single(c, s, n, mu, &cd);
        cudaError_t ec = cudaStreamEndCapture(c->stream, &graph);
        if (rc != F2GPU_OK) { if (graph) cudaGraphDestroy(graph); return rc; }
        if (ec != cudaSuccess) return set_err(F2GPU_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ec));
        cudaError_t ei = cudaGraphInstantiate(&g.exec, graph, 0);
        cudaGraphDestroy(graph);
        if (ei != cudaSuccess) { g.exec = nullptr; return set_err(F2GPU_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(ei)); }
        g.nodes = c->launches - l0;
        g.has_chain = cd.has;
        g.chain = cd.args;
        F2_TRY(launch());
    } else {
        if (graphs) {
            if (!g.match(w.p, w.stride, n, mu, s.st)) {
                g.reset();
                g.w = w.p; g.stride = w.stride; g.n = n; g.mu = mu; g.st = s.st;
            }
            g.seen += 1;
        }
        c->tl.mark(c->stream, "start");
        F2_TRY(enqueue_single(c, s, n, mu));
        c->tl.report("decompose_single");
    }
    return read_results(c, s, n, mu, perm, rj, rank);
}

// Broadcast hook: copies the owner's {state j, panel column} into every
// shard's landing buffer.  Virtual shards: device-to-device copies; NCCL: one
// ncclBroadcast of the header + column from the owner rank.
struct Exchange {
    virtual ~Exchange() = default;
    virtual int bcast(f2gpu_ctx* c, std::vector<Shard>& sh, int owner_local, int owner_global,
                      size_t n) = 0;
    // decompose_recursive: replicate panel j's state and its column rows [row_lo, n)
    // from the owner (local column lj) into every other shard's st[j] / land
    virtual int panel(f2gpu_ctx* c, std::vector<Shard>& sh, int owner_local, int owner_global, size_t j,
                      size_t lj, size_t row_lo, size_t n) = 0;
    // replicate global word-columns [c0, cm), rows [row_lo, n), into Lg (column
    // q - c0 of Lg holds global column q); shards hold columns round-robin
    virtual int gather(f2gpu_ctx* c, std::vector<Shard>& sh, int base, int G, size_t c0, size_t cm, size_t row_lo,
                       size_t n, View Lg) = 0;
};

// word-columns with global index < q owned by shard g of G (round-robin)
size_t lidx(int g, int G, size_t q) { return q <= size_t(g) ? 0 : (q - size_t(g) - 1) / size_t(G) + 1; }

struct LocalExchange : Exchange {
    int bcast(f2gpu_ctx* c, std::vector<Shard>& sh, int owner, int, size_t n) override {
        const size_t bytes = kBcastHdr + n * 8;
        for (size_t g = 0; g < sh.size(); ++g) {
            if (int(g) == owner) continue;
            CUDA_TRY(cudaMemcpyAsync(sh[g].bcast, sh[owner].bcast, bytes,
                                     cudaMemcpyDeviceToDevice, c->stream));
        }
        return F2GPU_OK;
    }
    int panel(f2gpu_ctx* c, std::vector<Shard>& sh, int owner, int, size_t j, size_t lj, size_t row_lo,
              size_t n) override {
        const Shard& o = sh[owner];
        for (size_t g = 0; g < sh.size(); ++g) {
            if (int(g) == owner) continue;
            CUDA_TRY(cudaMemcpyAsync(sh[g].st + j, o.st + j, kStateBytes, cudaMemcpyDeviceToDevice, c->stream));
            if (row_lo < n)
                CUDA_TRY(cudaMemcpyAsync(sh[g].land + row_lo, o.w.p + lj * o.w.stride + row_lo, (n - row_lo) * 8,
                                         cudaMemcpyDeviceToDevice, c->stream));
        }
        return F2GPU_OK;
    }
    int gather(f2gpu_ctx* c, std::vector<Shard>& sh, int base, int G, size_t c0, size_t cm, size_t row_lo,
               size_t n, View Lg) override {
        if (row_lo >= n) return F2GPU_OK;
        for (size_t i = 0; i < sh.size(); ++i) {
            const int g = base + int(i);
            const size_t l0 = lidx(g, G, c0), l1 = lidx(g, G, cm);
            if (l0 >= l1) continue;
            const size_t q0 = size_t(g) + l0 * size_t(G) - c0;  // Lg column of local column l0
            CUDA_TRY(cudaMemcpy2DAsync(Lg.p + q0 * Lg.stride + row_lo, size_t(G) * Lg.stride * 8,
                                       sh[i].w.p + l0 * sh[i].w.stride + row_lo, sh[i].w.stride * 8,
                                       (n - row_lo) * 8, l1 - l0, cudaMemcpyDeviceToDevice, c->stream));
        }
        return F2GPU_OK;
    }
};

int nccl_rc(int rc, const char* what) {
    if (rc == 0) return F2GPU_OK;
    NcclApi& api = nccl();
    return set_err(F2GPU_ENCCL, std::string(what) + ": " + (api.getErrorString ? api.getErrorString(rc) : "?"));
}

struct NcclExchange : Exchange {
    std::deque<DevBuf> scratch;  // gather staging (grown on demand)
    void* stage = nullptr;
    size_t stage_bytes = 0;
    int bcast(f2gpu_ctx* c, std::vector<Shard>& sh, int, int owner_global, size_t n) override {
        NcclApi& api = nccl();
        const size_t bytes = kBcastHdr + n * 8;
        return nccl_rc(api.broadcast(sh[0].bcast, sh[0].bcast, bytes, kNcclUint8, owner_global, c->comm, c->stream),
                       "ncclBroadcast");
    }
    // one grouped launch: the state (root: its st[j]) and the column rows
    // [row_lo, n) (root: straight from its W) -- (n - row_lo) * 8 + 1.5 KiB bytes
    int panel(f2gpu_ctx* c, std::vector<Shard>& sh, int owner_local, int owner_global, size_t j, size_t lj,
              size_t row_lo, size_t n) override {
        NcclApi& api = nccl();
        Shard& s = sh[0];
        const bool root = owner_local == 0;
        F2_TRY(nccl_rc(api.groupStart(), "ncclGroupStart"));
        int rc = api.broadcast(s.st + j, s.st + j, kStateBytes, kNcclUint8, owner_global, c->comm, c->stream);
        if (rc == 0 && row_lo < n)
            rc = api.broadcast(root ? static_cast<const void*>(s.w.p + lj * s.w.stride + row_lo)
                                    : static_cast<const void*>(s.land + row_lo),
                               s.land + row_lo, (n - row_lo) * 8, kNcclUint8, owner_global, c->comm, c->stream);
        const int re = api.groupEnd();
        F2_TRY(nccl_rc(rc, "ncclBroadcast(panel)"));
        return nccl_rc(re, "ncclGroupEnd");
    }
    // every rank broadcasts its packed block of the left columns (G broadcasts in
    // one group), then scatters the blocks into Lg
    int gather(f2gpu_ctx* c, std::vector<Shard>& sh, int base, int G, size_t c0, size_t cm, size_t row_lo,
               size_t n, View Lg) override {
        if (row_lo >= n) return F2GPU_OK;
        NcclApi& api = nccl();
        const size_t rows = n - row_lo;
        std::vector<size_t> off(size_t(G) + 1, 0);
        for (int g = 0; g < G; ++g) off[g + 1] = off[g] + (lidx(g, G, cm) - lidx(g, G, c0)) * rows;
        if (off[G] == 0) return F2GPU_OK;
        if (stage_bytes < off[G] * 8) {
            scratch.clear();
            scratch.emplace_back(c);
            F2_TRY(scratch.back().alloc(off[G] * 8));
            stage = scratch.back().p;
            stage_bytes = off[G] * 8;
        }
        uint64_t* st = static_cast<uint64_t*>(stage);
        const Shard& me = sh[0];
        const size_t l0 = lidx(base, G, c0), l1 = lidx(base, G, cm);
        if (l1 > l0)
            CUDA_TRY(cudaMemcpy2DAsync(st + off[base], rows * 8, me.w.p + l0 * me.w.stride + row_lo, me.w.stride * 8,
                                       rows * 8, l1 - l0, cudaMemcpyDeviceToDevice, c->stream));
        F2_TRY(nccl_rc(api.groupStart(), "ncclGroupStart"));
        int rc = 0;
        for (int g = 0; g < G && rc == 0; ++g)
            if (off[g + 1] > off[g])
                rc = api.broadcast(st + off[g], st + off[g], (off[g + 1] - off[g]) * 8, kNcclUint8, g, c->comm,
                                   c->stream);
        const int re = api.groupEnd();
        F2_TRY(nccl_rc(rc, "ncclBroadcast(gather)"));
        F2_TRY(nccl_rc(re, "ncclGroupEnd"));
        for (int g = 0; g < G; ++g) {
            const size_t a = lidx(g, G, c0), b = lidx(g, G, cm);
            if (a >= b) continue;
            const size_t q0 = size_t(g) + a * size_t(G) - c0;
            CUDA_TRY(cudaMemcpy2DAsync(Lg.p + q0 * Lg.stride + row_lo, size_t(G) * Lg.stride * 8, st + off[g],
                                       rows * 8, rows * 8, b - a, cudaMemcpyDeviceToDevice, c->stream));
        }
        return F2GPU_OK;
    }
};

// Sharded driver. `sh` holds the shards living in this process; global shard
// index of sh[i] is shard_base + i; G = total shards.
int decompose_sharded(f2gpu_ctx* c, std::vector<Shard>& sh, int shard_base, int G, size_t n,
                      size_t mu, Exchange& ex) {
    for (auto& s : sh) F2_TRY(check_launch(c, f2::launch_iota(s.perm, n, c->stream), "k_iota"));
    for (size_t j = 0; j < mu; ++j) {
        const int owner = int(j % size_t(G));
        const size_t lj = j / size_t(G);
        const int ol = owner - shard_base;  // local index of the owner (may be out of range)
        const bool have_owner = ol >= 0 && ol < int(sh.size());
        if (have_owner) {
            Shard& o = sh[ol];
            uint64_t* colj = o.w.p + lj * o.w.stride;
            F2_TRY(check_launch(c, f2::launch_panel(colj, n, o.st, int(j), c->stream), "k_panel"));
            F2_TRY(check_launch(c, f2::launch_post(o.w.p, o.w.stride, int(o.lw), int(lj), o.perm,
                                                   n, o.st + j, c->stream),
                                "k_post"));
            CUDA_TRY(cudaMemcpyAsync(o.bcast, o.st + j, kStateBytes, cudaMemcpyDeviceToDevice,
                                     c->stream));
            CUDA_TRY(cudaMemcpyAsync(o.bcast + kBcastHdr / 8, colj, n * 8,
                                     cudaMemcpyDeviceToDevice, c->stream));
        }
        F2_TRY(ex.bcast(c, sh, ol, owner, n));
        for (size_t g = 0; g < sh.size(); ++g) {
            Shard& s = sh[g];
            const int gg = shard_base + int(g);
            const f2::PanelState* stj = s.st + j;
            if (gg != owner) {
                CUDA_TRY(cudaMemcpyAsync(s.st + j, s.bcast, kStateBytes, cudaMemcpyDeviceToDevice,
                                         c->stream));
                F2_TRY(check_launch(c, f2::launch_swaps(s.w.p, s.w.stride, int(s.lw), -1, s.perm,
                                                        stj, c->stream),
                                    "k_swaps"));
            }
            const size_t l0 = first_local_after(j, gg, G);
            if (l0 < s.lw) {
                f2::UpdateArgs u{};
                u.C = s.w.p; u.sc = s.w.stride; u.c_wcol0 = l0; u.ncols = int(s.lw - l0);
                u.row_lo = 0; u.row_hi = n;
                u.a = (gg == owner) ? s.w.p + lj * s.w.stride : s.bcast + kBcastHdr / 8;
                u.B = s.w.p; u.sb = s.w.stride; u.b_wcol0 = l0;
                u.st = stj;
                F2_TRY(check_launch(c, f2::launch_update(u, c->num_sms, c->stream), "k_update"));
            }
        }
    }
    return F2GPU_OK;
}

int alloc_shard_aux(f2gpu_ctx* c, Shard& s, size_t n, size_t mu, std::deque<DevBuf>& keep) {
    keep.emplace_back(c);
    F2_TRY(keep.back().alloc(mu * kStateBytes));
    s.st = keep.back().as<f2::PanelState>();
    keep.emplace_back(c);
    F2_TRY(keep.back().alloc(n * 4));
    s.perm = keep.back().as<uint32_t>();
    keep.emplace_back(c);
    // landing column padded to the full stride (the bulk-copy update reads
    // 128-row segments of it) and zeroed once; broadcasts fill rows < n
    F2_TRY(keep.back().alloc(kBcastHdr + s.w.stride * 8));
    s.bcast = keep.back().as<uint64_t>();
    CUDA_TRY(cudaMemsetAsync(s.bcast, 0, kBcastHdr + s.w.stride * 8, c->stream));
    keep.emplace_back(c);
    F2_TRY(keep.back().alloc(s.w.stride * 8));
    s.land = keep.back().as<uint64_t>();
    CUDA_TRY(cudaMemsetAsync(s.land, 0, s.w.stride * 8, c->stream));
    return F2GPU_OK;
}

// ---- decompose_recursive over column shards ----
// The recursion's control flow is host-only and separate from the work it
// orders, so the GPU drivers below and the CPU protocol test
// (tests/test_dist_gloo.py through f2gpu_dist_schedule) run the SAME schedule:
//   leaf [c0, c1): per panel j, its owner (j mod G) factors it and the state +
//     column rows [R_lb, n) are replicated (R_lb <= R_j: the leaf's first R,
//     known on the host); every rank applies the row swaps and the Schur update
//     to its own columns in (j, c1);
//   split at cm: left half recursively; R0 / R1 read back; the left columns
//     rows [R0, n) replicated once (one gather per split); full rank -> every
//     rank solves X = L11^-1 C on its own right-half columns and forms
//     A' = D ^ L21 X on them (one product sharded by output word-columns, no
//     further exchange); otherwise the left panels are applied as rank-r_j
//     updates; then the right half.
int dist_schedule(size_t n, size_t mu, int world, size_t base, size_t tall_rows, size_t tall_base,
                  const f2gpu_dist_ops* o) {
    std::function<int(size_t, size_t, size_t)> rec = [&](size_t c0, size_t c1, size_t rlb) -> int {
        const size_t rows0 = n - std::min(n, 64 * c0);
        const size_t leaf = (tall_rows && rows0 >= tall_rows) ? std::min(base, tall_base) : base;
        if (c1 - c0 <= leaf && o->leaf) return o->leaf(o->user, c0, c1, rlb);
        if (c1 - c0 <= leaf) {
            for (size_t j = c0; j < c1; ++j) {
                const int owner = int(j % size_t(world));
                F2_TRY(o->panel(o->user, j, owner, rlb));
                F2_TRY(o->apply(o->user, j, owner, j + 1, c1));
            }
            return F2GPU_OK;
        }
        const size_t cm = c0 + (c1 - c0) / 2;
        F2_TRY(rec(c0, cm, rlb));
        size_t R0 = 0, r0 = 0, Rl = 0, rl = 0;
        F2_TRY(o->state(o->user, c0, &R0, &r0));
        F2_TRY(o->state(o->user, cm - 1, &Rl, &rl));
        const size_t R1 = Rl + rl;
        const bool full = R1 - R0 == 64 * (cm - c0) && R0 % 64 == 0;
        F2_TRY(o->gather(o->user, c0, cm, R0));
        if (full) {
            F2_TRY(o->solve(o->user, c0, cm, R0, cm, c1));
            if (R1 < n) F2_TRY(o->product(o->user, c0, cm, R0, R1, cm, c1));
        } else {
            F2_TRY(o->rank_update(o->user, c0, cm, cm, c1));
        }
        return rec(cm, c1, R1);
    };
    if (n == 0 || mu == 0) return F2GPU_OK;
    return rec(0, mu, 0);
}

// The GPU side of the schedule: shards sh (global index base + i of G), Lg = the
// replicated left columns of the current split (full n rows, one per process).
struct DistGpu {
    f2gpu_ctx* c = nullptr;
    std::vector<Shard>* sh = nullptr;
    int base = 0, G = 1;
    size_t n = 0, mu = 0;
    Exchange* ex = nullptr;
    View Lg{};
    std::deque<DevBuf> lg_keep;
    size_t lg_cols = 0;
    size_t tbase = 16, trsm_m4rm_k = 1024, cut = 16384, tc_cut = 8192;
    // whole-leaf mode: the leaf last factored on the gathered copy [lf_c0, lf_c1) (rows
    // >= lf_row valid); a split whose left half is exactly that leaf reuses it as Lg
    size_t lf_c0 = 0, lf_c1 = 0, lf_row = 0;
    bool lf_valid = false;
    bool whole_leaf = true;

    static DistGpu& of(void* u) { return *static_cast<DistGpu*>(u); }
    // Whole-leaf mode (default): a leaf is the latency-bound panel chain, which G GPUs
    // cannot speed up; replicating each panel (one NCCL launch on the chain per panel)
    // only slows it.  So the leaf's columns, rows [row_lo, n), are replicated ONCE
    // (the split's own gather primitive), every process factors the leaf on its copy
    // with the single-GPU schedule (fused lookahead, CUDA-graph replay) -- the kernels
    // are deterministic, so every copy, state and perm comes out identical with no
    // further exchange -- and then takes its own columns back and applies the leaf's
    // row swaps to its other columns in one launch.  Per-leaf traffic: (n - row_lo) x
    // leaf columns words; over a whole decomposition about half the matrix.
    static int leaf(void* u, size_t c0, size_t c1, size_t row_lo) {
        DistGpu& d = of(u);
        f2gpu_ctx* c = d.c;
        const size_t cols = c1 - c0, gs = dev_stride(d.n);
        if (c->leafbuf_words < gs * cols) {
            CUDA_TRY(cudaStreamSynchronize(c->stream));
            c->leaf_graphs.clear();  // graphs hold the old pointer
            cudaFree(c->leafbuf);
            c->leafbuf = nullptr;
            c->leafbuf_words = 0;
            CUDA_TRY(cudaMalloc(&c->leafbuf, gs * cols * 8));
            c->leafbuf_words = gs * cols;
        }
        const View lv{c->leafbuf, d.n, cols * 64, gs, gs};
        d.lf_valid = false;
        F2_TRY(d.ex->gather(c, *d.sh, d.base, d.G, c0, c1, row_lo, d.n, lv));
        Shard& s0 = (*d.sh)[0];
        Shard lf;
        lf.w = lv; lf.lw = cols; lf.st = s0.st; lf.perm = s0.perm;
        const bool la = lookahead_ok(c, lf, d.n);
        const std::array<uintptr_t, 8> key{uintptr_t(lv.p), gs, d.n, d.mu, c0, c1,
                                           uintptr_t(lf.st) ^ (la ? 1u : 0u), cols | (size_t(1) << 40)};
        F2_TRY(leaf_graph_run(c, key, [&](ChainDefer* cd) {
            return enqueue_panels(c, lf, d.n, d.mu, c0, c1, la, cols, c0, cd);
        }));
        for (size_t i = 0; i < d.sh->size(); ++i) {
            Shard& s = (*d.sh)[i];
            const int gg = d.base + int(i);
            if (i > 0)  // logical shards on one device: the states are factored once
                CUDA_TRY(cudaMemcpyAsync(s.st + c0, s0.st + c0, cols * kStateBytes, cudaMemcpyDeviceToDevice,
                                         c->stream));
            const size_t l0 = lidx(gg, d.G, c0), l1 = lidx(gg, d.G, c1);
            if (l1 > l0 && row_lo < d.n) {
                const size_t q0 = size_t(gg) + l0 * size_t(d.G) - c0;
                CUDA_TRY(cudaMemcpy2DAsync(s.w.p + l0 * s.w.stride + row_lo, s.w.stride * 8,
                                           lv.p + q0 * gs + row_lo, size_t(d.G) * gs * 8, (d.n - row_lo) * 8,
                                           l1 - l0, cudaMemcpyDeviceToDevice, c->stream));
            }
            F2_TRY(check_launch(c, f2::launch_swaps_range(s.w.p, s.w.stride, int(s.lw), int(l0), int(l1),
                                                          i == 0 ? nullptr : s.perm, s.st, int(c0), int(c1),
                                                          c->stream),
                                "k_swaps_range"));
        }
        d.lf_c0 = c0; d.lf_c1 = c1; d.lf_row = row_lo; d.lf_valid = true;
        return F2GPU_OK;
    }
    int local(int owner) const { return owner - base; }  // may be outside [0, sh.size())

    static int panel(void* u, size_t j, int owner, size_t row_lo) {
        DistGpu& d = of(u);
        const int ol = d.local(owner);
        const size_t lj = j / size_t(d.G);
        if (ol >= 0 && ol < int(d.sh->size())) {
            Shard& o = (*d.sh)[size_t(ol)];
            F2_TRY(check_launch(d.c, f2::launch_panel(o.w.p + lj * o.w.stride, d.n, o.st, int(j), d.c->stream),
                                "k_panel"));
            F2_TRY(check_launch(d.c, f2::launch_post(o.w.p, o.w.stride, int(o.lw), int(lj), o.perm, d.n, o.st + j,
                                                     d.c->stream),
                                "k_post"));
        }
        return d.ex->panel(d.c, *d.sh, ol, owner, j, lj, row_lo, d.n);
    }
    static int apply(void* u, size_t j, int owner, size_t col_lo, size_t col_hi) {
        DistGpu& d = of(u);
        for (size_t i = 0; i < d.sh->size(); ++i) {
            Shard& s = (*d.sh)[i];
            const int gg = d.base + int(i);
            if (gg != owner)
                F2_TRY(check_launch(d.c, f2::launch_swaps(s.w.p, s.w.stride, int(s.lw), -1, s.perm, s.st + j,
                                                          d.c->stream),
                                    "k_swaps"));
            const size_t l0 = lidx(gg, d.G, col_lo), l1 = lidx(gg, d.G, col_hi);
            if (l0 >= l1) continue;
            f2::UpdateArgs a{};
            a.C = s.w.p; a.sc = s.w.stride; a.c_wcol0 = l0; a.ncols = int(l1 - l0);
            a.row_lo = 0; a.row_hi = d.n;
            a.a = gg == owner ? s.w.p + (j / size_t(d.G)) * s.w.stride : s.land;
            a.B = s.w.p; a.sb = s.w.stride; a.b_wcol0 = l0;
            a.st = s.st + j;
            F2_TRY(check_launch(d.c, f2::launch_update(a, d.c->num_sms, d.c->stream), "k_update"));
        }
        return F2GPU_OK;
    }
    static int state(void* u, size_t j, size_t* R, size_t* r) {
        DistGpu& d = of(u);
        f2::PanelState h;
        CUDA_TRY(cudaStreamSynchronize(d.c->stream));
        CUDA_TRY(cudaMemcpy(&h, (*d.sh)[0].st + j, 16, cudaMemcpyDeviceToHost));
        *R = h.R;
        *r = h.r;
        return F2GPU_OK;
    }
    static int gather(void* u, size_t c0, size_t cm, size_t row_lo) {
        DistGpu& d = of(u);
        const size_t cols = cm - c0, gs = dev_stride(d.n);
        if (d.lf_valid && d.lf_c0 == c0 && d.lf_c1 == cm && d.lf_row <= row_lo) {
            // the left half is the leaf every process has just factored on its copy
            d.Lg = View{d.c->leafbuf, d.n, cols * 64, gs, gs};
            return F2GPU_OK;
        }
        if (cols > d.lg_cols) {
            d.lg_keep.clear();
            d.lg_keep.emplace_back(d.c);
            F2_TRY(d.lg_keep.back().alloc(gs * cols * 8));
            d.lg_cols = cols;
        }
        d.Lg = View{d.lg_keep.back().as<uint64_t>(), d.n, cols * 64, gs, gs};
        return d.ex->gather(d.c, *d.sh, d.base, d.G, c0, cm, row_lo, d.n, d.Lg);
    }
    // X = L11^-1 C on shard s's word-columns [l0, l1), panels [a, b) of the split
    // starting at c0 (L from Lg), rows [Ra, Ra + 64 (b - a))
    int trsm(Shard& s, size_t l0, size_t l1, size_t c0, size_t a, size_t b, size_t Ra) {
        const size_t nc = l1 - l0;
        if (b - a <= tbase)
            return check_launch(c, f2::launch_trsm_block_l(Lg.p + (a - c0) * Lg.stride + Ra, Lg.stride,
                                                           s.w.p + l0 * s.w.stride + Ra, s.w.stride, int(b - a),
                                                           int(nc), c->stream),
                                "k_trsm_block");
        const size_t m = a + (b - a) / 2, Rm = Ra + 64 * (m - a), Rb = Ra + 64 * (b - a);
        F2_TRY(trsm(s, l0, l1, c0, a, m, Ra));
        const View C = wview(s, Rm, Rb - Rm, l0, nc), A = Lg.sub(Rm, Rb - Rm, a - c0, m - a),
                   B = wview(s, Ra, Rm - Ra, l0, nc);
        if ((m - a) * 64 <= trsm_m4rm_k) F2_TRY(strassen_acc(c, C, A, B, cut));
        else F2_TRY(best_product(c, C, A, B, cut, tc_cut));
        return trsm(s, l0, l1, c0, m, b, Rm);
    }
    static int solve(void* u, size_t c0, size_t cm, size_t R0, size_t col_lo, size_t col_hi) {
        DistGpu& d = of(u);
        for (size_t i = 0; i < d.sh->size(); ++i) {
            const int gg = d.base + int(i);
            const size_t l0 = lidx(gg, d.G, col_lo), l1 = lidx(gg, d.G, col_hi);
            if (l0 < l1) F2_TRY(d.trsm((*d.sh)[i], l0, l1, c0, c0, cm, R0));
        }
        return F2GPU_OK;
    }
    static int product(void* u, size_t c0, size_t cm, size_t R0, size_t R1, size_t col_lo, size_t col_hi) {
        DistGpu& d = of(u);
        for (size_t i = 0; i < d.sh->size(); ++i) {
            Shard& s = (*d.sh)[i];
            const int gg = d.base + int(i);
            const size_t l0 = lidx(gg, d.G, col_lo), l1 = lidx(gg, d.G, col_hi);
            if (l0 >= l1) continue;
            F2_TRY(best_product(d.c, wview(s, R1, d.n - R1, l0, l1 - l0), d.Lg.sub(R1, d.n - R1, 0, cm - c0),
                                wview(s, R0, R1 - R0, l0, l1 - l0), d.cut, d.tc_cut));
        }
        return F2GPU_OK;
    }
    static int rank_update(void* u, size_t c0, size_t cm, size_t col_lo, size_t col_hi) {
        DistGpu& d = of(u);
        for (size_t i = 0; i < d.sh->size(); ++i) {
            Shard& s = (*d.sh)[i];
            const int gg = d.base + int(i);
            const size_t l0 = lidx(gg, d.G, col_lo), l1 = lidx(gg, d.G, col_hi);
            if (l0 >= l1) continue;
            for (size_t j = c0; j < cm; ++j) {
                f2::UpdateArgs a{};
                a.C = s.w.p; a.sc = s.w.stride; a.c_wcol0 = l0; a.ncols = int(l1 - l0);
                a.row_lo = 0; a.row_hi = d.n; a.a = d.Lg.p + (j - c0) * d.Lg.stride;
                a.B = s.w.p; a.sb = s.w.stride; a.b_wcol0 = l0;
                a.st = s.st + j;
                F2_TRY(check_launch(d.c, f2::launch_update(a, d.c->num_sms, d.c->stream), "k_update"));
            }
        }
        return F2GPU_OK;
    }
    f2gpu_dist_ops ops() {
        f2gpu_dist_ops o{};
        o.user = this;
        o.panel = &DistGpu::panel;
        o.apply = &DistGpu::apply;
        o.state = &DistGpu::state;
        o.gather = &DistGpu::gather;
        o.solve = &DistGpu::solve;
        o.product = &DistGpu::product;
        o.rank_update = &DistGpu::rank_update;
        if (whole_leaf) o.leaf = &DistGpu::leaf;
        return o;
    }
};

// leaf geometry shared with the single-GPU recursion (decompose_recursive)
void rec_leaf_params(size_t min_cols, size_t* base, size_t* tall_rows, size_t* tall_base) {
    *base = std::max<size_t>(1, (min_cols ? min_cols : 256 * 64) / 64);
    const f2::Options& o = f2::options();
    *tall_rows = size_t(o.rec_tall);
    *tall_base = std::max<size_t>(1, size_t(o.rec_tall_base));
    if (o.rec_base_set) *base = std::max<size_t>(1, size_t(o.rec_base));
}

int run_dist_recursive(f2gpu_ctx* c, std::vector<Shard>& sh, int base, int G, size_t n, size_t mu, size_t min_cols,
                       Exchange& ex) {
    DistGpu d;
    d.c = c; d.sh = &sh; d.base = base; d.G = G; d.n = n; d.mu = mu; d.ex = &ex;
    d.whole_leaf = f2::options().dist_leaf != 0;
    if (d.whole_leaf) {
        // the leaves replay captured graphs: their state array, perm and counters are
        // the context's persistent ones (stable addresses across calls)
        F2_TRY(ensure_scratch(c, n, mu));
        sh[0].st = static_cast<f2::PanelState*>(c->scr_st);
        sh[0].perm = c->scr_perm;
        CUDA_TRY(cudaMemsetAsync(c->scr_flags, 0, mu * 4 * kFlagsPerPanel, c->stream));
    }
    for (auto& s : sh) F2_TRY(check_launch(c, f2::launch_iota(s.perm, n, c->stream), "k_iota"));
    {  // the single-GPU recursion's TRSM base and product cutovers (options.h)
        const f2::Options& o = f2::options();
        d.tbase = std::min<size_t>(size_t(f2::trsm_max_panels()), std::max<size_t>(1, size_t(o.rec_tbase)));
        d.trsm_m4rm_k = size_t(o.trsm_m4rm_k);
        d.cut = size_t(o.rec_cut);
        d.tc_cut = size_t(o.rec_tc_cut);
    }
    if (!c->use_tc_cut_default) d.tc_cut = c->tc_cutover;
    size_t lb = 0, tr = 0, tb = 0;
    rec_leaf_params(min_cols, &lb, &tr, &tb);
    const f2gpu_dist_ops o = d.ops();
    return dist_schedule(n, mu, G, lb, tr, tb, &o);
}

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================
extern "C" {

const char* f2gpu_last_error(void) { return g_err.c_str(); }
const char* f2gpu_version(void) {
#if F2GPU_EXPERIMENTAL
    return F2GPU_VERSION " sm_100a +experimental";
#else
    return F2GPU_VERSION " sm_100a";
#endif
}

int f2gpu_options_describe(char* buf, size_t cap, size_t* len) {
    std::string t;
    const f2::Options& o = f2::options();
    char line[512];
#define F2_OPT_DESC(field, env, def, doc)                                                                  \
    snprintf(line, sizeof line, "%-24s %8lld%s  (default %lld)  %s\n", env, o.field, o.field##_set ? "*" : " ", \
             (long long)(def), doc);                                                                       \
    t += line;
    F2_OPTIONS(F2_OPT_DESC)
#undef F2_OPT_DESC
    if (len) *len = t.size();
    if (buf && cap) {
        const size_t k = std::min(cap - 1, t.size());
        memcpy(buf, t.data(), k);
        buf[k] = 0;
    }
    return F2GPU_OK;
}

int f2gpu_ctx_create(int device, f2gpu_ctx** out) {
    if (!out) return set_err(F2GPU_EINVAL, "ctx_create: null out");
    *out = nullptr;
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return set_err(F2GPU_ERANGE, "ctx_create: device index");
    CUDA_TRY(cudaSetDevice(device));
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return set_err(F2GPU_ECUDA, std::string("libf2gpu is built for sm_100a (B200); device is ") +
                                        prop.name);
    auto c = std::make_unique<f2gpu_ctx>();
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    {
        // scratch (B^T, Strassen arenas, broadcast buffers) comes from the stream-
        // ordered pool; keep freed blocks cached instead of returning them to the
        // OS at every synchronisation (release threshold 0 made each large scratch
        // allocation a fresh OS allocation inside the decomposition)
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t keep = ~uint64_t(0);
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    }
    {  // the schedule switches (options.h)
        const f2::Options& o = f2::options();
        c->tl.on = o.profile != 0;
        c->use_graphs = o.graphs != 0;
        c->lookahead = o.lookahead != 0;
        c->lookahead_col = o.lookahead_col != 0;
        c->fuse_post = o.postcol != 0;
        c->panel_early = o.panel_early != 0;
        c->poll_ns = uint32_t(std::max<long long>(0, o.poll_ns));
        c->u_first_col = o.u_firstcol != 0;
        c->u_fc_ctas = int(o.u_fc_ctas);
        c->u_fc_ctas_set = o.u_fc_ctas_set;
        c->u_fc_w_set = o.u_fc_w_set;
        c->u_fc_weight = int(std::max<long long>(1, std::min<long long>(4, o.u_fc_w)));
        c->panel_head = o.panel_head != 0;
        c->post_spin = o.post_spin != 0;
        c->pdl = o.pdl != 0;
        c->panel_hand = o.panel_hand != 0;
        c->panel_chain = o.panel_chain != 0;
        c->chain_sms = int(o.chain_sms);
        c->use_tc = o.tc != 0;
        if (o.tc_cut_set) {
            c->tc_cutover = size_t(o.tc_cut);
            c->use_tc_cut_default = false;
        }
    }
    if (f2::options().spin_diag && !g_diag) {
        void* h = nullptr;
        CUDA_TRY(cudaHostAlloc(&h, 64, cudaHostAllocMapped));
        memset(h, 0, 64);
        void* d = nullptr;
        CUDA_TRY(cudaHostGetDevicePointer(&d, h, 0));
        CUDA_TRY(f2::spin_diag_set(static_cast<unsigned long long*>(d)));
        g_diag = static_cast<unsigned long long*>(h);
    }
    CUDA_TRY(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&c->side2, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&c->ev_post, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&c->ev_panel2, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&c->ev_panel, cudaEventDisableTiming));
    CUDA_TRY(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
    c->stream = c->own_stream;
    CUDA_TRY(f2::init_kernel_attrs());
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    uint64_t jt[64 * 64];
    f2::host_jump_tables(jt);
    CUDA_TRY(cudaMalloc(&c->d_jump, sizeof(jt)));
    CUDA_TRY(cudaMemcpy(c->d_jump, jt, sizeof(jt), cudaMemcpyHostToDevice));
    *out = c.release();
    return F2GPU_OK;
}

int f2gpu_ctx_destroy(f2gpu_ctx* c) {
    if (!c) return F2GPU_OK;
    cudaSetDevice(c->device);
    if (c->comm && nccl().ok) nccl().commDestroy(c->comm);
    if (c->own_stream) cudaStreamSynchronize(c->own_stream);
    c->graph.reset();
    c->leaf_graphs.clear();
    if (c->side) { cudaStreamSynchronize(c->side); cudaStreamDestroy(c->side); }
    if (c->side2) { cudaStreamSynchronize(c->side2); cudaStreamDestroy(c->side2); }
    if (c->copy) { cudaStreamSynchronize(c->copy); cudaStreamDestroy(c->copy); }
    if (c->stage) { f2gpu_mat_free(c->stage); c->stage = nullptr; }
    cudaFree(c->scr_st);
    cudaFree(c->scr_perm);
    cudaFree(c->scr_flags);
    cudaFree(c->leafbuf);
    cudaFree(c->zero_flag);
    for (auto& e : c->desc_cache) {
        cudaFree(e.d);
        cudaEventDestroy(e.ready);
    }
    cudaFree(c->scr_hand);
    if (c->trace_buf) { f2::trace_set(nullptr, 0); cudaFree(c->trace_buf); }
    for (cudaEvent_t e : c->chunk_ev) cudaEventDestroy(e);
    cudaFree(c->pend);
    if (c->ev_post) cudaEventDestroy(c->ev_post);
    if (c->ev_panel2) cudaEventDestroy(c->ev_panel2);
    if (c->ev_panel) cudaEventDestroy(c->ev_panel);
    cudaFree(c->d_jump);
    if (c->own_stream) cudaStreamDestroy(c->own_stream);
    delete c;
    return F2GPU_OK;
}

int f2gpu_ctx_set_stream(f2gpu_ctx* c, void* s) {
    if (!c) return set_err(F2GPU_EINVAL, "null ctx");
    // F2GPU_OWN_STREAM selects the context's own stream; any other value is a CUDA
    // stream handle, including 0 / cudaStreamLegacy / cudaStreamPerThread (torch's
    // default stream is handle 0).  Stream capture is illegal on those, so the
    // CUDA-graph replay is off while one of them is selected.
    c->stream = s == F2GPU_OWN_STREAM ? c->own_stream : static_cast<cudaStream_t>(s);
    c->graphs_stream_ok = !(c->stream == nullptr || c->stream == cudaStreamLegacy ||
                            c->stream == cudaStreamPerThread);
    return F2GPU_OK;
}

int f2gpu_ctx_sync(f2gpu_ctx* c) {
    if (!c) return set_err(F2GPU_EINVAL, "null ctx");
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return F2GPU_OK;
}

uint64_t f2gpu_ctx_launches(const f2gpu_ctx* c) { return c ? c->launches : 0; }

int f2gpu_ctx_set_strassen_cutover(f2gpu_ctx* c, size_t v) {
    if (!c) return set_err(F2GPU_EINVAL, "null ctx");
    c->strassen_cutover = v ? v : 4096;
    return F2GPU_OK;
}

int f2gpu_ctx_set_tc(f2gpu_ctx* c, int on, size_t leaf) {
    if (!c) return set_err(F2GPU_EINVAL, "null ctx");
    c->use_tc = on != 0;
    c->tc_cutover = leaf ? leaf : 16384;
    c->use_tc_cut_default = leaf == 0;
    return F2GPU_OK;
}

// ---- device trace (diagnostics) ----
int f2gpu_debug_panel_chain(f2gpu_ctx* c, f2gpu_mat* a, size_t ncols) {
    if (!c || !a) return set_err(F2GPU_EINVAL, "debug_panel_chain: null argument");
    const size_t n = a->rows, mu = (a->cols + 63) / 64;
    if (ncols < 2 || ncols > mu) return set_err(F2GPU_ERANGE, "debug_panel_chain: ncols out of range");
    if (!f2::panel_link_ok()) return set_err(F2GPU_EINVAL, "debug_panel_chain: needs the k_panel_gj body");
    F2_TRY(ensure_scratch(c, n, mu));
    // every counter satisfied (waits are >= count or != 0), panel 0 "factored" with rank 0
    CUDA_TRY(cudaMemsetAsync(c->scr_flags, 0x3f, mu * 4 * kFlagsPerPanel, c->stream));
    CUDA_TRY(cudaMemsetAsync(c->scr_st, 0, kStateBytes, c->stream));
    f2::ChainArgs ca{};
    ca.w = a->d; ca.stride = a->stride; ca.n = n; ca.st = static_cast<f2::PanelState*>(c->scr_st);
    ca.flags = c->scr_flags; ca.flags_per_panel = int(kFlagsPerPanel);
    ca.leaf0 = 0; ca.c0 = 1; ca.c1 = int(ncols); ca.coff = 0;
    ca.yblocks = uint32_t(f2::post_col_yblocks(n));
    ca.upd_grid = uint32_t(c->num_sms);
    ca.poll_ns = uint32_t(c->poll_ns);
    ca.trace = false;
    return check_launch(c, f2::launch_panel_chain(ca, c->stream), "k_panel_chain");
}

int f2gpu_trace_enable(f2gpu_ctx* c, size_t cap) {
    if (!c) return set_err(F2GPU_EINVAL, "trace_enable: null ctx");
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    if ((cap != 0) != (c->trace_buf != nullptr)) {  // captured graphs hold the trace switch
        c->graph.reset();
        c->leaf_graphs.clear();
    }
    cudaFree(c->trace_buf);
    c->trace_buf = nullptr;
    c->trace_cap = 0;
    if (cap) {
        CUDA_TRY(cudaMalloc(&c->trace_buf, cap * 8));
        c->trace_cap = cap;
    }
    CUDA_TRY(f2::trace_set(c->trace_buf, uint32_t(c->trace_cap)));
    return F2GPU_OK;
}

int f2gpu_trace_read(f2gpu_ctx* c, uint64_t* out, size_t cap, size_t* n) {
    if (!c || !n) return set_err(F2GPU_EINVAL, "trace_read: null argument");
    CUDA_TRY(cudaDeviceSynchronize());
    uint32_t cnt = 0;
    CUDA_TRY(f2::trace_count(&cnt));
    const size_t k = std::min<size_t>({size_t(cnt), c->trace_cap, cap});
    if (k) CUDA_TRY(cudaMemcpy(out, c->trace_buf, k * 8, cudaMemcpyDeviceToHost));
    *n = k;
    return f2gpu_trace_enable(c, c->trace_cap);  // reset the count
}

// ---- one panel (Procedure buildZ) on a host column: kernel-level parity ----
int f2gpu_panel_build_z(f2gpu_ctx* c, const uint64_t* col, size_t n, uint64_t* col_out, uint64_t* z_out,
                        uint32_t* r_out, uint32_t* pairs_out, uint32_t* npairs_out) {
    if (!c || (!col && n) || (!col_out && n) || !z_out || !r_out)
        return set_err(F2GPU_EINVAL, "panel_build_z: null argument");
    uint64_t* d = nullptr;
    f2::PanelState* st = nullptr;
    auto fin = [&](int rc) {
        cudaFree(d);
        cudaFree(st);
        return rc;
    };
    if (cudaMalloc(&d, std::max<size_t>(n, 1) * 8) != cudaSuccess || cudaMalloc(&st, kStateBytes) != cudaSuccess)
        return fin(set_err(F2GPU_ENOMEM, "panel_build_z: device allocation"));
    if (n && cudaMemcpyAsync(d, col, n * 8, cudaMemcpyHostToDevice, c->stream) != cudaSuccess)
        return fin(set_err(F2GPU_ECUDA, "panel_build_z: upload"));
    if (int rc = check_launch(c, f2::launch_panel(d, n, st, 0, c->stream), "k_panel"); rc != F2GPU_OK) return fin(rc);
    f2::PanelState hs;
    if ((n && cudaMemcpyAsync(col_out, d, n * 8, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess) ||
        cudaMemcpyAsync(&hs, st, kStateBytes, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
        cudaStreamSynchronize(c->stream) != cudaSuccess)
        return fin(set_err(F2GPU_ECUDA, "panel_build_z: download"));
    std::copy(hs.Z, hs.Z + 64, z_out);
    *r_out = hs.r;
    if (npairs_out) *npairs_out = hs.npairs;
    if (pairs_out) {
        std::copy(hs.dst, hs.dst + 128, pairs_out);
        std::copy(hs.src, hs.src + 128, pairs_out + 128);
    }
    return fin(F2GPU_OK);
}

// ---- matrices ----
int f2gpu_mat_alloc(f2gpu_ctx* c, size_t n, size_t m, f2gpu_mat** out) {
    if (!c || !out) return set_err(F2GPU_EINVAL, "mat_alloc: null argument");
    *out = nullptr;
    auto M = std::make_unique<f2gpu_mat>();
    M->ctx = c; M->rows = n; M->cols = m; M->stride = dev_stride(n);
    const size_t words = ceil64(m) * M->stride;
    if (words) {
        cudaError_t e = cudaMalloc(&M->d, words * 8);
        if (e != cudaSuccess) return set_err(F2GPU_ENOMEM, std::string("mat_alloc: ") + cudaGetErrorString(e));
        CUDA_TRY(cudaMemsetAsync(M->d, 0, words * 8, c->stream));
    }
    *out = M.release();
    return F2GPU_OK;
}

int f2gpu_mat_free(f2gpu_mat* m) {
    if (!m) return F2GPU_OK;
    if (m->d) {
        cudaStreamSynchronize(m->ctx->stream);
        cudaFree(m->d);
    }
    delete m;
    return F2GPU_OK;
}

int f2gpu_mat_shape(const f2gpu_mat* m, size_t* r, size_t* cc, size_t* s) {
    if (!m) return set_err(F2GPU_EINVAL, "null mat");
    if (r) *r = m->rows;
    if (cc) *cc = m->cols;
    if (s) *s = m->stride;
    return F2GPU_OK;
}

int f2gpu_mat_device_ptr(const f2gpu_mat* m, uint64_t** p) {
    if (!m || !p) return set_err(F2GPU_EINVAL, "null argument");
    *p = m->d;
    return F2GPU_OK;
}

int f2gpu_mat_zero(f2gpu_ctx* c, f2gpu_mat* m) {
    if (!c || !m) return set_err(F2GPU_EINVAL, "null argument");
    if (m->d) CUDA_TRY(cudaMemsetAsync(m->d, 0, ceil64(m->cols) * m->stride * 8, c->stream));
    return F2GPU_OK;
}

int f2gpu_mat_upload(f2gpu_ctx* c, f2gpu_mat* m, const uint64_t* h, size_t hs) {
    if (!c || !m || (!h && m->rows && m->cols)) return set_err(F2GPU_EINVAL, "mat_upload: null argument");
    if (m->rows == 0 || m->cols == 0) return F2GPU_OK;
    if (hs < m->rows) return set_err(F2GPU_EINVAL, "mat_upload: host stride < rows");
    CUDA_TRY(cudaMemcpy2DAsync(m->d, m->stride * 8, h, hs * 8, m->rows * 8, ceil64(m->cols),
                               cudaMemcpyHostToDevice, c->stream));
    return F2GPU_OK;
}

int f2gpu_mat_download(f2gpu_ctx* c, const f2gpu_mat* m, uint64_t* h, size_t hs) {
    if (!c || !m || (!h && m->rows && m->cols)) return set_err(F2GPU_EINVAL, "mat_download: null argument");
    if (m->rows == 0 || m->cols == 0) return F2GPU_OK;
    if (hs < m->rows) return set_err(F2GPU_EINVAL, "mat_download: host stride < rows");
    CUDA_TRY(cudaMemcpy2DAsync(h, hs * 8, m->d, m->stride * 8, m->rows * 8, ceil64(m->cols),
                               cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return F2GPU_OK;
}

int f2gpu_mat_random_dense(f2gpu_ctx* c, f2gpu_mat* m, double density, uint64_t seed) {
    if (!c || !m) return set_err(F2GPU_EINVAL, "null argument");
    return check_launch(c, f2::launch_random_dense(m->d, m->rows, m->cols, m->stride, density, seed,
                                                   c->d_jump, c->stream),
                        "k_random_dense");
}

int f2gpu_mat_copy(f2gpu_ctx* c, f2gpu_mat* dst, const f2gpu_mat* src) {
    if (!c || !dst || !src) return set_err(F2GPU_EINVAL, "null argument");
    if (dst->rows != src->rows || dst->cols != src->cols)
        return set_err(F2GPU_EINVAL, "mat_copy: shape mismatch");
    if (dst->d && src->d)
        CUDA_TRY(cudaMemcpy2DAsync(dst->d, dst->stride * 8, src->d, src->stride * 8, src->rows * 8,
                                   ceil64(src->cols), cudaMemcpyDeviceToDevice, c->stream));
    return F2GPU_OK;
}

int f2gpu_mat_select_wcols(f2gpu_ctx* c, f2gpu_mat* dst, const f2gpu_mat* src, size_t first,
                           size_t step, int scatter) {
    if (!c || !dst || !src) return set_err(F2GPU_EINVAL, "null argument");
    if (dst->rows != src->rows || step == 0) return set_err(F2GPU_EINVAL, "select_wcols: shape");
    const f2gpu_mat* loc = scatter ? src : dst;   // the strided-over (local) side
    const f2gpu_mat* glob = scatter ? dst : src;
    const size_t nl = ceil64(loc->cols);
    if (nl && first + (nl - 1) * step >= ceil64(glob->cols))
        return set_err(F2GPU_ERANGE, "select_wcols: column outside matrix");
    if (!nl || !src->rows) return F2GPU_OK;
    // one strided 2D copy: rows*8 bytes per word-column, pitch step*stride on the global side
    if (scatter)
        CUDA_TRY(cudaMemcpy2DAsync(dst->d + first * dst->stride, step * dst->stride * 8, src->d,
                                   src->stride * 8, src->rows * 8, nl, cudaMemcpyDeviceToDevice,
                                   c->stream));
    else
        CUDA_TRY(cudaMemcpy2DAsync(dst->d, dst->stride * 8, src->d + first * src->stride,
                                   step * src->stride * 8, src->rows * 8, nl,
                                   cudaMemcpyDeviceToDevice, c->stream));
    return F2GPU_OK;
}

int f2gpu_mat_xor(f2gpu_ctx* c, f2gpu_mat* dst, const f2gpu_mat* src) {
    if (!c || !dst || !src) return set_err(F2GPU_EINVAL, "null argument");
    if (dst->rows != src->rows || dst->cols != src->cols)
        return set_err(F2GPU_EINVAL, "xor_with: shape mismatch");  // bit_matrix.hpp:243
    View s = view_of(src);
    return xor_views(c, view_of(dst), true, &s);
}

int f2gpu_mat_transpose(f2gpu_ctx* c, const f2gpu_mat* a, f2gpu_mat* out) {
    if (!c || !a || !out) return set_err(F2GPU_EINVAL, "null argument");
    if (out->rows != a->cols || out->cols != a->rows)
        return set_err(F2GPU_EINVAL, "transpose: output shape");
    return check_launch(c, f2::launch_transpose(a->d, a->rows, a->cols, a->stride, out->d,
                                                out->stride, c->stream),
                        "k_transpose");
}

// ---- products ----
namespace {
struct MatGuard {
    f2gpu_mat* m = nullptr;
    ~MatGuard() { f2gpu_mat_free(m); }
};
}  // namespace

int f2gpu_m4rm_mult_acc(f2gpu_ctx* c, const f2gpu_mat* a, const f2gpu_mat* b, f2gpu_mat* cm) {
    if (!c || !a || !b || !cm) return set_err(F2GPU_EINVAL, "null argument");
    if (a->cols != b->rows) return set_err(F2GPU_EINVAL, "m4rm_mult: shape mismatch");  // m4rm.hpp:181
    if (cm->rows != a->rows || cm->cols != b->cols)
        return set_err(F2GPU_EINVAL, "m4rm_mult: output shape mismatch");
    return gemm_acc(c, view_of(cm), view_of(a), view_of(b));
}

int f2gpu_m4rm_mult(f2gpu_ctx* c, const f2gpu_mat* a, const f2gpu_mat* b, f2gpu_mat* cm,
                    unsigned) {
    if (!c || !a || !b || !cm) return set_err(F2GPU_EINVAL, "null argument");
    if (a->cols != b->rows) return set_err(F2GPU_EINVAL, "m4rm_mult: shape mismatch");
    if (cm->rows != a->rows || cm->cols != b->cols)
        return set_err(F2GPU_EINVAL, "m4rm_mult: output shape mismatch");
    F2_TRY(f2gpu_mat_zero(c, cm));
    return gemm_acc(c, view_of(cm), view_of(a), view_of(b));
}

int f2gpu_gemm_tc(f2gpu_ctx* c, const f2gpu_mat* a, const f2gpu_mat* b, f2gpu_mat* cm, int acc) {
    if (!c || !a || !b || !cm) return set_err(F2GPU_EINVAL, "null argument");
    if (a->cols != b->rows || cm->rows != a->rows || cm->cols != b->cols)
        return set_err(F2GPU_EINVAL, "gemm_tc: shape mismatch");
#if F2GPU_EXPERIMENTAL
    static const int kind = [] {
        return f2::options().tc_kind == 8 ? 8 : 4;  // evaluation switch: the int8 leaf
    }();
#else
    constexpr int kind = 4;
#endif
    if (kind == 4 && f2::gemm_tc3_ok(a->rows, a->cols, b->cols)) {
        const size_t sbt = (b->cols + 127) / 128 * 128;
        DevBuf bt(c);
        if (int e = bt.alloc(sbt * ceil64(b->rows) * 8)) return e;
        if (int e = check_launch(c, f2::launch_transpose(b->d, b->rows, b->cols, b->stride, bt.as<uint64_t>(),
                                                         sbt, c->stream),
                                 "k_transpose"))
            return e;
        return check_launch(c, f2::launch_gemm_tc3(a->d, a->stride, a->rows, bt.as<uint64_t>(), sbt, cm->d,
                                                   cm->stride, a->cols, b->cols, acc != 0, c->stream),
                            "k_gemm_tc3");
    }
#if !F2GPU_EXPERIMENTAL
    return set_err(F2GPU_EINVAL, "gemm_tc: the fp4 leaf needs m % 256 == 0 (the int8 leaf is built only with "
                                 "F2GPU_EXPERIMENTAL=1)");
#else
    if (!f2::gemm_tc_ok(a->rows, a->cols, b->cols))
        return set_err(F2GPU_EINVAL, kind == 4 ? "gemm_tc: needs m % 256 == 0"
                                               : "gemm_tc: needs n % 256 == 0, m % 128 == 0, k % 64 == 0");
    if (f2::gemm_tc2_ok(a->rows, a->cols, b->cols)) {
        // B^T once (m x k), then the 256x256-tile kernel reads both operands as k-rows
        const size_t sbt = (b->cols + 127) / 128 * 128;
        DevBuf bt(c);
        if (int e = bt.alloc(sbt * ceil64(b->rows) * 8)) return e;
        if (int e = check_launch(c, f2::launch_transpose(b->d, b->rows, b->cols, b->stride, bt.as<uint64_t>(),
                                                         sbt, c->stream),
                                 "k_transpose"))
            return e;
        return check_launch(c, f2::launch_gemm_tc2(a->d, a->stride, bt.as<uint64_t>(), sbt, cm->d, cm->stride,
                                                   a->rows, a->cols, b->cols, acc != 0, c->stream),
                            "k_gemm_tc2");
    }
    return check_launch(c, f2::launch_gemm_tc(a->d, a->stride, b->d, b->stride, cm->d, cm->stride,
                                              a->rows, a->cols, b->cols, acc != 0, c->stream),
                        "k_gemm_tc");
#endif
}

int f2gpu_update_tc(f2gpu_ctx* c, f2gpu_mat* cm, size_t row_lo, size_t row_hi, size_t c_wcol0,
                    size_t n_wcols, const f2gpu_mat* a, size_t a_wcol0, size_t kwords, const f2gpu_mat* bt) {
    if (!c || !cm || !a || !bt) return set_err(F2GPU_EINVAL, "null argument");
    if (kwords < 1 || kwords > 2) return set_err(F2GPU_EINVAL, "update_tc: kwords must be 1 or 2");
    if (row_lo > row_hi || row_hi > cm->rows || a->rows != cm->rows)
        return set_err(F2GPU_ERANGE, "update_tc: row range outside C / A");
    if (c_wcol0 + n_wcols > ceil64(cm->cols) || a_wcol0 + kwords > ceil64(a->cols))
        return set_err(F2GPU_ERANGE, "update_tc: word-columns outside C / A");
    if (bt->rows < n_wcols * 64 || bt->cols < kwords * 64)
        return set_err(F2GPU_EINVAL, "update_tc: BT must be (n_wcols*64) x (kwords*64)");
    if (n_wcols == 0 || row_lo == row_hi) return F2GPU_OK;
#if !F2GPU_EXPERIMENTAL
    return set_err(F2GPU_EINVAL, "update_tc: the tensor-core update is built only with F2GPU_EXPERIMENTAL=1 "
                                 "(evaluated, not used: DESIGN.md)");
#else
    // B^T with the row padding the kernel's 192-row bulk loads read
    const size_t sbt = (f2::update_tc_bt_rows(int(n_wcols)) + 127) / 128 * 128;
    DevBuf pad(c);
    F2_TRY(pad.alloc(sbt * kwords * 8));
    CUDA_TRY(cudaMemcpy2DAsync(pad.p, sbt * 8, bt->d, bt->stride * 8, n_wcols * 64 * 8, kwords,
                               cudaMemcpyDeviceToDevice, c->stream));
    f2::TcUpdateArgs u{};
    u.C = cm->d; u.sc = cm->stride; u.q0 = c_wcol0; u.ncols = int(n_wcols);
    u.row_lo = row_lo; u.row_hi = row_hi;
    u.a = a->d + a_wcol0 * a->stride; u.sa = a->stride; u.kwords = int(kwords);
    u.bt = pad.as<uint64_t>(); u.sbt = sbt;
    if (!f2::update_tc_ok(u)) return set_err(F2GPU_EINVAL, "update_tc: operands not aligned");
    return check_launch(c, f2::launch_update_tc(u, c->num_sms, c->stream), "k_update_tc");
#endif
}

int f2gpu_mult_acc(f2gpu_ctx* c, f2gpu_mat* cm, size_t c_row0, size_t c_wcol0, size_t n_wcols,
                   const uint64_t* d_a, size_t n_rows, size_t k_bits, const f2gpu_mat* b,
                   size_t b_row0, size_t b_wcol0) {
    if (!c || !cm || !b || (!d_a && n_rows)) return set_err(F2GPU_EINVAL, "null argument");
    if (k_bits > 64) return set_err(F2GPU_EINVAL, "build_tables: block taller than a word");  // m4rm.hpp:97-98
    if (b_row0 + k_bits > b->rows || b_wcol0 + n_wcols > ceil64(b->cols))
        return set_err(F2GPU_ERANGE, "build_tables: block outside B");  // m4rm.hpp:99-100
    if (c_row0 + n_rows > cm->rows || c_wcol0 + n_wcols > ceil64(cm->cols))
        return set_err(F2GPU_ERANGE, "mult_acc: destination outside C");  // m4rm.hpp:144-145
    if (n_rows == 0 || n_wcols == 0 || k_bits == 0) return F2GPU_OK;
    f2::UpdateArgs u{};
    u.C = cm->d; u.sc = cm->stride; u.c_wcol0 = c_wcol0; u.ncols = int(n_wcols);
    u.row_lo = c_row0; u.row_hi = c_row0 + n_rows;
    u.a = d_a - c_row0;
    u.k_bits = int(k_bits);
    u.B = b->d; u.sb = b->stride; u.b_row0 = b_row0; u.b_wcol0 = b_wcol0;
    u.st = nullptr;
    return check_launch(c, f2::launch_update(u, c->num_sms, c->stream), "k_update");
}

// mult_acc over build_tables on HOST matrices in the reference layout: the
// destination block, the driving words and the B block are staged on the device,
// the fused table-build + XOR kernel runs, the destination block comes back.
// Validation and error codes follow m4rm.hpp:97-100 (build_tables) and :144-145
// (mult_acc).  Bits of a driving word at or above k_bits are ignored, as the
// reference's table lookups never read them.
int f2gpu_mult_acc_host(f2gpu_ctx* c, uint64_t* ch, size_t c_rows, size_t c_cols, size_t c_stride, size_t c_row0,
                        size_t c_wcol0, const uint64_t* a_words, size_t n_rows, const uint64_t* bh, size_t b_rows,
                        size_t b_cols, size_t b_stride, size_t b_row0, size_t k_bits, size_t b_wcol0,
                        size_t n_wcols) {
    if (!c) return set_err(F2GPU_EINVAL, "null ctx");
    if (k_bits > 64) return set_err(F2GPU_EINVAL, "build_tables: block taller than a word");  // m4rm.hpp:97-98
    if (b_row0 + k_bits > b_rows || b_wcol0 + n_wcols > ceil64(b_cols))
        return set_err(F2GPU_ERANGE, "build_tables: block outside B");  // m4rm.hpp:99-100
    if (c_row0 + n_rows > c_rows || c_wcol0 + n_wcols > ceil64(c_cols))
        return set_err(F2GPU_ERANGE, "mult_acc: destination outside C");  // m4rm.hpp:144-145
    if (n_rows == 0 || n_wcols == 0 || k_bits == 0) return F2GPU_OK;
    if (!ch || !a_words || !bh) return set_err(F2GPU_EINVAL, "mult_acc_host: null buffer");
    if (c_stride < c_rows || b_stride < b_rows) return set_err(F2GPU_EINVAL, "mult_acc_host: stride < rows");
    MatGuard Cd, Bd, Ad;
    F2_TRY(f2gpu_mat_alloc(c, n_rows, n_wcols * 64, &Cd.m));
    F2_TRY(f2gpu_mat_alloc(c, k_bits, n_wcols * 64, &Bd.m));
    F2_TRY(f2gpu_mat_alloc(c, n_rows, 64, &Ad.m));
    std::vector<uint64_t> a(a_words, a_words + n_rows);
    if (k_bits < 64)
        for (auto& x : a) x &= (uint64_t(1) << k_bits) - 1;
    CUDA_TRY(cudaMemcpy2DAsync(Cd.m->d, Cd.m->stride * 8, ch + c_wcol0 * c_stride + c_row0, c_stride * 8, n_rows * 8,
                               n_wcols, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(cudaMemcpy2DAsync(Bd.m->d, Bd.m->stride * 8, bh + b_wcol0 * b_stride + b_row0, b_stride * 8, k_bits * 8,
                               n_wcols, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(cudaMemcpyAsync(Ad.m->d, a.data(), n_rows * 8, cudaMemcpyHostToDevice, c->stream));
    F2_TRY(f2gpu_mult_acc(c, Cd.m, 0, 0, n_wcols, Ad.m->d, n_rows, k_bits, Bd.m, 0, 0));
    CUDA_TRY(cudaMemcpy2DAsync(ch + c_wcol0 * c_stride + c_row0, c_stride * 8, Cd.m->d, Cd.m->stride * 8, n_rows * 8,
                               n_wcols, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));  // `a` is a local; the caller's C is final on return
    return F2GPU_OK;
}

int f2gpu_strassen_mult(f2gpu_ctx* c, const f2gpu_mat* a, const f2gpu_mat* b, f2gpu_mat* cm,
                        size_t threshold) {
    if (!c || !a || !b || !cm) return set_err(F2GPU_EINVAL, "null argument");
    if (a->cols != b->rows) return set_err(F2GPU_EINVAL, "strassen_mult: shape mismatch");
    if (cm->rows != a->rows || cm->cols != b->cols)
        return set_err(F2GPU_EINVAL, "strassen_mult: output shape mismatch");
    F2_TRY(f2gpu_mat_zero(c, cm));
    c->tl.mark(c->stream, "start");
    // the paper's multiply: Strassen-Winograd over the fastest leaf (the fp4
    // tensor-core leaf when the shape allows, else M4RM); threshold = cutover
    F2_TRY(best_product(c, view_of(cm), view_of(a), view_of(b), threshold ? threshold : c->strassen_cutover,
                        threshold ? threshold : c->tc_cutover));
    c->tl.report("strassen");
    return F2GPU_OK;
}

// ---- decomposition ----
int f2gpu_decompose_block(f2gpu_ctx* c, f2gpu_mat* w, uint32_t* perm, uint32_t* rj, size_t* rank) {
    if (!c || !w) return set_err(F2GPU_EINVAL, "null argument");
    if (w->rows > 0xFFFFFFF0ull) return set_err(F2GPU_ERANGE, "decompose: too many rows for uint32 perm");
    return decompose_single(c, view_of(w), perm, rj, rank);
}

int f2gpu_decompose_recursive(f2gpu_ctx* c, f2gpu_mat* w, size_t min_cols, uint32_t* perm,
                              uint32_t* rj, size_t* rank) {
    if (!c || !w) return set_err(F2GPU_EINVAL, "null argument");
    if (w->rows > 0xFFFFFFF0ull) return set_err(F2GPU_ERANGE, "decompose: too many rows for uint32 perm");
    return decompose_recursive(c, view_of(w), min_cols, perm, rj, rank);
}

int f2gpu_decompose_block_sharded(f2gpu_ctx* c, f2gpu_mat* w, int G, uint32_t* perm, uint32_t* rj,
                                  size_t* rank) {
    if (!c || !w) return set_err(F2GPU_EINVAL, "null argument");
    if (G < 1) return set_err(F2GPU_EINVAL, "shards must be >= 1");
    const size_t n = w->rows, mu = ceil64(w->cols);
    if (n == 0 || mu == 0) return decompose_single(c, view_of(w), perm, rj, rank);
    // scatter word-columns round-robin into G local matrices
    std::deque<DevBuf> keep;
    std::vector<Shard> sh(G);
    for (int g = 0; g < G; ++g) {
        sh[g].lw = f2gpu_local_wcols(mu, g, G);
        keep.emplace_back(c);
        F2_TRY(keep.back().alloc(std::max<size_t>(1, sh[g].lw) * w->stride * 8));
        sh[g].w = View{keep.back().as<uint64_t>(), n, sh[g].lw * 64, w->stride, w->stride};
        for (size_t l = 0; l < sh[g].lw; ++l)
            CUDA_TRY(cudaMemcpyAsync(sh[g].w.p + l * w->stride, w->d + (g + l * G) * w->stride,
                                     w->stride * 8, cudaMemcpyDeviceToDevice, c->stream));
        F2_TRY(alloc_shard_aux(c, sh[g], n, mu, keep));
    }
    LocalExchange ex;
    F2_TRY(decompose_sharded(c, sh, 0, G, n, mu, ex));
    for (int g = 0; g < G; ++g)
        for (size_t l = 0; l < sh[g].lw; ++l)
            CUDA_TRY(cudaMemcpyAsync(w->d + (g + l * G) * w->stride, sh[g].w.p + l * w->stride,
                                     w->stride * 8, cudaMemcpyDeviceToDevice, c->stream));
    return read_results(c, sh[0], n, mu, perm, rj, rank);
}

int f2gpu_rank(f2gpu_ctx* c, const f2gpu_mat* a, size_t* rank) {
    if (!c || !a || !rank) return set_err(F2GPU_EINVAL, "null argument");
    const bool tr = a->rows < a->cols;
    f2gpu_mat* t = nullptr;
    F2_TRY(f2gpu_mat_alloc(c, tr ? a->cols : a->rows, tr ? a->rows : a->cols, &t));
    std::unique_ptr<f2gpu_mat, int (*)(f2gpu_mat*)> guard(t, f2gpu_mat_free);
    if (tr) {
        F2_TRY(f2gpu_mat_transpose(c, a, t));
    } else if (a->rows && a->cols) {
        CUDA_TRY(cudaMemcpyAsync(t->d, a->d, ceil64(a->cols) * a->stride * 8,
                                 cudaMemcpyDeviceToDevice, c->stream));
    }
    return decompose_single(c, view_of(t), nullptr, nullptr, rank);
}

// ---- null space / solve ---------------------------------
// Both are a PARTIAL block decomposition of an augmented matrix: the P panels of
// its left part are factored exactly as in decompose_block (buildZ, swaps on
// every word-column, Schur updates on every trailing word-column), the identity
// on the right records the row operations.  Non-pivot rows end with a zero left
// part, so their identity parts span the left null space of the left part.
//   null_space(A): left part A^T (m rows)        -> those rows, transposed, are N
//   solve(A, b):   left part [A^T; b^T] (m+1 rows) -> a null vector c with c_m = 1
//                                                    gives A * c[0..m) = b
namespace {
int partial_eliminate(f2gpu_ctx* c, f2gpu_mat* w, size_t panels, size_t* rank) {
    const size_t n = w->rows, mu = ceil64(w->cols);
    F2_TRY(ensure_scratch(c, n, mu));
    Shard s;
    s.w = view_of(w); s.lw = mu; s.st = static_cast<f2::PanelState*>(c->scr_st); s.perm = c->scr_perm;
    F2_TRY(check_launch(c, f2::launch_iota(s.perm, n, c->stream), "k_iota"));
    for (size_t j = 0; j < panels; ++j) F2_TRY(step_single(c, s, n, mu, j));
    return read_results(c, s, n, panels, nullptr, nullptr, rank);
}

// W (rows x (P + ceil64(rows)) word-cols): A^T in word-cols [0, P), I_rows after
int build_augmented(f2gpu_ctx* c, const f2gpu_mat* a, size_t rows, size_t P, f2gpu_mat** out) {
    F2_TRY(f2gpu_mat_alloc(c, rows, (P + ceil64(rows)) * 64, out));
    F2_TRY(f2gpu_mat_zero(c, *out));
    if (a->rows && a->cols)
        F2_TRY(check_launch(c, f2::launch_transpose(a->d, a->rows, a->cols, a->stride, (*out)->d, (*out)->stride,
                                                    c->stream),
                            "k_transpose"));
    return check_launch(c, f2::launch_set_diag((*out)->d, (*out)->stride, rows, P, c->stream), "k_set_diag");
}
}  // namespace

int f2gpu_null_space(f2gpu_ctx* c, const f2gpu_mat* a, f2gpu_mat** basis, size_t* nullity) {
    if (!c || !a || !basis) return set_err(F2GPU_EINVAL, "null argument");
    *basis = nullptr;
    const size_t n = a->rows, m = a->cols, P = ceil64(n);
    if (m > 0xFFFFFFF0ull) return set_err(F2GPU_ERANGE, "null_space: too many columns");
    f2gpu_mat* W = nullptr;
    F2_TRY(build_augmented(c, a, m, P, &W));
    std::unique_ptr<f2gpu_mat, int (*)(f2gpu_mat*)> guard(W, f2gpu_mat_free);
    size_t r = 0;
    if (m) F2_TRY(partial_eliminate(c, W, P, &r));
    const size_t nul = m - r;
    F2_TRY(f2gpu_mat_alloc(c, m, nul, basis));
    if (nul)
        F2_TRY(check_launch(c, f2::launch_transpose(W->d + P * W->stride + r, nul, m, W->stride, (*basis)->d,
                                                    (*basis)->stride, c->stream),
                            "k_transpose"));
    if (nullity) *nullity = nul;
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return F2GPU_OK;
}

int f2gpu_solve(f2gpu_ctx* c, const f2gpu_mat* a, const uint64_t* rhs, uint64_t* x, int* solvable) {
    if (!c || !a || !solvable || (!rhs && a->rows) || (!x && a->cols)) return set_err(F2GPU_EINVAL, "null argument");
    const size_t n = a->rows, m = a->cols, P = ceil64(n), m1 = m + 1;
    if (m1 > 0xFFFFFFF0ull) return set_err(F2GPU_ERANGE, "solve: too many columns");
    f2gpu_mat* W = nullptr;
    F2_TRY(build_augmented(c, a, m1, P, &W));  // row m of the A^T part stays 0 ...
    std::unique_ptr<f2gpu_mat, int (*)(f2gpu_mat*)> guard(W, f2gpu_mat_free);
    if (P) {  // ... and receives b^T (bits past n cleared)
        std::vector<uint64_t> b(rhs, rhs + P);
        if (n % 64) b[P - 1] &= (uint64_t(1) << (n % 64)) - 1;
        CUDA_TRY(cudaMemcpy2DAsync(W->d + m, W->stride * 8, b.data(), 8, 8, P, cudaMemcpyHostToDevice, c->stream));
        CUDA_TRY(cudaStreamSynchronize(c->stream));  // b is a local
    }
    size_t r = 0;
    F2_TRY(partial_eliminate(c, W, P, &r));
    *solvable = 0;
    const size_t mw = ceil64(m);
    if (x) std::fill(x, x + mw, 0ull);
    if (r >= m1) return F2GPU_OK;  // only the trivial combination: b not in the column space
    // the c_m bits of the null rows r .. m
    std::vector<uint64_t> tag(m1 - r);
    CUDA_TRY(cudaMemcpyAsync(tag.data(), W->d + (P + m / 64) * W->stride + r, tag.size() * 8, cudaMemcpyDeviceToHost,
                             c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    for (size_t i = 0; i < tag.size(); ++i) {
        if (!((tag[i] >> (m % 64)) & 1)) continue;
        std::vector<uint64_t> row(ceil64(m1));
        CUDA_TRY(cudaMemcpy2DAsync(row.data(), 8, W->d + P * W->stride + r + i, W->stride * 8, 8, row.size(),
                                   cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        for (size_t q = 0; q < mw; ++q) x[q] = row[q];
        if (m % 64) x[mw - 1] &= (uint64_t(1) << (m % 64)) - 1;  // drop c_m (and padding)
        *solvable = 1;
        break;
    }
    return F2GPU_OK;
}

// ---- host-buffer entry points ----

int f2gpu_m4rm_mult_host(f2gpu_ctx* c, const uint64_t* a, size_t n, size_t k, size_t sa,
                         const uint64_t* b, size_t m, size_t sb, uint64_t* out, size_t sc,
                         unsigned tc) {
    if (!c) return set_err(F2GPU_EINVAL, "null ctx");
    MatGuard A, B, C;
    F2_TRY(f2gpu_mat_alloc(c, n, k, &A.m));
    F2_TRY(f2gpu_mat_alloc(c, k, m, &B.m));
    F2_TRY(f2gpu_mat_alloc(c, n, m, &C.m));
    F2_TRY(f2gpu_mat_upload(c, A.m, a, sa));
    F2_TRY(f2gpu_mat_upload(c, B.m, b, sb));
    F2_TRY(f2gpu_m4rm_mult(c, A.m, B.m, C.m, tc));
    return f2gpu_mat_download(c, C.m, out, sc);
}

int f2gpu_strassen_mult_host(f2gpu_ctx* c, const uint64_t* a, size_t n, size_t k, size_t sa,
                             const uint64_t* b, size_t m, size_t sb, uint64_t* out, size_t sc,
                             size_t threshold) {
    if (!c) return set_err(F2GPU_EINVAL, "null ctx");
    MatGuard A, B, C;
    F2_TRY(f2gpu_mat_alloc(c, n, k, &A.m));
    F2_TRY(f2gpu_mat_alloc(c, k, m, &B.m));
    F2_TRY(f2gpu_mat_alloc(c, n, m, &C.m));
    F2_TRY(f2gpu_mat_upload(c, A.m, a, sa));
    F2_TRY(f2gpu_mat_upload(c, B.m, b, sb));
    F2_TRY(f2gpu_strassen_mult(c, A.m, B.m, C.m, threshold));
    return f2gpu_mat_download(c, C.m, out, sc);
}

// Host-buffer calls stage through a context-owned device matrix that is reused
// while the shape stays the same (no per-call 0.5 GiB cudaMalloc/cudaFree, and a
// stable pointer keeps the decomposition's CUDA graph cache warm).
int staging(f2gpu_ctx* c, size_t n, size_t m, f2gpu_mat** out) {
    if (c->stage && (c->stage->rows != n || c->stage->cols != m)) {
        f2gpu_mat_free(c->stage);
        c->stage = nullptr;
    }
    if (!c->stage) F2_TRY(f2gpu_mat_alloc(c, n, m, &c->stage));
    *out = c->stage;
    return F2GPU_OK;
}

int f2gpu_decompose_block_host(f2gpu_ctx* c, const uint64_t* a, size_t n, size_t m, size_t stride,
                               uint64_t* w_out, uint32_t* perm, uint32_t* rj, size_t* rank) {
    if (!c) return set_err(F2GPU_EINVAL, "null ctx");
    f2gpu_mat* W = nullptr;
    F2_TRY(staging(c, n, m, &W));
    F2_TRY(f2gpu_mat_upload(c, W, a, stride));
    F2_TRY(f2gpu_decompose_block(c, W, perm, rj, rank));
    if (w_out) F2_TRY(f2gpu_mat_download(c, W, w_out, stride));
    return F2GPU_OK;
}

int f2gpu_decompose_recursive_host(f2gpu_ctx* c, const uint64_t* a, size_t n, size_t m, size_t stride,
                                   size_t min_cols, uint64_t* w_out, uint32_t* perm, uint32_t* rj,
                                   size_t* rank) {
    if (!c) return set_err(F2GPU_EINVAL, "null ctx");
    f2gpu_mat* W = nullptr;
    F2_TRY(staging(c, n, m, &W));
    const size_t mu = ceil64(m);
    // Upload overlap: the first leaf's word-columns go straight into W; the rest
    // stream on the copy stream, chunk by chunk, into `pend` in the host's row
    // order, and the recursion materialises each chunk under the row permutation
    // of the panels factored so far when it first needs it (ensure_cols).
    // first chunk = the recursion's first leaf (tall leaves are narrower)
    size_t cw = std::max<size_t>(1, (min_cols ? min_cols : 256 * 64) / 64);
    {
        const f2::Options& o = f2::options();
        const size_t tall = size_t(o.rec_tall), tall_base = std::max<size_t>(1, size_t(o.rec_tall_base));
        if (o.rec_base_set) cw = std::max<size_t>(1, size_t(o.rec_base));
        if (tall && n >= tall) cw = std::min(cw, tall_base);
        // first leaf = upload chunk width (F2GPU_REC_FIRST; 65536^2 e2e: 128: 67.83 ms,
        // 64: 67.36, 32: 67.40-67.45, 16: 67.62 at the same 63.2 ms device time)
        const size_t first = std::max<size_t>(1, size_t(o.rec_first));
        cw = std::min(cw, first);
    }
    if (n == 0 || mu <= cw || !a || f2::options().no_upload_overlap) {
        F2_TRY(f2gpu_mat_upload(c, W, a, stride));
        F2_TRY(f2gpu_decompose_recursive(c, W, min_cols, perm, rj, rank));
    } else {
        if (n > 0xFFFFFFF0ull) return set_err(F2GPU_ERANGE, "decompose: too many rows for uint32 perm");
        const size_t ps = W->stride, nchunks = (mu - cw + cw - 1) / cw;
        const size_t bytes = (mu - cw) * ps * 8;
        if (!c->copy) CUDA_TRY(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
        while (c->chunk_ev.size() < nchunks + 1) {
            cudaEvent_t e;
            CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            c->chunk_ev.push_back(e);
        }
        if (c->pend_bytes < bytes) {
            CUDA_TRY(cudaStreamSynchronize(c->stream));
            cudaFree(c->pend);
            c->pend = nullptr;
            c->pend_bytes = 0;
            CUDA_TRY(cudaMalloc(&c->pend, bytes));
            c->pend_bytes = bytes;
        }
        // the copy stream may overwrite `pend` once earlier work on it is done
        CUDA_TRY(cudaEventRecord(c->chunk_ev[nchunks], c->stream));
        CUDA_TRY(cudaStreamWaitEvent(c->copy, c->chunk_ev[nchunks], 0));
        CUDA_TRY(cudaMemcpy2DAsync(W->d, W->stride * 8, a, stride * 8, n * 8, cw, cudaMemcpyHostToDevice,
                                   c->stream));
        uint64_t* pend = static_cast<uint64_t*>(c->pend);
        for (size_t i = 0; i < nchunks; ++i) {
            const size_t q0 = cw + i * cw, nq = std::min(cw, mu - q0);
            CUDA_TRY(cudaMemcpy2DAsync(pend + (q0 - cw) * ps, ps * 8, a + q0 * stride, stride * 8, n * 8, nq,
                                       cudaMemcpyHostToDevice, c->copy));
            CUDA_TRY(cudaEventRecord(c->chunk_ev[i], c->copy));
        }
        // download overlap: row blocks that are final go back on the copy stream
        // while the rest of the matrix is factored
        size_t done = 0;
        auto on_final = [&](size_t R) -> int {
            if (!w_out || R <= done) return F2GPU_OK;
            CUDA_TRY(cudaEventRecord(c->chunk_ev[nchunks], c->stream));
            CUDA_TRY(cudaStreamWaitEvent(c->copy, c->chunk_ev[nchunks], 0));
            CUDA_TRY(cudaMemcpy2DAsync(w_out + done, stride * 8, W->d + done, W->stride * 8, (R - done) * 8, mu,
                                       cudaMemcpyDeviceToHost, c->copy));
            done = R;
            return F2GPU_OK;
        };
        F2_TRY(decompose_recursive(c, view_of(W), min_cols, perm, rj, rank, cw, pend, ps, cw, on_final));
        if (w_out && done < n) {
            CUDA_TRY(cudaMemcpy2DAsync(w_out + done, stride * 8, W->d + done, W->stride * 8, (n - done) * 8, mu,
                                       cudaMemcpyDeviceToHost, c->stream));
        }
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        CUDA_TRY(cudaStreamSynchronize(c->copy));
        return F2GPU_OK;
    }
    if (w_out) F2_TRY(f2gpu_mat_download(c, W, w_out, stride));
    return F2GPU_OK;
}

int f2gpu_rank_host(f2gpu_ctx* c, const uint64_t* a, size_t n, size_t m, size_t stride,
                    size_t* rank) {
    if (!c) return set_err(F2GPU_EINVAL, "null ctx");
    MatGuard A;
    F2_TRY(f2gpu_mat_alloc(c, n, m, &A.m));
    F2_TRY(f2gpu_mat_upload(c, A.m, a, stride));
    return f2gpu_rank(c, A.m, rank);
}

// ---- multi-GPU ----
size_t f2gpu_local_wcols(size_t mu, int rank, int world) {
    if (world <= 0 || rank < 0 || size_t(rank) >= mu) return 0;
    return (mu - size_t(rank) + size_t(world) - 1) / size_t(world);
}

int f2gpu_nccl_unique_id(void* out) {
    NcclApi& api = nccl();
    if (!api.ok) return set_err(F2GPU_ENCCL, api.why);
    int rc = api.getUniqueId(out);
    if (rc) return set_err(F2GPU_ENCCL, "ncclGetUniqueId failed");
    return F2GPU_OK;
}

int f2gpu_ctx_init_comm(f2gpu_ctx* c, int rank, int world, const void* id) {
    if (!c || !id) return set_err(F2GPU_EINVAL, "null argument");
    if (world < 1 || rank < 0 || rank >= world) return set_err(F2GPU_ERANGE, "rank/world");
    c->rank = rank;
    c->world = world;
    // world == 1 needs no communicator; F2GPU_FORCE_NCCL=1 builds a 1-rank one so
    // the NCCL exchange path can be exercised on a single GPU.
    // read at each call (tests switch it per test within one process)
    long long force = 0;
    f2::env_value("F2GPU_FORCE_NCCL", &force);
    if (world == 1 && !force) return F2GPU_OK;
    NcclApi& api = nccl();
    if (!api.ok) return set_err(F2GPU_ENCCL, api.why);
    CUDA_TRY(cudaSetDevice(c->device));
    Id128 uid;
    std::memcpy(uid.b, id, 128);
    int rc = reinterpret_cast<CommInitRankFn>(api.commInitRankSym)(&c->comm, world, uid, rank);
    if (rc) return set_err(F2GPU_ENCCL, "ncclCommInitRank failed");
    return F2GPU_OK;
}

int f2gpu_mat_broadcast(f2gpu_ctx* c, f2gpu_mat* m, int root) {
    if (!c || !m) return set_err(F2GPU_EINVAL, "null argument");
    if (root < 0 || root >= c->world) return set_err(F2GPU_ERANGE, "broadcast: root rank");
    if (c->world == 1 && !c->comm) return F2GPU_OK;
    if (!c->comm) return set_err(F2GPU_ENCCL, "broadcast: communicator not initialised");
    NcclApi& api = nccl();
    const size_t bytes = ceil64(m->cols) * m->stride * 8;
    if (bytes == 0) return F2GPU_OK;
    int rc = api.broadcast(m->d, m->d, bytes, kNcclUint8, root, c->comm, c->stream);
    if (rc != 0)
        return set_err(F2GPU_ENCCL, std::string("ncclBroadcast: ") + (api.getErrorString ? api.getErrorString(rc) : "?"));
    return F2GPU_OK;
}

// Multiply sharded by column blocks: B and C word-columns are
// round-robin over the ranks, A is replicated by one broadcast from rank 0, and
// every rank computes its own C columns -- no per-step exchange.
int f2gpu_strassen_mult_dist(f2gpu_ctx* c, f2gpu_mat* a, const f2gpu_mat* b_local, f2gpu_mat* c_local,
                             size_t threshold) {
    if (!c || !a || !b_local || !c_local) return set_err(F2GPU_EINVAL, "null argument");
    F2_TRY(f2gpu_mat_broadcast(c, a, 0));
    return f2gpu_strassen_mult(c, a, b_local, c_local, threshold);
}

int f2gpu_decompose_block_dist(f2gpu_ctx* c, f2gpu_mat* w_local, size_t m_global, uint32_t* perm,
                               uint32_t* rj, size_t* rank) {
    if (!c || !w_local) return set_err(F2GPU_EINVAL, "null argument");
    const size_t n = w_local->rows, mu = ceil64(m_global);
    const size_t lw = f2gpu_local_wcols(mu, c->rank, c->world);
    if (ceil64(w_local->cols) != lw)
        return set_err(F2GPU_EINVAL, "decompose_dist: local matrix has the wrong number of word-columns");
    if (c->world == 1 && !c->comm) return decompose_single(c, view_of(w_local), perm, rj, rank);
    if (!c->comm) return set_err(F2GPU_ENCCL, "decompose_dist: communicator not initialised");
    std::deque<DevBuf> keep;
    std::vector<Shard> sh(1);
    sh[0].w = View{w_local->d, n, lw * 64, w_local->stride, w_local->stride};
    sh[0].lw = lw;
    F2_TRY(alloc_shard_aux(c, sh[0], n, mu, keep));
    NcclExchange ex;
    F2_TRY(decompose_sharded(c, sh, c->rank, c->world, n, mu, ex));
    return read_results(c, sh[0], n, mu, perm, rj, rank);
}

// ---- distributed decompose_recursive ----
int f2gpu_dist_schedule(size_t n_rows, size_t mu, int world, size_t leaf_panels, size_t tall_rows,
                        size_t tall_leaf_panels, const f2gpu_dist_ops* ops) {
    if (!ops || !ops->panel || !ops->apply || !ops->state || !ops->gather || !ops->solve || !ops->product ||
        !ops->rank_update)
        return set_err(F2GPU_EINVAL, "dist_schedule: null callback");
    if (world < 1) return set_err(F2GPU_EINVAL, "dist_schedule: world must be >= 1");
    return dist_schedule(n_rows, mu, world, std::max<size_t>(1, leaf_panels), tall_rows,
                         std::max<size_t>(1, tall_leaf_panels), ops);
}

int f2gpu_decompose_recursive_sharded(f2gpu_ctx* c, f2gpu_mat* w, int G, size_t min_cols, uint32_t* perm,
                                      uint32_t* rj, size_t* rank) {
    if (!c || !w) return set_err(F2GPU_EINVAL, "null argument");
    if (G < 1) return set_err(F2GPU_EINVAL, "shards must be >= 1");
    if (w->rows > 0xFFFFFFF0ull) return set_err(F2GPU_ERANGE, "decompose: too many rows for uint32 perm");
    const size_t n = w->rows, mu = ceil64(w->cols);
    if (n == 0 || mu == 0) return decompose_single(c, view_of(w), perm, rj, rank);
    std::deque<DevBuf> keep;
    std::vector<Shard> sh(G);
    for (int g = 0; g < G; ++g) {
        sh[g].lw = f2gpu_local_wcols(mu, g, G);
        keep.emplace_back(c);
        F2_TRY(keep.back().alloc(std::max<size_t>(1, sh[g].lw) * w->stride * 8));
        sh[g].w = View{keep.back().as<uint64_t>(), n, sh[g].lw * 64, w->stride, w->stride};
        if (sh[g].lw)
            CUDA_TRY(cudaMemcpy2DAsync(sh[g].w.p, w->stride * 8, w->d + size_t(g) * w->stride,
                                       size_t(G) * w->stride * 8, w->stride * 8, sh[g].lw, cudaMemcpyDeviceToDevice,
                                       c->stream));
        F2_TRY(alloc_shard_aux(c, sh[g], n, mu, keep));
    }
    LocalExchange ex;
    F2_TRY(run_dist_recursive(c, sh, 0, G, n, mu, min_cols, ex));
    for (int g = 0; g < G; ++g)
        if (sh[g].lw)
            CUDA_TRY(cudaMemcpy2DAsync(w->d + size_t(g) * w->stride, size_t(G) * w->stride * 8, sh[g].w.p,
                                       w->stride * 8, w->stride * 8, sh[g].lw, cudaMemcpyDeviceToDevice, c->stream));
    return read_results(c, sh[0], n, mu, perm, rj, rank);
}

int f2gpu_decompose_recursive_dist(f2gpu_ctx* c, f2gpu_mat* w_local, size_t m_global, size_t min_cols,
                                   uint32_t* perm, uint32_t* rj, size_t* rank) {
    if (!c || !w_local) return set_err(F2GPU_EINVAL, "null argument");
    if (w_local->rows > 0xFFFFFFF0ull) return set_err(F2GPU_ERANGE, "decompose: too many rows for uint32 perm");
    const size_t n = w_local->rows, mu = ceil64(m_global);
    const size_t lw = f2gpu_local_wcols(mu, c->rank, c->world);
    if (ceil64(w_local->cols) != lw)
        return set_err(F2GPU_EINVAL, "decompose_dist: local matrix has the wrong number of word-columns");
    if (c->world == 1 && !c->comm) return decompose_recursive(c, view_of(w_local), min_cols, perm, rj, rank);
    if (!c->comm) return set_err(F2GPU_ENCCL, "decompose_dist: communicator not initialised");
    if (n == 0 || mu == 0) {
        if (rank) *rank = 0;
        if (rj) std::fill(rj, rj + mu, 0u);
        if (perm) for (size_t i = 0; i < n; ++i) perm[i] = uint32_t(i);
        return F2GPU_OK;
    }
    std::deque<DevBuf> keep;
    std::vector<Shard> sh(1);
    sh[0].w = View{w_local->d, n, lw * 64, w_local->stride, w_local->stride};
    sh[0].lw = lw;
    F2_TRY(alloc_shard_aux(c, sh[0], n, mu, keep));
    NcclExchange ex;
    F2_TRY(run_dist_recursive(c, sh, c->rank, c->world, n, mu, min_cols, ex));
    return read_results(c, sh[0], n, mu, perm, rj, rank);
}

}  // extern "C"
