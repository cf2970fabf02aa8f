// kernels.cu — hand-written sm_100a kernels for the GF(2) decomposition hot path.
//
//   k_random_dense  bit-exact PackedMatrix::random_dense   (bit_matrix.hpp:125-142)
//   k_update        fused M4RM table build + XOR sweep     (m4rm.hpp:93-172) — the
//                   Schur update E ^= Y*C of decompose_block
//   k_gemm          stream-K M4RM product C ^= A*B         (m4rm.hpp:177-196)
//   k_panel         Procedure buildZ
//   k_panel_y       Y = D*Z written over D
//   k_swaps         mirror the panel's row transpositions  (bit_matrix.hpp:202-208)
//   k_xor           block XOR for Strassen-Winograd        (bit_matrix.hpp:241-250)
//   k_transpose     64x64 bit-tile transpose               (bit_matrix.hpp:59-70,220-238)
#include "kernels.cuh"
#include "options.h"

#include <algorithm>

#ifndef F2_PIPELINED_WRITEBACK
#define F2_PIPELINED_WRITEBACK 0
#endif
#ifndef F2_FENCE_IN_PRODUCER
#define F2_FENCE_IN_PRODUCER 0
#endif

namespace f2 {

// ---- device trace (diagnostics) ----
__device__ unsigned long long* g_trace = nullptr;
__device__ uint32_t g_trace_cap = 0;
__device__ uint32_t g_trace_n = 0;

// Cross-kernel waits (lookahead counters, release flags) are bounded: the fused
// schedule relies on its kernels being co-resident, which the CUDA model does not
// guarantee when other work holds the SMs (another stream, an MPS client).  A
// wait that exceeds kSpinLimitNs traps, so the call fails with a CUDA error
// instead of hanging the device.  Legitimate waits last microseconds.
constexpr uint64_t kSpinLimitNs = 20ull * 1000 * 1000 * 1000;
__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// F2GPU_SPIN_DIAG=1 (diagnostics): a timed-out wait records where it was stuck in
// host-mapped memory (readable after the trap killed the context; api.cu appends it
// to the error message):
//   [0] = 1 | site << 8, [1] = block, [2] = the counter's address, [3] = its last
//   value << 32 | the target
__device__ unsigned long long* g_spin_diag = nullptr;
struct SpinGuard {
    uint64_t t0 = 0;
    uint32_t polls = 0;
    __device__ __forceinline__ void tick(uint32_t site = 0, const void* addr = nullptr, uint32_t v = 0,
                                         uint32_t target = 0) {
        if ((++polls & 1023u) != 0) return;
        const uint64_t now = gtimer();
        if (t0 == 0) t0 = now;
        else if (now - t0 > kSpinLimitNs) {
            if (unsigned long long* d = g_spin_diag) {
                d[1] = blockIdx.x;
                d[2] = reinterpret_cast<unsigned long long>(addr);
                d[3] = (uint64_t(v) << 32) | target;
                __threadfence_system();
                d[0] = 1ull | (uint64_t(site) << 8);
                __threadfence_system();
            }
            __trap();
        }
    }
};

cudaError_t spin_diag_set(unsigned long long* mapped) {
    return cudaMemcpyToSymbol(g_spin_diag, &mapped, sizeof(mapped));
}

__device__ __forceinline__ void trace_ev(uint32_t ev, int j) {
    unsigned long long* b = g_trace;
    if (!b) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const uint32_t i = atomicAdd(&g_trace_n, 1u);
    if (i < g_trace_cap) b[i] = (t << 16) | (uint64_t(ev & 15) << 12) | uint64_t(uint32_t(j) & 4095u);
}

cudaError_t trace_set(unsigned long long* buf, uint32_t cap) {
    const uint32_t zero = 0;
    cudaError_t e = cudaMemcpyToSymbol(g_trace, &buf, sizeof(buf));
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_trace_cap, &cap, sizeof(cap));
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(g_trace_n, &zero, sizeof(zero));
    return e;
}

cudaError_t trace_count(uint32_t* n) { return cudaMemcpyFromSymbol(n, g_trace_n, sizeof(*n)); }


// ---------------------------------------------------------------------------
// small device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ void ld256(const uint64_t* p, uint64_t& a, uint64_t& b, uint64_t& c,
                                      uint64_t& d) {
    asm volatile("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
                 : "l"(p));
}
__device__ __forceinline__ void st256(uint64_t* p, uint64_t a, uint64_t b, uint64_t c,
                                      uint64_t d) {
    asm volatile("st.global.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(p), "l"(a), "l"(b), "l"(c),
                 "l"(d)
                 : "memory");
}

__device__ __forceinline__ uint64_t xs_step(uint64_t x) {  // prng.hpp:24-28
    x ^= x >> 12;
    x ^= x << 25;
    x ^= x >> 27;
    return x;
}

// ---------------------------------------------------------------------------
// K0: random_dense — jump-ahead xorshift64*
// ---------------------------------------------------------------------------
// The state map x -> step(x) is linear over GF(2); T^(2^s) (64 column images
// each) is precomputed on the host.  Thread (row i, segment g) jumps to draw
// i*m + 64*q0 and then steps serially, so the bits equal the reference's single
// serial stream (one draw per entry, row-major, prng.hpp:37-43).
constexpr int kRngSeg = 32;  // words per thread

__global__ void __launch_bounds__(256) k_random_dense(uint64_t* __restrict__ w, size_t n,
                                                      size_t m, size_t stride, uint64_t thr,
                                                      uint64_t s0,
                                                      const uint64_t* __restrict__ jump) {
    __shared__ uint64_t jt[64 * 64];
    for (int t = threadIdx.x; t < 64 * 64; t += blockDim.x) jt[t] = jump[t];
    __syncthreads();
    const size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const size_t mu = (m + 63) / 64;
    const size_t q0 = size_t(blockIdx.y) * kRngSeg;
    if (q0 >= mu) return;
    const size_t q1 = q0 + kRngSeg < mu ? q0 + kRngSeg : mu;
    uint64_t st = s0;
    uint64_t t = uint64_t(i) * m + 64 * q0;
    for (int s = 0; t; ++s, t >>= 1) {
        if (!(t & 1)) continue;
        const uint64_t* col = jt + s * 64;
        uint64_t y = 0;
#pragma unroll 16
        for (int b = 0; b < 64; ++b) y ^= col[b] & (0ull - ((st >> b) & 1));
        st = y;
    }
    for (size_t q = q0; q < q1; ++q) {
        const int kb = (q + 1 == mu) ? int(m - 64 * q) : 64;
        uint64_t word = 0;
        for (int k = 0; k < kb; ++k) {
            st = xs_step(st);
            const uint64_t v = st * 0x2545F4914F6CDD1Dull;
            word |= uint64_t(v < thr) << k;
        }
        w[q * stride + i] = word;
    }
}

__global__ void k_fill_ones(uint64_t* w, size_t n, size_t m, size_t stride) {
    const size_t mu = (m + 63) / 64;
    const size_t total = mu * n;
    for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += size_t(gridDim.x) * blockDim.x) {
        const size_t q = e / n, i = e % n;
        const size_t rem = m - 64 * q;
        w[q * stride + i] = rem >= 64 ? ~0ull : ((1ull << rem) - 1);
    }
}

static void host_mat_apply(const uint64_t* cols, uint64_t x, uint64_t* out) {
    uint64_t y = 0;
    for (int b = 0; b < 64; ++b)
        if ((x >> b) & 1) y ^= cols[b];
    *out = y;
}

void host_jump_tables(uint64_t out[64 * 64]) {
    for (int b = 0; b < 64; ++b) {
        uint64_t x = 1ull << b;
        x ^= x >> 12;
        x ^= x << 25;
        x ^= x >> 27;
        out[b] = x;
    }
    for (int s = 1; s < 64; ++s)
        for (int b = 0; b < 64; ++b)
            host_mat_apply(out + (s - 1) * 64, out[(s - 1) * 64 + b], out + s * 64 + b);
}

cudaError_t launch_random_dense(uint64_t* w, size_t n, size_t m, size_t stride, double density,
                                uint64_t seed, const uint64_t* d_jump, cudaStream_t s) {
    const size_t mu = (m + 63) / 64;
    if (n == 0 || m == 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(w, 0, mu * stride * 8, s);
    if (e != cudaSuccess || density <= 0.0) return e;   // bit_matrix.hpp:131
    if (density >= 1.0) {                               // :132-139 (no draws)
        k_fill_ones<<<1024, 256, 0, s>>>(w, n, m, stride);
        return cudaGetLastError();
    }
    const double scaled = density * 18446744073709551616.0;  // prng.hpp:41-42
    const uint64_t thr = static_cast<uint64_t>(scaled);
    const uint64_t s0 = seed != 0 ? seed : 0x9E3779B97F4A7C15ull;  // prng.hpp:20-21
    dim3 grid(unsigned((n + 255) / 256), unsigned((mu + kRngSeg - 1) / kRngSeg));
    k_random_dense<<<grid, 256, 0, s>>>(w, n, m, stride, thr, s0, d_jump);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// M4RM tables in shared memory
// ---------------------------------------------------------------------------
// Table t covers bits [7t, 7t+size_t) of the driving word; entry g of table t
// for CTA column col lives at tab[(128*t + g)*16 + col].  Entry g = XOR of the
// B rows selected by g's bits (M4rmTables, m4rm.hpp:21-35).  Each work item
// fills 32 consecutive entries of one (table, column) by doubling in
// registers: one 64-bit XOR per entry (cf. doubling fill, m4rm.hpp:74-88).
// Rows >= k_bits and columns >= ncols_valid read as zero.
__device__ __forceinline__ int tab_chunks(int nt) { return nt <= 8 ? 4 * nt : 40; }

template <int NTH>
__device__ __forceinline__ void build_tables(uint64_t* __restrict__ tab,
                                             const uint64_t* __restrict__ B, size_t sb,
                                             size_t b_row0, size_t bcol0, int ncols_valid,
                                             int k_bits, int nt) {
    const int total = tab_chunks(nt) * kTabCols;
    for (int it = threadIdx.x; it < total; it += NTH) {
        const int col = it & (kTabCols - 1);
        const int cg = it >> 4;
        const int t = cg < 32 ? (cg >> 2) : 8;
        const int chunk = cg < 32 ? (cg & 3) : cg - 32;
        const int sz = t < 8 ? 7 : 8;
        uint64_t rows[8];
        const bool cv = col < ncols_valid;
        const uint64_t* bp = B + (bcol0 + col) * sb + b_row0 + 7 * t;
#pragma unroll
        for (int b = 0; b < 8; ++b)
            rows[b] = (b < sz && cv && 7 * t + b < k_bits) ? __ldg(bp + b) : 0ull;
        uint64_t cur = 0;
#pragma unroll
        for (int hb = 0; hb < 3; ++hb)
            if ((chunk >> hb) & 1) cur ^= rows[5 + hb];
        uint64_t* dst = tab + (size_t(128 * t + chunk * 32) * kTabCols + col);
        uint64_t v[32];  // doubling in registers: v[g] = v[g - 2^b] ^ row b
        v[0] = cur;
#pragma unroll
        for (int b = 0; b < 5; ++b)
#pragma unroll
            for (int g = 1 << b; g < (2 << b); ++g) v[g] = v[g - (1 << b)] ^ rows[b];
#pragma unroll
        for (int g = 0; g < 32; ++g) dst[g * kTabCols] = v[g];
    }
}

// build_tables for a CTA of NTH >= 320 threads (at most two 32-entry items each)
// with B staged through shared memory first: the 16 columns x 64 rows are loaded
// coalesced into the start of the table region, each thread copies its rows to
// registers, and only then is the table written over the staging area.  Direct
// per-item __ldg touched 16 cache lines per warp load: 7.0k vs 3.5k cycles per
// group (tools/micro/tab_build.cu).  sync() must be a barrier of the NTH threads.
constexpr int kStagePitch = 66;  // words per staged column (conflict-free row reads)
template <int NTH, typename Sync>
__device__ __forceinline__ void build_tables_staged(uint64_t* __restrict__ tab, const uint64_t* __restrict__ B,
                                                    size_t sb, size_t b_row0, size_t bcol0, int ncols_valid,
                                                    int k_bits, Sync sync) {
    static_assert(NTH * 2 >= 640, "two items per thread");
    constexpr int total = 640;  // tab_chunks(9) * kTabCols
    uint64_t* stage = tab;
    for (int i = threadIdx.x; i < kTabCols * 64; i += NTH) {
        const int col = i >> 6, r = i & 63;
        stage[col * kStagePitch + r] =
            (col < ncols_valid && r < k_bits) ? __ldg(B + (bcol0 + col) * sb + b_row0 + r) : 0ull;
    }
    sync();
    uint64_t rows[2][8];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const int it = threadIdx.x + q * NTH;
        const int col = it & (kTabCols - 1);
        const int cg = it >> 4;
        const int t = cg < 32 ? (cg >> 2) : 8;
        const int sz = t < 8 ? 7 : 8;
#pragma unroll
        for (int b = 0; b < 8; ++b)
            rows[q][b] = (it < total && b < sz) ? stage[col * kStagePitch + 7 * t + b] : 0ull;
    }
    sync();
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const int it = threadIdx.x + q * NTH;
        if (it >= total) break;
        const int col = it & (kTabCols - 1);
        const int cg = it >> 4;
        const int t = cg < 32 ? (cg >> 2) : 8;
        const int chunk = cg < 32 ? (cg & 3) : cg - 32;
        uint64_t cur = 0;
#pragma unroll
        for (int hb = 0; hb < 3; ++hb)
            if ((chunk >> hb) & 1) cur ^= rows[q][5 + hb];
        uint64_t* dst = tab + (size_t(128 * t + chunk * 32) * kTabCols + col);
        uint64_t v[32];
        v[0] = cur;
#pragma unroll
        for (int b = 0; b < 5; ++b)
#pragma unroll
            for (int g = 1 << b; g < (2 << b); ++g) v[g] = v[g - (1 << b)] ^ rows[q][b];
#pragma unroll
        for (int g = 0; g < 32; ++g) dst[g * kTabCols] = v[g];
    }
}

// XOR of the nt table entries addressed by the groups of `a`
__device__ __forceinline__ uint64_t lookup(const uint64_t* __restrict__ tl, uint64_t a, int nt) {
    uint64_t acc = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t)
        if (t < nt) acc ^= tl[(128 * t + int((a >> (7 * t)) & 127)) * kTabCols];
    if (nt > 8) acc ^= tl[(1024 + int(a >> 56)) * kTabCols];
    return acc;
}

// Lookup with the table at a FIXED shared-window address (kTabAddr): the byte
// offset of entry g of table t for column col is t*16384 + g*128 + col*8, so a
// lookup is one shift + one LOP3 ((x & 0x3F80) | col*8) + LDS [reg + t*16384 + kTabAddr].
constexpr uint32_t kTabAddr = 0x10000;
template <int T>
__device__ __forceinline__ uint32_t tab_off(uint32_t lo, uint32_t hi, uint32_t colofs) {
    // byte offset of the entry selected by group T of the 64-bit word (hi:lo)
    uint32_t x;
    if (T == 0) x = lo << 7;
    else if (T == 1) x = lo;
    else if (T == 2) x = lo >> 7;
    else if (T == 3) x = lo >> 14;
    else if (T == 4) x = __funnelshift_r(lo, hi, 21);
    else if (T == 5) x = __funnelshift_r(lo, hi, 28);
    else if (T == 6) x = hi >> 3;
    else if (T == 7) x = hi >> 10;
    else x = hi >> 17;  // 8-bit group at bit 56
    return T == 8 ? ((x & 0x7F80u) | colofs) : ((x & 0x3F80u) | colofs);
}
template <int T>
__device__ __forceinline__ void lds_tab(uint32_t off, uint32_t& a, uint32_t& b) {
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2 + %3];"
                 : "=r"(a), "=r"(b)
                 : "r"(off), "n"(kTabAddr + T * 16384));
}
template <int T>
__device__ __forceinline__ void lds_tab2(uint32_t off, uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4 + %5];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                 : "r"(off), "n"(kTabAddr + T * 16384));
}
// two adjacent columns (colofs = 16-byte offset of the pair) from one 128-bit load per
// group: half the index arithmetic and half the shared-load instructions of two lookup9
template <int T>
__device__ __forceinline__ void lk2(uint32_t lo, uint32_t hi, uint32_t colofs, uint32_t (&acc)[4]) {
    uint32_t a, b, c, d;
    lds_tab2<T>(tab_off<T>(lo, hi, colofs), a, b, c, d);
    acc[0] ^= a; acc[1] ^= b; acc[2] ^= c; acc[3] ^= d;
}
__device__ __forceinline__ void lookup9x2(uint32_t colofs, uint64_t w, uint64_t& d0, uint64_t& d1) {
    const uint32_t lo = uint32_t(w), hi = uint32_t(w >> 32);
    uint32_t acc[4] = {0u, 0u, 0u, 0u};
    lk2<0>(lo, hi, colofs, acc); lk2<1>(lo, hi, colofs, acc); lk2<2>(lo, hi, colofs, acc);
    lk2<3>(lo, hi, colofs, acc); lk2<4>(lo, hi, colofs, acc); lk2<5>(lo, hi, colofs, acc);
    lk2<6>(lo, hi, colofs, acc); lk2<7>(lo, hi, colofs, acc); lk2<8>(lo, hi, colofs, acc);
    d0 = (uint64_t(acc[1]) << 32) | acc[0];
    d1 = (uint64_t(acc[3]) << 32) | acc[2];
}
// all 9 groups (full 64-bit k-block), branch-free
__device__ __forceinline__ uint64_t lookup9(uint32_t colofs, uint64_t w) {
    const uint32_t lo = uint32_t(w), hi = uint32_t(w >> 32);
    uint32_t a0, b0, a1, b1, a2, b2, a3, b3, a4, b4, a5, b5, a6, b6, a7, b7, a8, b8;
    lds_tab<0>(tab_off<0>(lo, hi, colofs), a0, b0);
    lds_tab<1>(tab_off<1>(lo, hi, colofs), a1, b1);
    lds_tab<2>(tab_off<2>(lo, hi, colofs), a2, b2);
    lds_tab<3>(tab_off<3>(lo, hi, colofs), a3, b3);
    lds_tab<4>(tab_off<4>(lo, hi, colofs), a4, b4);
    lds_tab<5>(tab_off<5>(lo, hi, colofs), a5, b5);
    lds_tab<6>(tab_off<6>(lo, hi, colofs), a6, b6);
    lds_tab<7>(tab_off<7>(lo, hi, colofs), a7, b7);
    lds_tab<8>(tab_off<8>(lo, hi, colofs), a8, b8);
    const uint32_t x = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7 ^ a8;
    const uint32_t y = b0 ^ b1 ^ b2 ^ b3 ^ b4 ^ b5 ^ b6 ^ b7 ^ b8;
    return (uint64_t(y) << 32) | x;
}

// XOR of the nt (<= 9) entries addressed by the groups of word (hi:lo)
__device__ __forceinline__ uint64_t lookup_fixed(uint32_t colofs, uint64_t w, int nt) {
    const uint32_t lo = uint32_t(w), hi = uint32_t(w >> 32);
    uint32_t a0, b0, a1, b1, a2, b2, a3, b3, a4, b4, a5, b5, a6, b6, a7, b7, a8, b8;
    if (nt == 9) {
        lds_tab<0>(tab_off<0>(lo, hi, colofs), a0, b0);
        lds_tab<1>(tab_off<1>(lo, hi, colofs), a1, b1);
        lds_tab<2>(tab_off<2>(lo, hi, colofs), a2, b2);
        lds_tab<3>(tab_off<3>(lo, hi, colofs), a3, b3);
        lds_tab<4>(tab_off<4>(lo, hi, colofs), a4, b4);
        lds_tab<5>(tab_off<5>(lo, hi, colofs), a5, b5);
        lds_tab<6>(tab_off<6>(lo, hi, colofs), a6, b6);
        lds_tab<7>(tab_off<7>(lo, hi, colofs), a7, b7);
        lds_tab<8>(tab_off<8>(lo, hi, colofs), a8, b8);
        const uint32_t x = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7 ^ a8;
        const uint32_t y = b0 ^ b1 ^ b2 ^ b3 ^ b4 ^ b5 ^ b6 ^ b7 ^ b8;
        return (uint64_t(y) << 32) | x;
    }
    uint32_t x = 0, y = 0;
#define F2_LK(T)                                                   \
    if (T < nt) {                                                  \
        lds_tab<T>(tab_off<T>(lo, hi, colofs), a##T, b##T);        \
        x ^= a##T;                                                 \
        y ^= b##T;                                                 \
    }
    F2_LK(0) F2_LK(1) F2_LK(2) F2_LK(3) F2_LK(4) F2_LK(5) F2_LK(6) F2_LK(7) F2_LK(8)
#undef F2_LK
    return (uint64_t(y) << 32) | x;
}

// ---------------------------------------------------------------------------
// K2: fused table build + XOR update (the Schur update / mult_acc)
// ---------------------------------------------------------------------------
// One CTA (512 threads, 160 KiB tables) per SM, persistent over a balanced
// range of 16-row units of the flattened (column group, row unit) space.
// Lane (h, col) of a warp owns rows [a0+8h, a0+8h+8) of column `col` of the
// group: C moves as two 32-byte loads/stores per lane; the two half-warps each
// read one 128-byte table row per lookup.
constexpr int kUpdThreads = 512;

__global__ void __launch_bounds__(kUpdThreads, 1) k_update(UpdateArgs p) {
    extern __shared__ __align__(128) uint64_t tab[];
    size_t row_lo = p.row_lo, b_row0 = p.b_row0;
    int k = p.k_bits;
    if (p.st) {
        const uint32_t R = p.st->R, r = p.st->r;
        row_lo = size_t(R) + r;
        k = int(r);
        b_row0 = R;
    }
    const size_t row_hi = p.row_hi;
    if (k <= 0 || row_lo >= row_hi || p.ncols <= 0) return;
    const int nt = k > 56 ? 9 : (k + 6) / 7;
    const size_t base16 = row_lo & ~size_t(15);
    const size_t U = (row_hi - base16 + 15) / 16;
    const size_t ncg = (size_t(p.ncols) + kTabCols - 1) / kTabCols;
    const size_t TU = U * ncg;
    const size_t u0 = TU * blockIdx.x / gridDim.x;
    const size_t u1 = TU * (blockIdx.x + 1) / gridDim.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int h = lane >> 4, col = lane & 15;

    for (size_t u = u0; u < u1;) {
        const size_t g = u / U;
        const size_t seg_end = u1 < (g + 1) * U ? u1 : (g + 1) * U;
        const int nvalid = int(size_t(p.ncols) - g * kTabCols) < kTabCols
                               ? int(size_t(p.ncols) - g * kTabCols)
                               : kTabCols;
        __syncthreads();
        build_tables<kUpdThreads>(tab, p.B, p.sb, b_row0, p.b_wcol0 + g * kTabCols, nvalid, k,
                                  nt);
        __syncthreads();
        const bool cv = col < nvalid;
        uint64_t* cp = p.C + (p.c_wcol0 + g * kTabCols + col) * p.sc;
        const uint64_t* tl = tab + col;
        for (size_t uu = u + warp; uu < seg_end; uu += kUpdThreads / 32) {
            const size_t a0 = base16 + (uu - g * U) * 16 + 8 * h;
            uint64_t c[8], aw[8];
            const bool full = a0 >= row_lo && a0 + 8 <= row_hi;
            if (cv) {
                ld256(cp + a0, c[0], c[1], c[2], c[3]);
                ld256(cp + a0 + 4, c[4], c[5], c[6], c[7]);
            }
            if (full) {
#pragma unroll
                for (int s = 0; s < 8; ++s) aw[s] = __ldg(p.a + a0 + s);
            } else {
#pragma unroll
                for (int s = 0; s < 8; ++s) {
                    const size_t row = a0 + s;
                    aw[s] = (row >= row_lo && row < row_hi) ? __ldg(p.a + row) : 0ull;
                }
            }
            if (!cv) continue;
#pragma unroll
            for (int s = 0; s < 8; ++s) c[s] ^= lookup(tl, aw[s], nt);
            if (full) {
                st256(cp + a0, c[0], c[1], c[2], c[3]);
                st256(cp + a0 + 4, c[4], c[5], c[6], c[7]);
            } else {
#pragma unroll
                for (int s = 0; s < 8; ++s) {
                    const size_t row = a0 + s;
                    if (row >= row_lo && row < row_hi) cp[row] = c[s];
                }
            }
        }
        u = seg_end;
    }
}

// ---------------------------------------------------------------------------
// bulk-copy helpers of the v3 update
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read1() {
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------------------
// K2 v3: table build + XOR sweep, C updated in place by bulk XOR-reduction
// ---------------------------------------------------------------------------
// ncu history: v1 (LSU loads/stores of C) is L1TEX-data-pipe bound, half of it
// global traffic at one wavefront per 32-byte sector; v2 (bulk-async C staging)
// was instruction/latency bound on the store-then-reload ring.  v3 never brings
// C into the SM: the consumers compute only the update delta
//   D[i, col] = XOR_t T_t[(y_i >> 7t) & mask][col]
// into a shared-memory ring, and the producer warp applies it with
// cp.reduce.async.bulk ... .xor.b64 (UBLKRED): the read-modify-write of C
// happens in L2, so DRAM still sees C once in and once out while the SM's data
// pipe carries only table lookups and the delta stores.  The 128 driving words
// of each tile come through a separate 8-deep bulk-load ring.  Rows outside
// [row_lo, row_hi) get a zero delta (the XOR leaves them unchanged).
#ifndef F2_UPDATE_COL2
#define F2_UPDATE_COL2 1  // consumer lanes own 2 rows x 2 columns (128-bit lookups); 0: 4 rows x 1 column
#endif
constexpr int kV3Warps = 16;                      // consumer warps
constexpr int kV3Threads = (kV3Warps + 1) * 32;   // + producer warp
constexpr int kV3Rows = 128;                      // tile rows (lane owns 4)
constexpr int kV3DStages = 3;
constexpr int kV3AStages = 8;
constexpr int kV3ColPitch = kV3Rows * 8 + 16;     // 1040 B: conflict-free 128-bit smem access
constexpr int kV3DBytes = kTabCols * kV3ColPitch; // 16640 B per delta tile
constexpr int kV3ABytes = kV3Rows * 8;            // 1 KiB of driving words
constexpr size_t kV3RingBytes = size_t(kV3DStages) * kV3DBytes + size_t(kV3AStages) * kV3ABytes + 256;
// dynamic smem: [rings + barriers | pad] below kTabAddr, then the tables at kTabAddr
// (the dynamic window starts at most 1 KiB into the shared address space)
constexpr size_t kV3Smem = kTabAddr + kTabBytes;
static_assert(kV3RingBytes + 1024 <= kTabAddr, "rings must fit below the table window");
static_assert(kV3Smem <= 232448, "exceeds the 227 KiB per-CTA limit");

__device__ __forceinline__ void bulk_red_xor(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.xor.b64 [%0], [%1], %2;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void v3_consumers_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(kV3Warps * 32) : "memory");
}

// per-CTA tile sequence: up to two contiguous segments of the flattened
// (group, tile) space, walked with incremental cursors (no per-tile divides)
struct TileCursor {
    size_t T, g, tt, i, len0, s1;
    __device__ void init(size_t T_, size_t s0, size_t len0_, size_t s1_) {
        T = T_; i = 0; len0 = len0_; s1 = s1_;
        const size_t u = len0 ? s0 : s1;
        g = u / T; tt = u % T;
    }
    __device__ void next() {
        if (++i == len0) { g = s1 / T; tt = s1 % T; }
        else if (++tt == T) { tt = 0; ++g; }
    }
};

__device__ __forceinline__ void release_signal(uint32_t* flag, int tag = -1) {
    __threadfence();
    if (tag >= 0) {  // tag >= 0 only while the device trace is on
        if (atomicAdd(flag, 1u) + 1 == gridDim.x) trace_ev(kTrUpdRelease, tag);
    } else {
        atomicAdd(flag, 1u);
    }
}

__global__ void __launch_bounds__(kV3Threads, 1) k_update_v3(UpdateArgs p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // programmatic dependent launch: no-op unless launched with p.pdl; every read
    // of the panel state, A, B or C comes after it
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (p.tag >= 0 && blockIdx.x == 0 && threadIdx.x == 0) trace_ev(kTrUpdBegin, p.tag);
    const uint32_t smem_base = smem_u32(smem_raw);
    if (smem_base > kTabAddr - kV3RingBytes) __trap();  // layout assumption violated
    uint64_t* tab = reinterpret_cast<uint64_t*>(smem_raw + (kTabAddr - smem_base));
    unsigned char* dring = smem_raw;
    unsigned char* aring = dring + size_t(kV3DStages) * kV3DBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(aring + size_t(kV3AStages) * kV3ABytes);
    uint64_t* a_full = bars;                       // [kV3AStages] tx barrier
    uint64_t* a_empty = a_full + kV3AStages;       // [kV3AStages] consumer warps
    uint64_t* d_done = a_empty + kV3AStages;       // [kV3DStages] consumer warps
    uint64_t* d_free = d_done + kV3DStages;        // [kV3DStages] producer

    size_t row_lo = p.row_lo, b_row0 = p.b_row0;
    int k = p.k_bits;
    if (p.st) {
        const uint32_t R = p.st->R, r = p.st->r;
        row_lo = size_t(R) + r;
        k = int(r);
        b_row0 = R;
    }
    const size_t row_hi = p.row_hi;
    if (p.tag >= 0 && blockIdx.x == 0 && threadIdx.x == 0) trace_ev(14, int(p.tag + 0 * k));
    if (k <= 0 || row_lo >= row_hi || p.ncols <= 0) {
        if (p.release && threadIdx.x == 0) release_signal(p.release, p.tag);
        return;
    }
    // first-column CTAs: [G - F, G) (F = 0: none, the split is uniform)
    const size_t G_all = gridDim.x;
    size_t fc_n = 0;
    if (p.release && p.first_col)
        fc_n = p.fc_ctas > 0 ? min(G_all, size_t(p.fc_ctas)) : G_all;
    const bool fc_mine = fc_n != 0 && blockIdx.x >= G_all - fc_n;
    if (fc_n != 0 && !fc_mine) {
        // never writes the first column: its arrival is vacuous
        if (threadIdx.x == 0) release_signal(p.release, p.tag);
        p.release = nullptr;
        ++p.c_wcol0;
        ++p.b_wcol0;
        if (--p.ncols <= 0) return;
    }
    if (fc_mine) {
        // the first column alone: one 256-entry 4-bit table over its 64 B rows,
        // rows split evenly over the first-column CTAs, plain loads/stores -- the
        // release the next panel kernel waits for comes ~2-3 us after launch instead
        // of after a whole 16-column group (table build + tile pipeline + bulk drain)
        uint64_t* t4 = tab;
        const uint64_t* Bc = p.B + p.b_wcol0 * p.sb + b_row0;
        if (threadIdx.x < 256) {
            const int g = threadIdx.x >> 4, v = threadIdx.x & 15;
            uint64_t x = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (((v >> q) & 1) && 4 * g + q < k) x ^= __ldg(Bc + 4 * g + q);
            t4[threadIdx.x] = x;
        }
        __syncthreads();
        uint64_t* Cc = p.C + p.c_wcol0 * p.sc;
        const size_t nrows = row_hi - row_lo, per = (nrows + fc_n - 1) / fc_n;
        const size_t r0 = row_lo + size_t(blockIdx.x - (G_all - fc_n)) * per, r1 = min(row_hi, r0 + per);
        // 4 rows per thread in flight (a first-column CTA has ~4096 rows at 65536)
        for (size_t i0 = r0 + threadIdx.x; i0 < r1; i0 += 4 * size_t(blockDim.x)) {
            uint64_t a[4], x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const size_t i = i0 + size_t(u) * blockDim.x;
                a[u] = i < r1 ? p.a[i] : 0;
                x[u] = i < r1 ? Cc[i] : 0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const size_t i = i0 + size_t(u) * blockDim.x;
#pragma unroll
                for (int g = 0; g < 16; ++g) x[u] ^= t4[16 * g + int((a[u] >> (4 * g)) & 15)];
                if (i < r1) Cc[i] = x[u];
            }
        }
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) release_signal(p.release, p.tag);
        __syncthreads();  // t4 lives where the group tables go
        p.release = nullptr;
        ++p.c_wcol0;
        ++p.b_wcol0;
        if (--p.ncols <= 0) return;
    }
    const int nt = 9;  // all tables built (rows >= k are zero); lookup9 is branch-free
    const size_t base = row_lo & ~size_t(kV3Rows - 1);
    const size_t T = (row_hi - base + kV3Rows - 1) / kV3Rows;  // tiles per column group
    const size_t ncg = (size_t(p.ncols) + kTabCols - 1) / kTabCols;
    const size_t G = gridDim.x, b = blockIdx.x;
    size_t s0, len0, s1, len1;
    if (p.release) {  // group 0 spread over every CTA first, then the rest
        s0 = T * b / G;
        len0 = T * (b + 1) / G - s0;
        const size_t TB = T * (ncg - 1);
        s1 = T + TB * b / G;
        len1 = T + TB * (b + 1) / G - s1;
    } else if (fc_n != 0 && fc_n < G && p.fc_weight < 4) {
        // weighted split: the first-column CTAs take fc_weight/4 of a share
        const size_t TU = T * ncg, d = size_t(4 - p.fc_weight), gf = G - fc_n;
        const size_t Wt = 4 * G - d * fc_n;
        auto W = [&](size_t x) { return 4 * x - d * (x > gf ? x - gf : 0); };
        s0 = TU * W(b) / Wt;
        len0 = TU * W(b + 1) / Wt - s0;
        s1 = s0 + len0;
        len1 = 0;
    } else {
        const size_t TU = T * ncg;
        s0 = TU * b / G;
        len0 = TU * (b + 1) / G - s0;
        s1 = s0 + len0;
        len1 = 0;
    }
    const size_t cnt = len0 + len1;
    if (cnt == 0) {
        if (p.release && threadIdx.x == 0) release_signal(p.release, p.tag);
        return;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kV3AStages; ++s) {
            mbar_init(&a_full[s], 1);
            mbar_init(&a_empty[s], kV3Warps);
        }
        for (int s = 0; s < kV3DStages; ++s) {
            mbar_init(&d_done[s], kV3Warps);
            mbar_init(&d_free[s], 1);
        }
        fence_async_smem();
    }
    __syncthreads();
    if (p.tag >= 0 && blockIdx.x == 0 && threadIdx.x == 0) trace_ev(15, p.tag);

    if (warp == kV3Warps) {
        // ===== producer warp =====
        TileCursor ac;
        ac.init(T, s0, len0, s1);
        uint32_t a_stage = 0;
        auto issue_a = [&]() {
            if (lane == 0) {
                mbar_expect_tx(&a_full[a_stage], kV3ABytes);
                bulk_g2s(aring + size_t(a_stage) * kV3ABytes, p.a + base + ac.tt * kV3Rows,
                         kV3ABytes, &a_full[a_stage]);
            }
            ac.next();
            if (++a_stage == kV3AStages) a_stage = 0;
        };
        if (p.release && len0 == 0 && lane == 0) release_signal(p.release, p.tag);
        const size_t pre = cnt < size_t(kV3AStages) ? cnt : size_t(kV3AStages);
        for (size_t i = 0; i < pre; ++i) issue_a();
        TileCursor dc;
        dc.init(T, s0, len0, s1);
        int s = 0, ae = 0;
        uint32_t dph = 0, aph = 0;
        // Pipelined write-back: tile t's reductions are committed, and the stage of
        // tile t-1 is released once ITS reductions have read shared memory
        // (wait_group.read 1), so the producer never blocks on the tile it just issued.
#if F2_PIPELINED_WRITEBACK
        int sprev = -1;
#endif
        for (size_t t = 0; t < cnt; ++t) {
            const size_t r0 = base + dc.tt * kV3Rows;
            const int nvalid = min(kTabCols, int(size_t(p.ncols) - dc.g * kTabCols));
            mbar_wait(&d_done[s], dph);
            // consumers' generic-proxy smem writes (released by their d_done arrivals,
            // acquired by the wait above) -> ordered before the async-proxy reads of
            // the bulk reductions by one cumulative proxy fence here
#if F2_FENCE_IN_PRODUCER
            fence_async_smem();
#endif
            const bool issued = lane < nvalid;
            if (issued) {
                bulk_red_xor(p.C + (p.c_wcol0 + dc.g * kTabCols + lane) * p.sc + r0,
                             dring + size_t(s) * kV3DBytes + lane * kV3ColPitch, kV3ABytes);
                bulk_commit();
            }
            const bool rel_point = p.release && t + 1 == len0;
            if (t == 0 && p.tag >= 0 && blockIdx.x == 0 && lane == 0) trace_ev(11, p.tag);
#if F2_PIPELINED_WRITEBACK
            if (rel_point) bulk_wait0();          // group-0 writes complete in memory
            else if (issued) bulk_wait_read1();   // previous tile's reads done
            else bulk_wait_read0();
            __syncwarp();
            if (rel_point && lane == 0) release_signal(p.release, p.tag);
            if (lane == 0) {
                if (rel_point) mbar_arrive(&d_free[s]);  // everything drained
                if (sprev >= 0) mbar_arrive(&d_free[sprev]);
            }
            sprev = rel_point ? -1 : s;
#else
            if (rel_point) bulk_wait0();          // group-0 writes complete in memory
            else bulk_wait_read0();               // this tile's reads done
            __syncwarp();
            if (rel_point && lane == 0) release_signal(p.release, p.tag);
            if (lane == 0) mbar_arrive(&d_free[s]);
#endif
            if (t + kV3AStages < cnt) {
                mbar_wait(&a_empty[ae], aph);
                issue_a();
            }
            if (++ae == kV3AStages) { ae = 0; aph ^= 1; }
            if (++s == kV3DStages) { s = 0; dph ^= 1; }
            dc.next();
        }
        bulk_wait0();
        if (p.tag >= 0 && blockIdx.x == 0 && lane == 0) trace_ev(12, p.tag);
        // (the last tile's stage needs no release: no consumer waits for it)
        return;
    }

    // ===== consumer warps =====
#if F2_UPDATE_COL2
    // lane = (row pair r4 = lane >> 3, column pair c8 = lane & 7): rows 8 w + 2 r4 (+1),
    // columns 2 c8 (+1) -- one 128-bit table load serves two columns; a quarter-warp
    // reads one whole 128-byte entry (conflict-free)
    const int r4 = lane >> 3, c8 = lane & 7;
    const uint32_t colofs = uint32_t(c8) * 16u;
    const int rl = 8 * warp + 2 * r4;
#else
    const int h = lane >> 4, col = lane & 15;
    const uint32_t colofs = uint32_t(col) * 8u;
    const int rl = 8 * warp + 4 * h;  // this lane's 4 rows within the tile
#endif
    size_t gcur = ~size_t(0);
    TileCursor cc;
    cc.init(T, s0, len0, s1);
    int as = 0, s = 0;
    uint32_t aph = 0, dph = 0;
    for (size_t t = 0; t < cnt; ++t) {
        const size_t g = cc.g;
        if (g != gcur) {
            v3_consumers_sync();
            const int nvalid = min(kTabCols, int(size_t(p.ncols) - g * kTabCols));
            build_tables_staged<kV3Warps * 32>(tab, p.B, p.sb, b_row0, p.b_wcol0 + g * kTabCols, nvalid, k,
                                               [] { v3_consumers_sync(); });
            v3_consumers_sync();
            if (p.tag >= 0 && gcur == ~size_t(0) && blockIdx.x == 0 && threadIdx.x == 0) trace_ev(10, p.tag);
            gcur = g;
        }
        mbar_wait(&a_full[as], aph);
#if F2_UPDATE_COL2
        const ulonglong2 av = *(reinterpret_cast<const ulonglong2*>(aring + size_t(as) * kV3ABytes) + rl / 2);
        uint64_t x[2] = {av.x, av.y};
        const size_t row = base + cc.tt * kV3Rows + rl;
        if (row < row_lo || row + 2 > row_hi) {
#pragma unroll
            for (int q = 0; q < 2; ++q)
                if (row + q < row_lo || row + q >= row_hi) x[q] = 0;
        }
        uint64_t d[2][2];
#pragma unroll
        for (int q = 0; q < 2; ++q) lookup9x2(colofs, x[q], d[q][0], d[q][1]);
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_empty[as]);
        if (t >= size_t(kV3DStages)) mbar_wait(&d_free[s], dph ^ 1);
        // store j writes column 2 c8 + (j ^ hb): the 8 lanes of a quarter-warp then hit 8
        // distinct column residues mod 8, i.e. 8 distinct 16-byte bank groups at the
        // 1040-byte column pitch (j alone would pair columns c and c + 8: 2-way conflicts)
        const int hb = (c8 >> 2) & 1;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int c = j ^ hb;
            ulonglong2* dp = reinterpret_cast<ulonglong2*>(dring + size_t(s) * kV3DBytes +
                                                           (2 * c8 + c) * kV3ColPitch) + rl / 2;
            dp[0] = c ? make_ulonglong2(d[0][1], d[1][1]) : make_ulonglong2(d[0][0], d[1][0]);
        }
#else
        const ulonglong2* ap = reinterpret_cast<const ulonglong2*>(aring + size_t(as) * kV3ABytes) + rl / 2;
        uint64_t x[4];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const ulonglong2 v = ap[q];
            x[2 * q] = v.x;
            x[2 * q + 1] = v.y;
        }
        const size_t row = base + cc.tt * kV3Rows + rl;
        if (row < row_lo || row + 4 > row_hi) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (row + q < row_lo || row + q >= row_hi) x[q] = 0;
        }
        uint64_t d[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) d[q] = lookup9(colofs, x[q]);
        // release the A stage only once every lane has CONSUMED its words: an
        // mbarrier arrive is not ordered behind the warp's outstanding shared loads,
        // so arriving right after the LDS could let the next bulk load overwrite them
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_empty[as]);
        if (t >= size_t(kV3DStages)) mbar_wait(&d_free[s], dph ^ 1);
        ulonglong2* dp = reinterpret_cast<ulonglong2*>(dring + size_t(s) * kV3DBytes + col * kV3ColPitch) + rl / 2;
        dp[0] = make_ulonglong2(d[0], d[1]);
        dp[1] = make_ulonglong2(d[2], d[3]);
#endif
#if !F2_FENCE_IN_PRODUCER
        fence_async_smem();  // generic-proxy smem writes -> async-proxy bulk reductions
#endif
        __syncwarp();
        if (lane == 0) mbar_arrive(&d_done[s]);
        if (++as == kV3AStages) { as = 0; aph ^= 1; }
        if (++s == kV3DStages) { s = 0; dph ^= 1; }
        cc.next();
    }
}

// ---------------------------------------------------------------------------
// K2 v4: the same delta + bulk-XOR design over 8-column groups with 8-bit tables
// ---------------------------------------------------------------------------
// v3 is bound by the shared-memory data pipe: 9 table lookups of 8 B per output
// word (16 columns x 1280 entries = 160 KiB).  With 8 columns per group the same
// space holds eight 8-bit tables (8 x 256 entries x 64 B = 128 KiB): 8 lookups
// per output word, and 32 KiB more for the delta ring.  A 64-byte entry is half a
// bank row, so tables 2p and 2p+1 share region p, one in each half:
//   byte offset of entry g of table t, column c = (t>>1)*32 KiB + g*128 + (t&1)*64 + 8c.
// A quarter-warp (8 lanes x 16 B) holds two row slots of 4 lanes; at step s the even
// slot reads table s and the odd slot table s^1, i.e. the two halves of one
// region: every 128-bit lookup is conflict-free, and each slot still visits all
// eight tables.  The odd slot's driving word has its adjacent bytes swapped
// (PRMT) so both slots take byte s.  The table sits at a 32 KiB-aligned shared
// address, so base, half and column fold into one LOP3 with the index.
// Measured at the north-star unit (C 65536^2 ^= A(65536x64) B(64x65536), tools/upd_time.py):
//   v3 243.9 us; v4 16 warps 243 -> 222 us (producer loop restructured); 20 warps 213.5;
//   24 warps 193-194 us = 5.55 TB/s (0.85 of the measured HBM copy peak); 28 / 30 warps
//   (64 registers) 205 / 211.  Two delta stages beat three or four (206 vs 213 at 20 warps),
//   one is slower (196.8).  Write-back depth > 0 (F2_V4_PIPE) and one producer-side proxy
//   fence per tile (F2_V4_FENCE_PRODUCER) were slower (246 / 228.6 us at 16 warps).
//   Diagnostic modes at 16 warps: no lookups 205 us (the write-back alone), no write-back
//   185 us (the lookups alone), no delta stores 226 us.
#ifndef F2_V4_PIPE
#define F2_V4_PIPE 0  // tiles whose write-back reductions may still read shared memory (< stages)
#endif
#ifndef F2_V4_FENCE_PRODUCER
#define F2_V4_FENCE_PRODUCER 0  // one proxy fence per tile in the producer instead of one per consumer warp
#endif
#ifndef F2_V4_DSTAGES
#define F2_V4_DSTAGES 2
#endif
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
#ifndef F2_V4_MODE
#define F2_V4_MODE 0  // diagnostics: 1 no lookups, 2 no write-back, 3 no delta stores
#endif
constexpr int kV4Cols = 8;
#ifndef F2_V4_WARPS
#define F2_V4_WARPS 24
#endif
constexpr int kV4Warps = F2_V4_WARPS;              // consumer warps
constexpr int kV4Threads = (kV4Warps + 1) * 32;
constexpr int kV4Rows = 16 * kV4Warps;             // tile rows: 8 slots x 2 rows per warp
constexpr int kV4DStages = F2_V4_DSTAGES;
static_assert(F2_V4_PIPE < F2_V4_DSTAGES && F2_V4_DSTAGES <= 4, "pipelined write-back depth");
constexpr int kV4AStages = 6;
constexpr int kV4ColPitch = kV4Rows * 8 + 16;      // 2064 B: conflict-free 128-bit delta stores
constexpr int kV4DBytes = kV4Cols * kV4ColPitch;   // 16512 B per delta tile
constexpr int kV4ABytes = kV4Rows * 8;             // 2 KiB of driving words
constexpr uint32_t kV4TabAddr = 0x8000;            // 32 KiB-aligned (bits disjoint from the index)
constexpr uint32_t kV4TabBytes = 4u * 32768u;      // 128 KiB
constexpr uint32_t kV4LowBytes = uint32_t(kV4AStages) * kV4ABytes + 256;  // A ring + barriers, below
constexpr size_t kV4Smem = size_t(kV4TabAddr) + kV4TabBytes + size_t(kV4DStages) * kV4DBytes;
static_assert(kV4LowBytes + 1024 <= kV4TabAddr, "A ring must fit below the table window");
static_assert(kV4Smem <= 232448, "exceeds the 227 KiB per-CTA limit");

__device__ __forceinline__ void v4_consumers_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(kV4Warps * 32) : "memory");
}

// one lookup of step S: byte S of the (byte-pair-swapped for odd slots) word,
// table region S/2, half and column pair in `co` (with the table base bit)
template <int S>
__device__ __forceinline__ void lk8(uint32_t lo, uint32_t hi, uint32_t co, uint32_t (&acc)[4]) {
    const uint32_t u = S < 4 ? lo : hi;
    uint32_t x;
    if ((S & 3) == 0) x = u << 7;
    else if ((S & 3) == 1) x = u >> 1;
    else if ((S & 3) == 2) x = u >> 9;
    else x = u >> 17;
    const uint32_t off = (x & 0x7F80u) | co;
    uint32_t a, b, c, d;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4 + %5];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                 : "r"(off), "n"((S >> 1) * 32768));
    acc[0] ^= a; acc[1] ^= b; acc[2] ^= c; acc[3] ^= d;
}
__device__ __forceinline__ void lookup8x2(uint32_t sel, uint32_t co_e, uint32_t co_o, uint64_t w,
                                          uint64_t& d0, uint64_t& d1) {
    const uint32_t lo = __byte_perm(uint32_t(w), 0u, sel), hi = __byte_perm(uint32_t(w >> 32), 0u, sel);
    uint32_t acc[4] = {0u, 0u, 0u, 0u};
    lk8<0>(lo, hi, co_e, acc); lk8<1>(lo, hi, co_o, acc); lk8<2>(lo, hi, co_e, acc); lk8<3>(lo, hi, co_o, acc);
    lk8<4>(lo, hi, co_e, acc); lk8<5>(lo, hi, co_o, acc); lk8<6>(lo, hi, co_e, acc); lk8<7>(lo, hi, co_o, acc);
    d0 = (uint64_t(acc[1]) << 32) | acc[0];
    d1 = (uint64_t(acc[3]) << 32) | acc[2];
}

// the eight 8-bit tables of one 8-column group (512 consumer threads, one
// 32-entry item each: column, half, region, chunk), B staged through the table
// space first (coalesced), doubling in registers (m4rm.hpp:74-88)
__device__ __forceinline__ void build_tables8(unsigned char* tabb, const uint64_t* __restrict__ B, size_t sb,
                                              size_t b_row0, size_t bcol0, int ncols_valid, int k_bits) {
    static_assert(kV4Warps * 32 >= 512, "one item per consumer thread");
    uint64_t* stage = reinterpret_cast<uint64_t*>(tabb);
    const int it = threadIdx.x;
    if (it < 512) {
        const int col = it >> 6, r = it & 63;
        stage[col * kStagePitch + r] =
            (col < ncols_valid && r < k_bits) ? __ldg(B + (bcol0 + col) * sb + b_row0 + r) : 0ull;
    }
    v4_consumers_sync();
    const int col = it & 7, half = (it >> 3) & 1, reg = (it >> 4) & 3, chunk = it >> 6;
    const int t = 2 * reg + half;
    uint64_t rows[8];
#pragma unroll
    for (int b = 0; b < 8; ++b) rows[b] = it < 512 ? stage[col * kStagePitch + 8 * t + b] : 0ull;
    v4_consumers_sync();
    if (it >= 512) return;
    uint64_t cur = 0;
#pragma unroll
    for (int hb = 0; hb < 3; ++hb)
        if ((chunk >> hb) & 1) cur ^= rows[5 + hb];
    uint64_t* dst = reinterpret_cast<uint64_t*>(tabb + size_t(reg) * 32768 + size_t(chunk * 32) * 128 +
                                                half * 64 + col * 8);
    uint64_t v[32];
    v[0] = cur;
#pragma unroll
    for (int b = 0; b < 5; ++b)
#pragma unroll
        for (int g = 1 << b; g < (2 << b); ++g) v[g] = v[g - (1 << b)] ^ rows[b];
#pragma unroll
    for (int g = 0; g < 32; ++g) dst[g * 16] = v[g];
}

__global__ void __launch_bounds__(kV4Threads, 1) k_update_v4(UpdateArgs p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (p.tag >= 0 && blockIdx.x == 0 && threadIdx.x == 0) trace_ev(kTrUpdBegin, p.tag);
    const uint32_t smem_base = smem_u32(smem_raw);
    if (smem_base > kV4TabAddr - kV4LowBytes) __trap();  // layout assumption violated
    unsigned char* tabb = smem_raw + (kV4TabAddr - smem_base);
    unsigned char* aring = tabb - kV4LowBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(aring + size_t(kV4AStages) * kV4ABytes);
    unsigned char* dring = tabb + kV4TabBytes;
    uint64_t* a_full = bars;
    uint64_t* a_empty = a_full + kV4AStages;
    uint64_t* d_done = a_empty + kV4AStages;
    uint64_t* d_free = d_done + kV4DStages;

    size_t row_lo = p.row_lo, b_row0 = p.b_row0;
    int k = p.k_bits;
    if (p.st) {
        const uint32_t R = p.st->R, r = p.st->r;
        row_lo = size_t(R) + r;
        k = int(r);
        b_row0 = R;
    }
    const size_t row_hi = p.row_hi;
    if (k <= 0 || row_lo >= row_hi || p.ncols <= 0) {
        if (p.release && threadIdx.x == 0) release_signal(p.release, p.tag);
        return;
    }
    const size_t G_all = gridDim.x;
    size_t fc_n = 0;
    if (p.release && p.first_col)
        fc_n = p.fc_ctas > 0 ? min(G_all, size_t(p.fc_ctas)) : G_all;
    const bool fc_mine = fc_n != 0 && blockIdx.x >= G_all - fc_n;
    if (fc_n != 0 && !fc_mine) {
        if (threadIdx.x == 0) release_signal(p.release, p.tag);
        p.release = nullptr;
        ++p.c_wcol0;
        ++p.b_wcol0;
        if (--p.ncols <= 0) return;
    }
    if (fc_mine) {
        // the first column alone (as in k_update_v3): 4-bit table, rows split over
        // the first-column CTAs, plain loads/stores, then the release
        uint64_t* t4 = reinterpret_cast<uint64_t*>(tabb);
        const uint64_t* Bc = p.B + p.b_wcol0 * p.sb + b_row0;
        if (threadIdx.x < 256) {
            const int g = threadIdx.x >> 4, v = threadIdx.x & 15;
            uint64_t x = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (((v >> q) & 1) && 4 * g + q < k) x ^= __ldg(Bc + 4 * g + q);
            t4[threadIdx.x] = x;
        }
        __syncthreads();
        uint64_t* Cc = p.C + p.c_wcol0 * p.sc;
        const size_t nrows = row_hi - row_lo, per = (nrows + fc_n - 1) / fc_n;
        const size_t r0 = row_lo + size_t(blockIdx.x - (G_all - fc_n)) * per, r1 = min(row_hi, r0 + per);
        for (size_t i0 = r0 + threadIdx.x; i0 < r1; i0 += 4 * size_t(blockDim.x)) {
            uint64_t a[4], x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const size_t i = i0 + size_t(u) * blockDim.x;
                a[u] = i < r1 ? p.a[i] : 0;
                x[u] = i < r1 ? Cc[i] : 0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const size_t i = i0 + size_t(u) * blockDim.x;
#pragma unroll
                for (int g = 0; g < 16; ++g) x[u] ^= t4[16 * g + int((a[u] >> (4 * g)) & 15)];
                if (i < r1) Cc[i] = x[u];
            }
        }
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) release_signal(p.release, p.tag);
        __syncthreads();
        p.release = nullptr;
        ++p.c_wcol0;
        ++p.b_wcol0;
        if (--p.ncols <= 0) return;
    }
    const size_t base = row_lo & ~size_t(127);
    const size_t T = (row_hi - base + kV4Rows - 1) / kV4Rows;
    const size_t ncg = (size_t(p.ncols) + kV4Cols - 1) / kV4Cols;
    const size_t row_end = (row_hi + 1) & ~size_t(1);  // bulk sizes in 16-byte units
    const size_t G = gridDim.x, b = blockIdx.x;
    size_t s0, len0, s1, len1;
    if (p.release) {
        s0 = T * b / G;
        len0 = T * (b + 1) / G - s0;
        const size_t TB = T * (ncg - 1);
        s1 = T + TB * b / G;
        len1 = T + TB * (b + 1) / G - s1;
    } else if (fc_n != 0 && fc_n < G && p.fc_weight < 4) {
        const size_t TU = T * ncg, d = size_t(4 - p.fc_weight), gf = G - fc_n;
        const size_t Wt = 4 * G - d * fc_n;
        auto W = [&](size_t x) { return 4 * x - d * (x > gf ? x - gf : 0); };
        s0 = TU * W(b) / Wt;
        len0 = TU * W(b + 1) / Wt - s0;
        s1 = s0 + len0;
        len1 = 0;
    } else {
        const size_t TU = T * ncg;
        s0 = TU * b / G;
        len0 = TU * (b + 1) / G - s0;
        s1 = s0 + len0;
        len1 = 0;
    }
    const size_t cnt = len0 + len1;
    if (cnt == 0) {
        if (p.release && threadIdx.x == 0) release_signal(p.release, p.tag);
        return;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kV4AStages; ++s) {
            mbar_init(&a_full[s], 1);
            mbar_init(&a_empty[s], kV4Warps);
        }
        for (int s = 0; s < kV4DStages; ++s) {
            mbar_init(&d_done[s], kV4Warps);
            mbar_init(&d_free[s], 1);
        }
        fence_async_smem();
    }
    __syncthreads();

    if (warp == kV4Warps) {
        // ===== producer warp =====
        TileCursor ac;
        ac.init(T, s0, len0, s1);
        uint32_t a_stage = 0;
        auto issue_a = [&]() {
            if (lane == 0) {
                const size_t r0 = base + ac.tt * kV4Rows;
                const uint32_t bytes = uint32_t(min(size_t(kV4Rows), row_end - r0) * 8);
                mbar_expect_tx(&a_full[a_stage], bytes);
                bulk_g2s(aring + size_t(a_stage) * kV4ABytes, p.a + r0, bytes, &a_full[a_stage]);
            }
            ac.next();
            if (++a_stage == kV4AStages) a_stage = 0;
        };
        if (p.release && len0 == 0 && lane == 0) release_signal(p.release, p.tag);
        const size_t pre = cnt < size_t(kV4AStages) ? cnt : size_t(kV4AStages);
        for (size_t i = 0; i < pre; ++i) issue_a();
        TileCursor dc;
        dc.init(T, s0, len0, s1);
        int s = 0, ae = 0;
        uint32_t dph = 0, aph = 0;
        int pq[4], pq0 = 0, npend = 0;
        for (size_t t = 0; t < cnt; ++t) {
            const size_t r0 = base + dc.tt * kV4Rows;
            const uint32_t bytes = uint32_t(min(size_t(kV4Rows), row_end - r0) * 8);
            const int nvalid = min(kV4Cols, int(size_t(p.ncols) - dc.g * kV4Cols));
            mbar_wait(&d_done[s], dph);
#if F2_V4_FENCE_PRODUCER
            fence_async_smem();
#endif
            const bool issued = lane < nvalid && F2_V4_MODE != 2;
            if (issued) {
                bulk_red_xor(p.C + (p.c_wcol0 + dc.g * kV4Cols + lane) * p.sc + r0,
                             dring + size_t(s) * kV4DBytes + lane * kV4ColPitch, bytes);
                bulk_commit();
            }
            const bool rel_point = p.release && t + 1 == len0;
            // pipelined write-back: the reductions of the last F2_V4_PIPE tiles may
            // still be reading shared memory; a stage is freed once its reads are done
            pq[(pq0 + npend) & 3] = s;
            ++npend;
            if (rel_point) {
                bulk_wait0();  // group-0 writes complete in memory
                __syncwarp();
                if (lane == 0) {
                    release_signal(p.release, p.tag);
                    for (int q = 0; q < npend; ++q) mbar_arrive(&d_free[pq[(pq0 + q) & 3]]);
                }
                pq0 = (pq0 + npend) & 3;
                npend = 0;
            } else if (npend > F2_V4_PIPE) {
                bulk_wait_read<F2_V4_PIPE>();
                __syncwarp();
                if (lane == 0) mbar_arrive(&d_free[pq[pq0]]);
                pq0 = (pq0 + 1) & 3;
                --npend;
            }
            if (t + kV4AStages < cnt) {
                mbar_wait(&a_empty[ae], aph);
                issue_a();
            }
            if (++ae == kV4AStages) { ae = 0; aph ^= 1; }
            if (++s == kV4DStages) { s = 0; dph ^= 1; }
            dc.next();
        }
        bulk_wait0();
        return;
    }

    // ===== consumer warps =====
    // lane = (row slot sl = lane >> 2, column pair cp = lane & 3): rows 16 w + 2 sl (+1),
    // columns 2 cp (+1); odd slots read the other half of each table region
    const int sl = lane >> 2, cp = lane & 3, hsl = sl & 1;
    const uint32_t sel = hsl ? 0x2301u : 0x3210u;
    const uint32_t co_e = kV4TabAddr | uint32_t(hsl * 64 + cp * 16);
    const uint32_t co_o = kV4TabAddr | uint32_t((hsl ^ 1) * 64 + cp * 16);
    const int rl = 16 * warp + 2 * sl;
    size_t gcur = ~size_t(0);
    TileCursor cc;
    cc.init(T, s0, len0, s1);
    int as = 0, s = 0;
    uint32_t aph = 0, dph = 0;
    for (size_t t = 0; t < cnt; ++t) {
        const size_t g = cc.g;
        if (g != gcur) {
            v4_consumers_sync();
            const int nvalid = min(kV4Cols, int(size_t(p.ncols) - g * kV4Cols));
            build_tables8(tabb, p.B, p.sb, b_row0, p.b_wcol0 + g * kV4Cols, nvalid, k);
            v4_consumers_sync();
            gcur = g;
        }
        mbar_wait(&a_full[as], aph);
        const ulonglong2 av = *(reinterpret_cast<const ulonglong2*>(aring + size_t(as) * kV4ABytes) + rl / 2);
        uint64_t x[2] = {av.x, av.y};
        const size_t row = base + cc.tt * kV4Rows + rl;
        if (row < row_lo || row + 2 > row_hi) {
#pragma unroll
            for (int q = 0; q < 2; ++q)
                if (row + q < row_lo || row + q >= row_hi) x[q] = 0;
        }
        uint64_t d[2][2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
#if F2_V4_MODE == 1
            d[q][0] = x[q]; d[q][1] = x[q] ^ co_o;
#else
            lookup8x2(sel, co_e, co_o, x[q], d[q][0], d[q][1]);
#endif
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_empty[as]);
        if (t >= size_t(kV4DStages)) mbar_wait(&d_free[s], dph ^ 1);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
#if F2_V4_MODE == 3
            if (d[0][c] != 0x123456789ull) continue;
#endif
            ulonglong2* dp = reinterpret_cast<ulonglong2*>(dring + size_t(s) * kV4DBytes +
                                                           (2 * cp + c) * kV4ColPitch) + rl / 2;
            dp[0] = make_ulonglong2(d[0][c], d[1][c]);
        }
#if !F2_V4_FENCE_PRODUCER
        fence_async_smem();
#endif
        __syncwarp();
        if (lane == 0) mbar_arrive(&d_done[s]);
        if (++as == kV4AStages) { as = 0; aph ^= 1; }
        if (++s == kV4DStages) { s = 0; dph ^= 1; }
        cc.next();
    }
}

bool update_fast_ok(const UpdateArgs& a);
bool update_v3_ok(const UpdateArgs& a) {
    return (a.sc % kV3Rows) == 0 && (reinterpret_cast<uintptr_t>(a.C) % 16) == 0 &&
           (reinterpret_cast<uintptr_t>(a.a) % 16) == 0 && a.row_hi <= a.sc;
}

bool update_fast_ok(const UpdateArgs& a) { return update_v3_ok(a); }

cudaError_t launch_update(const UpdateArgs& a, int num_sms, cudaStream_t s) {
    if (a.ncols <= 0) return cudaSuccess;
    if (a.release && !update_v3_ok(a)) return cudaErrorInvalidValue;
    if (update_v3_ok(a)) {
        const bool v4 = options().update == 4;
        if (a.pdl) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(num_sms);
            cfg.blockDim = dim3(v4 ? kV4Threads : kV3Threads);
            cfg.dynamicSmemBytes = v4 ? kV4Smem : kV3Smem;
            cfg.stream = s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            return v4 ? cudaLaunchKernelEx(&cfg, k_update_v4, a) : cudaLaunchKernelEx(&cfg, k_update_v3, a);
        }
        if (v4) k_update_v4<<<num_sms, kV4Threads, kV4Smem, s>>>(a);
        else k_update_v3<<<num_sms, kV3Threads, kV3Smem, s>>>(a);
        return cudaGetLastError();
    }
    k_update<<<num_sms, kUpdThreads, kTabBytes, s>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K1+K2 for products: stream-K M4RM GEMM, C ^= A*B
// ---------------------------------------------------------------------------
// Tile = 16 word-columns x 1024 rows, accumulated in registers over the
// k-blocks (32 words per lane).  The (tile, k-block) unit space is split into
// one contiguous range per CTA (stream-K) so every SM gets the same work;
// tiles finished by one CTA are XOR-stored, shared tiles use atomicXor.
constexpr int kGemmThreads = 512;
constexpr int kGemmRows = 1024;

__global__ void __launch_bounds__(kGemmThreads, 1) k_gemm(GemmArgs p) {
    extern __shared__ __align__(128) uint64_t tab[];
    const size_t KB = (p.k + 63) / 64;
    const size_t ntr = (p.n + kGemmRows - 1) / kGemmRows;
    const size_t ncg = (size_t(p.mcols) + kTabCols - 1) / kTabCols;
    const size_t TU = ntr * ncg * KB;
    const size_t u0 = TU * blockIdx.x / gridDim.x;
    const size_t u1 = TU * (blockIdx.x + 1) / gridDim.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int h = lane >> 4, col = lane & 15;
    const uint64_t* tl = tab + col;

    for (size_t u = u0; u < u1;) {
        const size_t tile = u / KB;
        const size_t kb0 = u % KB;
        const size_t kb1 = (u1 - u) < (KB - kb0) ? kb0 + (u1 - u) : KB;
        const size_t cg = tile % ncg, rt = tile / ncg;
        const int nvalid = int(size_t(p.mcols) - cg * kTabCols) < kTabCols
                               ? int(size_t(p.mcols) - cg * kTabCols)
                               : kTabCols;
        const size_t row0 = rt * kGemmRows + size_t(warp) * 64 + 32 * h;  // lane's 32 rows
        uint64_t acc[32];
#pragma unroll
        for (int s = 0; s < 32; ++s) acc[s] = 0;
        for (size_t kb = kb0; kb < kb1; ++kb) {
            const int kbits = int(p.k - kb * 64 < 64 ? p.k - kb * 64 : 64);
            const int nt = kbits > 56 ? 9 : (kbits + 6) / 7;
            __syncthreads();
            build_tables<kGemmThreads>(tab, p.B, p.sb, kb * 64, cg * kTabCols, nvalid, kbits,
                                       nt);
            __syncthreads();
            const uint64_t* ap = p.A + kb * p.sa + row0;
            if (row0 >= p.n) continue;
            const bool fullrows = row0 + 32 <= p.n;
#pragma unroll
            for (int g8 = 0; g8 < 4; ++g8) {
                uint64_t aw[8];
                if (fullrows) {
                    ld256(ap + 8 * g8, aw[0], aw[1], aw[2], aw[3]);
                    ld256(ap + 8 * g8 + 4, aw[4], aw[5], aw[6], aw[7]);
                } else {
#pragma unroll
                    for (int s = 0; s < 8; ++s)
                        aw[s] = (row0 + 8 * g8 + s < p.n) ? ap[8 * g8 + s] : 0ull;
                }
#pragma unroll
                for (int s = 0; s < 8; ++s) acc[8 * g8 + s] ^= lookup(tl, aw[s], nt);
            }
        }
        // epilogue
        if (col < nvalid && row0 < p.n) {
            uint64_t* cp = p.C + (cg * kTabCols + col) * p.sc + row0;
            const bool alone = (kb0 == 0 && kb1 == KB);
            if (alone && row0 + 32 <= p.n) {
#pragma unroll
                for (int g4 = 0; g4 < 8; ++g4) {
                    uint64_t x0, x1, x2, x3;
                    ld256(cp + 4 * g4, x0, x1, x2, x3);
                    st256(cp + 4 * g4, x0 ^ acc[4 * g4], x1 ^ acc[4 * g4 + 1],
                          x2 ^ acc[4 * g4 + 2], x3 ^ acc[4 * g4 + 3]);
                }
            } else {
#pragma unroll
                for (int s = 0; s < 32; ++s)
                    if (row0 + s < p.n && acc[s])
                        atomicXor(reinterpret_cast<unsigned long long*>(cp + s),
                                  (unsigned long long)acc[s]);
            }
        }
        u += kb1 - kb0;
    }
}

// ---------------------------------------------------------------------------
// K1+K2 v2 for products: producer-fed stream-K M4RM GEMM, C ^= A*B
// ---------------------------------------------------------------------------
// ncu on v1 (profiles/r1_gemm_r1_summary.txt): instruction-bound (3.55 G
// instructions for 16384^3, issue 39%) on guarded lookups, with the global-load
// latency of every k-block's table build exposed.  v2: a producer warp streams
// each (tile, k-block) unit's A segment (1024 driving words) and B block
// (64 rows x 16 word-columns) into a 3-stage shared ring with bulk copies; the
// 16 consumer warps build the tables from shared memory at the fixed table
// address and run the 3-instruction lookups; accumulators stay in registers
// across the k-blocks of a tile (stream-K split, atomicXor for shared tiles).
constexpr int kG2Warps = 16;
constexpr int kG2Threads = kG2Warps * 32;
constexpr int kG2Rows = 1024;                     // tile rows (lane owns 32)
constexpr int kG2Stages = 3;
constexpr int kG2ABytes = kG2Rows * 8;            // 8 KiB driving words
constexpr int kG2BPitch = 64 * 8 + 16;            // 528 B: conflict-free 128-bit row-pair loads
constexpr int kG2BBytes = kTabCols * kG2BPitch;   // 16 columns x 64 rows (padded)
constexpr int kG2StageBytes = kG2ABytes + kG2BBytes;
constexpr size_t kG2RingBytes = size_t(kG2Stages) * kG2StageBytes + 64;
constexpr size_t kG2Smem = kTabAddr + kTabBytes;
static_assert(kG2RingBytes + 1024 <= kTabAddr, "gemm ring must fit below the table window");

// table build from a shared-memory B block (column c at bs + 64*c, k-row r)
// 16-entry chunks (smaller register footprint: the GEMM keeps 32 accumulators live)
__device__ __forceinline__ int tab_chunks16(int nt) { return nt <= 8 ? 8 * nt : 80; }

template <int NTH>
__device__ __forceinline__ void build_tables_smem(uint64_t* __restrict__ tab,
                                                  const uint64_t* __restrict__ bs, int ncols_valid,
                                                  int k_bits, int nt, int tid) {
    const int total = tab_chunks16(nt) * kTabCols;
    for (int it = tid; it < total; it += NTH) {
        const int col = it & (kTabCols - 1);
        const int cg = it >> 4;
        const int t = cg < 64 ? (cg >> 3) : 8;
        const int chunk = cg < 64 ? (cg & 7) : cg - 64;  // high bits (>= 4) of the entry index
        const int sz = t < 8 ? 7 : 8;
        uint64_t rows[8];
        const bool cv = col < ncols_valid;
        // rows 7t..7t+sz-1 of this column via 4 aligned 128-bit loads from row (7t & ~1)
        const int r0 = (7 * t) & ~1, sh = (7 * t) & 1;
        const ulonglong2* bp = reinterpret_cast<const ulonglong2*>(
            reinterpret_cast<const unsigned char*>(bs) + col * kG2BPitch) + r0 / 2;
        uint64_t raw[9];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const ulonglong2 v = bp[q];
            raw[2 * q] = v.x;
            raw[2 * q + 1] = v.y;
        }
        raw[8] = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const uint64_t x = sh ? raw[b + 1] : raw[b];
            rows[b] = (b < sz && cv && 7 * t + b < k_bits) ? x : 0ull;
        }
        uint64_t cur = 0;
#pragma unroll
        for (int hb = 0; hb < 4; ++hb)
            if ((chunk >> hb) & 1) cur ^= rows[4 + hb];
        uint64_t* dst = tab + (size_t(128 * t + chunk * 16) * kTabCols + col);
        uint64_t v[16];
        v[0] = cur;
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int g = 1 << b; g < (2 << b); ++g) v[g] = v[g - (1 << b)] ^ rows[b];
#pragma unroll
        for (int g = 0; g < 16; ++g) dst[g * kTabCols] = v[g];
    }
}

__device__ __forceinline__ size_t gemm_units(const GemmArgs& p) {
    return ((p.n + kG2Rows - 1) / kG2Rows) * ((size_t(p.mcols) + kTabCols - 1) / kTabCols) *
           ((p.k + 63) / 64);
}

// units [u0, u1) of problem p; the ring stage/phase cursor (s, ph) carries over
// between calls (every stage is drained at the end of a call)
__device__ __forceinline__ void gemm_range(const GemmArgs& p, size_t u0, size_t u1,
                                           unsigned char* ring, uint64_t* full, uint64_t* tab,
                                           int& s, uint32_t& ph) {
    const size_t KB = (p.k + 63) / 64;
    const size_t ncg = (size_t(p.mcols) + kTabCols - 1) / kTabCols;
    if (u0 >= u1) return;
    const size_t cnt = u1 - u0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s0 = s;

    // producer role (thread 0): bulk loads of unit `i` into stage i % kG2Stages.  A
    // stage is reused only after the CTA-wide barrier that ends its previous unit.
    size_t ptile = u0 / KB, pkb = u0 % KB;
    auto produce = [&](size_t i) {
        const int st = int((size_t(s0) + i) % kG2Stages);
        const size_t cg = ptile % ncg, rt = ptile / ncg;
        const int nvalid = min(kTabCols, int(size_t(p.mcols) - cg * kTabCols));
        const size_t row0 = rt * kG2Rows;
        const size_t arows = min(size_t(kG2Rows), p.a_cap - row0);
        const size_t brows = min(size_t(64), p.b_cap - pkb * 64);
        unsigned char* sb = ring + size_t(st) * kG2StageBytes;
        mbar_expect_tx(&full[st], uint32_t(arows * 8 + size_t(nvalid) * brows * 8));
        bulk_g2s(sb, p.A + pkb * p.sa + row0, uint32_t(arows * 8), &full[st]);
        for (int c = 0; c < nvalid; ++c)
            bulk_g2s(sb + kG2ABytes + c * kG2BPitch, p.B + (cg * kTabCols + c) * p.sb + pkb * 64,
                     uint32_t(brows * 8), &full[st]);
        if (++pkb == KB) { pkb = 0; ++ptile; }
    };
    __syncthreads();  // previous range fully consumed
    if (threadIdx.x == 0)
        for (size_t i = 0; i < cnt && i + 1 < size_t(kG2Stages); ++i) produce(i);

    const int h = lane >> 4, col = lane & 15;
    const uint32_t colofs = uint32_t(col) * 8u;
    const int rl = 64 * warp + 32 * h;  // lane's 32 rows within the tile
    size_t tile = u0 / KB, kb0 = u0 % KB;
    for (size_t i = 0; i < cnt;) {
        // one tile segment: k-blocks [kb0, kb0 + seg) of tile `tile`
        const size_t seg = min(KB - kb0, cnt - i);
        const size_t cg = tile % ncg, rt = tile / ncg;
        const int nvalid = min(kTabCols, int(size_t(p.mcols) - cg * kTabCols));
        uint64_t acc[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) acc[q] = 0;
        for (size_t j = 0; j < seg; ++j, ++i) {
            const size_t kb = kb0 + j;
            const int kbits = int(p.k - kb * 64 < 64 ? p.k - kb * 64 : 64);
            const unsigned char* sb = ring + size_t(s) * kG2StageBytes;
            __syncthreads();  // every warp finished unit i-1: its stage and the tables are free
            if (threadIdx.x == 0 && i + kG2Stages - 1 < cnt) produce(i + kG2Stages - 1);
            mbar_wait(&full[s], ph);
            build_tables_smem<kG2Threads>(tab, reinterpret_cast<const uint64_t*>(sb + kG2ABytes),
                                          nvalid, kbits, 9, threadIdx.x);
            __syncthreads();
            // all 9 tables are always built (groups beyond k are all-zero tables and the
            // driving words' bits beyond k are zero), so the lookup is branch-free
            const ulonglong2* ap = reinterpret_cast<const ulonglong2*>(sb) + rl / 2;
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const ulonglong2 v = ap[q];
                acc[2 * q] ^= lookup9(colofs, v.x);
                acc[2 * q + 1] ^= lookup9(colofs, v.y);
            }
            if (++s == kG2Stages) { s = 0; ph ^= 1; }
        }
        // epilogue: XOR into C (exclusive tile -> plain RMW, shared tile -> atomicXor)
        const size_t row0 = rt * kG2Rows + rl;
        if (col < nvalid && row0 < p.n) {
            uint64_t* cp = p.C + (cg * kTabCols + col) * p.sc + row0;
            const bool alone = (kb0 == 0 && seg == KB) && row0 + 32 <= p.n;
#pragma unroll
            for (int g4 = 0; g4 < 8; ++g4) {
                if (alone) {
                    uint64_t x0, x1, x2, x3;
                    ld256(cp + 4 * g4, x0, x1, x2, x3);
                    st256(cp + 4 * g4, x0 ^ acc[4 * g4], x1 ^ acc[4 * g4 + 1],
                          x2 ^ acc[4 * g4 + 2], x3 ^ acc[4 * g4 + 3]);
                } else {
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const int q = 4 * g4 + t;
                        if (row0 + q < p.n && acc[q])
                            atomicXor(reinterpret_cast<unsigned long long*>(cp + q),
                                      (unsigned long long)acc[q]);
                    }
                }
            }
        }
        kb0 = 0;
        ++tile;
    }
}

__device__ __forceinline__ uint64_t* g2_setup(unsigned char* smem_raw, unsigned char*& ring,
                                               uint64_t*& full) {
    const uint32_t smem_base = smem_u32(smem_raw);
    if (smem_base > kTabAddr - kG2RingBytes) __trap();
    ring = smem_raw;
    full = reinterpret_cast<uint64_t*>(ring + size_t(kG2Stages) * kG2StageBytes);
    if (threadIdx.x == 0) {
        for (int s = 0; s < kG2Stages; ++s) mbar_init(&full[s], 1);
        fence_async_smem();
    }
    __syncthreads();
    return reinterpret_cast<uint64_t*>(smem_raw + (kTabAddr - smem_base));
}

__global__ void __launch_bounds__(kG2Threads, 1) k_gemm_v2(GemmArgs p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const size_t TU = gemm_units(p);
    const size_t u0 = TU * blockIdx.x / gridDim.x;
    const size_t u1 = TU * (blockIdx.x + 1) / gridDim.x;
    if (u0 >= u1) return;
    unsigned char* ring;
    uint64_t* full;
    uint64_t* tab = g2_setup(smem_raw, ring, full);
    int s = 0;
    uint32_t ph = 0;
    gemm_range(p, u0, u1, ring, full, tab, s, ph);
}

// Batched products (Strassen-Winograd leaves): the concatenated unit spaces of
// nprob problems are split evenly over the CTAs (one launch, no tail effects
// per leaf).  offs[q] = first unit of problem q, offs[nprob] = total.
__global__ void __launch_bounds__(kG2Threads, 1)
    k_gemm_batched(const GemmArgs* __restrict__ probs, const size_t* __restrict__ offs, int nprob) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const size_t TU = offs[nprob];
    const size_t u0 = TU * blockIdx.x / gridDim.x;
    const size_t u1 = TU * (blockIdx.x + 1) / gridDim.x;
    if (u0 >= u1) return;
    unsigned char* ring;
    uint64_t* full;
    uint64_t* tab = g2_setup(smem_raw, ring, full);
    int s = 0;
    uint32_t ph = 0;
    int q = 0;
    while (q + 1 < nprob && offs[q + 1] <= u0) ++q;
    for (; q < nprob && offs[q] < u1; ++q) {
        const GemmArgs p = probs[q];
        const size_t a = u0 > offs[q] ? u0 - offs[q] : 0;
        const size_t b = (u1 < offs[q + 1] ? u1 : offs[q + 1]) - offs[q];
        gemm_range(p, a, b, ring, full, tab, s, ph);
    }
}

// Batched XOR jobs: dst = (acc ? dst : 0) ^ src0 ^ src1 ^ src2 ^ src3 (null srcs
// skipped); blockIdx.y = job, blockIdx.z = word-column, 32-byte vector accesses.
__global__ void __launch_bounds__(256) k_xor_batched(const XorJob* __restrict__ jobs) {
    const XorJob& J = jobs[blockIdx.y];
    const size_t q = blockIdx.z;
    if (q >= J.wcols) return;
    uint64_t* dp = J.dst + q * J.sd;
    const uint64_t* sp[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) sp[t] = J.src[t] ? J.src[t] + q * J.ss[t] : nullptr;
    const size_t nq = J.rows / 4;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nq;
         i += size_t(gridDim.x) * blockDim.x) {
        uint64_t v0 = 0, v1 = 0, v2 = 0, v3 = 0, x0, x1, x2, x3;
        if (J.acc) ld256(dp + 4 * i, v0, v1, v2, v3);
#pragma unroll
        for (int t = 0; t < 4; ++t)
            if (sp[t]) {
                ld256(sp[t] + 4 * i, x0, x1, x2, x3);
                v0 ^= x0; v1 ^= x1; v2 ^= x2; v3 ^= x3;
            }
        st256(dp + 4 * i, v0, v1, v2, v3);
    }
}

cudaError_t launch_xor_batched(const XorJob* d_jobs, int njobs, size_t max_rows, size_t max_wcols,
                               cudaStream_t s) {
    if (njobs == 0) return cudaSuccess;
    const unsigned bx = unsigned(std::min<size_t>((max_rows / 4 + 255) / 256, 16));
    dim3 grid(bx ? bx : 1, unsigned(njobs), unsigned(max_wcols));
    k_xor_batched<<<grid, 256, 0, s>>>(d_jobs);
    return cudaGetLastError();
}

cudaError_t launch_gemm_batched(const GemmArgs* d_probs, const size_t* d_offs, int nprob,
                                size_t total_units, int num_sms, cudaStream_t s) {
    if (nprob == 0 || total_units == 0) return cudaSuccess;
    const int grid = int(total_units < size_t(num_sms) ? total_units : size_t(num_sms));
    k_gemm_batched<<<grid, kG2Threads, kG2Smem, s>>>(d_probs, d_offs, nprob);
    return cudaGetLastError();
}

size_t gemm_units_host(const GemmArgs& p) {
    return ((p.n + kG2Rows - 1) / kG2Rows) * ((size_t(p.mcols) + kTabCols - 1) / kTabCols) *
           ((p.k + 63) / 64);
}

bool gemm_fast_ok(const GemmArgs& g) {
    return g.a_cap >= g.n && g.b_cap >= g.k && (g.sa % 2) == 0 && (g.sb % 2) == 0 &&
           (reinterpret_cast<uintptr_t>(g.A) % 16) == 0 && (reinterpret_cast<uintptr_t>(g.B) % 16) == 0;
}

cudaError_t launch_gemm(const GemmArgs& g, int num_sms, cudaStream_t s) {
    if (g.n == 0 || g.k == 0 || g.mcols <= 0) return cudaSuccess;
    const size_t KB = (g.k + 63) / 64;
    const size_t units = ((g.n + kGemmRows - 1) / kGemmRows) *
                         ((size_t(g.mcols) + kTabCols - 1) / kTabCols) * KB;
    const int grid = int(units < size_t(num_sms) ? units : size_t(num_sms));
    const bool v2 = g.a_cap >= g.n && g.b_cap >= g.k && (g.sa % 2) == 0 && (g.sb % 2) == 0 &&
                    (reinterpret_cast<uintptr_t>(g.A) % 16) == 0 &&
                    (reinterpret_cast<uintptr_t>(g.B) % 16) == 0;
    if (v2) {
        k_gemm_v2<<<grid, kG2Threads, kG2Smem, s>>>(g);
        return cudaGetLastError();
    }
    k_gemm<<<grid, kGemmThreads, kTabBytes, s>>>(g);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K4: panel kernel — Procedure buildZ
// ---------------------------------------------------------------------------
// The 64 steps are strictly sequential, so the whole procedure runs in ONE
// warp with no block barriers.  Z and M are held TRANSPOSED in registers: lane
// l owns columns l and l+32 (zt_l bit j = bit l of Z_j).  In that form every
// Gauss-Jordan update of the procedure is lane-local:
//   c   = 2^k | (mt_k & low(k))                       (:989-992, one shuffle)
//   M_k <- A_ib            : bit k of mt_l = bit l of A_ib              (:997)
//   Z_k ^= sum_{j<k,y_j}Z_j: bit k of zt_l ^= parity(zt_l & y & low(k)) (:1001-1006)
//   Z_j ^= Z_k (c_j, j<k)  : zt_l ^= c & low(k)  if bit k of zt_l      (:1007-1010)
// and likewise for M.  The pivot search (:993-1000) tests 32 candidate rows
// per ballot from a shared-memory window of the first kPanelWin rows (first
// odd-parity row wins: the reference's lowest-index tie-break);
// misses fall back to a 256-rows-per-iteration scan that also ORs the rows it
// sees — when nothing nonzero remains, the remaining steps are insertions that
// only touch bit positions the final compression removes, so the loop ends.
// orig[] tracks the source row of every window slot, giving the composite
// permutation that k_swaps mirrors on every other word-column.
constexpr int kPanelThreads = 256;  // all warps load the window; warp 0 runs buildZ
constexpr int kPanelWin = 2048;
constexpr uint32_t kNone = 0xFFFFFFFFu;

struct PanelSmem {
    uint64_t win[kPanelWin];
    uint32_t orig[kPanelWin];
    uint32_t ext_pos[64];
    uint32_t ext_orig[64];
};

__device__ __forceinline__ uint64_t low_mask64(int k) {
    return k >= 64 ? ~0ull : ((1ull << k) - 1);
}

// software pext: gather the bits of x at the set positions of sel (ascending)
__device__ __forceinline__ uint64_t pext64(uint64_t x, uint64_t sel) {
    uint64_t out = 0;
    int cnt = 0;
    while (sel) {
        const int b = __ffsll(static_cast<long long>(sel)) - 1;
        out |= ((x >> b) & 1ull) << cnt++;
        sel &= sel - 1;
    }
    return out;
}

__global__ void __launch_bounds__(kPanelThreads, 1)
    k_panel(uint64_t* __restrict__ col, size_t n, PanelState* __restrict__ st_all, int j,
            const uint32_t* wait_flag, uint32_t wait_count) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    PanelSmem& S = *reinterpret_cast<PanelSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31;
    if (wait_flag) {
        // lookahead: the previous panel's update releases this column early
        if (tid == 0) {
            uint32_t v;
            SpinGuard g;
            while (true) {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(wait_flag) : "memory");
                if (v >= wait_count) break;
                __nanosleep(64);
                g.tick(1, wait_flag, v, wait_count);
            }
        }
        __syncthreads();
    }
    const size_t R = j == 0 ? 0 : size_t(st_all[j - 1].R) + st_all[j - 1].r;
    PanelState* st = st_all + j;
    const size_t rows = R < n ? n - R : 0;
    if (rows == 0) {
        if (tid == 0) { st->R = uint32_t(R < n ? R : n); st->r = 0; st->npairs = 0; st->flags = 0; }
        if (tid < 64) st->Z[tid] = 0;
        return;
    }
    uint64_t* A = col + R;
    const uint32_t winrows = rows < size_t(kPanelWin) ? uint32_t(rows) : uint32_t(kPanelWin);
    for (uint32_t x = tid; x < winrows; x += kPanelThreads) {
        S.win[x] = A[x];
        S.orig[x] = x;
    }
    __syncthreads();
    if (tid >= 32) return;

    // transposed Z, M: lane owns columns lane (lo) and lane+32 (hi)
    uint64_t zlo = 1ull << lane, zhi = 1ull << (lane + 32);
    uint64_t mlo = zlo, mhi = zhi;
    uint64_t sel = 0;        // bit k: step k selected a row (P_k != -1)
    uint32_t ib = 0;         // next pivot slot (relative row)
    uint32_t n_ext = 0;      // beyond-window rows touched (lane 0 bookkeeping, uniform count)
    uint32_t max_touch = 0;  // highest window slot touched
    // Fast path: lane L holds candidate slot ib + L in registers (cv, co) and the
    // window advances by one shuffle per selection instead of a shared-memory
    // round trip; shared memory stays authoritative (the swaps are stored) and
    // the search below is the slow path (pivot outside the 32 candidates, window
    // exhausted).  Measured 20.5 -> 19.5 us per panel; the remaining ~17 us are
    // the 64-step chain at ~180 instructions per step in one warp.
    uint64_t cv = 0;
    uint32_t co = 0;
    bool regwin = false;
    auto load_regwin = [&]() {
        regwin = ib + 33u <= winrows;  // the slot entering after a selection must be in the window
        if (regwin) {
            cv = S.win[ib + lane];
            co = S.orig[ib + lane];
        }
    };
    load_regwin();
    for (int k = 0; k < 64; ++k) {
        const uint64_t lowk = low_mask64(k);
        const uint64_t mtk = __shfl_sync(0xffffffffu, k < 32 ? mlo : mhi, k & 31);
        const uint64_t c = (1ull << k) | (mtk & lowk);
        uint32_t found = kNone;
        uint64_t newrow = 0;
        bool fast = false;
        if (regwin) {
            uint64_t pv = 0;
            uint32_t po = 0;
            if (lane == 31) {  // the slot entering the window after a selection
                pv = S.win[ib + 32];
                po = S.orig[ib + 32];
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, __popcll(c & cv) & 1);
            if (bal) {
                fast = true;
                const int f = __ffs(bal) - 1;
                found = ib + uint32_t(f);
                newrow = __shfl_sync(0xffffffffu, cv, f);
                const uint32_t of = __shfl_sync(0xffffffffu, co, f);
                const uint64_t vb = __shfl_sync(0xffffffffu, cv, 0);
                const uint32_t ob = __shfl_sync(0xffffffffu, co, 0);
                if (lane == 0) { S.win[ib] = newrow; S.orig[ib] = of; }
                const bool mv = lane == f && f != 0;
                if (mv) { S.win[found] = vb; S.orig[found] = ob; }
                // slots ib+1 .. ib+32 (slot ib+f now holds the old slot ib)
                cv = __shfl_down_sync(0xffffffffu, mv ? vb : cv, 1);
                co = __shfl_down_sync(0xffffffffu, mv ? ob : co, 1);
                if (lane == 31) { cv = pv; co = po; }
            }
        }
        if (!fast) {
            __syncwarp();  // the fast path's swap stores are visible to every lane
            // ---- pivot search: first row i >= ib with odd popcount(c & A_i) ----
            {
                const uint32_t i = ib + lane;
                uint64_t v = 0;
                uint32_t o = 0;
                if (i < winrows) { v = S.win[i]; o = S.orig[i]; }
                else if (i < rows) { v = A[i]; }
                const uint32_t bal = __ballot_sync(0xffffffffu, i < rows && (__popcll(c & v) & 1));
                if (bal) {
                    const int f = __ffs(bal) - 1;
                    found = ib + f;
                    newrow = __shfl_sync(0xffffffffu, v, f);
                    if (found < winrows) {  // fast path: both slots are in the window
                        const uint64_t vb = __shfl_sync(0xffffffffu, v, 0);
                        const uint32_t of = __shfl_sync(0xffffffffu, o, f);
                        const uint32_t ob = __shfl_sync(0xffffffffu, o, 0);
                        if (lane == 0) { S.win[ib] = newrow; S.orig[ib] = of; }
                        if (lane == f && f != 0) { S.win[found] = vb; S.orig[found] = ob; }
                        __syncwarp();
                    }
                } else {
                    // slow path: scan the rest 256 rows at a time, OR-ing what we see
                    uint64_t orr = v;
                    for (size_t base = size_t(ib) + 32; base < rows && found == kNone; base += 256) {
                        uint32_t hits[8];
    #pragma unroll
                        for (int t = 0; t < 8; ++t) {
                            const size_t ii = base + 32 * t + lane;
                            uint64_t vv = 0;
                            if (ii < winrows) vv = S.win[ii];
                            else if (ii < rows) vv = A[ii];
                            orr |= vv;
                            hits[t] = __ballot_sync(0xffffffffu, ii < rows && (__popcll(c & vv) & 1));
                        }
    #pragma unroll
                        for (int t = 0; t < 8; ++t)
                            if (found == kNone && hits[t]) found = uint32_t(base + 32 * t + __ffs(hits[t]) - 1);
                    }
                    if (found == kNone) {
                        orr = __reduce_or_sync(0xffffffffu, uint32_t(orr)) |
                              (uint64_t(__reduce_or_sync(0xffffffffu, uint32_t(orr >> 32))) << 32);
                        if (orr == 0) break;  // only zero rows remain: no further selections
                    } else {
                        if (lane == 0) {
                            const uint64_t vb = S.win[ib];
                            const uint32_t ob = S.orig[ib];
                            if (found < winrows) {
                                newrow = S.win[found];
                                S.win[ib] = newrow;
                                S.orig[ib] = S.orig[found];
                                S.win[found] = vb;
                                S.orig[found] = ob;
                            } else {
                                newrow = A[found];
                                A[found] = vb;
                                S.win[ib] = newrow;
                                uint32_t e = 0;
                                while (e < n_ext && S.ext_pos[e] != found) ++e;
                                if (e == n_ext) { S.ext_pos[e] = found; S.ext_orig[e] = found; }
                                S.orig[ib] = S.ext_orig[e];
                                S.ext_orig[e] = ob;
                            }
                        }
                        __syncwarp();
                        newrow = __shfl_sync(0xffffffffu, newrow, 0);
                        if (found >= winrows) {
                            const uint32_t e0 = n_ext;  // uniform recount
                            uint32_t present = 0;
                            for (uint32_t e = 0; e < e0; ++e) present |= (S.ext_pos[e] == found);
                            if (!present) ++n_ext;
                        }
                    }
                }
            }
        }
        if (found == kNone) {
            // insertion (P_k = -1): M_k stays 2^k, y = 2^k -> only Z_j/M_j ^= 2^k for c_j
            const uint64_t cm = c & lowk;
            if ((zlo >> k) & 1) zlo ^= cm;
            if ((zhi >> k) & 1) zhi ^= cm;
            if ((mlo >> k) & 1) mlo ^= cm;
            if ((mhi >> k) & 1) mhi ^= cm;
            continue;  // no swap happened: the register window is still valid
        }
        if (found < winrows && found > max_touch) max_touch = found;
        sel |= 1ull << k;
        // M_k <- newrow (bit k of mt_l = bit l of newrow; it was [l==k] before)
        const uint64_t bk = 1ull << k;
        mlo = (mlo & ~bk) | (((newrow >> lane) & 1ull) << k);
        mhi = (mhi & ~bk) | (((newrow >> (lane + 32)) & 1ull) << k);
        // Z_k ^= sum_{j<k, y_j} Z_j and M_k likewise, y = newrow
        const uint64_t yk = newrow & lowk;
        zlo ^= uint64_t(__popcll(zlo & yk) & 1) << k;
        zhi ^= uint64_t(__popcll(zhi & yk) & 1) << k;
        mlo ^= uint64_t(__popcll(mlo & yk) & 1) << k;
        mhi ^= uint64_t(__popcll(mhi & yk) & 1) << k;
        // Z_j ^= Z_k, M_j ^= M_k for j < k with c_j
        const uint64_t cm = c & lowk;
        if ((zlo >> k) & 1) zlo ^= cm;
        if ((zhi >> k) & 1) zhi ^= cm;
        if ((mlo >> k) & 1) mlo ^= cm;
        if ((mhi >> k) & 1) mhi ^= cm;
        ++ib;
        if (fast) {
            regwin = ib + 33u <= winrows;
            if (!regwin) __syncwarp();
        } else {
            load_regwin();
        }
    }
    __syncwarp();
    // ---- composite permutation: window slots with orig != slot, then ext rows ----
    uint32_t np = 0;
    const uint32_t span = (ib > 0 ? max(max_touch + 1, ib) : 0);
    for (uint32_t x0 = 0; x0 < span; x0 += 32) {
        const uint32_t x = x0 + lane;
        const bool moved = x < span && S.orig[x] != x;
        const uint32_t bal = __ballot_sync(0xffffffffu, moved);
        if (moved) {
            const uint32_t e = np + __popc(bal & ((1u << lane) - 1));
            A[x] = S.win[x];
            st->dst[e] = x;
            st->src[e] = S.orig[x];
        }
        np += __popc(bal);
    }
    for (uint32_t e0 = 0; e0 < n_ext; e0 += 32) {
        const uint32_t e = e0 + lane;
        const bool moved = e < n_ext && S.ext_orig[e] != S.ext_pos[e];
        const uint32_t bal = __ballot_sync(0xffffffffu, moved);
        if (moved) {
            const uint32_t d = np + __popc(bal & ((1u << lane) - 1));
            st->dst[d] = S.ext_pos[e];
            st->src[d] = S.ext_orig[e];
        }
        np += __popc(bal);
    }
    // ---- Z rows back from the transposed form, compressed (:1011-1015) ----
    uint64_t zr0 = 0, zr1 = 0;  // rows lane, lane+32
    for (int r = 0; r < 64; ++r) {
        const uint64_t row = uint64_t(__ballot_sync(0xffffffffu, (zlo >> r) & 1)) |
                             (uint64_t(__ballot_sync(0xffffffffu, (zhi >> r) & 1)) << 32);
        if (r == lane) zr0 = row;
        if (r == lane + 32) zr1 = row;
    }
    if (sel != ~0ull) { zr0 = pext64(zr0, sel); zr1 = pext64(zr1, sel); }
    st->Z[lane] = zr0;
    st->Z[lane + 32] = zr1;
    if (lane == 0) {
        st->R = uint32_t(R);
        st->r = ib;
        st->npairs = np;
        st->flags = 0;
    }
}

// 64x64 bit-matrix transpose held in a warp: lane L holds rows L (x0) and L+32
// (x1) on entry and columns L / L+32 on exit.  One register swap for the 32-bit
// halves, then five shuffle butterflies -- no shared memory, no bank conflicts.
__device__ __forceinline__ void warp_transpose64(uint64_t& x0, uint64_t& x1, int lane) {
    {
        const uint64_t t = ((x0 >> 32) ^ x1) & 0x00000000FFFFFFFFull;
        x1 ^= t;
        x0 ^= t << 32;
    }
    const uint64_t masks[5] = {0x0000FFFF0000FFFFull, 0x00FF00FF00FF00FFull, 0x0F0F0F0F0F0F0F0Full,
                               0x3333333333333333ull, 0x5555555555555555ull};
#pragma unroll
    for (int st = 0; st < 5; ++st) {
        const int j = 16 >> st;
        const uint64_t msk = masks[st];
        const uint64_t y0 = __shfl_xor_sync(0xffffffffu, x0, j);
        const uint64_t y1 = __shfl_xor_sync(0xffffffffu, x1, j);
        if (!(lane & j)) {
            x0 ^= (((x0 >> j) ^ y0) & msk) << j;
            x1 ^= (((x1 >> j) ^ y1) & msk) << j;
        } else {
            x0 ^= ((y0 >> j) ^ x0) & msk;
            x1 ^= ((y1 >> j) ^ x1) & msk;
        }
    }
}

// ---------------------------------------------------------------------------
// K4': buildZ as Gauss-Jordan on a TRANSPOSED register block
// ---------------------------------------------------------------------------
// buildZ's pivot test at step k is parity(c_k & A_i) with c_k = e_k + {j < k :
// M_j[k]}.  M stays in reduced row-echelon form (every
// update of :1001-1010 is a Gauss-Jordan step), so that parity is bit k of
//   rho_i = A_i + sum_{j<k} A_i[j] M_j,
// and rho evolves by plain Gauss-Jordan: after step k selects p,
//   rho_i ^= rho_i[k] * rho_p   for every other row, earlier pivots included.
// (Insertion steps only change M at column k, which no later test reads.)
//
// The first kGjPos candidate positions are held reduced and TRANSPOSED in warp
// 0: lane l owns columns l and l+32 as kGjWords 32-bit words over the positions.
// One step is then
//   broadcast column k (3 shuffles) -> f = first live set position (every lane
//   computes it) -> per own column: bit f, xor the column mask, swap bits ib/f
// -- lane-local except the broadcast, ~70 instructions and one shuffle of
// dependent latency per step.  The reference's tie-break (first row at or after
// ib in the CURRENT order) is kept exactly: positions are swapped
// as the reference swaps rows.
//
// Z.  With rho_i = A_i + y_i*P (P = the selected rows in order), the pivot at
// position u ends as the RREF row M_u = (e_u + y_u)*P, so Z row k_u = e_u + y_u
// and the other Z rows are 0.  That Z is not the reference's bit for bit, but
// Y = D*Z is only formed for rows below the pivots (panel_y_body), all of which
// lie in span(P) (every step either selected a pivot or found bit k clear in
// ALL remaining rows), where coordinates are unique -- so Y is identical.  Warp
// 1 tracks y in the same transposed form from a per-step log, off the chain.
//
// Positions >= kGjPos take the slow path: rows are tested against c_k and the
// pivot is reduced by the RREF rows (popcounts per own column).  Warp 2 replays
// the swaps on win/orig (the composite permutation) from the same log.
// ---------------------------------------------------------------------------
#ifndef GJ_POLL_NS
#define GJ_POLL_NS 0
#endif
constexpr int kGjWords = 3;
constexpr uint32_t kGjPos = 32 * kGjWords;
constexpr uint32_t kLogValid = 0x80000000u, kLogSlow = 0x40000000u, kLogEnd = 0x20000000u;

struct PanelGjSmem {
    uint64_t win[kPanelWin];
    uint32_t orig[kPanelWin];
    uint32_t ext_pos[64];
    uint32_t ext_orig[64];
    uint4 log[66];      // per selection t: column-k mask over positions (3 words), meta
    uint2 logu[66];     // slow selections: dead positions u with x[k_u] (the reduction set)
    uint64_t rows0[kGjPos];  // hand-in: this panel's first kGjPos rows after the previous panel's update
    uint64_t dh[kGjPos];     // hand-in: the previous panel's D rows
    uint32_t pd[128];   // composite pair list (dst, src), also kept here for the next-column swaps
    uint32_t ps[128];
    uint32_t fin;       // warps 0-2 finished (done_out)
    uint64_t z[64];     // Z rows (head chunk)
    uint64_t bs[64];    // next column's pivot rows after the swaps (head chunk)
    uint64_t zt[256];   // 4-bit tables over Z and B (head chunk)
    uint64_t bt[256];
    uint32_t want;  // warp 0's slow path needs entries < want - 1 applied to win/orig
    uint32_t done;  // = want once they are (published by warp 2 on request)
    uint32_t r_fin; // chain kernel: this panel's r, for the helper warps
    // chain kernel: the window stays as loaded and slot[p] = where position p's row sits
    // in it (swapped like orig), so the replay moves indices only; win_ready = j + 1
    // once the window of panel j is in shared memory
    uint32_t win_ready;
    uint32_t slot[kPanelWin];
};
// Chain kernel (k_panel_chain): the next panel's first kGjPos rows, already updated by
// this panel (x ^= (D*Z)*B), and its first row R + r -- the in-CTA hand-off
struct ChainHand {
    uint64_t rows0[kGjPos];
    uint32_t R;
};
static_assert(kGjWords == 3, "log entries carry three position words");

// meta = valid | slow | end | k << 8 | f  (f < kGjPos for fast entries; r for the end entry)
__device__ __forceinline__ uint32_t gj_meta(bool slow, int k, uint32_t f) {
    return kLogValid | (slow ? kLogSlow : 0u) | (uint32_t(k) << 8) | f;
}

__device__ __forceinline__ uint32_t pick3(const uint32_t (&a)[kGjWords], uint32_t w) {
    return w == 0 ? a[0] : (w == 1 ? a[1] : a[2]);
}

__device__ __forceinline__ uint64_t warp_or64(uint64_t v) {
    return uint64_t(__reduce_or_sync(0xffffffffu, uint32_t(v))) |
           (uint64_t(__reduce_or_sync(0xffffffffu, uint32_t(v >> 32))) << 32);
}

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) { return *reinterpret_cast<const volatile uint32_t*>(p); }
__device__ __forceinline__ void st_volatile(uint32_t* p, uint32_t v) { *reinterpret_cast<volatile uint32_t*>(p) = v; }

__device__ __forceinline__ uint4 ld_log(const uint4* p) {
    uint4 v;
    asm volatile("ld.volatile.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))) : "memory");
    return v;
}
__device__ __forceinline__ void st_log(uint4* p, uint32_t a, uint32_t b, uint32_t c, uint32_t m) {
    asm volatile("st.volatile.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))), "r"(a), "r"(b), "r"(c), "r"(m)
                 : "memory");
}

// position masks of one step: the pivot column's positions minus f, and the
// two-bit swap mask {ib, f}
struct GjStep {
    uint32_t E[kGjWords];
    uint32_t sw[kGjWords];
};

__device__ __forceinline__ void wait_count_ge(const uint32_t* flag, uint32_t count, uint32_t site = 2) {
    if (!flag) return;
    uint32_t v;
    SpinGuard g;
    while (true) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
        if (v >= count) break;
        __nanosleep(32);
        g.tick(site, flag, v, count);
    }
}

// the whole warp spins (no lane-divergent loop: a warp that diverged around a
// long spin can stay split afterwards and run every later shuffle twice)
__device__ __forceinline__ void wait_count_ge_warp(const uint32_t* flag, uint32_t count, uint32_t site = 3) {
    if (!flag) return;
    SpinGuard g;
    while (true) {
        uint32_t v;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
        if (__all_sync(0xffffffffu, v >= count)) break;
        __nanosleep(32);
        g.tick(site, flag, v, count);
    }
}

// Named barriers of the panel body: ids 2..7 (+ boff in the chain kernel, whose two
// teams of kPanelThreads threads each run one body at a time).
#define GJ_BAR_SYNC(id, cnt) asm volatile("bar.sync %0, %1;" ::"r"((id) + boff), "n"(cnt) : "memory")
#define GJ_BAR_ARRIVE(id, cnt) asm volatile("bar.arrive %0, %1;" ::"r"((id) + boff), "n"(cnt) : "memory")
// the barriers both variants use: literal ids in k_panel_gj (its code stays as it was)
#define GJ_SYNC(id, cnt)                                                     \
    do {                                                                     \
        if constexpr (CHAIN) GJ_BAR_SYNC(id, cnt);                           \
        else asm volatile("bar.sync " #id ", " #cnt ";" ::: "memory");       \
    } while (0)
#define GJ_ARRIVE(id, cnt)                                                   \
    do {                                                                     \
        if constexpr (CHAIN) GJ_BAR_ARRIVE(id, cnt);                         \
        else asm volatile("bar.arrive " #id ", " #cnt ";" ::: "memory");     \
    } while (0)
constexpr int kChainHelpers = kPanelThreads - 96;  // warps 3..7
static_assert(kChainHelpers == 64 + int(kGjPos), "one helper thread per gathered row");

// One panel.  CHAIN = false: the whole k_panel_gj kernel (tid = threadIdx.x).  CHAIN =
// true: one iteration of a team of k_panel_chain -- the panel starts on the hand-off
// of the team that ran panel j-1 (hin, named barrier hb_in) instead of on counters of
// k_post_col, and its warps 3..7 prepare the same hand-off for panel j+1 (hout, hb_out).
template <bool CHAIN>
__device__ __forceinline__ void panel_gj_body(uint64_t* __restrict__ col, size_t n, PanelState* __restrict__ st_all,
                                              int j, const PanelLink& link, PanelGjSmem& S, const int tid,
                                              const int boff, const ChainHand* hin, ChainHand* hout,
                                              const int hb_in, const int hb_out) {
    const int lane = tid & 31, warp = tid >> 5;
    // F2GPU_SPIN_DIAG=1: the chain kernel's progress, words 4 (team 0) and 5 (team 1) of
    // the host-mapped record: panel << 8 | stage
    auto mark = [&](int stage) {
        if constexpr (CHAIN) {
            if (unsigned long long* d = g_spin_diag)
                *reinterpret_cast<volatile unsigned long long*>(d + 4 + (boff ? 1 : 0)) =
                    (uint64_t(j) << 8) | uint64_t(stage);
        }
    };
    if (tid == 0) mark(1);
    // every warp waits for the previous panel's head chunk (or the fused post's
    // head) before reading its state: the kernel may be queued on another stream
    // and resident while the previous panel kernel still runs
    if constexpr (CHAIN) {
        // ... or, in the chain kernel, for the other team's hand-off (also the
        // iteration barrier of this team: every warp is done with the panel before)
        if (hin) asm volatile("bar.sync %0, %1;" ::"r"(hb_in), "n"(kPanelThreads + kChainHelpers) : "memory");
        else wait_count_ge_warp(link.head, link.head_count, 10);  // the chain's first panel
    } else {
        wait_count_ge_warp(link.head, link.head_count, 10);
    }
    if (tid == 0) mark(2);
    const size_t R = (CHAIN && hin) ? size_t(hin->R)
                                    : (j == 0 ? 0 : size_t(st_all[j - 1].R) + st_all[j - 1].r);
    PanelState* st = st_all + j;
    const size_t rows = R < n ? n - R : 0;
    if (rows == 0) {
        if (tid == 0) { st->R = uint32_t(R < n ? R : n); st->r = 0; st->npairs = 0; st->flags = 0; }
        if (tid < 64) st->Z[tid] = 0;
        if (link.head_out || link.done_out) {  // counters other kernels wait on
            __threadfence();
            if constexpr (CHAIN) GJ_BAR_SYNC(2, kPanelThreads);
            else __syncthreads();
            if (tid == 0 && link.head_out) atomicAdd(link.head_out, 1u);
            if (tid == 0 && link.done_out) atomicAdd(link.done_out, 1u);
        }
        if constexpr (CHAIN) {
            if (hout) {  // no rows left for the next panel either
                if (tid == 96) hout->R = uint32_t(R < n ? R : n);
                __threadfence_block();
                if (tid >= 96)
                    asm volatile("bar.arrive %0, %1;" ::"r"(hb_out), "n"(kPanelThreads + kChainHelpers) : "memory");
            }
        }
        return;
    }
    uint64_t* A = col + R;
    if (!CHAIN && link.hand_in && warp < 3) {
        // the previous panel's update of this panel's first kGjPos rows, from its
        // hand-off block: Y = D*Z, rows ^= Y*B (4-bit tables), warps 0-2
        const int t3 = tid;
        for (int i2 = t3; i2 < kHandWords; i2 += 96) {
            const uint64_t v = link.hand_in[i2];
            if (i2 < 64) S.bs[i2] = v;
            else if (i2 < 64 + int(kGjPos)) S.rows0[i2 - 64] = v;
            else S.dh[i2 - 64 - kGjPos] = v;
        }
        if (t3 < 64) S.z[t3] = link.prev->Z[t3];
        asm volatile("bar.sync 5, 96;" ::: "memory");
        for (int e = t3; e < 256; e += 96) {
            const int g = e >> 4, v = e & 15;
            uint64_t za = 0, zb = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if ((v >> q) & 1) { za ^= S.z[4 * g + q]; zb ^= S.bs[4 * g + q]; }
            S.zt[e] = za;
            S.bt[e] = zb;
        }
        asm volatile("bar.sync 5, 96;" ::: "memory");
        if (t3 < int(kGjPos)) {
            const uint64_t d = S.dh[t3];
            uint64_t y = 0;
#pragma unroll
            for (int g = 0; g < 16; ++g) y ^= S.zt[16 * g + int((d >> (4 * g)) & 15)];
            uint64_t x = S.rows0[t3];
#pragma unroll
            for (int g = 0; g < 16; ++g) x ^= S.bt[16 * g + int((y >> (4 * g)) & 15)];
            S.rows0[t3] = x;
        }
        asm volatile("bar.sync 5, 96;" ::: "memory");
    }
    const uint32_t winrows = rows < size_t(kPanelWin) ? uint32_t(rows) : uint32_t(kPanelWin);
    const uint32_t npos = winrows < kGjPos ? winrows : kGjPos;
#ifdef GJ_PROFILE
    const long long t_start = clock64();
#endif
    // Chain kernel, warps 3..7 after the window load: the hand-off for panel j+1.  Once
    // the chain has ended (r, Z, win/orig final: barrier 4) one thread per row gathers
    // column j+1's pivot rows and its next kGjPos rows through orig (= after this
    // panel's swaps, which warp 2 applies to the column only after barrier 6), and the
    // rows get this panel's update (Y = D*Z, x ^= Y*B by 4-bit tables) in shared
    // memory: the next panel's selection starts ~2 us after this one's ends, without
    // the round trip through the done counter and k_post_col's first rows.
    auto chain_helper = [&]() {
        const int h = tid - 96;  // 0..159
        GJ_BAR_SYNC(4, kPanelThreads);
        if (!hout) return;
        // device trace (diagnostics): code 0, panel | stage << 8 (leaves of <= 256 panels)
        auto stamp = [&](int stage) {
            if (link.trace && h == 0) trace_ev(0, (j & 255) | (stage << 8));
        };
        stamp(1);
        if (h == 0) mark(4);
        const uint32_t r = S.r_fin;
        // column j+1 is final for the earlier panels once update j-1 released it
        if (warp == 3) wait_count_ge_warp(link.next_ready, link.next_count, 15);
        GJ_BAR_SYNC(5, kChainHelpers);
        stamp(2);
        const uint64_t* nx0 = link.next + R;
        uint64_t x = 0;
        if (h < 64) {
            S.bs[h] = uint32_t(h) < r ? __ldcg(nx0 + S.orig[h]) : 0ull;
        } else {
            const size_t pos = size_t(r) + (h - 64);
            if (pos < rows) x = __ldcg(nx0 + S.orig[pos]);
            S.rows0[h - 64] = x;  // keeps the load ahead of the arrival below
        }
        __threadfence_block();
        GJ_BAR_ARRIVE(6, kChainHelpers + 32);  // warp 2 may now swap column j+1
        GJ_BAR_SYNC(5, kChainHelpers);
        stamp(3);
        for (int e = h; e < 256; e += kChainHelpers) {
            const int g = e >> 4, v = e & 15;
            uint64_t za = 0, zb = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if ((v >> q) & 1) { za ^= S.z[4 * g + q]; zb ^= S.bs[4 * g + q]; }
            S.zt[e] = za;
            S.bt[e] = zb;
        }
        GJ_BAR_SYNC(5, kChainHelpers);
        if (h >= 64) {
            const size_t pos = size_t(r) + (h - 64);
            if (pos < rows) {
                const uint64_t d = S.win[S.slot[pos]];
                uint64_t y = 0;
#pragma unroll
                for (int g = 0; g < 16; ++g) y ^= S.zt[16 * g + int((d >> (4 * g)) & 15)];
#pragma unroll
                for (int g = 0; g < 16; ++g) x ^= S.bt[16 * g + int((y >> (4 * g)) & 15)];
            }
            hout->rows0[h - 64] = x;
        } else if (h == 0) {
            hout->R = uint32_t(R + r);
        }
        __threadfence_block();
        stamp(4);
        if (h == 0) mark(5);
        asm volatile("bar.arrive %0, %1;" ::"r"(hb_out), "n"(kPanelThreads + kChainHelpers) : "memory");
    };
    if (warp == 0) {
        // warp 0 starts on its own rows (loaded below) without waiting for the
        // window; it zeroes the log, then releases the two consumer warps
        for (int t = lane; t < 66; t += 32) S.log[t] = make_uint4(0, 0, 0, 0);
        if (lane == 0) { S.done = 0; S.want = 0; S.fin = 0; }
        GJ_ARRIVE(3, 96);
        if (link.trace && lane == 0) trace_ev(kTrPanelBegin, j);
        __syncwarp();
    } else if (warp == 1) {
        GJ_SYNC(3, 96);  // the log is zeroed
    } else if constexpr (CHAIN) {
        // The chain's panels start before their window is in memory (it comes with
        // k_post_col(j-1), ~3 us into the selection), and a replay that starts late
        // trails the selection to its end.  So the replay (warp 2) moves indices only and
        // starts with the selection: orig[p] = the original row at position p, slot[p] =
        // where its value sits in the window, which warps 3..7 load whenever it arrives
        // and nobody permutes.
        for (uint32_t x = tid - 64; x < winrows; x += kPanelThreads - 64) S.orig[x] = S.slot[x] = x;
        GJ_BAR_SYNC(2, 192);
        if (warp > 2) {
            if (warp == 3) wait_count_ge_warp(link.win, link.win_count, 11);
            GJ_BAR_SYNC(5, kChainHelpers);
            // one kernel over many panels: not through L1
            for (uint32_t x = tid - 96; x < winrows; x += kChainHelpers) S.win[x] = __ldcg(A + x);
            __threadfence_block();
            GJ_BAR_SYNC(5, kChainHelpers);
            if (tid == 96) st_volatile(&S.win_ready, uint32_t(j) + 1);  // warp 0's slow path
            GJ_BAR_ARRIVE(7, kChainHelpers + 32);                       // warp 2's write-back
            chain_helper();
            return;
        }
        GJ_BAR_SYNC(3, 96);
    } else {
        // warps 2..7 load the window; warp 2 then replays the swaps on it
        if (warp == 2) wait_count_ge_warp(link.win, link.win_count, 11);
        GJ_SYNC(2, 192);
        for (uint32_t x = tid - 64; x < winrows; x += kPanelThreads - 64) {
            S.win[x] = A[x];
            S.orig[x] = x;
        }
        GJ_SYNC(2, 192);
        if (warp > 2) {
            if (warp == 7) wait_count_ge_warp(link.chain_up, 1, 16);
            return;
        }
        GJ_SYNC(3, 96);
    }
#ifdef GJ_PROFILE
    const long long t_loaded = clock64();
#endif

    // Head chunk (warps 0-2 after their own work, link.head_out set): Y = D*Z for
    // the first kPanelHeadRows rows below the pivots (D from the swapped window)
    // and next[i] ^= Y_i * B, B = the next column's pivot rows (swapped by warp 2
    // just before), then the head counter the next panel kernel waits on.  This
    // takes the fused post's launch and first chunk off the panel chain.
    auto head_chunk = [&](uint32_t r) {
        const int t3 = tid;  // 0..95
        asm volatile("bar.sync 4, 96;" ::: "memory");
        const size_t lo = R + r;
        const uint32_t H = (r != 0 && lo < n) ? uint32_t(min(size_t(kPanelHeadRows), n - lo)) : 0u;
        if (H) {
            if (t3 < 64) S.bs[t3] = uint32_t(t3) < r ? link.next[R + t3] : 0ull;
            asm volatile("bar.sync 4, 96;" ::: "memory");
            for (int e = t3; e < 256; e += 96) {
                const int g = e >> 4, v = e & 15;
                uint64_t za = 0, zb = 0;
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if ((v >> q) & 1) { za ^= S.z[4 * g + q]; zb ^= S.bs[4 * g + q]; }
                S.zt[e] = za;
                S.bt[e] = zb;
            }
            asm volatile("bar.sync 4, 96;" ::: "memory");
            for (uint32_t p = r + t3; p < r + H; p += 96) {
                const uint64_t d = S.win[p];
                uint64_t y = 0;
#pragma unroll
                for (int g = 0; g < 16; ++g) y ^= S.zt[16 * g + int((d >> (4 * g)) & 15)];
                uint64_t x = link.next[R + p];
#pragma unroll
                for (int g = 0; g < 16; ++g) x ^= S.bt[16 * g + int((y >> (4 * g)) & 15)];
                A[p] = y;
                link.next[R + p] = x;
            }
        }
        __threadfence();
        asm volatile("bar.sync 4, 96;" ::: "memory");
        if (t3 == 0) atomicAdd(link.head_out, 1u);
    };
    // each of warps 0-2 calls this once, after its last global write.  Warp 2 ends
    // last (the pair list and the next column's swaps): it waits for the other two
    // (long done), so one device fence orders its own stores -- and, cumulatively,
    // theirs -- before the done counter (one fence on the chain instead of two)
    auto finish = [&]() {
        if (!link.done_out) return;
        __syncwarp();
        if (lane != 0) return;
        if (warp != 2) {
            __threadfence();
            atomicAdd(&S.fin, 1u);
            return;
        }
        while (atomicAdd(&S.fin, 0u) < 2u) {
        }
        __threadfence();
        atomicAdd(link.done_out, 1u);
        mark(6);
        if (link.trace) trace_ev(13, j);
    };

    if (warp == 2) {
        // ---- win/orig bookkeeping: replay the fast swaps ----
        uint32_t t = 0;
        uint32_t max_touch = 0, n_ext = 0;
        uint32_t live[kGjWords], tm[kGjWords] = {1u, 0u, 0u};
#pragma unroll
        for (int w = 0; w < kGjWords; ++w) {
            const uint32_t b0 = 32 * w;
            live[w] = npos >= b0 + 32 ? 0xffffffffu : (npos > b0 ? (1u << (npos - b0)) - 1 : 0u);
        }
        for (;; ++t) {
            // warp-uniform polling: every lane must see the entry before any acts
            // (lanes that diverge here would pair with different __syncwarp /
            // ballot instances and read win/orig while lane 0 still swaps)
            uint4 e;
            while (true) {
                e = ld_log(&S.log[t]);
                if (__all_sync(0xffffffffu, e.w != 0)) break;
                if (link.poll_ns) __nanosleep(link.poll_ns);
                // warp 0's slow path waits for entries < t: publish them
                const bool wanted = __shfl_sync(0xffffffffu, lane == 0 && ld_volatile(&S.want) == t + 1, 0);
                if (wanted) {
                    __threadfence_block();
                    if (lane == 0) st_volatile(&S.done, t + 1);
                }
            }
            if (e.w & kLogEnd) {
                n_ext = e.x;
                break;
            }
            const uint32_t m0 = e.x & live[0], m1 = e.y & live[1], m2 = e.z & live[2];
            const uint32_t f = (e.w & kLogSlow) ? e.z
                               : (m0 ? __ffs(m0) - 1 : (m1 ? 31 + __ffs(m1) : 63 + __ffs(m2)));
            if (f < winrows && f > max_touch) max_touch = f;
#pragma unroll
            for (int w = 0; w < kGjWords; ++w) live[w] &= ~tm[w];
            tm[2] = (tm[2] << 1) | (tm[1] >> 31);
            tm[1] = (tm[1] << 1) | (tm[0] >> 31);
            tm[0] = tm[0] << 1;
            if (CHAIN && !(e.w & kLogSlow) && lane == 1 && f != t) {
                const uint32_t st2 = S.slot[t], sf = S.slot[f];
                S.slot[t] = sf;
                S.slot[f] = st2;
            }
            if (!(e.w & kLogSlow) && lane == 0) {
                if (f != t) {
                    if constexpr (CHAIN) {  // indices only (lane 1 below: slot)
                        const uint32_t ot = S.orig[t], of = S.orig[f];
                        S.orig[t] = of;
                        S.orig[f] = ot;
                    } else {
                        const uint64_t vt = S.win[t], vf = S.win[f];
                        const uint32_t ot = S.orig[t], of = S.orig[f];
                        S.win[t] = vf; S.orig[t] = of;
                        S.win[f] = vt; S.orig[f] = ot;
                    }
                }
            }
            __syncwarp();
        }
        if constexpr (CHAIN) {  // orig / slot are final: the helper warps may gather through them
            if (link.trace && lane == 0) trace_ev(0, (j & 255) | (6 << 8));
            __threadfence_block();
            GJ_BAR_ARRIVE(4, kPanelThreads);
            GJ_BAR_SYNC(7, kChainHelpers + 32);  // the window is loaded (the write-back below)
        }
        // ---- composite permutation: window slots with orig != slot, then ext rows ----
        // every position < r may hold a moved row (pivots brought in from beyond
        // the window do not show in max_touch)
        const uint32_t span = t > 0 ? max(max_touch + 1, t) : 0;
        uint32_t np = 0;
        for (uint32_t x0 = 0; x0 < span; x0 += 32) {
            const uint32_t x = x0 + lane;
            const bool moved = x < span && S.orig[x] != x;
            const uint32_t bal = __ballot_sync(0xffffffffu, moved);
            if (moved) {
                const uint32_t e = np + __popc(bal & ((1u << lane) - 1));
                A[x] = CHAIN ? S.win[S.slot[x]] : S.win[x];
                st->dst[e] = S.pd[e] = x;
                st->src[e] = S.ps[e] = S.orig[x];
            }
            np += __popc(bal);
        }
        for (uint32_t e0 = 0; e0 < n_ext; e0 += 32) {
            const uint32_t e = e0 + lane;
            const bool moved = e < n_ext && S.ext_orig[e] != S.ext_pos[e];
            const uint32_t bal = __ballot_sync(0xffffffffu, moved);
            if (moved) {
                const uint32_t d = np + __popc(bal & ((1u << lane) - 1));
                st->dst[d] = S.pd[d] = S.ext_pos[e];
                st->src[d] = S.ps[d] = S.ext_orig[e];
            }
            np += __popc(bal);
        }
        __syncwarp();
        if (lane == 0) st->npairs = np;
        // column j+1 is final for the earlier panels once the previous update has
        // released it: needed by the swaps below AND by the head chunk's reads
        if (link.next) wait_count_ge_warp(link.next_ready, link.next_count, 13);
        if (link.next && np) {
            // this panel's row swaps on column j+1 (the fused POST skips it)
            __threadfence_block();
            uint64_t* nx = link.next + R;
            uint32_t d[4], sv[4];
            uint64_t v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t e = lane + 32 * q;
                if (e < np) { d[q] = S.pd[e]; sv[q] = S.ps[e]; }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (lane + 32 * q < np) v[q] = CHAIN ? __ldcg(nx + sv[q]) : nx[sv[q]];
            __syncwarp();
            // the helper warps gather the unswapped column: wait for their loads
            if constexpr (CHAIN) GJ_BAR_SYNC(6, kChainHelpers + 32);
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (lane + 32 * q < np) nx[d[q]] = v[q];
        } else {
            if constexpr (CHAIN) {
                if (hout) GJ_BAR_SYNC(6, kChainHelpers + 32);
            }
        }
        if (link.trace && lane == 0) trace_ev(kTrPanelEnd, j);
#ifdef GJ_PROFILE
        if (lane == 0) reinterpret_cast<long long*>(st->src)[56] = clock64() - t_start;
#endif
        if (link.hand_out) {
            // hand-off for the next panel kernel: the next column's pivot rows and its
            // next kGjPos rows (swapped, before this panel's update) and this
            // column's kGjPos rows below the pivots
            __syncwarp();
            __threadfence_block();
            const uint32_t r = t;
            const uint64_t* nx = link.next + R;
            for (int i2 = lane; i2 < kHandWords; i2 += 32) {
                uint64_t v = 0;
                if (i2 < 64) {
                    if (uint32_t(i2) < r) v = nx[i2];
                } else if (i2 < 64 + int(kGjPos)) {
                    const size_t p = size_t(r) + (i2 - 64);
                    if (p < rows) v = nx[p];
                } else {
                    const size_t p = size_t(r) + (i2 - 64 - kGjPos);
                    if (p < rows) v = S.win[p];
                }
                link.hand_out[i2] = v;
            }
        }
        if (link.head_out) {
            __threadfence_block();
            head_chunk(t);
        }
        finish();
        return;
    }

    if (warp == 1) {
        // ---- coordinates y (rho = A + y*P), transposed: lane owns coordinates
        //      lane and lane+32 as position words; then Z ----
        uint32_t y0[kGjWords] = {0, 0, 0}, y1[kGjWords] = {0, 0, 0};
        uint32_t tm[kGjWords] = {1u, 0u, 0u};  // one-hot position t
        uint32_t live[kGjWords];
#pragma unroll
        for (int w = 0; w < kGjWords; ++w) {
            const uint32_t b0 = 32 * w;
            live[w] = npos >= b0 + 32 ? 0xffffffffu : (npos > b0 ? (1u << (npos - b0)) - 1 : 0u);
        }
        uint32_t t = 0;
        for (;; ++t) {
            uint4 e;
            while (true) {
                e = ld_log(&S.log[t]);
                if (e.w) break;
                if (link.poll_ns) __nanosleep(link.poll_ns);
            }
            if (e.w & kLogEnd) break;
            uint32_t D[kGjWords] = {e.x, e.y, e.z};
            if (!(e.w & kLogSlow)) {
                const uint32_t m0 = D[0] & live[0], m1 = D[1] & live[1], m2 = D[2] & live[2];
                uint32_t fm[kGjWords], E[kGjWords], sw[kGjWords];
                fm[0] = m0 & (0u - m0);
                fm[1] = m0 ? 0u : m1 & (0u - m1);
                fm[2] = (m0 | m1) ? 0u : m2 & (0u - m2);
#pragma unroll
                for (int w = 0; w < kGjWords; ++w) {
                    E[w] = D[w] ^ fm[w];
                    sw[w] = fm[w] ^ tm[w];
                }
                auto upd = [&](uint32_t (&yc)[kGjWords], uint32_t tc) {
                    const uint32_t yf = 0u - uint32_t(((yc[0] & fm[0]) | (yc[1] & fm[1]) | (yc[2] & fm[2])) != 0);
                    const uint32_t flip = yf ^ (0u - uint32_t(tc == t));
#pragma unroll
                    for (int w = 0; w < kGjWords; ++w) yc[w] ^= E[w] & flip;
                    const uint32_t d = yf ^ (0u - uint32_t(((yc[0] & tm[0]) | (yc[1] & tm[1]) | (yc[2] & tm[2])) != 0));
#pragma unroll
                    for (int w = 0; w < kGjWords; ++w) yc[w] ^= sw[w] & d;
                };
                upd(y0, uint32_t(lane));
                if (t >= 32) upd(y1, uint32_t(lane) + 32);  // coordinates > t are still zero
            } else {
                D[2] = 0;  // carries found
                const uint2 u = S.logu[t];
                auto upd = [&](uint32_t (&yc)[kGjWords], uint32_t tc) {
                    const uint32_t um = tc < 32 ? (u.x >> tc) & 1u : (u.y >> (tc - 32)) & 1u;
                    const uint32_t yf = ((__popc(yc[0] & u.x) + __popc(yc[1] & u.y)) & 1u) ^ um;
#pragma unroll
                    for (int w = 0; w < kGjWords; ++w) yc[w] = (yc[w] & ~tm[w]) | (yf ? tm[w] : 0u);
                    const uint32_t flip = 0u - (yf ^ uint32_t(tc == t));
#pragma unroll
                    for (int w = 0; w < kGjWords; ++w) yc[w] ^= D[w] & flip;
                };
                upd(y0, uint32_t(lane));
                upd(y1, uint32_t(lane) + 32);
            }
#pragma unroll
            for (int w = 0; w < kGjWords; ++w) live[w] &= ~tm[w];
            tm[2] = (tm[2] << 1) | (tm[1] >> 31);
            tm[1] = (tm[1] << 1) | (tm[0] >> 31);
            tm[0] = tm[0] << 1;
        }
        // t = r.  Z row k_u = e_u + y_u for u < r: transpose so lane u holds y_u.
        const uint32_t r = t;
        uint64_t x0 = uint64_t(y0[0]) | (uint64_t(y0[1]) << 32);
        uint64_t x1 = uint64_t(y1[0]) | (uint64_t(y1[1]) << 32);
        warp_transpose64(x0, x1, lane);
        if (uint32_t(lane) < r) {
            const uint32_t kz = (S.log[lane].w >> 8) & 63u;
            st->Z[kz] = S.z[kz] = (1ull << lane) ^ x0;
        }
        if (uint32_t(lane) + 32 < r) {
            const uint32_t kz = (S.log[lane + 32].w >> 8) & 63u;
            st->Z[kz] = S.z[kz] = (1ull << (lane + 32)) ^ x1;
        }
        if constexpr (CHAIN) {
            if (link.trace && lane == 0) trace_ev(0, (j & 255) | (5 << 8));
            __threadfence_block();
            GJ_BAR_ARRIVE(4, kPanelThreads);
        }
#ifdef GJ_PROFILE
        if (lane == 0) reinterpret_cast<long long*>(st->src)[57] = clock64() - t_start;
#endif
        if (link.head_out) head_chunk(r);
        finish();
        return;
    }

    // ---- warp 0: the selection chain ----
    uint32_t c0[kGjWords], c1[kGjWords], live[kGjWords];
    {
        const uint64_t* src0 = CHAIN ? (hin ? hin->rows0 : A) : (link.hand_in ? S.rows0 : A);
        uint64_t x0 = uint32_t(lane) < npos ? src0[lane] : 0;
        uint64_t x1 = uint32_t(lane) + 32 < npos ? src0[lane + 32] : 0;
        uint64_t z0 = uint32_t(lane) + 64 < npos ? src0[lane + 64] : 0;
        uint64_t z1 = 0;
        warp_transpose64(x0, x1, lane);
        warp_transpose64(z0, z1, lane);
        c0[0] = uint32_t(x0); c0[1] = uint32_t(x0 >> 32); c0[2] = uint32_t(z0);
        c1[0] = uint32_t(x1); c1[1] = uint32_t(x1 >> 32); c1[2] = uint32_t(z1);
#pragma unroll
        for (int w = 0; w < kGjWords; ++w) {
            const uint32_t b0 = 32 * w;
            live[w] = npos >= b0 + 32 ? 0xffffffffu : (npos > b0 ? (1u << (npos - b0)) - 1 : 0u);
        }
    }
    uint32_t ib = 0, n_ext = 0;
    uint64_t sel = 0;
    bool stop = false;
#ifdef GJ_PROFILE
    uint32_t n_slow = 0;
#endif

    // one-hot mask of position ib over the three words
    uint32_t ibm[kGjWords] = {1u, 0u, 0u};

    auto step = [&](const int k, const bool hi) {
        const int kl = k & 31;
        uint32_t ck[kGjWords], m[kGjWords];
#pragma unroll
        for (int w = 0; w < kGjWords; ++w) {
            ck[w] = __shfl_sync(0xffffffffu, hi ? c1[w] : c0[w], kl);
            m[w] = ck[w] & live[w];
        }
        const uint32_t iw = ib >> 5, ibit = 1u << (ib & 31);
        if (m[0] | m[1] | m[2]) {
            // ---- fast: the pivot is a register position; fm = its one-hot mask ----
            uint32_t fm[kGjWords], E[kGjWords], sw[kGjWords];
            fm[0] = m[0] & (0u - m[0]);
            fm[1] = m[0] ? 0u : m[1] & (0u - m[1]);
            fm[2] = (m[0] | m[1]) ? 0u : m[2] & (0u - m[2]);
#pragma unroll
            for (int w = 0; w < kGjWords; ++w) {
                E[w] = ck[w] ^ fm[w];
                sw[w] = fm[w] ^ ibm[w];
            }
            auto upd = [&](uint32_t (&c)[kGjWords]) {
                const uint32_t bf = 0u - uint32_t(((c[0] & fm[0]) | (c[1] & fm[1]) | (c[2] & fm[2])) != 0);
#pragma unroll
                for (int w = 0; w < kGjWords; ++w) c[w] ^= E[w] & bf;
                const uint32_t d = bf ^ (0u - uint32_t(((c[0] & ibm[0]) | (c[1] & ibm[1]) | (c[2] & ibm[2])) != 0));
#pragma unroll
                for (int w = 0; w < kGjWords; ++w) c[w] ^= sw[w] & d;
            };
            // columns < k are never tested again: from k = 32 on only c1 matters
            if (!hi) upd(c0);
            upd(c1);
            // the consumers recover f as the first live position of ck
            if (lane == 0) st_log(&S.log[ib], ck[0], ck[1], ck[2], gj_meta(false, k, 0));
        } else {
            // ---- slow: search the positions beyond the register block ----
#ifdef GJ_PROFILE
            ++n_slow;
#endif
            if (lane == 0) st_volatile(&S.want, ib + 1);
            wait_count_ge_warp(link.all, link.all_count, 14);  // rows beyond the window
            while (!__all_sync(0xffffffffu, ld_volatile(&S.done) == ib + 1 &&
                                                (!CHAIN || ld_volatile(&S.win_ready) == uint32_t(j) + 1))) {}
            __syncwarp();
            __threadfence_block();
            // ck holds only dead positions (no live one has bit k): the RREF rows
            // with a 1 in column k.  c_k = e_k + their pivot columns.
            const uint64_t dk = uint64_t(ck[0]) | (uint64_t(ck[1]) << 32);
            uint64_t cacc = 0;
            if ((dk >> lane) & 1) cacc |= 1ull << ((S.log[lane].w >> 8) & 63u);
            if ((dk >> (lane + 32)) & 1) cacc |= 1ull << ((S.log[lane + 32].w >> 8) & 63u);
            const uint64_t c = (1ull << k) | warp_or64(cacc);
            uint32_t found = kNone;
            uint64_t orr = 0;
            for (size_t base = npos; base < rows && found == kNone; base += 256) {
                uint32_t hits[8];
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                    const size_t ii = base + 32 * t + lane;
                    uint64_t vv = 0;
                    if (ii < winrows) vv = CHAIN ? S.win[S.slot[ii]] : S.win[ii];
                    else if (ii < rows) vv = A[ii];
                    orr |= vv;
                    hits[t] = __ballot_sync(0xffffffffu, ii < rows && (__popcll(c & vv) & 1));
                }
#pragma unroll
                for (int t = 0; t < 8; ++t)
                    if (found == kNone && hits[t]) found = uint32_t(base + 32 * t + __ffs(hits[t]) - 1);
            }
            if (found == kNone) {
                // insertion; when every remaining row is zero no later step selects
                uint32_t anyl = 0;
#pragma unroll
                for (int w = 0; w < kGjWords; ++w) anyl |= ((hi ? 0u : c0[w]) | c1[w]) & live[w];
                if (warp_or64(orr) == 0 && !__any_sync(0xffffffffu, anyl != 0)) stop = true;
                return;
            }
            const uint64_t x = found < winrows ? (CHAIN ? S.win[S.slot[found]] : S.win[found]) : A[found];
            // reduction set: dead positions u with x[k_u] = 1
            const bool u0 = uint32_t(lane) < ib && ((x >> ((S.log[lane].w >> 8) & 63u)) & 1);
            const bool u1 = uint32_t(lane) + 32 < ib && ((x >> ((S.log[lane + 32].w >> 8) & 63u)) & 1);
            const uint32_t U0 = __ballot_sync(0xffffffffu, u0), U1 = __ballot_sync(0xffffffffu, u1);
            auto upd = [&](uint32_t (&c)[kGjWords], int l) {
                const uint32_t rx = uint32_t((x >> l) & 1) ^ ((__popc(c[0] & U0) + __popc(c[1] & U1)) & 1u);
#pragma unroll
                for (int w = 0; w < kGjWords; ++w)
                    if (uint32_t(w) == iw) c[w] = (c[w] & ~ibit) | (rx ? ibit : 0u);
                const uint32_t m = 0u - rx;
#pragma unroll
                for (int w = 0; w < kGjWords; ++w) c[w] ^= ck[w] & m;
            };
            if (!hi) upd(c0, lane);
            upd(c1, lane + 32);
            if (lane == 0) {
                const uint32_t sb = CHAIN ? S.slot[ib] : ib;  // where position ib's value sits
                const uint64_t vb = S.win[sb];
                const uint32_t ob = S.orig[ib];
                if (found < winrows) {
                    if constexpr (CHAIN) {
                        S.slot[ib] = S.slot[found];
                        S.slot[found] = sb;
                    } else {
                        S.win[ib] = x;
                        S.win[found] = vb;
                    }
                    S.orig[ib] = S.orig[found];
                    S.orig[found] = ob;
                } else {
                    A[found] = vb;
                    S.win[sb] = x;
                    uint32_t e = 0;
                    while (e < n_ext && S.ext_pos[e] != found) ++e;
                    if (e == n_ext) { S.ext_pos[e] = found; S.ext_orig[e] = found; }
                    S.orig[ib] = S.ext_orig[e];
                    S.ext_orig[e] = ob;
                }
                S.logu[ib] = make_uint2(U0, U1);
            }
            __syncwarp();
            if (found >= winrows) {
                const uint32_t e0 = n_ext;  // uniform recount
                uint32_t present = 0;
                for (uint32_t e = 0; e < e0; ++e) present |= (S.ext_pos[e] == found);
                if (!present) ++n_ext;
            }
            __threadfence_block();
            // dead positions are < 64, so ck[2] == 0: the third word carries found
            if (lane == 0) st_log(&S.log[ib], ck[0], ck[1], found, gj_meta(true, k, 0));
        }
#pragma unroll
        for (int w = 0; w < kGjWords; ++w) live[w] &= ~ibm[w];
        ibm[2] = (ibm[2] << 1) | (ibm[1] >> 31);
        ibm[1] = (ibm[1] << 1) | (ibm[0] >> 31);
        ibm[0] = ibm[0] << 1;
        sel |= 1ull << k;
        ++ib;
    };
    for (int k = 0; k < 32 && !stop; ++k) step(k, false);
    for (int k = 32; k < 64 && !stop; ++k) step(k, true);

    __threadfence_block();
    if (lane == 0) st_log(&S.log[ib], n_ext, 0, 0, kLogValid | kLogEnd | ib);
    if (lane == 0) mark(3);
    if (link.trace && lane == 0) trace_ev(kTrPanelChainEnd, j);
#ifdef GJ_PROFILE
    const long long t_chain = clock64();
#endif
    if (!((sel >> lane) & 1)) st->Z[lane] = S.z[lane] = 0;
    if (!((sel >> (lane + 32)) & 1)) st->Z[lane + 32] = S.z[lane + 32] = 0;
    if constexpr (CHAIN) {
        if (lane == 0) S.r_fin = ib;
        __threadfence_block();
        GJ_BAR_ARRIVE(4, kPanelThreads);
    }
    if (lane == 0) {
        st->R = uint32_t(R);
        st->r = ib;
        st->flags = 0;
    }
#ifdef GJ_PROFILE
    if (lane == 0) {
        long long* pr = reinterpret_cast<long long*>(st->src);
        pr[61] = t_loaded - t_start; pr[62] = t_chain - t_loaded; pr[63] = clock64() - t_chain;
        pr[59] = ib;
        pr[58] = n_slow;
        pr[60] = 0;
    }
#endif
    if (link.head_out) head_chunk(ib);
    finish();
}
#undef GJ_SYNC
#undef GJ_ARRIVE
#undef GJ_BAR_SYNC
#undef GJ_BAR_ARRIVE

__global__ void __launch_bounds__(kPanelThreads, 1)
    k_panel_gj(uint64_t* __restrict__ col, size_t n, PanelState* __restrict__ st_all, int j,
               const PanelLink link) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    PanelGjSmem& S = *reinterpret_cast<PanelGjSmem*>(smem_raw);
    panel_gj_body<false>(col, n, st_all, j, link, S, threadIdx.x, 0, nullptr, nullptr, 0, 0);
}

// ---------------------------------------------------------------------------
// K4'': the panel chain of a whole leaf in ONE persistent CTA
// ---------------------------------------------------------------------------
// Panels [c0, c1) of a leaf, one launch (c0 = the leaf's second panel: the first one is
// a k_panel_gj launch in stream order, during which this CTA becomes resident -- a
// chain queued beside the first k_post_col could find every SM holding one of its
// spinning blocks).  Two teams of kPanelThreads threads take the
// panels alternately (team = (j - c0) & 1), each running the k_panel_gj body on its
// own shared-memory block, so panel j's tail (pair list, next-column swaps, state,
// done counter) overlaps panel j+1's selection exactly as two resident k_panel_gj
// kernels did -- but the hand-off between them stays inside the CTA: the helper warps
// of panel j gather and update the next column's first rows in shared memory and
// release the other team through a named barrier (panel_gj_body, CHAIN = true).
// Every other wait (k_post_col's window / all-rows counters, the update's
// first-column release) and every output (PanelState, pair list, swaps on column j+1,
// done counter for k_post_col(j)) is the same as with per-panel launches, so the
// fused post and the updates on the main stream are unchanged.
struct ChainSmem {
    PanelGjSmem S[2];
    ChainHand H[2];
};

__global__ void __launch_bounds__(2 * kPanelThreads, 1) k_panel_chain(const ChainArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    ChainSmem& M = *reinterpret_cast<ChainSmem*>(smem_raw);
    const int team = threadIdx.x / kPanelThreads, tid = threadIdx.x % kPanelThreads;
    if (threadIdx.x < 2) M.S[threadIdx.x].win_ready = 0;  // epochs j + 1 > 0
    if (threadIdx.x == 0 && g_spin_diag)
        *reinterpret_cast<volatile unsigned long long*>(g_spin_diag + 6) = (uint64_t(a.c0) << 32) | uint32_t(a.c1);
    // resident: the leaf's first panel kernel (PanelLink::chain_up) may exit
    if (threadIdx.x == 0) atomicAdd(a.flags + size_t(a.leaf0) * a.flags_per_panel + 5, 1u);
    __syncthreads();
    // named barriers: team-local ids 2..7 (+ 6 * team), hand-off barriers 14 + team
    for (int j = a.c0 + team; j < a.c1; j += 2) {
        PanelLink l{};
        if (j > a.leaf0) {
            const uint32_t* f = a.flags + size_t(j - 1) * a.flags_per_panel;
            if (j == a.c0) { l.head = f; l.head_count = 1; }  // k_post_col(j-1)'s first rows
            l.win = f + 1; l.win_count = 8;
            l.all = f + 2; l.all_count = a.yblocks;
            if (j + 1 < a.c1) { l.next_ready = f + 3; l.next_count = a.upd_grid; }
        }
        if (j + 1 < a.c1) l.next = a.w + size_t(j + 1 - a.coff) * a.stride;
        l.poll_ns = a.poll_ns;
        l.trace = a.trace;
        l.done_out = a.flags + size_t(j) * a.flags_per_panel + 4;
        panel_gj_body<true>(a.w + size_t(j - a.coff) * a.stride, a.n, a.st, j, l, M.S[team], tid, 6 * team,
                            j > a.c0 ? &M.H[team] : nullptr, j + 1 < a.c1 ? &M.H[team ^ 1] : nullptr,
                            14 + team, 14 + (team ^ 1));
    }
}

static bool g_panel_gj = true;  // F2GPU_PANEL=0: the transposed-M k_panel
// The panel kernel reserves (nearly) a whole SM's shared memory: it is queued
// ahead and spins until its column is ready, and any CTA placed beside it (a
// persistent update CTA, post blocks) would slow its single-warp chain ~4x.
constexpr size_t kPanelGjSmemMax = 227 * 1024;
static_assert(sizeof(PanelGjSmem) <= kPanelGjSmemMax, "panel smem");
static size_t kPanelGjSmemBytes = kPanelGjSmemMax;  // F2GPU_PANEL_SMEM=0: only what the kernel uses

cudaError_t launch_panel(uint64_t* col, size_t n, PanelState* st_all, int j, cudaStream_t s,
                         const uint32_t* wait_flag, uint32_t wait_count) {
    if (g_panel_gj) {
        PanelLink l{};
        l.head = l.win = l.all = wait_flag;
        l.head_count = l.win_count = l.all_count = wait_count;
        k_panel_gj<<<1, kPanelThreads, kPanelGjSmemBytes, s>>>(col, n, st_all, j, l);
    } else {
        k_panel<<<1, kPanelThreads, sizeof(PanelSmem), s>>>(col, n, st_all, j, wait_flag, wait_count);
    }
    return cudaGetLastError();
}

cudaError_t launch_panel_link(uint64_t* col, size_t n, PanelState* st_all, int j, const PanelLink& link,
                              cudaStream_t s) {
    if (!g_panel_gj) return cudaErrorNotSupported;
    k_panel_gj<<<1, kPanelThreads, kPanelGjSmemBytes, s>>>(col, n, st_all, j, link);
    return cudaGetLastError();
}

bool panel_link_ok() { return g_panel_gj; }

cudaError_t launch_panel_chain(const ChainArgs& a, cudaStream_t s) {
    if (!g_panel_gj) return cudaErrorNotSupported;
    if (a.c1 <= a.c0) return cudaSuccess;
    k_panel_chain<<<1, 2 * kPanelThreads, kPanelGjSmemMax, s>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Y = D*Z over D (rows R+r .. n of the panel column), written in place
// ---------------------------------------------------------------------------
__device__ __forceinline__ void panel_y_body(uint64_t* __restrict__ col, size_t n,
                                             const PanelState* __restrict__ st, uint64_t* zt,
                                             unsigned blk, unsigned nblk) {
    // every load this block needs up front: the state header, Z, and the block's
    // first row word (one round trip instead of a chain)
    __shared__ uint64_t zs[64];
    const uint32_t R = st->R, r = st->r;
    if (threadIdx.x < 64) zs[threadIdx.x] = st->Z[threadIdx.x];
    const size_t lo = size_t(R) + r;
    const size_t i0 = lo + size_t(blk) * blockDim.x + threadIdx.x;
    const uint64_t d0 = (r != 0 && i0 < n) ? col[i0] : 0;
    __syncthreads();
    if (r == 0 || lo >= n) return;
    // single-column tables over the 64 Z words, all entries in parallel:
    // groups 0-7 cover bits 7t..7t+6 (128 entries), group 8 bits 56..63 (256)
    for (int e = threadIdx.x; e < kTabEntries; e += blockDim.x) {
        const int t = e < 1024 ? e >> 7 : 8;
        const int idx = e < 1024 ? e & 127 : e - 1024;
        uint64_t v = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b)
            if ((idx >> b) & 1) v ^= zs[7 * t + b];
        zt[e] = v;
    }
    __syncthreads();
    uint64_t d = d0;
    for (size_t i = i0; i < n; i += size_t(nblk) * blockDim.x) {
        if (i != i0) d = col[i];
        uint64_t y = 0;
#pragma unroll
        for (int t = 0; t < 8; ++t) y ^= zt[128 * t + int((d >> (7 * t)) & 127)];
        y ^= zt[1024 + int(d >> 56)];
        col[i] = y;
    }
}

// Lookahead column update: the next panel's column only,
//   next[i] ^= Y_j[i] * B   for i >= R_j + r_j,   B = next[R_j .. R_j + r_j)
// (panel j's Schur update restricted to word-column j+1).  Many
// small CTAs, a 1280-entry table per CTA; every CTA increments *done when its
// rows are in memory, and the next panel kernel spins on the count -- so the
// panel chain no longer waits for a full column group of the persistent update.
__global__ void __launch_bounds__(256) k_update_col(uint64_t* __restrict__ next, const uint64_t* __restrict__ ycol,
                                                    size_t n, const PanelState* __restrict__ st,
                                                    uint32_t* __restrict__ done) {
    __shared__ uint64_t bs[64];
    __shared__ uint64_t tab[kTabEntries];
    const uint32_t R = st->R, r = st->r;
    const size_t lo = size_t(R) + r;
    if (threadIdx.x < 64) bs[threadIdx.x] = (threadIdx.x < r && R + threadIdx.x < n) ? next[R + threadIdx.x] : 0;
    __syncthreads();
    if (r != 0 && lo < n) {
        for (int e = threadIdx.x; e < kTabEntries; e += blockDim.x) {
            const int t = e < 1024 ? e >> 7 : 8;
            const int idx = e < 1024 ? e & 127 : e - 1024;
            uint64_t v = 0;
#pragma unroll
            for (int b = 0; b < 8; ++b)
                if ((idx >> b) & 1) v ^= bs[7 * t + b];
            tab[e] = v;
        }
        __syncthreads();
        for (size_t i = lo + size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
            const uint64_t y = ycol[i];
            uint64_t x = 0;
#pragma unroll
            for (int t = 0; t < 8; ++t) x ^= tab[128 * t + int((y >> (7 * t)) & 127)];
            x ^= tab[1024 + int(y >> 56)];
            next[i] ^= x;
        }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(done, 1u);
}

int update_col_grid(size_t n, int num_sms) {
    return int(std::max<size_t>(1, std::min<size_t>((n + 255) / 256, size_t(4) * size_t(num_sms))));
}
cudaError_t launch_update_col(uint64_t* next, const uint64_t* ycol, size_t n, const PanelState* st, uint32_t* done,
                              int grid, cudaStream_t s) {
    k_update_col<<<grid, 256, 0, s>>>(next, ycol, n, st, done);
    return cudaGetLastError();
}

__global__ void __launch_bounds__(256) k_panel_y(uint64_t* __restrict__ col, size_t n,
                                                 const PanelState* __restrict__ st) {
    __shared__ uint64_t zt[kTabEntries];
    panel_y_body(col, n, st, zt, blockIdx.x, gridDim.x);
}

cudaError_t launch_panel_y(uint64_t* col, size_t n, const PanelState* st, int num_sms,
                           cudaStream_t s) {
    k_panel_y<<<num_sms, 256, 0, s>>>(col, n, st);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K6: apply the panel's composite row permutation to word-columns (+ perm)
// ---------------------------------------------------------------------------
// One warp per word-column; column index == ncols handles the uint32 perm.
__device__ __forceinline__ void swaps_body(uint64_t* __restrict__ w, size_t stride, int ncols,
                                           int skip_col, uint32_t* __restrict__ perm,
                                           const PanelState* __restrict__ st, int gw, int skip_col2 = -1) {
    const int lane = threadIdx.x & 31;
    if (gw > ncols || gw == skip_col || gw == skip_col2) return;
    // header and pair lists are loaded together (independent addresses), so the
    // swap costs two dependent global round trips: state, then the rows
    const uint32_t np = st->npairs;
    const uint32_t R = st->R;
    uint32_t sidx[4], didx[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        sidx[e] = st->src[lane + 32 * e];
        didx[e] = st->dst[lane + 32 * e];
    }
    if (np == 0) return;
    if (gw == ncols) {
        if (!perm) return;
        uint32_t v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (lane + 32 * e < int(np)) v[e] = perm[R + sidx[e]];
        __syncwarp();
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (lane + 32 * e < int(np)) perm[R + didx[e]] = v[e];
        return;
    }
    uint64_t* cp = w + size_t(gw) * stride + R;
    uint64_t v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e)
        if (lane + 32 * e < int(np)) v[e] = cp[sidx[e]];
    __syncwarp();
#pragma unroll
    for (int e = 0; e < 4; ++e)
        if (lane + 32 * e < int(np)) cp[didx[e]] = v[e];
}

__global__ void __launch_bounds__(256) k_swaps(uint64_t* __restrict__ w, size_t stride,
                                               int ncols, int skip_col,
                                               uint32_t* __restrict__ perm,
                                               const PanelState* __restrict__ st) {
    swaps_body(w, stride, ncols, skip_col, perm, st,
               int((size_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5));
}

cudaError_t launch_swaps(uint64_t* w, size_t stride, int ncols, int skip_col, uint32_t* perm,
                         const PanelState* st, cudaStream_t s) {
    const int warps = ncols + 1;
    k_swaps<<<(warps + 7) / 8, 256, 0, s>>>(w, stride, ncols, skip_col, perm, st);
    return cudaGetLastError();
}

// Rank-deficient inputs (decompose_recursive): is the block rows [row0, n) x nwc
// word-columns all zero?  *flag |= 1 otherwise.  One pass over the block (HBM-bound),
// run only after a split whose left half was not at full rank.
__global__ void __launch_bounds__(256) k_any_nonzero(const uint64_t* __restrict__ w, size_t stride, size_t row0,
                                                     size_t n, size_t nwc, uint32_t* __restrict__ flag) {
    const size_t rows = n - row0, total = rows * nwc;
    uint64_t acc = 0;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += size_t(gridDim.x) * blockDim.x) {
        const size_t q = i / rows, r = i - q * rows;
        acc |= w[q * stride + row0 + r];
    }
    if (__syncthreads_or(acc != 0) && threadIdx.x == 0) atomicOr(flag, 1u);
}

cudaError_t launch_any_nonzero(const uint64_t* w, size_t stride, size_t row0, size_t n, size_t nwc, uint32_t* flag,
                               int num_sms, cudaStream_t s) {
    if (row0 >= n || nwc == 0) return cudaSuccess;
    const size_t total = (n - row0) * nwc;
    const int grid = int(std::min<size_t>(size_t(num_sms) * 8, (total + 255) / 256));
    k_any_nonzero<<<grid, 256, 0, s>>>(w, stride, row0, n, nwc, flag);
    return cudaGetLastError();
}

// ... and when it is: panels [j0, j1) have rank 0 and no swaps -- exactly what the
// panel kernel writes for an all-zero column (R, r = 0, npairs = 0, Z = 0)
__global__ void __launch_bounds__(64) k_fill_zero_states(PanelState* __restrict__ st, int j0, uint32_t R) {
    PanelState* p = st + j0 + blockIdx.x;
    if (threadIdx.x == 0) { p->R = R; p->r = 0; p->npairs = 0; p->flags = 0; }
    p->Z[threadIdx.x] = 0;
}

cudaError_t launch_fill_zero_states(PanelState* st, int j0, int j1, uint32_t R, cudaStream_t s) {
    if (j1 <= j0) return cudaSuccess;
    k_fill_zero_states<<<j1 - j0, 64, 0, s>>>(st, j0, R);
    return cudaGetLastError();
}

// Distributed recursion: the row swaps of a whole leaf (panels [j0, j1), in order)
// on the word-columns outside [skip_lo, skip_hi) and on perm, one launch.  One warp
// per column; panel j+1's header and pair list are loaded while panel j's rows move,
// so a panel costs one dependent round trip (the rows), not two.
__global__ void __launch_bounds__(256) k_swaps_range(uint64_t* __restrict__ w, size_t stride, int ncols,
                                                     int skip_lo, int skip_hi, uint32_t* __restrict__ perm,
                                                     const PanelState* __restrict__ st, int j0, int j1) {
    const int gw = int((size_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (gw > ncols || (gw >= skip_lo && gw < skip_hi) || j0 >= j1) return;
    if (gw == ncols && !perm) return;
    uint32_t np = st[j0].npairs, R = st[j0].R;
    uint32_t sidx[4], didx[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        sidx[e] = st[j0].src[lane + 32 * e];
        didx[e] = st[j0].dst[lane + 32 * e];
    }
    for (int j = j0; j < j1; ++j) {
        const uint32_t cnp = np, cR = R;
        uint32_t cs[4], cd[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) { cs[e] = sidx[e]; cd[e] = didx[e]; }
        if (j + 1 < j1) {
            np = st[j + 1].npairs;
            R = st[j + 1].R;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                sidx[e] = st[j + 1].src[lane + 32 * e];
                didx[e] = st[j + 1].dst[lane + 32 * e];
            }
        }
        if (cnp == 0) continue;
        if (gw == ncols) {
            uint32_t v[4];
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (lane + 32 * e < int(cnp)) v[e] = perm[cR + cs[e]];
            __syncwarp();
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (lane + 32 * e < int(cnp)) perm[cR + cd[e]] = v[e];
        } else {
            uint64_t* cp = w + size_t(gw) * stride + cR;
            uint64_t v[4];
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (lane + 32 * e < int(cnp)) v[e] = cp[cs[e]];
            __syncwarp();
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (lane + 32 * e < int(cnp)) cp[cd[e]] = v[e];
        }
        __syncwarp();  // panel j's writes are visible to the warp before panel j+1's reads
    }
}

cudaError_t launch_swaps_range(uint64_t* w, size_t stride, int ncols, int skip_lo, int skip_hi, uint32_t* perm,
                               const PanelState* st, int j0, int j1, cudaStream_t s) {
    const int warps = ncols + 1;
    k_swaps_range<<<(warps + 7) / 8, 256, 0, s>>>(w, stride, ncols, skip_lo, skip_hi, perm, st, j0, j1);
    return cudaGetLastError();
}

// Swaps on every other word-column (+perm) and Y = D*Z on the panel column in
// ONE launch: the two touch disjoint data (skip_col is the panel column).
constexpr int kPostYBlocks = 64;
__global__ void __launch_bounds__(256) k_post(uint64_t* __restrict__ w, size_t stride, int ncols,
                                              int panel_col, uint32_t* __restrict__ perm,
                                              size_t n, const PanelState* __restrict__ st,
                                              int swap_blocks, int yblocks) {
    __shared__ uint64_t zt[kTabEntries];
    if (int(blockIdx.x) < swap_blocks) {
        swaps_body(w, stride, ncols, panel_col, perm, st,
                   int((size_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5));
        return;
    }
    panel_y_body(w + size_t(panel_col) * stride, n, st, zt, blockIdx.x - swap_blocks, yblocks);
}

cudaError_t launch_post(uint64_t* w, size_t stride, int ncols, int panel_col, uint32_t* perm,
                        size_t n, const PanelState* st, cudaStream_t s) {
    const int swap_blocks = (ncols + 1 + 7) / 8;
    // Y blocks: about one row per thread (latency-bound), at least kPostYBlocks
    const int yblocks = int(std::min<size_t>(1024, std::max<size_t>(kPostYBlocks, (n + 255) / 256)));
    k_post<<<swap_blocks + yblocks, 256, 0, s>>>(w, stride, ncols, panel_col, perm, n, st,
                                                   swap_blocks, yblocks);
    return cudaGetLastError();
}

// POST fused with the next column's update (lookahead).  Row blocks: 4-bit
// tables over Z (16 groups x 16) and over B = the next column's pivot rows
// (already swapped by the panel kernel), 256 entries each -- one entry per
// thread, so the tables cost one round of shared-memory reads instead of the
// five of a 1280-entry table; each row then takes 16 + 16 lookups:
//   y = D_i * Z -> panel column,   next_i ^= y * B.
// Counters for the next panel kernel (k_panel_gj link): block 0 after its first
// 256 rows, blocks < 8 after theirs (the 2048-row window), every block at end.
constexpr int kPcMinYBlocks = 64;
int post_col_yblocks(size_t n) {
    return int(std::min<size_t>(1024, std::max<size_t>(kPcMinYBlocks, (n + 255) / 256)));
}

__global__ void __launch_bounds__(256) k_post_col(uint64_t* __restrict__ w, size_t stride, int ncols,
                                                  int panel_col, int next_col, uint32_t* __restrict__ perm,
                                                  size_t n, const PanelState* __restrict__ st,
                                                  int swap_blocks, uint32_t* __restrict__ flags, bool trace,
                                                  int skip, const uint32_t* wait_panel) {
    __shared__ uint64_t zs[64], bs[64];
    __shared__ uint64_t zt[256], bt[256];
    // launched as a programmatic dependent of the previous update (pdl): placed as its
    // CTAs retire, then waits for its completion before touching any column
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (wait_panel) {  // queued ahead: the panel kernel's writes are complete
        if (threadIdx.x < 32) {
            SpinGuard g;
            while (true) {
                uint32_t v;
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(wait_panel) : "memory");
                if (__all_sync(0xffffffffu, v != 0)) break;
                __nanosleep(128);
                g.tick(4, wait_panel, v, 1);
            }
        }
        __syncthreads();
    }
    // the update that follows (UpdateArgs::pdl) may start placing its CTAs now (it
    // waits for this grid's completion before touching data).  Not before the panel
    // kernel is done: 146 update CTAs placed early could take the SM it still needs
    // (its post would wait for it forever -- seen with the post launched early too)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (int(blockIdx.x) < swap_blocks) {
        swaps_body(w, stride, ncols, panel_col, perm, st,
                   int((size_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5), next_col);
        return;
    }
    const unsigned blk = blockIdx.x - swap_blocks, nblk = gridDim.x - swap_blocks;
    const int tid = threadIdx.x;
    if (trace && blk == 0 && tid == 0) trace_ev(kTrPostBegin, panel_col);
    uint64_t* col = w + size_t(panel_col) * stride;
    uint64_t* nx = next_col >= 0 ? w + size_t(next_col) * stride : nullptr;
    const uint32_t R = st->R, r = st->r;
    const size_t lo = size_t(R) + r;
    if (tid < 64) {
        zs[tid] = st->Z[tid];
        bs[tid] = (nx && uint32_t(tid) < r) ? nx[R + tid] : 0;
    }
    // rows [lo, lo + skip) were done by the panel kernel (its head chunk), which
    // also signals flags[0]; the window counter then covers blocks < 8 - skip/256
    const size_t i0 = lo + size_t(skip) + size_t(blk) * blockDim.x + tid;
    const unsigned nwin = 8u - unsigned(skip) / 256u;
    const bool work = r != 0 && lo + size_t(skip) < n;
    const uint64_t d0 = (work && i0 < n) ? col[i0] : 0;
    const uint64_t x0 = (work && nx && i0 < n) ? nx[i0] : 0;
    __syncthreads();
    if (work) {
        {
            const int g = tid >> 4, v = tid & 15;
            uint64_t a = 0, b = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if ((v >> q) & 1) { a ^= zs[4 * g + q]; b ^= bs[4 * g + q]; }
            zt[tid] = a;
            bt[tid] = b;
        }
        __syncthreads();
        auto row = [&](size_t i, uint64_t d, uint64_t x) {
            uint64_t y = 0;
#pragma unroll
            for (int g = 0; g < 16; ++g) y ^= zt[16 * g + int((d >> (4 * g)) & 15)];
            col[i] = y;
            if (nx) {
#pragma unroll
                for (int g = 0; g < 16; ++g) x ^= bt[16 * g + int((y >> (4 * g)) & 15)];
                nx[i] = x;
            }
        };
        if (i0 < n) row(i0, d0, x0);
        if (flags && blk < nwin) {  // every writer fences, then one arrival per block
            __threadfence();
            __syncthreads();
            if (tid == 0) {
                if (blk == 0 && skip == 0) {
                    atomicAdd(flags + 0, 1u);
                    if (trace) trace_ev(kTrPostHead, panel_col);
                }
                atomicAdd(flags + 1, 1u);
            }
        }
        for (size_t i = i0 + size_t(nblk) * blockDim.x; i < n; i += size_t(nblk) * blockDim.x)
            row(i, col[i], nx ? nx[i] : 0);
        if (flags) {
            __threadfence();
            __syncthreads();
            if (tid == 0) {
                if (!trace) atomicAdd(flags + 2, 1u);
                else if (atomicAdd(flags + 2, 1u) == nblk - 1) trace_ev(kTrPostEnd, panel_col);
            }
        }
    } else if (tid == 0 && flags) {
        if (blk == 0 && skip == 0) atomicAdd(flags + 0, 1u);
        if (blk < nwin) atomicAdd(flags + 1, 1u);
        atomicAdd(flags + 2, 1u);
    }
}

cudaError_t launch_post_col(uint64_t* w, size_t stride, int ncols, int panel_col, int next_col, uint32_t* perm,
                            size_t n, const PanelState* st, uint32_t* flags, cudaStream_t s, bool trace,
                            int skip, const uint32_t* wait_panel, bool pdl) {
    const int swap_blocks = (ncols + 1 + 7) / 8;
    if (pdl) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(swap_blocks + post_col_yblocks(n));
        cfg.blockDim = dim3(256);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, k_post_col, w, stride, ncols, panel_col, next_col, perm, n, st, swap_blocks,
                                  flags, trace, skip, wait_panel);
    }
    k_post_col<<<swap_blocks + post_col_yblocks(n), 256, 0, s>>>(w, stride, ncols, panel_col, next_col, perm, n,
                                                                  st, swap_blocks, flags, trace, skip, wait_panel);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// block TRSM base case of decompose_recursive (full rank): panels a .. a+P-1
// own pivot rows Ra .. Ra+64P; on word-columns [col0, col0+ncols) of those rows
//   for t = 0..P-1:  rows of panel u > t  ^=  Y_t[row] * (pivot rows of t)
// (the in-place X = L11^-1 C of SPEC.md:328-345 restricted to a 64P-row block).
// One 128-thread CTA per word-column: the column segment (<= 1024 words) sits in
// shared memory; per panel a 4-bit lookup table of its 64 final pivot words (16
// groups x 16 entries, one 128-byte group per lookup step -> conflict-free)
// turns each row update into 16 lookups, and each thread loads all of its
// multiplier words for the panel at once.  Replaces P launches of the rank-64
// update.
// ---------------------------------------------------------------------------
// NT threads per CTA (one CTA per word-column), up to MAXP panels, the multiplier
// words prefetched PF panels ahead (their L2 round trip is the step's latency floor).
template <int NT, int MAXP, int PF>
__global__ void __launch_bounds__(NT) k_trsm_block(const uint64_t* __restrict__ L, size_t ls,
                                                   uint64_t* __restrict__ C, size_t sc, int P) {
    constexpr int RPT = 64 * MAXP / NT;  // row slots per thread
    __shared__ uint64_t cs[64 * MAXP];
    __shared__ uint64_t tb[256];
    const int tid = threadIdx.x;
    uint64_t* col = C + size_t(blockIdx.x) * sc;
    const int rows = 64 * P;
    // multiplier words of panel t for this thread's rows (rows of panels > t)
    auto load_y = [&](int t, uint64_t (&y)[RPT]) {
        const uint64_t* Y = L + size_t(t) * ls;
        const int r0 = 64 * (t + 1) + tid;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            const int r = r0 + NT * i;
            y[i] = (t < P && r < rows) ? Y[r] : 0;
        }
    };
    uint64_t yq[PF][RPT];
#pragma unroll
    for (int f = 0; f < PF; ++f) load_y(f, yq[f]);
    for (int i = tid; i < rows; i += NT) cs[i] = col[i];
    __syncthreads();
    for (int t = 0; t < P; ++t) {
        const int r0 = 64 * (t + 1) + tid;
        uint64_t y[RPT];
#pragma unroll
        for (int i = 0; i < RPT; ++i) y[i] = yq[0][i];
#pragma unroll
        for (int f = 0; f + 1 < PF; ++f)
#pragma unroll
            for (int i = 0; i < RPT; ++i) yq[f][i] = yq[f + 1][i];
        if (t + PF < P) load_y(t + PF, yq[PF - 1]);
        // 4-bit table of panel t's final pivot words
        const uint64_t* B = cs + 64 * t;
        for (int e = tid; e < 256; e += NT) {
            const int g = e >> 4, v = e & 15;
            uint64_t x = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if ((v >> i) & 1) x ^= B[4 * g + i];
            tb[e] = x;
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            const int r = r0 + NT * i;
            if (r < rows) {
                uint64_t x = 0;
#pragma unroll
                for (int g = 0; g < 16; ++g) x ^= tb[16 * g + int((y[i] >> (4 * g)) & 15)];
                cs[r] ^= x;
            }
        }
        __syncthreads();
    }
    for (int i = 64 + tid; i < rows; i += NT) col[i] = cs[i];  // panel 0's rows are unchanged
}

cudaError_t launch_trsm_block(uint64_t* W, size_t stride, int a, int P, size_t Ra, size_t col0, int ncols,
                              cudaStream_t s) {
    return launch_trsm_block_l(W + size_t(a) * stride + Ra, stride, W + col0 * stride + Ra, stride, P, ncols, s);
}

int trsm_max_panels() { return 64; }

cudaError_t launch_trsm_block_l(const uint64_t* L, size_t ls, uint64_t* C, size_t sc, int P, int ncols,
                                cudaStream_t s) {
    if (P < 1 || P > trsm_max_panels() || ncols < 1) return cudaErrorInvalidValue;
    // F2GPU_TRSM_KERNEL=1: the multiplier words two panels ahead / 512 threads at P > 32
    // (65536^2, TRSM base 32: no faster -- at the top split the base is bound by the
    // shared-memory lookups, 16 per row and panel, not by the L2 round trips)
    const bool alt = options().trsm_kernel == 1;
    if (P <= 16) {
        if (alt) k_trsm_block<128, 16, 2><<<ncols, 128, 0, s>>>(L, ls, C, sc, P);
        else k_trsm_block<128, 16, 1><<<ncols, 128, 0, s>>>(L, ls, C, sc, P);
    } else if (P <= 32) {
        if (alt) k_trsm_block<256, 32, 2><<<ncols, 256, 0, s>>>(L, ls, C, sc, P);
        else k_trsm_block<256, 32, 1><<<ncols, 256, 0, s>>>(L, ls, C, sc, P);
    } else {
        if (alt) k_trsm_block<512, 64, 1><<<ncols, 512, 0, s>>>(L, ls, C, sc, P);
        else k_trsm_block<256, 64, 1><<<ncols, 256, 0, s>>>(L, ls, C, sc, P);
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// block XOR (Strassen-Winograd additions)
// ---------------------------------------------------------------------------
// 2D grid: blockIdx.y = word-column, threads stride over 4-word (32 B) row chunks
// with 256-bit accesses when every operand is 32-byte aligned (Strassen views are:
// strides are multiples of 128 rows and quadrant offsets multiples of 64 rows).
__global__ void __launch_bounds__(256) k_xor(uint64_t* __restrict__ dst, size_t sd,
                                             const uint64_t* __restrict__ a, size_t sa,
                                             const uint64_t* __restrict__ b, size_t sb,
                                             const uint64_t* __restrict__ c, size_t sc,
                                             const uint64_t* __restrict__ d, size_t sdd,
                                             size_t rows, bool acc, bool vec) {
    const size_t q = blockIdx.y;
    uint64_t* dp = dst + q * sd;
    const uint64_t* ap = a ? a + q * sa : nullptr;
    const uint64_t* bp = b ? b + q * sb : nullptr;
    const uint64_t* cp = c ? c + q * sc : nullptr;
    const uint64_t* ep = d ? d + q * sdd : nullptr;
    if (vec) {
        const size_t nq = rows / 4;
        for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nq;
             i += size_t(gridDim.x) * blockDim.x) {
            uint64_t v0 = 0, v1 = 0, v2 = 0, v3 = 0, x0, x1, x2, x3;
            if (acc) ld256(dp + 4 * i, v0, v1, v2, v3);
            if (ap) { ld256(ap + 4 * i, x0, x1, x2, x3); v0 ^= x0; v1 ^= x1; v2 ^= x2; v3 ^= x3; }
            if (bp) { ld256(bp + 4 * i, x0, x1, x2, x3); v0 ^= x0; v1 ^= x1; v2 ^= x2; v3 ^= x3; }
            if (cp) { ld256(cp + 4 * i, x0, x1, x2, x3); v0 ^= x0; v1 ^= x1; v2 ^= x2; v3 ^= x3; }
            if (ep) { ld256(ep + 4 * i, x0, x1, x2, x3); v0 ^= x0; v1 ^= x1; v2 ^= x2; v3 ^= x3; }
            st256(dp + 4 * i, v0, v1, v2, v3);
        }
        return;
    }
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < rows;
         i += size_t(gridDim.x) * blockDim.x) {
        uint64_t v = acc ? dp[i] : 0ull;
        if (ap) v ^= ap[i];
        if (bp) v ^= bp[i];
        if (cp) v ^= cp[i];
        if (ep) v ^= ep[i];
        dp[i] = v;
    }
}

cudaError_t launch_xor(uint64_t* dst, size_t sd, const uint64_t* a, size_t sa, const uint64_t* b,
                       size_t sb, const uint64_t* c, size_t scc, const uint64_t* d, size_t sdd,
                       size_t rows, size_t wcols, bool acc, cudaStream_t s) {
    if (rows == 0 || wcols == 0) return cudaSuccess;
    auto al = [](const void* p, size_t st) {
        return !p || ((reinterpret_cast<uintptr_t>(p) % 32) == 0 && st % 4 == 0);
    };
    const bool vec = rows % 4 == 0 && al(dst, sd) && al(a, sa) && al(b, sb) && al(c, scc) &&
                     al(d, sdd);
    const size_t work = vec ? rows / 4 : rows;
    const unsigned bx = unsigned(std::min<size_t>((work + 255) / 256, 64));
    dim3 grid(bx, unsigned(wcols));
    k_xor<<<grid, 256, 0, s>>>(dst, sd, a, sa, b, sb, c, scc, d, sdd, rows, acc, vec);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// bit transpose: one warp per 64x64 tile (transpose_tile, bit_matrix.hpp:59-70)
// ---------------------------------------------------------------------------
// out (m x n) = a (n x m)^T.  Grid: blockIdx.y = input word-column q, each warp
// transposes kTrTilesPerWarp consecutive 64-row tiles of it (loads issued
// together); no integer division in the kernel.
constexpr int kTrTilesPerWarp = 2;
__global__ void __launch_bounds__(256) k_transpose(const uint64_t* __restrict__ a, size_t n,
                                                   size_t m, size_t sa, uint64_t* __restrict__ out,
                                                   size_t so) {
    const int lane = threadIdx.x & 31;
    const size_t q = blockIdx.y, mt = (n + 63) / 64;
    const size_t tr0 = (size_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5)) * kTrTilesPerWarp;
    const uint64_t* col = a + q * sa;
    uint64_t x0[kTrTilesPerWarp], x1[kTrTilesPerWarp];
#pragma unroll
    for (int u = 0; u < kTrTilesPerWarp; ++u) {
        const size_t i0 = (tr0 + u) * 64;
        x0[u] = (i0 + lane < n) ? col[i0 + lane] : 0;
        x1[u] = (i0 + lane + 32 < n) ? col[i0 + lane + 32] : 0;
    }
    const size_t orow = q * 64;
#pragma unroll
    for (int u = 0; u < kTrTilesPerWarp; ++u) {
        const size_t tr = tr0 + u;
        if (tr >= mt) break;  // warp-uniform
        warp_transpose64(x0[u], x1[u], lane);
        uint64_t* o = out + tr * so + orow;
        if (orow + lane < m) o[lane] = x0[u];
        if (orow + lane + 32 < m) o[lane + 32] = x1[u];
    }
}

cudaError_t launch_transpose(const uint64_t* a, size_t n, size_t m, size_t sa, uint64_t* out,
                             size_t so, cudaStream_t s) {
    const size_t mu = (m + 63) / 64, mt = (n + 63) / 64;
    if (mu == 0 || mt == 0) return cudaSuccess;
    if (mu > 65535) return cudaErrorInvalidValue;
    const size_t per_block = 8 * kTrTilesPerWarp;
    dim3 grid(unsigned((mt + per_block - 1) / per_block), unsigned(mu));
    k_transpose<<<grid, 256, 0, s>>>(a, n, m, sa, out, so);
    return cudaGetLastError();
}

// dst word-column q, row i  <-  src word-column q, row perm[i]   (i < n, q < nq):
// materialises a column chunk uploaded in original row order under the
// composite row permutation of the panels already factored
__global__ void __launch_bounds__(256) k_gather_rows(uint64_t* __restrict__ dst, size_t sd,
                                                     const uint64_t* __restrict__ src, size_t ss,
                                                     const uint32_t* __restrict__ perm, size_t n) {
    const size_t q = blockIdx.y;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        dst[q * sd + i] = src[q * ss + perm[i]];
}
cudaError_t launch_gather_rows(uint64_t* dst, size_t sd, const uint64_t* src, size_t ss, const uint32_t* perm,
                               size_t n, size_t nq, cudaStream_t s) {
    if (n == 0 || nq == 0) return cudaSuccess;
    if (nq > 65535) return cudaErrorInvalidValue;
    dim3 grid(unsigned(std::min<size_t>((n + 255) / 256, 64)), unsigned(nq));
    k_gather_rows<<<grid, 256, 0, s>>>(dst, sd, src, ss, perm, n);
    return cudaGetLastError();
}

// identity block: bit (i, 64*wcol0 + i) = 1 for i < rows (the matrix is zeroed)
__global__ void k_set_diag(uint64_t* w, size_t stride, size_t rows, size_t wcol0) {
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < rows; i += size_t(gridDim.x) * blockDim.x)
        w[(wcol0 + i / 64) * stride + i] |= uint64_t(1) << (i % 64);
}
cudaError_t launch_set_diag(uint64_t* w, size_t stride, size_t rows, size_t wcol0, cudaStream_t s) {
    if (rows == 0) return cudaSuccess;
    k_set_diag<<<256, 256, 0, s>>>(w, stride, rows, wcol0);
    return cudaGetLastError();
}

__global__ void k_iota(uint32_t* p, size_t n) {
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x)
        p[i] = uint32_t(i);
}
cudaError_t launch_iota(uint32_t* p, size_t n, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_iota<<<256, 256, 0, s>>>(p, n);
    return cudaGetLastError();
}

__global__ void k_mask_cols(uint64_t* w, size_t stride, size_t n, uint64_t mask) {
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x)
        w[i] &= mask;
}
// re-zero the padding bits of the last word-column (mask_padding, bit_matrix.hpp:312-318)
cudaError_t launch_mask_cols(uint64_t* w, size_t stride, size_t n, size_t m, cudaStream_t s) {
    const size_t mu = (m + 63) / 64;
    if (mu == 0 || n == 0 || m % 64 == 0) return cudaSuccess;
    const uint64_t mask = (1ull << (m % 64)) - 1;
    k_mask_cols<<<64, 256, 0, s>>>(w + (mu - 1) * stride, stride, n, mask);
    return cudaGetLastError();
}

cudaError_t init_kernel_attrs() {
    cudaError_t e = cudaFuncSetAttribute(k_update, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(kTabBytes));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_update_v3, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(kV3Smem));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_update_v4, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(kV4Smem));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(kTabBytes));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_gemm_v2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(kG2Smem));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_gemm_batched, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(kG2Smem));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_panel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(sizeof(PanelSmem)));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_panel_gj, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(kPanelGjSmemMax));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_panel_chain, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(kPanelGjSmemMax));
    static_assert(sizeof(ChainSmem) <= kPanelGjSmemMax, "chain smem");
    // CUDA loads kernels lazily, and a first launch that has to load can wait for the
    // device to go idle.  k_panel_chain spins on counters of kernels launched after it,
    // so every kernel of the fused schedule is loaded here, before any launch (the ones
    // above by their attribute calls, the fused post by this query).
    if (e == cudaSuccess) {
        cudaFuncAttributes fa;
        e = cudaFuncGetAttributes(&fa, k_post_col);
    }
    kPanelGjSmemBytes = options().panel_smem ? kPanelGjSmemMax : sizeof(PanelGjSmem);
    g_panel_gj = options().panel != 0;
    return e;
}

}  // namespace f2
