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

namespace f2 {

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

// XOR of the nt table entries addressed by the groups of `a`
__device__ __forceinline__ uint64_t lookup(const uint64_t* __restrict__ tl, uint64_t a, int nt) {
    uint64_t acc = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t)
        if (t < nt) acc ^= tl[(128 * t + int((a >> (7 * t)) & 127)) * kTabCols];
    if (nt > 8) acc ^= tl[(1024 + int(a >> 56)) * kTabCols];
    return acc;
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

cudaError_t launch_update(const UpdateArgs& a, int num_sms, cudaStream_t s) {
    if (a.ncols <= 0) return cudaSuccess;
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

cudaError_t launch_gemm(const GemmArgs& g, int num_sms, cudaStream_t s) {
    if (g.n == 0 || g.k == 0 || g.mcols <= 0) return cudaSuccess;
    const size_t KB = (g.k + 63) / 64;
    const size_t units = ((g.n + kGemmRows - 1) / kGemmRows) *
                         ((size_t(g.mcols) + kTabCols - 1) / kTabCols) * KB;
    const int grid = int(units < size_t(num_sms) ? units : size_t(num_sms));
    k_gemm<<<grid, kGemmThreads, kTabBytes, s>>>(g);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K4: panel kernel — Procedure buildZ
// ---------------------------------------------------------------------------
// One CTA of 512 threads.  The first kPanelWin rows of the panel are cached in
// shared memory (loaded lazily, 512 rows at a time, only as far as the pivot
// search reaches); rows beyond are read/written in place in global memory.
// Each of the 64 sequential steps: warp 0 forms the mask c from M (two
// ballots), the CTA finds the FIRST row i >= i_b with odd popcount(c & A_i)
// (ballot + per-warp first index, min over warps) — the reference's
// lowest-index tie-break — and warp 0 performs the swap and the
// Gauss-Jordan update of Z and M with __reduce_xor_sync.  An orig[] array
// tracks where each row came from, giving the composite permutation that the
// swap kernel applies to every other word-column.
constexpr int kPanelThreads = 512;
constexpr int kPanelWin = 8192;
constexpr uint32_t kNone = 0xFFFFFFFFu;

struct PanelSmem {
    uint64_t win[kPanelWin];
    uint32_t orig[kPanelWin];
    uint32_t ext_pos[64];
    uint32_t ext_orig[64];
    uint32_t wfirst[2][kPanelThreads / 32];
    uint64_t c;
    uint32_t n_ext;
    uint32_t npairs;
};

__device__ __forceinline__ uint64_t xor_reduce64(uint64_t v) {
    const uint32_t lo = __reduce_xor_sync(0xffffffffu, uint32_t(v));
    const uint32_t hi = __reduce_xor_sync(0xffffffffu, uint32_t(v >> 32));
    return (uint64_t(hi) << 32) | lo;
}

__global__ void __launch_bounds__(kPanelThreads, 1)
    k_panel(uint64_t* __restrict__ col, size_t n, PanelState* __restrict__ st_all, int j) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    PanelSmem& S = *reinterpret_cast<PanelSmem*>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const size_t R = j == 0 ? 0 : size_t(st_all[j - 1].R) + st_all[j - 1].r;
    PanelState* st = st_all + j;
    const size_t rows = R < n ? n - R : 0;
    if (rows == 0) {
        if (tid == 0) { st->R = uint32_t(R < n ? R : n); st->r = 0; st->npairs = 0; st->flags = 0; }
        if (tid < 64) st->Z[tid] = 0;
        return;
    }
    uint64_t* A = col + R;
    if (tid == 0) { S.n_ext = 0; S.npairs = 0; }

    // warp-0 registers: Z_l, Z_{l+32}, M_l, M_{l+32}
    uint64_t z0 = 1ull << lane, z1 = 1ull << (lane + 32);
    uint64_t m0 = z0, m1 = z1;
    uint64_t sel = 0;  // bit k set iff step k selected a row (P_k != -1)
    size_t ib = 0, loaded = 0;
    int par = 0;
    const size_t winrows = rows < size_t(kPanelWin) ? rows : size_t(kPanelWin);

    for (int k = 0; k < 64; ++k) {
        if (warp == 0) {  // c = 2^k xor sum_{i<k, M_i bit k} 2^i   (:989-992)
            const uint32_t lo = __ballot_sync(0xffffffffu, lane < k && ((m0 >> k) & 1));
            const uint32_t hi = __ballot_sync(0xffffffffu, lane + 32 < k && ((m1 >> k) & 1));
            if (lane == 0) S.c = (1ull << k) | lo | (uint64_t(hi) << 32);
        }
        __syncthreads();
        const uint64_t c = S.c;
        size_t found = kNone;
        for (size_t base = ib; base < rows; base += kPanelThreads) {  // (:993-1000)
            const size_t need = (base + kPanelThreads < winrows) ? base + kPanelThreads : winrows;
            while (loaded < need) {
                const size_t x = loaded + tid;
                if (x < winrows) { S.win[x] = A[x]; S.orig[x] = uint32_t(x); }
                loaded += kPanelThreads;
                if (loaded > winrows) loaded = winrows;
                __syncthreads();
            }
            const size_t i = base + tid;
            bool hit = false;
            if (i < rows) {
                const uint64_t v = i < size_t(kPanelWin) ? S.win[i] : A[i];
                hit = __popcll(c & v) & 1;
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, hit);
            if (lane == 0)
                S.wfirst[par][warp] = bal ? uint32_t(base + warp * 32 + __ffs(bal) - 1) : kNone;
            __syncthreads();
            uint32_t f = kNone;
#pragma unroll
            for (int w = 0; w < kPanelThreads / 32; ++w) f = min(f, S.wfirst[par][w]);
            par ^= 1;
            if (f != kNone) { found = f; break; }
        }
        if (warp == 0) {
            const int kl = k & 31;
            const bool khi = k >= 32;
            if (found != kNone) {
                if (lane == 0) {  // A_i <-> A_ib   (:996)
                    const uint64_t vb = S.win[ib];
                    uint32_t ob = S.orig[ib];
                    if (found < size_t(kPanelWin)) {
                        S.win[ib] = S.win[found];
                        S.orig[ib] = S.orig[found];
                        S.win[found] = vb;
                        S.orig[found] = ob;
                    } else {
                        S.win[ib] = A[found];
                        A[found] = vb;
                        uint32_t e = 0;
                        while (e < S.n_ext && S.ext_pos[e] != uint32_t(found)) ++e;
                        if (e == S.n_ext) {
                            S.ext_pos[e] = uint32_t(found);
                            S.ext_orig[e] = uint32_t(found);
                            S.n_ext = e + 1;
                        }
                        S.orig[ib] = S.ext_orig[e];
                        S.ext_orig[e] = ob;
                    }
                }
                __syncwarp();
                const uint64_t newrow = S.win[ib];  // M_k <- A_ib   (:997)
                if (lane == kl) { if (khi) m1 = newrow; else m0 = newrow; }
                sel |= 1ull << k;
            }
            // Z_k ^= sum_{j<k, y_j} Z_j ; M_k likewise   (:1001-1006)
            const uint64_t y = __shfl_sync(0xffffffffu, khi ? m1 : m0, kl);
            uint64_t zc = 0, mc = 0;
            if (lane < k && ((y >> lane) & 1)) { zc ^= z0; mc ^= m0; }
            if (lane + 32 < k && ((y >> (lane + 32)) & 1)) { zc ^= z1; mc ^= m1; }
            const uint64_t zx = xor_reduce64(zc), mx = xor_reduce64(mc);
            if (lane == kl) {
                if (khi) { z1 ^= zx; m1 ^= mx; } else { z0 ^= zx; m0 ^= mx; }
            }
            const uint64_t zk = __shfl_sync(0xffffffffu, khi ? z1 : z0, kl);
            const uint64_t mk = __shfl_sync(0xffffffffu, khi ? m1 : m0, kl);
            // Z_j ^= Z_k, M_j ^= M_k for j<k with c_j   (:1007-1010)
            if (lane < k && ((c >> lane) & 1)) { z0 ^= zk; m0 ^= mk; }
            if (lane + 32 < k && ((c >> (lane + 32)) & 1)) { z1 ^= zk; m1 ^= mk; }
        }
        if (found != kNone) ++ib;
    }
    __syncthreads();
    // write back touched window rows and collect the composite permutation
    for (size_t x = tid; x < loaded; x += kPanelThreads) {
        const uint32_t o = S.orig[x];
        if (o != uint32_t(x)) {
            A[x] = S.win[x];
            const uint32_t e = atomicAdd(&S.npairs, 1u);
            st->dst[e] = uint32_t(x);
            st->src[e] = o;
        }
    }
    __syncthreads();
    if (tid < int(S.n_ext)) {
        const uint32_t pos = S.ext_pos[tid], o = S.ext_orig[tid];
        if (o != pos) {
            const uint32_t e = atomicAdd(&S.npairs, 1u);
            st->dst[e] = pos;
            st->src[e] = o;
        }
    }
    if (warp == 0) {
        // compression: drop the bit positions of inserted rows   (:1011-1015)
        uint64_t msk = 0;
        for (int i = 0; i < 64; ++i) {
            if (!((sel >> i) & 1)) {
                z0 = ((z0 >> 1) & ~msk) ^ (z0 & msk);
                z1 = ((z1 >> 1) & ~msk) ^ (z1 & msk);
            } else {
                msk = 2 * msk + 1;
            }
        }
        st->Z[lane] = z0;
        st->Z[lane + 32] = z1;
    }
    __syncthreads();
    if (tid == 0) {
        st->R = uint32_t(R);
        st->r = uint32_t(ib);
        st->npairs = S.npairs;
        st->flags = 0;
    }
}

cudaError_t launch_panel(uint64_t* col, size_t n, PanelState* st_all, int j, cudaStream_t s) {
    k_panel<<<1, kPanelThreads, sizeof(PanelSmem), s>>>(col, n, st_all, j);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Y = D*Z over D (rows R+r .. n of the panel column), written in place
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_panel_y(uint64_t* __restrict__ col, size_t n,
                                                 const PanelState* __restrict__ st) {
    __shared__ uint64_t zt[kTabEntries];
    const size_t R = st->R, r = st->r;
    const size_t lo = R + r;
    if (r == 0 || lo >= n) return;
    // single-column tables over the 64 Z words
    for (int it = threadIdx.x; it < 40; it += blockDim.x) {
        const int t = it < 32 ? (it >> 2) : 8;
        const int chunk = it < 32 ? (it & 3) : it - 32;
        const int sz = t < 8 ? 7 : 8;
        uint64_t rows[8];
#pragma unroll
        for (int b = 0; b < 8; ++b) rows[b] = b < sz ? st->Z[7 * t + b] : 0ull;
        uint64_t cur = 0;
#pragma unroll
        for (int hb = 0; hb < 3; ++hb)
            if ((chunk >> hb) & 1) cur ^= rows[5 + hb];
        uint64_t* dst = zt + 128 * t + chunk * 32;
        uint64_t v[32];
        v[0] = cur;
#pragma unroll
        for (int b = 0; b < 5; ++b)
#pragma unroll
            for (int g = 1 << b; g < (2 << b); ++g) v[g] = v[g - (1 << b)] ^ rows[b];
#pragma unroll
        for (int g = 0; g < 32; ++g) dst[g] = v[g];
    }
    __syncthreads();
    for (size_t i = lo + size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x) {
        const uint64_t d = col[i];
        uint64_t y = 0;
#pragma unroll
        for (int t = 0; t < 8; ++t) y ^= zt[128 * t + int((d >> (7 * t)) & 127)];
        y ^= zt[1024 + int(d >> 56)];
        col[i] = y;
    }
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
__global__ void __launch_bounds__(256) k_swaps(uint64_t* __restrict__ w, size_t stride,
                                               int ncols, int skip_col,
                                               uint32_t* __restrict__ perm,
                                               const PanelState* __restrict__ st) {
    const int gw = int((size_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (gw > ncols || gw == skip_col) return;
    const uint32_t np = st->npairs;
    if (np == 0) return;
    const size_t R = st->R;
    if (gw == ncols) {
        if (!perm) return;
        uint32_t v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (lane + 32 * e < int(np)) v[e] = perm[R + st->src[lane + 32 * e]];
        __syncwarp();
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (lane + 32 * e < int(np)) perm[R + st->dst[lane + 32 * e]] = v[e];
        return;
    }
    uint64_t* cp = w + size_t(gw) * stride + R;
    uint64_t v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e)
        if (lane + 32 * e < int(np)) v[e] = cp[st->src[lane + 32 * e]];
    __syncwarp();
#pragma unroll
    for (int e = 0; e < 4; ++e)
        if (lane + 32 * e < int(np)) cp[st->dst[lane + 32 * e]] = v[e];
}

cudaError_t launch_swaps(uint64_t* w, size_t stride, int ncols, int skip_col, uint32_t* perm,
                         const PanelState* st, cudaStream_t s) {
    const int warps = ncols + 1;
    k_swaps<<<(warps + 7) / 8, 256, 0, s>>>(w, stride, ncols, skip_col, perm, st);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// block XOR (Strassen-Winograd additions)
// ---------------------------------------------------------------------------
__global__ void k_xor(uint64_t* __restrict__ dst, size_t sd, const uint64_t* __restrict__ a,
                      size_t sa, const uint64_t* __restrict__ b, size_t sb,
                      const uint64_t* __restrict__ c, size_t sc, const uint64_t* __restrict__ d,
                      size_t sdd, size_t rows, size_t wcols, bool acc) {
    const size_t rq = (rows + 3) / 4;  // 4-word (32 B) chunks per column
    const size_t total = rq * wcols;
    for (size_t e = size_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += size_t(gridDim.x) * blockDim.x) {
        const size_t q = e / rq, i0 = (e % rq) * 4;
        const int cnt = rows - i0 >= 4 ? 4 : int(rows - i0);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            if (t >= cnt) break;
            const size_t i = i0 + t;
            uint64_t v = acc ? dst[q * sd + i] : 0ull;
            if (a) v ^= a[q * sa + i];
            if (b) v ^= b[q * sb + i];
            if (c) v ^= c[q * sc + i];
            if (d) v ^= d[q * sdd + i];
            dst[q * sd + i] = v;
        }
    }
}

cudaError_t launch_xor(uint64_t* dst, size_t sd, const uint64_t* a, size_t sa, const uint64_t* b,
                       size_t sb, const uint64_t* c, size_t scc, const uint64_t* d, size_t sdd,
                       size_t rows, size_t wcols, bool acc, cudaStream_t s) {
    if (rows == 0 || wcols == 0) return cudaSuccess;
    const size_t total = (rows + 3) / 4 * wcols;
    size_t blocks = (total + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_xor<<<unsigned(blocks), 256, 0, s>>>(dst, sd, a, sa, b, sb, c, scc, d, sdd, rows, wcols, acc);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// bit transpose: one warp per 64x64 tile (transpose_tile, bit_matrix.hpp:59-70)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_transpose(const uint64_t* __restrict__ a, size_t n,
                                                   size_t m, size_t sa, uint64_t* __restrict__ out,
                                                   size_t so) {
    __shared__ uint64_t tiles[8][64];
    const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t mu = (m + 63) / 64, mt = (n + 63) / 64;
    const size_t tile = size_t(blockIdx.x) * 8 + wl;
    if (tile >= mu * mt) return;
    const size_t q = tile / mt, tr = tile % mt;
    uint64_t* x = tiles[wl];
    const size_t i0 = tr * 64;
    x[lane] = (i0 + lane < n) ? a[q * sa + i0 + lane] : 0ull;
    x[lane + 32] = (i0 + lane + 32 < n) ? a[q * sa + i0 + lane + 32] : 0ull;
    __syncwarp();
    uint64_t msk = 0x00000000FFFFFFFFull;
    for (int jj = 32; jj != 0; jj >>= 1, msk ^= (msk << jj)) {
        const int k = ((lane & ~(jj - 1)) << 1) | (lane & (jj - 1));
        const uint64_t t = ((x[k] >> jj) ^ x[k + jj]) & msk;
        __syncwarp();
        x[k + jj] ^= t;
        x[k] ^= t << jj;
        __syncwarp();
    }
    const size_t orow = q * 64;
    if (orow + lane < m) out[tr * so + orow + lane] = x[lane];
    if (orow + lane + 32 < m) out[tr * so + orow + lane + 32] = x[lane + 32];
}

cudaError_t launch_transpose(const uint64_t* a, size_t n, size_t m, size_t sa, uint64_t* out,
                             size_t so, cudaStream_t s) {
    const size_t tiles = ((m + 63) / 64) * ((n + 63) / 64);
    if (tiles == 0) return cudaSuccess;
    k_transpose<<<unsigned((tiles + 7) / 8), 256, 0, s>>>(a, n, m, sa, out, so);
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
        e = cudaFuncSetAttribute(k_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(kTabBytes));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_panel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(sizeof(PanelSmem)));
    return e;
}

}  // namespace f2
