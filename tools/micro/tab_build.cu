// Cost of building one 16-column M4RM table group (9 groups x 1280 entries x 16
// word-columns = 160 KB of shared memory) in a 512-thread CTA, as k_update_v3
// does before each column group: loads of the 64 B rows from global (L2), the
// doubling XORs and the 20480 stores.  147 CTAs read the same B block (as the
// update's group 0 does).  Prints per-phase clock64 medians of CTA 0.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
constexpr int kTabCols = 16;
constexpr int NTH = 512;

__global__ void __launch_bounds__(NTH, 1) k_tab(const uint64_t* __restrict__ B, size_t sb, long long* out, int mode) {
    extern __shared__ __align__(1024) uint64_t tab[];
    __shared__ uint64_t bs[kTabCols * 66];
    const long long t0 = clock64();
    const int total = 640;
    uint64_t rows[2][8];
    int its[2];
    if (mode == 1) {  // stage B (16 cols x 64 rows) in smem first
        for (int i = threadIdx.x; i < kTabCols * 64; i += NTH) {
            const int col = i >> 6, r = i & 63;
            bs[col * 66 + r] = __ldg(B + size_t(col) * sb + r);
        }
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const int it = threadIdx.x + q * NTH;
        its[q] = it;
        const int col = it & (kTabCols - 1);
        const int cg = it >> 4;
        const int t = cg < 32 ? (cg >> 2) : 8;
        const int sz = t < 8 ? 7 : 8;
        const bool cv = it < total;
        if (mode == 1) {
#pragma unroll
            for (int b = 0; b < 8; ++b) rows[q][b] = (b < sz && cv) ? bs[col * 66 + 7 * t + b] : 0ull;
        } else {
            const uint64_t* bp = B + size_t(col) * sb + 7 * t;
#pragma unroll
            for (int b = 0; b < 8; ++b) rows[q][b] = (b < sz && cv) ? __ldg(bp + b) : 0ull;
        }
    }
    long long t1 = 0;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const int it = its[q];
        if (it >= total) break;
        if (q == 0 && threadIdx.x == 0) t1 = clock64();
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
    __syncthreads();
    const long long t2 = clock64();
    if (threadIdx.x == 0) { out[blockIdx.x * 3] = t1 - t0; out[blockIdx.x * 3 + 1] = t2 - t1; out[blockIdx.x * 3 + 2] = t2 - t0; }
}

int main() {
    const size_t sb = 65536;
    uint64_t* B; long long* out;
    cudaMalloc(&B, 16 * sb * 8); cudaMemset(B, 0x5a, 16 * sb * 8);
    cudaMalloc(&out, 148 * 3 * 8);
    const int smem = 160 * 1024;
    cudaFuncSetAttribute(k_tab, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int mode = 0; mode < 2; ++mode) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            k_tab<<<147, NTH, smem>>>(B, sb, out, mode);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            std::vector<long long> h(147 * 3);
            cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
            std::vector<long long> a, b, c;
            for (int i = 0; i < 147; ++i) { a.push_back(h[3*i]); b.push_back(h[3*i+1]); c.push_back(h[3*i+2]); }
            std::sort(a.begin(), a.end()); std::sort(b.begin(), b.end()); std::sort(c.begin(), c.end());
            printf("mode %d (%s): loads %lld  build+store %lld  total %lld cycles (median; max total %lld)  kernel %.2f us  %s\n",
                   mode, mode ? "staged" : "direct", a[73], b[73], c[73], c[146], ms * 1000, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
