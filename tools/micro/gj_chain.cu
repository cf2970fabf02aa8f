// Selection-chain microbenchmark of the transposed Gauss-Jordan panel step
// (k_panel_gj warp 0, fast path only): the current step, which broadcasts
// column k with a shuffle at the start of every step (on the chain), against a
// recurrence that derives column k+1 from column k+1 as it stood before step k
// (shuffled one step ahead, off the chain) with uniform mask arithmetic.
// Both write the same log (column-k position mask per selection); the host
// compares the logs of every window and prints cycles per step.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gj_chain.bin gj_chain.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

constexpr int W = 3;
constexpr uint32_t kPos = 96;

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

template <bool REC>
__global__ void __launch_bounds__(32) k_chain(const uint64_t* __restrict__ rows, uint4* __restrict__ log_out,
                                              long long* __restrict__ cyc) {
    const int lane = threadIdx.x;
    const uint64_t* A = rows + size_t(blockIdx.x) * kPos;
    uint32_t c0[W], c1[W], live[W];
    {
        uint64_t x0 = A[lane], x1 = A[lane + 32], z0 = A[lane + 64], z1 = 0;
        warp_transpose64(x0, x1, lane);
        warp_transpose64(z0, z1, lane);
        c0[0] = uint32_t(x0); c0[1] = uint32_t(x0 >> 32); c0[2] = uint32_t(z0);
        c1[0] = uint32_t(x1); c1[1] = uint32_t(x1 >> 32); c1[2] = uint32_t(z1);
        live[0] = live[1] = live[2] = 0xffffffffu;
    }
    uint32_t ibm[W] = {1u, 0u, 0u};
    uint32_t ib = 0;
    bool bad = false;
    __shared__ uint4 lg[64];
    // REC: ck = column k after step k-1 (uniform), o = column k+1 after step k-1
    uint32_t ck[W], o[W];
#pragma unroll
    for (int w = 0; w < W; ++w) {
        ck[w] = __shfl_sync(0xffffffffu, c0[w], 0);
        o[w] = __shfl_sync(0xffffffffu, c0[w], 1);
    }
    __syncwarp();
    const long long t0 = clock64();
#pragma unroll
    for (int k = 0; k < 64; ++k) {
        const bool hi = k >= 32;
        const int kl = k & 31;
        if (!REC) {
#pragma unroll
            for (int w = 0; w < W; ++w) ck[w] = __shfl_sync(0xffffffffu, hi ? c1[w] : c0[w], kl);
        }
        uint32_t m[W];
#pragma unroll
        for (int w = 0; w < W; ++w) m[w] = ck[w] & live[w];
        if (!(m[0] | m[1] | m[2])) { bad = true; break; }
        uint32_t fm[W], E[W], sw[W];
        fm[0] = m[0] & (0u - m[0]);
        fm[1] = m[0] ? 0u : m[1] & (0u - m[1]);
        fm[2] = (m[0] | m[1]) ? 0u : m[2] & (0u - m[2]);
#pragma unroll
        for (int w = 0; w < W; ++w) {
            E[w] = ck[w] ^ fm[w];
            sw[w] = fm[w] ^ ibm[w];
        }
        auto upd = [&](uint32_t (&c)[W]) {
            const uint32_t bf = 0u - uint32_t(((c[0] & fm[0]) | (c[1] & fm[1]) | (c[2] & fm[2])) != 0);
#pragma unroll
            for (int w = 0; w < W; ++w) c[w] ^= E[w] & bf;
            const uint32_t d = bf ^ (0u - uint32_t(((c[0] & ibm[0]) | (c[1] & ibm[1]) | (c[2] & ibm[2])) != 0));
#pragma unroll
            for (int w = 0; w < W; ++w) c[w] ^= sw[w] & d;
        };
        if (lane == 0) lg[ib] = make_uint4(ck[0], ck[1], ck[2], 0x80000000u | (uint32_t(k) << 8));
        if (REC && k < 63) {
            upd(o);  // column k+1 after this step: the next step's ck (uniform, on the chain)
#pragma unroll
            for (int w = 0; w < W; ++w) ck[w] = o[w];
        }
        if (!hi) upd(c0);
        upd(c1);
        if (REC && k < 62) {
            // column k+2 after this step, one step ahead of its use (off the chain)
            const int k2 = k + 2;
#pragma unroll
            for (int w = 0; w < W; ++w) o[w] = __shfl_sync(0xffffffffu, k2 >= 32 ? c1[w] : c0[w], k2 & 31);
        }
#pragma unroll
        for (int w = 0; w < W; ++w) live[w] &= ~ibm[w];
        ibm[2] = (ibm[2] << 1) | (ibm[1] >> 31);
        ibm[1] = (ibm[1] << 1) | (ibm[0] >> 31);
        ibm[0] = ibm[0] << 1;
        ++ib;
    }
    const long long t1 = clock64();
    __syncwarp();
    for (int t = lane; t < 64; t += 32) log_out[size_t(blockIdx.x) * 64 + t] = uint32_t(t) < ib ? lg[t] : make_uint4(0, 0, 0, 0);
    if (lane == 0) cyc[blockIdx.x] = bad ? -1 : t1 - t0;
}

int main(int argc, char** argv) {
    const int nb = argc > 1 ? atoi(argv[1]) : 2048;
    std::vector<uint64_t> h(size_t(nb) * kPos);
    uint64_t x = 0x9E3779B97F4A7C15ull;
    for (auto& v : h) { x ^= x >> 12; x ^= x << 25; x ^= x >> 27; v = x * 0x2545F4914F6CDD1Dull; }
    // a few windows with structure: duplicate rows and rows that are sums of earlier ones
    for (int b = 0; b < nb; b += 7) {
        uint64_t* w = h.data() + size_t(b) * kPos;
        w[5] = w[2]; w[9] = w[1] ^ w[3]; w[0] = w[1] ^ w[2] ^ w[4];
    }
    uint64_t* d; uint4 *l0, *l1; long long *y0, *y1;
    cudaMalloc(&d, h.size() * 8);
    cudaMalloc(&l0, size_t(nb) * 64 * 16); cudaMalloc(&l1, size_t(nb) * 64 * 16);
    cudaMalloc(&y0, nb * 8); cudaMalloc(&y1, nb * 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 2; ++rep) {
        k_chain<false><<<nb, 32>>>(d, l0, y0);
        k_chain<true><<<nb, 32>>>(d, l1, y1);
    }
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<uint4> a(size_t(nb) * 64), b(size_t(nb) * 64);
    std::vector<long long> ca(nb), cb(nb);
    cudaMemcpy(a.data(), l0, a.size() * 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), l1, b.size() * 16, cudaMemcpyDeviceToHost);
    cudaMemcpy(ca.data(), y0, nb * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(cb.data(), y1, nb * 8, cudaMemcpyDeviceToHost);
    size_t mism = 0, bad = 0;
    double sa = 0, sb = 0;
    for (int i = 0; i < nb; ++i) {
        if (ca[i] < 0 || cb[i] < 0) { ++bad; continue; }
        sa += ca[i]; sb += cb[i];
        for (int t = 0; t < 64; ++t) {
            const uint4 p = a[size_t(i) * 64 + t], q = b[size_t(i) * 64 + t];
            if (p.x != q.x || p.y != q.y || p.z != q.z || p.w != q.w) { ++mism; break; }
        }
    }
    const double ok = double(nb - bad);
    printf("err=%s windows=%d slow(skipped)=%zu log mismatches=%zu  shuffle-on-chain %.1f cyc/step  recurrence %.1f cyc/step\n",
           cudaGetErrorString(e), nb, bad, mism, sa / ok / 64, sb / ok / 64);
    return mism ? 1 : 0;
}
