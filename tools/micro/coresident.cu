// Can a small CTA (256 threads, S bytes of static shared memory, ~32 registers) be
// placed on an SM that runs a k_update_v3-sized CTA (544 threads, 224 KiB dynamic
// shared memory, 96 registers)?  A "big" kernel (one CTA per SM, spinning 2 ms)
// runs, then "small" blocks launch on another stream and record their start time
// and SM id; started-during-big = co-resident.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o coresident.bin coresident.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include "../../paper_1209_5198_b200/csrc/kernels.cuh"

__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ uint32_t smid() { uint32_t s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s)); return s; }

__global__ void __launch_bounds__(544, 1) k_big(uint64_t* t_end, uint64_t ns) {
    extern __shared__ uint64_t sm[];
    const uint64_t t0 = gt();
    uint64_t acc = 0;
    while (gt() - t0 < ns) acc += sm[threadIdx.x & 1023];
    if (threadIdx.x == 0) t_end[blockIdx.x] = gt() + (acc == 12345 ? 1 : 0);
}

template <int S>
__global__ void __launch_bounds__(256) k_small(uint64_t* rec) {
    __shared__ uint64_t sm[S / 8 > 0 ? S / 8 : 1];
    constexpr int W = S / 8 > 0 ? S / 8 : 1;
    for (int i = threadIdx.x; i < W; i += 256) sm[i] = i;
    __syncthreads();
    if (threadIdx.x == 0) {
        sm[0] += gt() + sm[(rec[0] & 0xff) % W];
        rec[2 * blockIdx.x] = sm[0];
        rec[2 * blockIdx.x + 1] = smid();
    }
}

__global__ void k_mark(uint64_t* m) { *m = gt(); }

// panel-kernel-like: one CTA, 227 KiB of shared memory, triggers its dependents then spins a bit
__global__ void __launch_bounds__(256, 1) k_pan(uint64_t ns) {
    extern __shared__ uint64_t sm[];
    const uint64_t t0 = gt();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    uint64_t acc = 0;
    while (gt() - t0 < ns) acc += sm[threadIdx.x];
    if (acc == 12345) sm[0] = 1;
}
template <int S>
__global__ void __launch_bounds__(256) k_small_pdl(uint64_t* rec) {
    __shared__ uint64_t sm[S / 8 > 0 ? S / 8 : 1];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) {
        sm[0] = gt();
        rec[2 * blockIdx.x] = sm[0];
        rec[2 * blockIdx.x + 1] = smid();
    }
}

template <int S>
void run_upd(int nsm, int carve, int pdl, int mode) {
    cudaFuncSetAttribute(k_pan, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (carve >= 0) cudaFuncSetAttribute(k_small_pdl<S>, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
    // the real k_update_v3 on a 65536 x 8192 update, then small blocks beside it
    if (carve >= 0) cudaFuncSetAttribute(k_small<S>, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
    const size_t n = 65536, m = 8192, mu = m / 64;
    static uint64_t *C = nullptr, *A = nullptr;
    if (!C) { cudaMalloc(&C, n * mu * 8); cudaMalloc(&A, n * 8); cudaMemset(C, 1, n * mu * 8); cudaMemset(A, 3, n * 8); }
    f2::UpdateArgs u{};
    u.C = C; u.sc = n; u.c_wcol0 = 1; u.ncols = int(mu - 1); u.row_lo = 64; u.row_hi = n; u.a = A; u.k_bits = 64;
    u.B = C; u.sb = n; u.b_row0 = 0; u.b_wcol0 = 1; u.pdl = pdl != 0;
    uint64_t* rec; const int nb = 4 * nsm; cudaMalloc(&rec, nb * 16);
    cudaStream_t a, b;
    cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    uint64_t* mk; cudaMalloc(&mk, 16);
    for (int it = 0; it < 2; ++it) {
        k_mark<<<1, 1, 0, a>>>(mk);
        cudaEventRecord(e0, a);
        f2::launch_update(u, nsm - 2, a);
        cudaEventRecord(e1, a);
        k_mark<<<1, 1, 0, a>>>(mk + 1);
        cudaStreamWaitEvent(b, e0, 0);
        if (mode == 0) {
            k_small<S><<<nb, 256, 0, b>>>(rec);
        } else {
            k_pan<<<1, 256, 227 * 1024, b>>>(2000);
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(nb); cfg.blockDim = dim3(256); cfg.stream = b;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at; cfg.numAttrs = mode == 2 ? 1 : 0;
            cudaLaunchKernelEx(&cfg, k_small_pdl<S>, rec);
        }
        cudaDeviceSynchronize();
    }
    uint64_t hm[2]; cudaMemcpy(hm, mk, 16, cudaMemcpyDeviceToHost);
    float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
    std::vector<uint64_t> hr(nb * 2);
    cudaMemcpy(hr.data(), rec, nb * 16, cudaMemcpyDeviceToHost);
    uint64_t lo = ~0ull, hi = 0;
    for (int i = 0; i < nb; ++i) { lo = hr[2 * i] < lo ? hr[2 * i] : lo; hi = hr[2 * i] > hi ? hr[2 * i] : hi; }
    printf("mode %d pdl %d real update %.1f us (marks %.1f us apart); carveout %3d small smem %5d B: small blocks start %.1f .. %.1f us after the first mark (%s)\n",
           mode, pdl, ms * 1e3, (hm[1] - hm[0]) / 1e3, carve, S, (double(lo) - double(hm[0])) / 1e3, (double(hi) - double(hm[0])) / 1e3,
           cudaGetErrorString(cudaGetLastError()));
}

template <int S>
void run(int nsm, int big_smem, int carve) {
    if (carve >= 0) cudaFuncSetAttribute(k_small<S>, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
    uint64_t *tend, *rec;
    cudaMalloc(&tend, nsm * 8);
    const int nb = 4 * nsm;
    cudaMalloc(&rec, nb * 16);
    cudaStream_t a, b;
    cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
    k_big<<<nsm, 544, big_smem, a>>>(tend, 2000000);
    // let the big CTAs get placed
    uint64_t* d; cudaMalloc(&d, 8);
    k_small<S><<<nb, 256, 0, b>>>(rec);
    cudaDeviceSynchronize();
    std::vector<uint64_t> he(nsm), hr(nb * 2);
    cudaMemcpy(he.data(), tend, nsm * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hr.data(), rec, nb * 16, cudaMemcpyDeviceToHost);
    uint64_t big_end = 0;
    for (auto v : he) big_end = v > big_end ? v : big_end;
    int during = 0;
    for (int i = 0; i < nb; ++i) during += hr[2 * i] < big_end - 100000;
    printf("carveout %3d small static smem %6d B: %d of %d small blocks started while the big CTAs ran (%s)\n", carve, S, during, nb,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int nsm = 0, smsm = 0, rsv = 0, optin = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&smsm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, 0);
    cudaDeviceGetAttribute(&rsv, cudaDevAttrReservedSharedMemoryPerBlock, 0);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
    printf("SMs %d, smem/SM %d, reserved/block %d, opt-in max/block %d\n", nsm, smsm, rsv, optin);
    const int big = 224 * 1024;
    cudaFuncSetAttribute(k_big, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    run<0>(nsm, big, -1);
    run<0>(nsm, big, 100);
    run<1024>(nsm, big, 100);
    run<2048>(nsm, big, 100);
    run<4096>(nsm, big, 100);
    f2::init_kernel_attrs();
    run_upd<0>(nsm, 100, 0, 0);
    run_upd<1024>(nsm, 100, 0, 0);
    run_upd<2048>(nsm, 100, 0, 0);
    run_upd<3072>(nsm, 100, 0, 0);
    run_upd<4096>(nsm, 100, 0, 0);
    run_upd<2048>(nsm, -1, 0, 0);
    return 0;
}
