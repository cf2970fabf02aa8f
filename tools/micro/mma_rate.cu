// Issue-rate ceiling of the kind::mxf4 MMA shapes the fp4 leaves use: one thread
// issues `iters` MMAs back to back (operands fixed, contents irrelevant), one
// commit at the end.  Prints cycles per MMA and the implied fraction of the
// 16384 fp4 MAC/clk/SM peak.  Variants: cta_group::1 / ::2, A operand from
// shared memory (ss) or TMEM (ts), N = 224 / 240 / 256.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o mma_rate.bin mma_rate.cu
#include <cstdio>
#include <cstdint>
#include "../../paper_1209_5198_b200/csrc/tc_common.cuh"

using namespace f2;

template <int CG, bool TS, int N>
__global__ void __cluster_dims__(2, 1, 1) rate(long long* out, int iters) {
    __shared__ __align__(1024) unsigned char a[128 * 64];
    __shared__ __align__(1024) unsigned char b[256 * 64];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    const uint32_t rank = cluster_rank();
    if (threadIdx.x == 0) { mbar_init_n(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) a[i] = 0x22;
    for (int i = threadIdx.x; i < 256 * 64; i += blockDim.x) b[i] = 0x22;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        if (CG == 2) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sm_u32(&slot)), "r"(512u));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sm_u32(&slot)), "r"(512u));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    cluster_sync_all();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = slot;
    const uint32_t idesc = idesc_f4(CG == 2 ? 256 : 128, N);
    const uint32_t tsf = tmem + 480, ta = tmem + 448;
    if (threadIdx.x == 0 && (CG == 1 || rank == 0)) {
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint64_t db = umma_desc(sm_u32(b) + 32 * (i & 1));
            const uint32_t acc = i > 0;
            if (CG == 2) {
                if (TS)
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
                                 "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.scale_vec::2X [%0], [%1], %2, %4, [%5], [%5], p;\n\t}\n" ::"r"(tmem),
                                 "r"(ta), "l"(db), "r"(acc), "r"(idesc), "r"(tsf));
                else
                    mma_f4_pair(tmem, umma_desc(sm_u32(a) + 32 * (i & 1)), db, idesc, acc, tsf);
            } else {
                if (TS)
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], [%1], %2, %4, [%5], [%5], p;\n\t}\n" ::"r"(tmem),
                                 "r"(ta), "l"(db), "r"(acc), "r"(idesc), "r"(tsf));
                else
                    mma_f4(tmem, umma_desc(sm_u32(a) + 32 * (i & 1)), db, idesc, acc, tsf);
            }
        }
        const long long t1 = clock64();
        if (CG == 2) tc_commit_pair(&bar, 0x3); else tc_commit(&bar);
        mbar_wait1(&bar, 0);
        const long long t2 = clock64();
        if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
    } else if (CG == 2 && threadIdx.x == 0) {
        mbar_wait1(&bar, 0);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    cluster_sync_all();
    if (warp == 0) {
        if (CG == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
        else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
    }
}

template <int CG, bool TS, int N>
void run(const char* name, long long* d, int grid) {
    const int iters = 4096;
    rate<CG, TS, N><<<grid, 128>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[2];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    const double macs_sm = double(CG == 2 ? 128 : 128) * N * 64;  // per SM per MMA
    const double cyc = double(h[1]) / iters;
    printf("%-22s grid %3d: issue %.1f cyc/MMA, complete %.1f cyc/MMA -> %.0f%% of 16384 MAC/clk/SM (%s)\n", name, grid,
           double(h[0]) / iters, cyc, 100.0 * macs_sm / cyc / 16384.0, cudaGetErrorString(e));
}

int main() {
    long long* d;
    cudaMalloc(&d, 16);
    for (int grid : {2, 148}) {
        run<2, true, 224>("2cta ts N=224", d, grid);
        run<2, false, 224>("2cta ss N=224", d, grid);
        run<2, true, 256>("2cta ts N=256", d, grid);
        run<2, false, 256>("2cta ss N=256", d, grid);
        run<1, false, 240>("1cta ss N=240", d, grid);
        run<1, true, 240>("1cta ts N=240", d, grid);
        run<1, false, 256>("1cta ss N=256", d, grid);
    }
    return 0;
}
