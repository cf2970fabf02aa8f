// Micro-benchmark: latency of tcgen05.commit -> mbarrier completion (no MMA in
// flight, and after one small fp4 MMA), and of an mbarrier arrive -> try_wait
// wake-up across warps.  Prints cycles per round trip.
#include <cstdio>
#include <cstdint>
#include "../../paper_1209_5198_b200/csrc/tc_common.cuh"
using namespace f2;

__global__ void k(long long* out, int iters) {
    __shared__ __align__(1024) unsigned char tile[2][16384];
    __shared__ uint64_t bar[4];
    __shared__ uint32_t tm;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sm_u32(&tm)), "r"(512u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) { for (int i = 0; i < 4; ++i) mbar_init_n(&bar[i], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    for (int i = tid; i < 2 * 16384; i += blockDim.x) (&tile[0][0])[i] = 0;
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tm;
    // 1) commit with nothing in flight
    if (tid == 0) {
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) { tc_commit(&bar[0]); mbar_wait1(&bar[0], i & 1); }
        out[0] = (clock64() - t0) / iters;
        // 2) one fp4 MMA 128x192x64 + commit
        t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            mma_f4(tmem, umma_desc(sm_u32(tile[0])), umma_desc(sm_u32(tile[1])), idesc_f4(128, 192), 1u, tmem + 448);
            tc_commit(&bar[1]); mbar_wait1(&bar[1], i & 1);
        }
        out[1] = (clock64() - t0) / iters;
        // 3) two MMAs + commit
        t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            mma_f4(tmem, umma_desc(sm_u32(tile[0])), umma_desc(sm_u32(tile[1])), idesc_f4(128, 192), 1u, tmem + 448);
            mma_f4(tmem, umma_desc(sm_u32(tile[0]) + 32), umma_desc(sm_u32(tile[1]) + 32), idesc_f4(128, 192), 1u, tmem + 448);
            tc_commit(&bar[2]); mbar_wait1(&bar[2], i & 1);
        }
        out[2] = (clock64() - t0) / iters;
        // 4) throughput: 64 back-to-back MMA pairs then one commit
        t0 = clock64();
        for (int i = 0; i < iters; ++i)
            mma_f4(tmem + 192 * (i & 1), umma_desc(sm_u32(tile[0])), umma_desc(sm_u32(tile[1])), idesc_f4(128, 192), 1u, tmem + 448);
        tc_commit(&bar[3]); mbar_wait1(&bar[3], 0);
        out[3] = (clock64() - t0) / iters;
    }
    __syncthreads();
    // 5) ping-pong between warp 0 and warp 1 through two mbarriers
    __shared__ uint64_t pp[2];
    if (tid == 0) { mbar_init_n(&pp[0], 1); mbar_init_n(&pp[1], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncthreads();
    if (warp < 2 && lane == 0) {
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            if (warp == 0) { mbar_arrive1(&pp[0]); mbar_wait1(&pp[1], i & 1); }
            else { mbar_wait1(&pp[0], i & 1); mbar_arrive1(&pp[1]); }
        }
        if (warp == 0) out[4] = (clock64() - t0) / iters;
    }
    // 5b) ping-pong with a non-blocking test_wait spin
    __shared__ uint64_t pq[2];
    __syncthreads();
    if (tid == 0) { mbar_init_n(&pq[0], 1); mbar_init_n(&pq[1], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncthreads();
    auto spin = [](uint64_t* b, uint32_t ph) {
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok) : "r"(sm_u32(b)), "r"(ph) : "memory");
    };
    if (warp < 2 && lane == 0) {
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            if (warp == 0) { mbar_arrive1(&pq[0]); spin(&pq[1], i & 1); }
            else { spin(&pq[0], i & 1); mbar_arrive1(&pq[1]); }
        }
        if (warp == 0) out[6] = (clock64() - t0) / iters;
    }
    // 6) tcgen05.ld 32x32b.x32 x2 + wait
    if (warp == 2) {
        uint32_t v[32];
        long long t0 = clock64();
        uint32_t acc = 0;
        for (int i = 0; i < iters; ++i) {
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31]) : "r"(tmem + (64u << 16) + (i & 7) * 32));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            acc ^= v[0] ^ v[31];
        }
        out[5] = (clock64() - t0) / iters;
        if (acc == 12345) out[7] = acc;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
}

int main() {
    long long* d; cudaMalloc(&d, 8 * sizeof(long long)); cudaMemset(d, 0, 64);
    k<<<1, 128>>>(d, 256);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[8]; cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
    printf("err=%s\ncommit_empty=%lld\nmma1_commit=%lld\nmma2_commit=%lld\nmma_tput=%lld\nmbar_pingpong=%lld\nldtm_x32=%lld\npingpong_testwait=%lld\n",
           cudaGetErrorString(e), h[0], h[1], h[2], h[3], h[4], h[5], h[6]);
    return 0;
}
