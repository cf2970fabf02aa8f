// Ceiling of the Schur update's memory pattern on one B200: C (512 MiB) read and
// written once.  Variants:
//   copy      : plain 16-byte LSU copy src -> dst (the measured-peak pattern)
//   rmw_lsu   : C[i] ^= pattern with 16-byte LSU loads/stores (in place)
//   red_bulk  : cp.reduce.async.bulk .xor.b64 from a shared buffer (k_update_v3/v4's
//               write-back), CHUNK bytes per request, DEPTH groups in flight per lane
//   bulk_rt   : cp.async.bulk C tile -> smem, then cp.async.bulk smem -> C (in place)
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rmw_bw.bin rmw_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void k_copy(const uint4* __restrict__ s, uint4* __restrict__ d, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        d[i] = s[i];
}
__global__ void k_rmw(uint4* __restrict__ d, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        uint4 v = d[i];
        v.x ^= 0x9e3779b9u; v.y ^= 1u; v.z ^= 2u; v.w ^= 3u;
        d[i] = v;
    }
}
// unrolled x4: 4 loads in flight per thread before the stores
__global__ void k_rmw4(uint4* __restrict__ d, size_t n) {
    const size_t T = size_t(gridDim.x) * blockDim.x;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += 4 * T) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) if (i + u * T < n) v[u] = d[i + u * T];
#pragma unroll
        for (int u = 0; u < 4; ++u) if (i + u * T < n) { v[u].x ^= 0x9e3779b9u; d[i + u * T] = v[u]; }
    }
}

template <int CHUNK, int DEPTH>
__global__ void k_red(uint64_t* __restrict__ C, size_t bytes) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int lane = threadIdx.x;
    for (int i = lane; i < CHUNK * 8 / 8; i += 32) reinterpret_cast<uint64_t*>(sm)[i] = 0x0101010101010101ull * i;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    const size_t nchunks = bytes / CHUNK;
    // CTA b owns a contiguous range; lane l issues chunks l, l+32, ...
    const size_t c0 = nchunks * blockIdx.x / gridDim.x, c1 = nchunks * (blockIdx.x + 1) / gridDim.x;
    int k = 0;
    for (size_t c = c0 + lane; c < c1; c += 32) {
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.xor.b64 [%0], [%1], %2;" ::"l"(
                         reinterpret_cast<unsigned char*>(C) + c * CHUNK),
                     "r"(smem_u32(sm + (k % 8) * CHUNK)), "r"(CHUNK)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(DEPTH) : "memory");
        ++k;
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
            smem_u32(b)),
        "r"(ph)
        : "memory");
}
// bulk round trip: STAGES buffers of CHUNK bytes; lane 0 of warp 0 loads, then
// writes the same tile back (no compute), one bulk group per tile
template <int CHUNK, int STAGES>
__global__ void k_bulk_rt(uint64_t* __restrict__ C, size_t bytes) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + STAGES * CHUNK);
    if (threadIdx.x != 0) return;
    for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const size_t nchunks = bytes / CHUNK;
    const size_t c0 = nchunks * blockIdx.x / gridDim.x, c1 = nchunks * (blockIdx.x + 1) / gridDim.x;
    auto load = [&](size_t c, int s) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(CHUNK)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(sm + s * CHUNK)),
            "l"(reinterpret_cast<unsigned char*>(C) + c * CHUNK), "r"(CHUNK), "r"(smem_u32(&bar[s]))
            : "memory");
    };
    for (int s = 0; s < STAGES && c0 + s < c1; ++s) load(c0 + s, s);
    uint32_t ph = 0;
    int s = 0;
    for (size_t c = c0; c < c1; ++c) {
        mbar_wait(&bar[s], ph);
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                         reinterpret_cast<unsigned char*>(C) + c * CHUNK),
                     "r"(smem_u32(sm + s * CHUNK)), "r"(CHUNK)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        if (c + STAGES < c1) load(c + STAGES, s);
        if (++s == STAGES) { s = 0; ph ^= 1; }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    const size_t bytes = size_t(512) << 20;
    uint64_t *a, *b;
    cudaMalloc(&a, bytes);
    cudaMalloc(&b, bytes);
    cudaMemset(a, 1, bytes);
    cudaMemset(b, 2, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](const char* name, double traffic, auto&& f) {
        for (int i = 0; i < 3; ++i) f();
        cudaDeviceSynchronize();
        const int reps = 10;
        cudaEventRecord(e0);
        for (int i = 0; i < reps; ++i) f();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double us = ms * 1e3 / reps;
        printf("%-28s %8.1f us  %7.1f GB/s  %s\n", name, us, traffic / (us * 1e-6) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    };
    const size_t n16 = bytes / 16;
    timeit("copy 148x8x256", 2.0 * bytes, [&] { k_copy<<<sms * 8, 256>>>((uint4*)a, (uint4*)b, n16); });
    timeit("copy 148x4x1024", 2.0 * bytes, [&] { k_copy<<<sms * 4, 1024>>>((uint4*)a, (uint4*)b, n16); });
    timeit("rmw 148x8x256", 2.0 * bytes, [&] { k_rmw<<<sms * 8, 256>>>((uint4*)a, n16); });
    timeit("rmw4 148x8x256", 2.0 * bytes, [&] { k_rmw4<<<sms * 8, 256>>>((uint4*)a, n16); });
    timeit("rmw4 148x4x512", 2.0 * bytes, [&] { k_rmw4<<<sms * 4, 512>>>((uint4*)a, n16); });
#define RED(CH, D)                                                                                   \
    cudaFuncSetAttribute(k_red<CH, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * CH);          \
    timeit("red_bulk " #CH " depth " #D, 2.0 * bytes, [&] { k_red<CH, D><<<sms, 32, 8 * CH>>>(a, bytes); });
    RED(1024, 0) RED(1024, 2) RED(1024, 4) RED(2048, 0) RED(2048, 2) RED(2048, 4) RED(4096, 2) RED(8192, 1)
#define RT(CH, S)                                                                                     \
    cudaFuncSetAttribute(k_bulk_rt<CH, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * CH + 256); \
    timeit("bulk_rt " #CH " x" #S, 2.0 * bytes, [&] { k_bulk_rt<CH, S><<<sms, 32, S * CH + 256>>>(a, bytes); });
    RT(8192, 8) RT(16384, 8) RT(16384, 12)
    // grid = 2 CTAs per SM for the reductions
    cudaFuncSetAttribute(k_red<2048, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 2048);
    timeit("red_bulk 2048 d2 x2 CTAs", 2.0 * bytes, [&] { k_red<2048, 2><<<2 * sms, 32, 8 * 2048>>>(a, bytes); });
    return 0;
}
