// Dependent-chain latency (cycles per op) of warp primitives on one warp.
#include <cstdio>
#include <cstdint>
__global__ void k(long long* out, uint32_t seed) {
    const int lane = threadIdx.x;
    uint32_t x = seed + lane;
    uint64_t y = seed * 0x9E3779B97F4A7C15ull + lane;
    const int N = 1024;
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (x + i) & 31);
    long long t1 = clock64();
    for (int i = 0; i < N; ++i) x = __ballot_sync(0xffffffffu, (x >> (i & 31)) & 1) + i;
    long long t2 = clock64();
    for (int i = 0; i < N; ++i) x = __reduce_xor_sync(0xffffffffu, x) + lane + i;
    long long t3 = clock64();
    for (int i = 0; i < N; ++i) y = __shfl_sync(0xffffffffu, y, int(y + i) & 31);
    long long t4 = clock64();
    for (int i = 0; i < N; ++i) x = __popc(x) + x * 3 + i;
    long long t5 = clock64();
    for (int i = 0; i < N; ++i) y = (y >> 1) ^ (y << 3) ^ i;
    long long t6 = clock64();
    if (lane == 0) {
        out[0] = (t1 - t0) / N; out[1] = (t2 - t1) / N; out[2] = (t3 - t2) / N;
        out[3] = (t4 - t3) / N; out[4] = (t5 - t4) / N; out[5] = (t6 - t5) / N;
        out[6] = x + y;
    }
}
int main() {
    long long* d; cudaMalloc(&d, 64);
    k<<<1, 32>>>(d, 7); cudaDeviceSynchronize();
    long long h[8]; cudaMemcpy(h, d, 56, cudaMemcpyDeviceToHost);
    printf("shfl32 %lld  vote %lld  redux_xor %lld  shfl64 %lld  popc+imad %lld  u64 shift/xor %lld (cycles/iter)\n",
           h[0], h[1], h[2], h[3], h[4], h[5]);
    return 0;
}
