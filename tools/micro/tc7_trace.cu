// Event trace of k_gemm_tc7 cluster 0 (F2GPU_TC7_MODE=8): per stage, when the
// leader finished waiting for `full`, finished issuing, and when the expansion
// warps (warp 0 / 8 of each CTA) saw `empty` and arrived on `full`.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_1209_5198_b200/csrc/kernels.cuh"
namespace f2 { int tc7_trace_read(unsigned long long* out, int cap); }
int main() {
    if (!getenv("F2GPU_TC7_MODE")) setenv("F2GPU_TC7_MODE", "8", 1);
    const size_t n = 16384, k = 16384, m = 16384;
    uint64_t *A, *BT, *C;
    cudaMalloc(&A, (k / 64) * n * 8); cudaMalloc(&BT, (k / 64) * m * 8); cudaMalloc(&C, (m / 64) * n * 8);
    f2::TcGemmArgs p{A, n, n, BT, m, C, n, k, m, 0};
    std::vector<unsigned long long> ev(8192);
    int cnt = 0;
    for (int rep = 0; rep < 2; ++rep) {
        f2::tc7_trace_read(ev.data(), 8192);
        f2::launch_gemm_tc7(p, 0);
        cudaDeviceSynchronize();
        cnt = f2::tc7_trace_read(ev.data(), 8192); (void)cnt;
    }
    std::map<int, std::map<int, long long>> tm;
    for (int code = 0; code < 16; ++code)
        for (int sq = 0; sq < 512; ++sq)
            if (ev[code * 512 + sq]) tm[code][sq] = (long long)ev[code * 512 + sq];
    const char* names[] = {"L.wait", "L.full", "L.issued", "r0w0", "r0w1", "r0w2", "r0w3", "r0w4", "r0w5", "r0w6",
                           "r0w7", "r0w8", "r0w12", "r1w0", "r1w8", "r1w15"};
    long long base = tm[0].count(0) ? tm[0][0] : 0;
    printf("stage:");
    for (int c = 0; c < 16; ++c) printf(" %8s", names[c]);
    printf("   (ns)\n");
    for (int sidx = 100; sidx < 120; ++sidx) {
        printf("%5d:", sidx);
        for (int c = 0; c < 16; ++c) {
            auto it = tm[c].find(sidx);
            if (it == tm[c].end()) printf(" %8s", "-");
            else printf(" %8lld", it->second - base);
        }
        printf("\n");
    }
    return 0;
}
