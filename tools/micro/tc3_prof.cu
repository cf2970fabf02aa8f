// Phases of one k_gemm_tc3 CTA (tile (0,0)) for a given k, with clock64 stamps
// (build: nvcc -DTC3_PROFILE ... this file includes tc_leaf.cu).
#include <cstdio>
#include <cstdlib>
#define TC3_PROFILE 1
#include "../../paper_1209_5198_b200/csrc/tc_leaf.cu"

int main(int argc, char** argv) {
    const size_t n = 2400, m = 37888;
    for (size_t k : {64, 256, 1024, 4096, 16384}) {
        const size_t KB = (k + 63) / 64;
        uint64_t *A, *BT, *C;
        cudaMalloc(&A, KB * n * 8); cudaMalloc(&BT, KB * m * 8); cudaMalloc(&C, (m / 64) * n * 8);
        cudaMemset(A, 0x35, KB * n * 8); cudaMemset(BT, 0x53, KB * m * 8);
        for (int rep = 0; rep < 3; ++rep) {
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            cudaError_t e = f2::launch_gemm_tc3(A, n, n, BT, m, C, n, k, m, false, 0);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            long long pr[8];
            cudaMemcpyFromSymbol(pr, f2::g_tc3_prof, sizeof pr);
            if (rep == 2)
                printf("k=%5zu total %.1f us | setup %lld  first-stage %lld  mma-issue %lld  mma-drain %lld  epilogue %lld  teardown %lld cycles  %s %s\n",
                       k, ms * 1000, pr[1] - pr[0], pr[2] - pr[1], pr[3] - pr[2], pr[4] - pr[3], pr[5] - pr[4], pr[6] - pr[5],
                       cudaGetErrorString(e), cudaGetErrorString(cudaGetLastError()));
        }
        cudaFree(A); cudaFree(BT); cudaFree(C);
    }
    return 0;
}
