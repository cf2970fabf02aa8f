// Cycle accounting of k_gemm_tc7 (F2GPU_TC7_MODE=7): where cluster 0's agents wait.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tc7_prof.bin tc7_prof.cu ../../paper_1209_5198_b200/csrc/tc_pair.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../../paper_1209_5198_b200/csrc/kernels.cuh"
namespace f2 { void tc7_prof_read(unsigned long long* out16, bool reset); }
int main() {
    if (!getenv("F2GPU_TC7_MODE")) setenv("F2GPU_TC7_MODE", "7", 1);
    const size_t n = 16384, k = 16384, m = 16384;
    uint64_t *A, *BT, *C;
    cudaMalloc(&A, (k / 64) * n * 8); cudaMalloc(&BT, (k / 64) * m * 8); cudaMalloc(&C, (m / 64) * n * 8);
    cudaMemset(A, 0x35, (k / 64) * n * 8); cudaMemset(BT, 0x53, (k / 64) * m * 8);
    f2::TcGemmArgs p{A, n, n, BT, m, C, n, k, m, 0};
    for (int rep = 0; rep < 3; ++rep) {
        unsigned long long pr[16];
        f2::tc7_prof_read(pr, true);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        cudaError_t e = f2::launch_gemm_tc7(p, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        f2::tc7_prof_read(pr, false);
        const double st = double(pr[15]);
        printf("%s %.3f ms, %llu stages (cluster 0): per stage cycles\n", cudaGetErrorString(e), ms, pr[15]);
        printf("  leader MMA per stage: wait full %.0f  issue %.0f  commit %.0f  | per tile wait acc_empty %.0f\n",
               pr[0] / st, pr[1] / st, pr[2] / st, pr[3] / st);
        const double es = double(pr[14]);
        printf("  M-side warp0 per stage: rfull %.0f  empty %.0f  load+expand %.0f  wait::st+arrive %.0f\n", pr[4] / es, pr[5] / es, pr[6] / es, pr[7] / es);
        printf("  N-side warp8 per stage: rfull %.0f  empty %.0f  load+expand %.0f  fence+arrive %.0f\n", pr[9] / es, pr[10] / es, pr[11] / es, pr[12] / es);
    }
    return 0;
}
