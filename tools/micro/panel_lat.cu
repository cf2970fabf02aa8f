// Warm duration of the panel kernel (k_panel, buildZ on one 64-column panel) on
// an n-row random column, launched back to back; links against libf2gpu.so.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_1209_5198_b200/csrc/kernels.cuh"

int main(int argc, char** argv) {
    const size_t n = argc > 1 ? size_t(atol(argv[1])) : 65536;
    const int reps = 200;
    std::vector<uint64_t> h(n);
    uint64_t x = 0x9E3779B97F4A7C15ull;
    for (auto& v : h) { x ^= x >> 12; x ^= x << 25; x ^= x >> 27; v = x * 0x2545F4914F6CDD1Dull; }
    uint64_t* col; f2::PanelState* st;
    cudaMalloc(&col, n * 8); cudaMalloc(&st, 2 * sizeof(f2::PanelState));
    cudaMemcpy(col, h.data(), n * 8, cudaMemcpyHostToDevice);
    f2::init_kernel_attrs();
    cudaStream_t s; cudaStreamCreate(&s);
    for (int i = 0; i < 10; ++i) f2::launch_panel(col, n, st, 0, s, nullptr, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int i = 0; i < reps; ++i) f2::launch_panel(col, n, st, 0, s, nullptr, 0);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("n=%zu k_panel %.2f us per launch (back to back) err=%s\n", n, ms * 1000 / reps,
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}
