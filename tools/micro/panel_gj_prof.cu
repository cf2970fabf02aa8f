// clock64 phases of k_panel_gj (build with -DGJ_PROFILE together with kernels.cu):
// window load, selection chain (warp 0), bookkeeping replay (warp 1), tail.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_1209_5198_b200/csrc/kernels.cuh"

int main(int argc, char** argv) {
    const size_t n = argc > 1 ? size_t(atol(argv[1])) : 65536;
    std::vector<uint64_t> h(n);
    uint64_t x = 0x9E3779B97F4A7C15ull;
    for (auto& v : h) { x ^= x >> 12; x ^= x << 25; x ^= x >> 27; v = x * 0x2545F4914F6CDD1Dull; }
    uint64_t* col; f2::PanelState* st;
    cudaMalloc(&col, n * 8); cudaMalloc(&st, 2 * sizeof(f2::PanelState));
    f2::init_kernel_attrs();
    cudaStream_t s; cudaStreamCreate(&s);
    for (int i = 0; i < 5; ++i) {
        cudaMemcpy(col, h.data(), n * 8, cudaMemcpyHostToDevice);
        f2::launch_panel(col, n, st, 0, s, nullptr, 0);
        cudaStreamSynchronize(s);
        f2::PanelState hs;
        cudaMemcpy(&hs, st, sizeof hs, cudaMemcpyDeviceToHost);
        const long long* pr = reinterpret_cast<const long long*>(hs.src);
        printf("n=%zu r=%u slow=%lld load %lld chain %lld w1end %lld w2end %lld tail %lld cycles  err=%s\n", n, hs.r, pr[58], pr[61], pr[62], pr[57], pr[56],
               pr[63], cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
