// Probe: kind::mxf4 MMA with the A operand in TMEM.
//  (1) k-order: which TMEM nibble of an A row meets which k of the B operand
//      (B staged by store_row_f4, the leaf's SWIZZLE_64B K-major layout);
//  (2) how many scale-factor columns the MMA reads (M = 128, scale_vec::2X):
//      columns [sf, sf + x) hold 0x7F (1.0), the rest of the SF window 0x00.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o tmem_a_probe.bin tmem_a_probe.cu
#include <cstdio>
#include <cstdint>
#include "../../paper_1209_5198_b200/csrc/tc_common.cuh"

using namespace f2;

constexpr int N = 64;             // B rows (one per k)
constexpr uint32_t kD = 0, kA = 128, kSF = 256;

__global__ void probe(uint32_t* out, int sf_cols, int a_mode) {
    __shared__ __align__(1024) unsigned char bt[N * 64];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sm_u32(&slot)), "r"(512u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) { mbar_init_n(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    // B row r = bit r only (k = r in the leaf's logical order)
    if (tid < N) store_row_f4(bt, tid, 0, uint64_t(1) << tid);
    if (tid < N) store_row_f4(bt, tid, 1, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = slot;
    // A row i (TMEM lane i): a_mode 0 -> single 1.0 nibble at position p = i % 64
    // (column p / 8, nibble p % 8); a_mode 1 -> all 64 nibbles 1.0
    {
        const int i = 32 * warp + lane;
        uint32_t v[8];
        for (int c = 0; c < 8; ++c) v[c] = 0;
        if (a_mode == 0) {
            const int p = i % 64;
            v[p / 8] = 0x2u << (4 * (p % 8));
        } else {
            for (int c = 0; c < 8; ++c) v[c] = 0x22222222u;
        }
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(
                         tmem + (uint32_t(32 * warp) << 16) + kA),
                     "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                     : "memory");
        uint32_t s[32];
        for (int c = 0; c < 32; ++c) s[c] = c < sf_cols ? 0x7F7F7F7Fu : 0u;
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
            "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(
                tmem + (uint32_t(32 * warp) << 16) + kSF),
            "r"(s[0]), "r"(s[1]), "r"(s[2]), "r"(s[3]), "r"(s[4]), "r"(s[5]), "r"(s[6]), "r"(s[7]), "r"(s[8]),
            "r"(s[9]), "r"(s[10]), "r"(s[11]), "r"(s[12]), "r"(s[13]), "r"(s[14]), "r"(s[15]), "r"(s[16]),
            "r"(s[17]), "r"(s[18]), "r"(s[19]), "r"(s[20]), "r"(s[21]), "r"(s[22]), "r"(s[23]), "r"(s[24]),
            "r"(s[25]), "r"(s[26]), "r"(s[27]), "r"(s[28]), "r"(s[29]), "r"(s[30]), "r"(s[31])
            : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (tid == 0) {
        const uint32_t idesc = idesc_f4(128, N);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], [%1], %2, %3, [%5], [%5], p;\n\t}\n" ::"r"(
                tmem + kD),
            "r"(tmem + kA), "l"(umma_desc(sm_u32(bt))), "r"(idesc), "r"(0u), "r"(tmem + kSF));
        tc_commit(&bar);
    }
    mbar_wait1(&bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    // D: lane i, column r -> out[i * N + r]
    for (int c0 = 0; c0 < N; c0 += 16) {
        uint32_t v[16];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
            "%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(tmem + (uint32_t(32 * warp) << 16) + kD + c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int q = 0; q < 16; ++q) out[(32 * warp + lane) * N + c0 + q] = v[q];
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
}

int main() {
    uint32_t* d;
    cudaMalloc(&d, 128 * N * 4);
    static uint32_t h[128 * N];
    // (1) k-order with all SF columns set
    probe<<<1, 128>>>(d, 32, 0);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("probe(k-order): %s\n", cudaGetErrorString(e));
    int perm[64];
    bool ok = true;
    for (int p = 0; p < 64; ++p) {
        int hit = -1, cnt = 0;
        for (int r = 0; r < N; ++r) {
            const float f = *reinterpret_cast<float*>(&h[p * N + r]);
            if (f != 0.f) { ++cnt; hit = r; if (f != 1.f) printf("  p=%d r=%d value %g\n", p, r, f); }
        }
        perm[p] = cnt == 1 ? hit : -1;
        ok = ok && cnt == 1;
        // rows p + 64 must agree
        for (int r = 0; r < N; ++r) ok = ok && h[(p + 64) * N + r] == h[p * N + r];
    }
    printf("nibble position p -> k:");
    for (int p = 0; p < 64; ++p) printf(" %d", perm[p]);
    printf("\n%s\n", ok ? "k-order: one hit per position" : "k-order: AMBIGUOUS");
    // (2) SF columns: all-ones A x single-bit B rows -> D = 1.0 everywhere when every read SF is 1.0
    for (int x : {0, 1, 2, 4, 8, 16, 32}) {
        probe<<<1, 128>>>(d, x, 1);
        e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        int good = 0;
        for (int i = 0; i < 128 * N; ++i) good += *reinterpret_cast<float*>(&h[i]) == 1.f;
        printf("sf_cols=%2d: %d of %d entries == 1.0 (%s)\n", x, good, 128 * N, cudaGetErrorString(e));
    }
    return 0;
}
