// tc_update.cu -- the trailing update of a blocked decomposition on the tensor
// cores:  C[lo..hi) x [q0, q0+ncols) ^= A * B, rank <= 128.
//
// EVALUATED, NOT ON THE DECOMPOSITION PATH.  It is bit-exact (tests/
// test_gpu_parity.py::test_update_tc) but it cannot beat the M4RM update
// (k_update_v3) for rank <= 128 on B200: every output bit costs one f32 TMEM
// accumulator word, TMEM reads run at 64 B/cycle/SM (B300_MICROARCH.md, TMEM
// table), so a 128 x 192 tile needs ~1500 cycles of tcgen05.ld alone --
// 16 output bits/cycle/SM against M4RM's ~59 per panel.  The measured per-tile
// period (clock64 timeline of CTA 0, profiles/r1_update_tc_summary.txt) is
// ~1300 cycles; rank-128 C(65536^2) takes 0.68-1.1 ms vs 0.50 ms for two M4RM
// rank-64 passes.  The tensor-core leaf wins only for large K (tc_leaf.cu).
//
// A (hi-lo rows x KB words) are the multiplier columns of the block's panels
// (Y of panel j, j+1: word (i, kb) at a[kb*sa + i]); B^T (ncols*64 rows x KB
// words: word (c, kb) at bt[kb*sbt + c]) are the block's final pivot rows,
// transposed.  This is the GEMM step A22 ^= L21 * U12 of a right-looking
// blocked LU (block width 64*KB) -- the per-panel Schur updates of PAPER.md
// Algorithm 2 applied two panels at a time, which halves the
// HBM traffic of the trailing matrix (deferred updates commute with the later
// row swaps, SURVEY Probe P5, so the result is bit-identical).
//
// Mapping: MMA M = 128 C rows (TMEM lanes), N = 192 C columns (3 word-columns,
// TMEM columns), K = 64 bits per fp4 MMA (kind::mxf4, bits as E2M1 1.0/0.0,
// E8M0 scales all 1.0).  The accumulators start at 2^23 (f32), so after the
// MMAs bit 0 of each accumulator word IS the running parity.  The buffers are
// never reset: every MMA accumulates, each tile adds at most 128, so a buffer
// stays in [2^23, 2^24) for 2^16 tiles (a launch uses < 2^12 per buffer) and
// the tile's GF(2) result is the packed parity XOR the packed parity the same
// thread read from the same buffer two tiles earlier (kept in a register).  No
// reset traffic, no extra MMA.  A funnel-shift chain packs 32 of them into a C
// half-word with one instruction per bit.  Every epilogue thread owns one C
// word (row, word-column) per tile and a warp covers 32 consecutive rows, so it
// read-modify-writes C directly with 256-byte coalesced accesses; the C word of
// its next tile is loaded one tile ahead, which hides the HBM latency without
// any staging, barrier or proxy fence between the epilogue warps.
//
// Persistent CTAs (one per SM), warp-specialised:
//   warps 0-11  epilogue: warp w reads TMEM lane quarter w & 3 (32 tile rows) of
//               word-column w >> 2; double-buffered accumulators
//   warps 12-15 expansion of the raw words into the fp4 K-major tiles
//   warp  16    MMA issue (one elected thread)
//   warp  17    bulk loads of the raw A / B^T words
// Work unit = (column tile c of 3 word-columns, row segment s); the B^T tile is
// expanded once per unit and the unit walks its 128-row tiles.  Units with
// c == 0 (the next block's panel columns) come first; every epilogue warp
// increments *release once its share of such a unit is in memory (lookahead:
// update_tc_release_count() increments in total).
#include <cstdint>
#include <cstdlib>
#include "../options.h"

#include "../kernels.cuh"
#include "../tc_common.cuh"

#if F2GPU_EXPERIMENTAL  // evaluated, not used: built only with F2GPU_EXPERIMENTAL=1
namespace f2 {

namespace {

constexpr int kUtRows = 128;                  // C rows per tile (M)
constexpr int kUtCols = 192;                  // C columns per tile (N)
constexpr int kUtWc = kUtCols / 64;           // word-columns per tile
constexpr int kUtKB = 2;                      // max k-words (rank 128)
constexpr int kUtATile = kUtRows * 64;        // expanded A tile: 64-byte rows (2 k-words of fp4)
constexpr int kUtBTile = kUtCols * 64;        // expanded B^T tile
constexpr int kUtAStages = 6;                 // expanded A tiles
constexpr int kUtARaw = 8;                    // raw A words (L2 latency + two mbarrier hops)
constexpr int kUtPf = 4;                      // C prefetch distance (tiles) in the epilogue
constexpr int kUtARawBytes = kUtRows * 8 * kUtKB;
constexpr int kUtBRawBytes = kUtCols * 8 * kUtKB;
constexpr int kUtStg = kUtRows * 8 * kUtWc;   // staging: 3 word-columns x 128 rows
constexpr uint32_t kUtAcc = kUtCols;          // TMEM columns per accumulator buffer
constexpr uint32_t kUtSf = 2 * kUtAcc;        // 32 columns of E8M0 1.0 scale factors
constexpr int kUtEpi = 4 * kUtWc;             // epilogue warps
constexpr int kUtExp0 = kUtEpi;               // first expansion warp
constexpr int kUtMmaW = kUtExp0 + 4;
constexpr int kUtLoadW = kUtMmaW + 1;
constexpr int kUtThreads = 32 * (kUtLoadW + 1);
constexpr uint32_t kUtIdesc = idesc_f4(kUtRows, kUtCols);

struct UtSmem {
    unsigned char btile[2][kUtBTile];         // 1024-aligned (offsets multiples of 1024)
    unsigned char atile[kUtAStages][kUtATile];
    uint64_t araw[kUtARaw][kUtRows * kUtKB];
    uint64_t braw[2][kUtCols * kUtKB];
    uint64_t a_rfull[kUtARaw], a_rempty[kUtARaw], a_full[kUtAStages], a_empty[kUtAStages];
    uint64_t b_rfull[2], b_rempty[2], b_full[2], b_empty[2];
    uint64_t t_full[2], t_empty[2];
    uint32_t tmem;
};

// unit u -> (column tile, row-tile range); identical in every role
struct UtPlan {
    size_t t0, T;      // first 128-row tile, number of row tiles (from lo, hi)
    int ct, S;         // column tiles, row segments per column tile
    __device__ void unit(int u, int& c, size_t& r0, size_t& r1) const {
        c = u / S;
        const int s = u % S;
        r0 = t0 + T * size_t(s) / size_t(S);
        r1 = t0 + T * size_t(s + 1) / size_t(S);
    }
};

// this CTA's tiles in order: units u = first, first + G, ... (empty ones skipped)
struct TileIter {
    const UtPlan* pl;
    int u, G, units;
    int c = 0;
    size_t t = 0, r1 = 0;
    bool valid = false;
    __device__ void seek() {
        for (; u < units; u += G) {
            size_t r0;
            pl->unit(u, c, r0, r1);
            if (r0 < r1) {
                t = r0;
                valid = true;
                return;
            }
        }
        valid = false;
    }
    __device__ void next() {
        if (++t < r1) return;
        u += G;
        seek();
    }
};

__device__ __forceinline__ uint64_t ld_cg(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
        "%28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
          "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
          "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32_const(uint32_t taddr, uint32_t x) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, "
        "%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(taddr),
        "r"(x)
        : "memory");
}
// bit q of the result = bit 0 of v[q]
__device__ __forceinline__ uint32_t pack_lsb32(const uint32_t (&v)[32]) {
    uint32_t w = 0;
#pragma unroll
    for (int q = 0; q < 32; ++q) w = __funnelshift_r(w, v[q], 1);
    return w;
}


// MODE (diagnostic, F2GPU_UT_MODE, timing only): bit 1 skips the C
// stores, bit 2 skips the MMAs (results wrong in every mode but 0)
template <int MODE>
__global__ void __launch_bounds__(kUtThreads, 1)
    k_update_tc(TcUpdateArgs p, int S) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    UtSmem& sm = *reinterpret_cast<UtSmem*>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int KB = p.kwords;

    size_t lo = p.row_lo;
    if (p.st) lo = size_t(p.st->R) + p.st->r;
    const size_t hi = p.row_hi;
    UtPlan plan;
    plan.t0 = lo / kUtRows;
    plan.T = hi > lo ? (hi + kUtRows - 1) / kUtRows - plan.t0 : 0;
    plan.ct = (p.ncols + kUtWc - 1) / kUtWc;
    plan.S = S;
    const int units = plan.ct * plan.S;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sm_u32(&sm.tmem)),
                     "r"(512u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int s = 0; s < kUtARaw; ++s) {
            mbar_init_n(&sm.a_rfull[s], 1);
            mbar_init_n(&sm.a_rempty[s], 4);
        }
        for (int s = 0; s < kUtAStages; ++s) {
            mbar_init_n(&sm.a_full[s], 4);
            mbar_init_n(&sm.a_empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init_n(&sm.b_rfull[s], 1);
            mbar_init_n(&sm.b_rempty[s], 4);
            mbar_init_n(&sm.b_full[s], 4);
            mbar_init_n(&sm.b_empty[s], 1);
            mbar_init_n(&sm.t_full[s], 1);
            mbar_init_n(&sm.t_empty[s], kUtEpi);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = sm.tmem;
    if (warp < 4) {  // accumulators <- 2^23 (once), scale factors <- E8M0 1.0
        const uint32_t lq = uint32_t(32 * warp) << 16;
        for (uint32_t c = 0; c < 2 * kUtAcc; c += 32) tmem_st32_const(tmem + lq + c, 0x4B000000u);
        tmem_st32_const(tmem + lq + kUtSf, 0x7F7F7F7Fu);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");

    if (warp == kUtLoadW) {
        // ===== bulk loads =====
        if (lane == 0) {
            size_t g = 0;
            int lu = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                int c;
                size_t r0, r1;
                plan.unit(u, c, r0, r1);
                if (r0 == r1) continue;
                const int ub = lu & 1;
                if (lu >= 2) mbar_wait1(&sm.b_rempty[ub], ((lu >> 1) - 1) & 1);
                ++lu;  // buffers and phases count processed units only
                mbar_expect(&sm.b_rfull[ub], uint32_t(KB * kUtCols * 8));
                for (int kb = 0; kb < KB; ++kb)
                    bulk_g2s(&sm.braw[ub][kb * kUtCols], p.bt + size_t(kb) * p.sbt + size_t(c) * kUtCols,
                             kUtCols * 8, &sm.b_rfull[ub]);
                for (size_t t = r0; t < r1; ++t, ++g) {
                    const int s = int(g % kUtARaw);
                    if (g >= size_t(kUtARaw)) mbar_wait1(&sm.a_rempty[s], ((g / kUtARaw) - 1) & 1);
                    mbar_expect(&sm.a_rfull[s], uint32_t(KB * kUtRows * 8));
                    for (int kb = 0; kb < KB; ++kb)
                        bulk_g2s(&sm.araw[s][kb * kUtRows], p.a + size_t(kb) * p.sa + t * kUtRows,
                                 kUtRows * 8, &sm.a_rfull[s]);
                }
            }
        }
        __syncwarp();
    } else if (warp >= kUtExp0 && warp < kUtMmaW) {
        // ===== expansion: 128 threads =====
        const int et = tid - 32 * kUtExp0;
        size_t g = 0;
        int lu = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x) {
            int c;
            size_t r0, r1;
            plan.unit(u, c, r0, r1);
            if (r0 == r1) continue;
            const int ub = lu & 1;
            mbar_wait1(&sm.b_rfull[ub], (lu >> 1) & 1);
            if (lu >= 2) mbar_wait1(&sm.b_empty[ub], ((lu >> 1) - 1) & 1);
            ++lu;
            const size_t cbase = size_t(c) * kUtCols;
            const size_t cmax = size_t(p.ncols) * 64;
            for (int r = et; r < kUtCols; r += 128) {
                const bool ok = cbase + r < cmax;
                for (int kb = 0; kb < KB; ++kb)
                    store_row_f4(sm.btile[ub], r, kb, ok ? sm.braw[ub][kb * kUtCols + r] : 0ull);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive1(&sm.b_rempty[ub]);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive1(&sm.b_full[ub]);
            for (size_t t = r0; t < r1; ++t, ++g) {
                const int rs = int(g % kUtARaw);
                const int s = int(g % kUtAStages);
                const uint32_t ph = uint32_t(g / kUtAStages) & 1;
                mbar_wait1(&sm.a_rfull[rs], uint32_t(g / kUtARaw) & 1);
                if (g >= size_t(kUtAStages)) mbar_wait1(&sm.a_empty[s], ph ^ 1);
                const size_t row = t * kUtRows + et;
                const bool ok = row >= lo && row < hi;
                if (!(MODE & 16))
                    for (int kb = 0; kb < KB; ++kb)
                        store_row_f4(sm.atile[s], et, kb, ok ? sm.araw[rs][kb * kUtRows + et] : 0ull);
                __syncwarp();
                if (lane == 0) mbar_arrive1(&sm.a_rempty[rs]);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive1(&sm.a_full[s]);
            }
        }
    } else if (warp == kUtMmaW) {
        // ===== MMA issue =====
        if (lane == 0) {
            const uint32_t tsf = tmem + kUtSf;
            size_t g = 0;
            int lu = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                int c;
                size_t r0, r1;
                plan.unit(u, c, r0, r1);
                if (r0 == r1) continue;
                const int ub = lu & 1;
                mbar_wait1(&sm.b_full[ub], (lu >> 1) & 1);
                ++lu;
                const uint32_t bt = sm_u32(sm.btile[ub]);
                for (size_t t = r0; t < r1; ++t, ++g) {
                    const int s = int(g % kUtAStages);
                    const int tb = int(g & 1);
                    mbar_wait1(&sm.a_full[s], uint32_t(g / kUtAStages) & 1);
                    if (g >= 2) mbar_wait1(&sm.t_empty[tb], uint32_t((g >> 1) - 1) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t at = sm_u32(sm.atile[s]);
                    const uint32_t td = tmem + uint32_t(tb) * kUtAcc;
                    if (!(MODE & 4))
                        for (int kb = 0; kb < KB; ++kb)
                            mma_f4(td, umma_desc(at + kKHalf * kb), umma_desc(bt + kKHalf * kb), kUtIdesc, 1u,
                                   tsf);
                    tc_commit(&sm.a_empty[s]);
                    tc_commit(&sm.t_full[tb]);
                }
                tc_commit(&sm.b_empty[ub]);
            }
        }
        __syncwarp();
    } else {
        // ===== epilogue: warp w -> rows 32(w&3).. of the tile, word-column j = w >> 2 =====
        const uint32_t lq = uint32_t(32 * (warp & 3)) << 16;
        const int row = 32 * (warp & 3) + lane;
        const int j = warp >> 2;
        if (p.release) {  // empty row segments of column tile 0 owe their signal now
            for (int u = blockIdx.x; u < plan.S; u += gridDim.x) {
                int c;
                size_t r0, r1;
                plan.unit(u, c, r0, r1);
                if (r0 == r1 && lane == 0) atomicAdd(p.release, 1u);
            }
        }
        TileIter it{&plan, int(blockIdx.x), int(gridDim.x), units};
        it.seek();
        auto cptr = [&](const TileIter& x) -> uint64_t* {
            return x.valid && x.c * kUtWc + j < p.ncols
                       ? p.C + (p.q0 + size_t(x.c) * kUtWc + j) * p.sc + x.t * kUtRows + row
                       : nullptr;
        };
        // C words of the next kUtPf tiles are in flight.  Slot i of cp/cv always
        // holds tile g with g % kUtPf == i (the loop is unrolled by kUtPf), so no
        // register ever moves while its load is outstanding.
        TileIter pf = it;
        uint64_t* cp[kUtPf];
        uint64_t cv[kUtPf];
#pragma unroll
        for (int i = 0; i < kUtPf; ++i) {
            cp[i] = cptr(pf);
            cv[i] = cp[i] ? ld_cg(cp[i]) : 0;
            if (pf.valid) pf.next();
        }
        uint64_t prev0 = 0, prev1 = 0;  // packed parity last read from accumulator buffer 0 / 1
        size_t g = 0;
        while (it.valid) {
#pragma unroll
            for (int i = 0; i < kUtPf; ++i, ++g) {
                if (!it.valid) break;
                const int tb = i & 1;  // == g & 1 (kUtPf is even)
                mbar_wait1(&sm.t_full[tb], uint32_t(g >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t ta = tmem + lq + uint32_t(tb) * kUtAcc + uint32_t(64 * j);
                uint64_t word = 0;
                if (MODE & 8) {
                    asm volatile("tcgen05.fence::before_thread_sync;");
                    __syncwarp();
                    if (lane == 0) mbar_arrive1(&sm.t_empty[tb]);
                } else {
                    uint32_t v0[32], v1[32];
                    tmem_ld32(ta, v0);
                    tmem_ld32(ta + 32, v1);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    // the values are in registers: release the buffer before packing
                    asm volatile("tcgen05.fence::before_thread_sync;");
                    __syncwarp();
                    if (lane == 0) mbar_arrive1(&sm.t_empty[tb]);
                    word = uint64_t(pack_lsb32(v0)) | (uint64_t(pack_lsb32(v1)) << 32);
                }
                const uint64_t delta = word ^ (tb ? prev1 : prev0);
                if (tb) prev1 = word; else prev0 = word;
                if (cp[i] && !(MODE & 2)) *cp[i] = cv[i] ^ delta;
                if (p.release && it.c == 0 && it.t + 1 == it.r1) {
                    // last tile of a column-tile-0 unit: publish this warp's share
                    __threadfence();
                    __syncwarp();
                    if (lane == 0) atomicAdd(p.release, 1u);
                }
                cp[i] = cptr(pf);  // refill the slot kUtPf tiles ahead
                cv[i] = cp[i] ? ld_cg(cp[i]) : 0;
                if (pf.valid) pf.next();
                it.next();
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
}

}  // namespace

bool update_tc_ok(const TcUpdateArgs& a) {
    return a.kwords >= 1 && a.kwords <= kUtKB && a.ncols >= 1 && (a.sc % kUtRows) == 0 &&
           (a.sa % 2) == 0 && (a.sbt % 2) == 0 && a.row_hi <= a.sc &&
           (reinterpret_cast<uintptr_t>(a.C) % 16) == 0 && (reinterpret_cast<uintptr_t>(a.a) % 16) == 0 &&
           (reinterpret_cast<uintptr_t>(a.bt) % 16) == 0;
}

int update_tc_release_count(const TcUpdateArgs& a, int grid) { return update_tc_segments(a, grid) * kUtEpi; }

int update_tc_segments(const TcUpdateArgs& a, int grid) {
    const size_t tmax = (a.row_hi + kUtRows - 1) / kUtRows;
    const int ct = (a.ncols + kUtWc - 1) / kUtWc;
    const size_t want = (size_t(4) * size_t(grid) + size_t(ct) - 1) / size_t(ct);
    return int(std::max<size_t>(1, std::min<size_t>(tmax, want)));
}

cudaError_t launch_update_tc(const TcUpdateArgs& a, int grid, cudaStream_t s) {
    static bool attr = false;
    static int mode = 0;
    using Fn = void (*)(TcUpdateArgs, int);
    static const Fn fns[32] = {
        k_update_tc<0>,  k_update_tc<1>,  k_update_tc<2>,  k_update_tc<3>,  k_update_tc<4>,  k_update_tc<5>,
        k_update_tc<6>,  k_update_tc<7>,  k_update_tc<8>,  k_update_tc<9>,  k_update_tc<10>, k_update_tc<11>,
        k_update_tc<12>, k_update_tc<13>, k_update_tc<14>, k_update_tc<15>, k_update_tc<16>, k_update_tc<17>,
        k_update_tc<18>, k_update_tc<19>, k_update_tc<20>, k_update_tc<21>, k_update_tc<22>, k_update_tc<23>,
        k_update_tc<24>, k_update_tc<25>, k_update_tc<26>, k_update_tc<27>, k_update_tc<28>, k_update_tc<29>,
        k_update_tc<30>, k_update_tc<31>};
    if (!attr) {
        for (Fn f : fns) {
            cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(UtSmem)));
            if (e != cudaSuccess) return e;
        }
        mode = int(options().ut_mode) & 31;
        attr = true;
    }
    if (!update_tc_ok(a)) return cudaErrorInvalidValue;
    fns[mode]<<<grid, kUtThreads, sizeof(UtSmem), s>>>(a, update_tc_segments(a, grid));
    return cudaGetLastError();
}

size_t update_tc_bt_rows(int ncols) {
    return (size_t(ncols) * 64 + kUtCols - 1) / kUtCols * kUtCols;
}

}  // namespace f2

#endif  // F2GPU_EXPERIMENTAL
