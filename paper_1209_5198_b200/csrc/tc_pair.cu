// tc_pair.cu — k_gemm_tc7: the fp4 tensor-core GF(2) product leaf on CTA PAIRS,
// persistent, with the M-side operand expanded straight into TMEM.
//
// Product formulation as in tc_leaf.cu: D^T = B^T * A^T, bits as E2M1 1.0 / 0.0,
// unit E8M0 scales, exact f32 sums (|sum| <= k < 2^23), parity = LSB of v + 2^23.
// MMA M (TMEM lanes) = output COLUMNS (rows of B^T), N (TMEM columns) = output
// ROWS (rows of A).
//
// Why this shape (profiles/r1f_tc3_summary.txt): the single-CTA leaf k_gemm_tc3
// moves ~47 KB of shared memory per 64-bit k-block (raw words in, E2M1 tiles of
// both operands out, both tiles read again by two M = 128 MMAs) against ~240
// tensor cycles, i.e. ~196 B/clk on a 128 B/clk pipe: the tensor pipe idles ~45%.
// Here, per CTA and k-block:
//   * a 2-CTA cluster issues ONE M = 256 x N = NN MMA (tcgen05.mma.cta_group::2):
//     each SM computes 128 output columns x NN rows and holds half of the N-side
//     operand (NN/2 A rows); the pair shares it, so no B-side row is read twice;
//   * the M-side operand (128 B^T rows of this CTA) is expanded by four warps
//     directly into TMEM with tcgen05.st (the MMA's A operand may live in TMEM),
//     so it never touches shared memory;
//   * shared memory carries only the raw words (1.9 KB in, 1.9 KB out), the
//     N-side E2M1 tile (3.5 KB) and its MMA read (3.5 KB): ~10.8 KB per 112
//     tensor cycles (~96 B/clk) at NN = 224.
// Raw words arrive by 2-D TMA tensor copies, 8 k-blocks x 128 (or NN/2) rows per
// request: small 1-D bulk copies (two per k-block) measured ~360 cycles per
// k-block for the feed alone -- a per-request cost, not bandwidth.
// The kernel is persistent (one CTA pair per two SMs, tiles strided over the
// clusters) with two TMEM accumulators, so a tile's epilogue (TMEM reads +
// ballots) overlaps the next tile's MMAs: short-k products no longer pay the
// ~10k-cycle per-tile setup + epilogue of k_gemm_tc3.
//
// TMEM (512 columns): accumulators at 0 and NN, scale factors (0x7F = 1.0) at
// 2NN..2NN+7, the M-side operand ring after them (16 columns per stage of two
// k-blocks).  The A-operand k-order inside a 64-bit k-block is the one
// store_row_f4 gives the smem operand: TMEM column c, nibble q holds bit
// 32*(c/4) + 4*q + c%4 (measured, tools/micro/tmem_a_probe.cu).
//
// Warps (per CTA): 0-3 M-side expansion (lane quarter = warp; warp 0 allocates
// TMEM), 4-7 N-side expansion, 8-15 epilogue (two per lane quarter), 16 MMA issue
// (leader CTA) / stage forwarding (peer), 17 TMA loads of raw words.
#include <cuda.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <vector>

#include "kernels.cuh"
#include "options.h"
#include "tc_common.cuh"

namespace f2 {

namespace {

constexpr int kP7M = 256;             // output columns per pair tile (MMA M)
constexpr int kP7MH = kP7M / 2;       // M rows per CTA (its TMEM lanes)
constexpr int kP7Grp = 8;             // k-blocks per TMA request (box height)
constexpr int kP7Threads = 27 * 32;
constexpr int kP7EpiW0 = 16, kP7EpiWarps = 8;
constexpr int kP7Mma = 24, kP7Mma2 = 25, kP7Load = 26;

// NN: output rows per pair tile (MMA N); NACC: TMEM accumulators (2 = the next
// tile's MMAs overlap this tile's epilogue); STG x KPS: the operand ring, STG
// stages of KPS k-blocks; RG: raw TMA groups (kP7Grp k-blocks) in flight.
template <int NN, int NACC, int STG, int KPS, int RG>
struct P7 {
    static constexpr int N = NN, NH = NN / 2, Stages = STG, Kps = KPS;
    static constexpr int Slot = (NH * 64 + 1023) / 1024 * 1024;  // NH rows x 64 B: 2 k-blocks, SWIZZLE_64B
    static constexpr int RawM = kP7Grp * kP7MH * 8;            // M-side box: 8 kb x 128 rows
    static constexpr int RawN = kP7Grp * NH * 8;               // N-side box: 8 kb x NH rows
    static constexpr int RawGroup = (RawM + RawN + 1023) / 1024 * 1024;
    static constexpr int BStage = Slot * (KPS / 2);
    static constexpr uint32_t AccCol = NN, SfCol = NACC * NN, ACol = NACC * NN + 8;
    static constexpr size_t RawOff = size_t(STG) * BStage;
    static constexpr size_t BarOff = RawOff + size_t(RG) * RawGroup;
    static constexpr size_t Smem = BarOff + 1024;
    static constexpr uint32_t Idesc = idesc_f4(kP7M, NN);
    static_assert(ACol + STG * KPS * 8 <= 512, "TMEM budget");
    static_assert(KPS % 2 == 0 && kP7Grp % KPS == 0, "stage / TMA group geometry");
    static_assert(NH % 8 == 0 && NH <= 128, "SWIZZLE_64B atoms");
    static_assert(Smem <= 227 * 1024, "shared memory");
};

// per problem: the TMA descriptors of its raw operands (box 128 rows of B^T,
// box NH rows of A; 8 k-blocks each) and the problem itself
struct alignas(64) Tc7Prob {
    CUtensorMap mbt;  // B^T: dims {m, KB}
    CUtensorMap ma;   // A:   dims {n, KB}
    TcGemmArgs P;
};

__device__ __forceinline__ void mma_f4_pair_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t acc,
                                               uint32_t idesc, uint32_t tsf) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %3, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.scale_vec::2X [%0], [%1], %2, %4, [%5], [%5], p;\n\t}\n" ::"r"(
            tmem_d),
        "r"(tmem_a), "l"(db), "r"(acc), "r"(idesc), "r"(tsf));
}

// Arrive on the barrier at the same shared offset in CTA `rank` of the pair,
// relaxed: a .release.cluster arrive compiles to ERRBAR + CGAERRBAR (a drain of
// the SM's outstanding memory traffic) and measured ~900 cycles per call.  What
// it signals -- an expanded operand stage in this CTA's shared memory / TMEM --
// is completed and published to the async proxy (fence.proxy.async, or
// tcgen05.wait::st + tcgen05.fence::before_thread_sync) by the arriving warp.
__device__ __forceinline__ void arrive_in(uint64_t* bar, uint32_t rank) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(mapa_shared(bar, rank))
                 : "memory");
}

__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            sm_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(sm_u32(bar))
        : "memory");
}

// Wait by polling mbarrier.test_wait (never suspends).  try_wait parks the thread
// and, measured here, the wake-up after the phase completes adds several hundred
// cycles to every commit -> expansion -> MMA round trip of the operand ring.
__device__ __forceinline__ void mbar_poll(uint64_t* b, uint32_t ph) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "L_%=:\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra L_%=;\n}" ::"r"(sm_u32(b)),
        "r"(ph)
        : "memory");
}

// MODE 7: cycle accounting of cluster 0's MMA thread (clock64 deltas summed)
__device__ unsigned long long g_p7_prof[16];
__device__ __forceinline__ void p7_acc(int i, long long& t) {
    const long long now = clock64();
    atomicAdd(&g_p7_prof[i], (unsigned long long)(now - t));
    t = now;
}

// MODE 8: event trace of cluster 0 (globaltimer ns): code << 56 | seq << 32 | ns (low 32)
__device__ unsigned long long g_p7_trace[8192];
__device__ unsigned int g_p7_ntrace;
__device__ __forceinline__ void p7_ev(uint32_t code, uint32_t seq) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (seq < 512 && code < 16) g_p7_trace[code * 512 + seq] = t;  // plain store: no round trip
}

struct P7Tile {
    const Tc7Prob* Q;
    size_t c0, i0;  // pair tile origin: output column c0, output row i0
};

template <int NN>
__device__ __forceinline__ bool p7_tile(uint32_t t, const Tc7Prob* probs, uint32_t GX, uint32_t GY, P7Tile& T) {
    const uint32_t per = GX * GY;
    const uint32_t z = t / per, rem = t - z * per, by = rem / GX, bx = rem - by * GX;
    T.Q = probs + z;
    T.c0 = size_t(bx) * kP7M;
    T.i0 = size_t(by) * NN;
    return T.c0 < T.Q->P.m && T.i0 < T.Q->P.n;
}

// MODE (diagnostics): 0 product; 1 no MMA (commits only); 7 cycle accounting
// DUAL: two MMA-issuing warps take alternate stages.  A tcgen05.mma issue blocks
// until the tensor pipe takes it (a one-deep queue, tools/micro/mma_rate.cu), so
// one issuing thread idles the pipe while it commits a stage and waits for the
// next one (~270 of every ~1300 cycles at 8 k-blocks per stage); with two, one
// thread's waits overlap the other's MMAs.  The MMAs of a tile interleave in any
// order (sums commute) except its first (accumulate = 0), which the stage-0
// thread issues before it publishes the tile as started.
template <int NN, int NACC, int STG, int KPS, int RG, int MODE, bool POLL = false, bool DUAL = true>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kP7Threads, 1)
    k_gemm_tc7(const Tc7Prob* __restrict__ probs, uint32_t GX, uint32_t GY, uint32_t NT) {
    using G = P7<NN, NACC, STG, KPS, RG>;
    constexpr int kN = G::N, kNH = G::NH, kStages = G::Stages;
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char* btile = smem;
    unsigned char* raw = smem + G::RawOff;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + G::BarOff);
    uint64_t* full = bars;                   // [stages] leader: 16 expansion warps of EACH CTA
    uint64_t* empty = full + kStages;        // [stages] MMA commit (multicast to the pair)
    uint64_t* rfull = empty + kStages;       // [RG] TMA boxes landed
    uint64_t* rempty = rfull + RG;           // [RG] 16 expansion warps consumed the group
    uint64_t* acc_full = rempty + RG;        // [NACC] MMA commit of a tile (multicast)
    uint64_t* acc_empty = acc_full + NACC;   // [NACC] leader: 16 epilogue warps (both CTAs) read it
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + NACC);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = cluster_rank();
    const uint32_t cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

    if (tid == 0) {
        tmem_slot[1] = 0;  // tiles whose first MMA is issued (DUAL)
        for (int s = 0; s < kStages; ++s) {
            mbar_init_n(&full[s], 32);
            mbar_init_n(&empty[s], 1);
        }
        for (int g = 0; g < RG; ++g) {
            mbar_init_n(&rfull[g], 1);
            mbar_init_n(&rempty[g], 16);
        }
        for (int b = 0; b < NACC; ++b) {
            mbar_init_n(&acc_full[b], DUAL ? 2 : 1);
            mbar_init_n(&acc_empty[b], 2 * kP7EpiWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sm_u32(tmem_slot)),
                     "r"(512u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;
    if (warp < 4) {  // scale factors: 8 columns of E8M0 1.0 (4 are read for M = 128 per CTA)
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(
                         tmem + (uint32_t(32 * warp) << 16) + G::SfCol),
                     "r"(0x7F7F7F7Fu)
                     : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync_all();  // both CTAs: barriers initialised, TMEM allocated, scales set
    asm volatile("tcgen05.fence::after_thread_sync;");

    if (warp == kP7Load) {
        // ---- raw words: per group of 8 k-blocks, one box of this CTA's 128 B^T rows
        //      and one of its NH A rows (rows past n are zero-filled by the TMA) ----
        if (lane == 0) {
            int g = 0;
            uint32_t ph = 0;
            size_t issued = 0;
            for (uint32_t t = cid; t < NT; t += ncl) {
                P7Tile T;
                if (!p7_tile<NN>(t, probs, GX, GY, T)) continue;
                const int cm = int(T.c0 + size_t(kP7MH) * rank);
                const int ia = int(T.i0 + size_t(kNH) * rank);
                const size_t KB = (T.Q->P.k + 63) / 64;
                for (size_t kb = 0; kb < KB; kb += kP7Grp, ++issued) {
                    if (issued >= size_t(RG)) mbar_wait1(&rempty[g], ph ^ 1);
                    unsigned char* r = raw + size_t(g) * G::RawGroup;
                    mbar_expect(&rfull[g], uint32_t(G::RawM + G::RawN));
                    tma_2d(r, &T.Q->mbt, cm, int(kb), &rfull[g]);
                    tma_2d(r + G::RawM, &T.Q->ma, ia, int(kb), &rfull[g]);
                    if (++g == RG) { g = 0; ph ^= 1; }
                }
            }
        }
        __syncwarp();
    } else if (warp == kP7Mma || warp == kP7Mma2) {
        const int me = warp - kP7Mma;
        if (lane == 0 && rank == 0 && (DUAL || me == 0)) {
            const uint32_t tsf = tmem + G::SfCol;
            const bool prof = MODE == 7 && cid == 0 && me == 0;
            volatile uint32_t* tstart = reinterpret_cast<volatile uint32_t*>(tmem_slot + 1);  // tiles started
            uint32_t nst = 0, gs = 0;
            int s = 0;
            uint32_t ph = 0, it = 0;
            for (uint32_t t = cid; t < NT; t += ncl, ++it) {
                P7Tile T;
                if (!p7_tile<NN>(t, probs, GX, GY, T)) { --it; continue; }
                const uint32_t buf = it % NACC;
                const uint32_t d = tmem + buf * G::AccCol;
                const size_t KB = (T.Q->P.k + 63) / 64;
                for (size_t kb = 0; kb < KB; kb += KPS, ++gs) {
                    const bool mine = !DUAL || int(gs & 1) == me;
                    if (mine) {
                        long long tt = prof ? clock64() : 0;
                        if (kb == 0) {
                            if (it >= NACC) {  // both CTAs' epilogues have drained this accumulator
                                // DUAL: the other thread may still be behind on this barrier;
                                // a parity wait is only unambiguous once the previous tile
                                // has started (its owner passed the phase before ours)
                                if (DUAL) while (*tstart < it) {}
                                mbar_wait1(&acc_empty[buf], ((it / NACC) - 1) & 1);
                                asm volatile("tcgen05.fence::after_thread_sync;");
                            }
                        } else if (DUAL) {
                            while (*tstart <= it) {}  // the tile's first MMA is issued
                        }
                        if (prof) p7_acc(3, tt);
                        if ((MODE == 8 || MODE == 10) && cid == 0) p7_ev(0, nst);
                        if (POLL) mbar_poll(&full[s], ph);
                        else mbar_wait1(&full[s], ph);
                        asm volatile("tcgen05.fence::after_thread_sync;");
                        if ((MODE == 8 || MODE == 10) && cid == 0) p7_ev(1, nst);
                        if (prof) p7_acc(0, tt);
                        const uint32_t bs = sm_u32(btile + size_t(s) * G::BStage);
#pragma unroll
                        for (int j = 0; j < KPS; ++j) {
                            if (kb + j >= KB) break;
                            if (MODE != 1)
                                mma_f4_pair_ts(d, tmem + G::ACol + uint32_t(8 * (KPS * s + j)),
                                               umma_desc(bs + (j >> 1) * G::Slot + 32 * (j & 1)),
                                               kb + j > 0 ? 1u : 0u, G::Idesc, tsf);
                            if (DUAL && kb == 0 && j == 0) *tstart = it + 1;
                        }
                        if (prof) p7_acc(1, tt);
                        if ((MODE == 8 || MODE == 10) && cid == 0) p7_ev(2, nst);
                        tc_commit_pair(&empty[s], 0x3);
                        ++nst;
                        if (prof) { p7_acc(2, tt); atomicAdd(&g_p7_prof[15], 1ull); }
                    }
                    if (++s == kStages) { s = 0; ph ^= 1; }
                }
                // every issuing thread commits every tile (no MMA pending: immediate)
                tc_commit_pair(&acc_full[buf], 0x3);
            }
        }
        __syncwarp();
    } else if (warp < 16) {
        // ---- expansion: warps 0-7 -> M-side operand in TMEM (lane = B^T row),
        //      warps 8-15 -> N-side operand tile in shared memory (A row 32 (w & 3) + lane);
        //      warp w takes the k-blocks j of a stage with j % 2 == (w >> 2) & 1 ----
        const bool mside = warp < 8;
        const int par = (warp >> 2) & 1;
        const int row = 32 * (warp & 3) + lane;
        const int roff = mside ? row : G::RawM / 8 + row;  // word offset of k-block 0 in a group
        const int kstride = mside ? kP7MH : kNH;            // words per k-block in the box
        const bool has_row = mside || row < kNH;
        const uint32_t tlane = uint32_t(32 * (warp & 3)) << 16;
        int s = 0, g = 0;
        uint32_t ph = 0, gph = 0;
        size_t staged = 0;
        for (uint32_t t = cid; t < NT; t += ncl) {
            P7Tile T;
            if (!p7_tile<NN>(t, probs, GX, GY, T)) continue;
            const size_t KB = (T.Q->P.k + 63) / 64;
            const bool prof = MODE == 7 && cid == 0 && rank == 0 && (tid == 0 || tid == 256);
            const int pb = mside ? 4 : 9;
            for (size_t kg = 0; kg < KB; kg += kP7Grp) {
                long long tt = prof ? clock64() : 0;
                mbar_wait1(&rfull[g], gph);
                if (prof) p7_acc(pb, tt);
                const uint64_t* rw = reinterpret_cast<const uint64_t*>(raw + size_t(g) * G::RawGroup) + roff;
                const size_t kend = min(KB, kg + kP7Grp);
                for (size_t kb = kg; kb < kend; kb += KPS, ++staged) {
                    if (prof) tt = clock64();
                    if (staged >= size_t(kStages)) mbar_wait1(&empty[s], ph ^ 1);
                    if (mside) asm volatile("tcgen05.fence::after_thread_sync;");
                    if (prof) p7_acc(pb + 1, tt);

                    uint64_t x[KPS / 2];
#pragma unroll
                    for (int i = 0; i < KPS / 2; ++i) {
                        const size_t k = kb + 2 * i + par;
                        x[i] = (MODE != 3 && MODE != 8 && k < kend && has_row) ? rw[int(k - kg) * kstride] : 0;
                    }
#pragma unroll
                    for (int i = 0; i < KPS / 2; ++i) {
                        const int j = 2 * i + par;
                        if (kb + j >= kend || MODE == 3 || MODE == 8) break;
                        if (mside && MODE == 2) {
                            if (x[i] == 0x123456789ull) btile[0] = 1;
                        } else if (mside) {
                            constexpr uint32_t M = 0x22222222u;
                            const uint32_t x0 = uint32_t(x[i]), x1 = uint32_t(x[i] >> 32);
                            asm volatile(
                                "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(
                                    tmem + tlane + G::ACol + uint32_t(8 * (KPS * s + j))),
                                "r"((x0 << 1) & M), "r"(x0 & M), "r"((x0 >> 1) & M), "r"((x0 >> 2) & M),
                                "r"((x1 << 1) & M), "r"(x1 & M), "r"((x1 >> 1) & M), "r"((x1 >> 2) & M)
                                : "memory");
                        } else if (has_row) {
                            store_row_f4(btile + size_t(s) * G::BStage + (j >> 1) * G::Slot, row, j & 1, x[i]);
                        }
                    }
                    if (prof) p7_acc(pb + 2, tt);
                    if (mside) {
                        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                        asm volatile("tcgen05.fence::before_thread_sync;");
                    } else {
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    }
                    __syncwarp();
                    if (lane == 0) {
                        if (rank == 0) mbar_arrive1(&full[s]);
                        else arrive_in(&full[s], 0);
                    }
                    if (prof) { p7_acc(pb + 3, tt); if (mside) atomicAdd(&g_p7_prof[14], 1ull); }
                    if ((MODE == 8 || MODE == 10) && cid == 0 && lane == 0) {
                        const int code = rank == 0 ? (warp < 8 ? 3 + warp : (warp == 8 ? 11 : (warp == 12 ? 12 : -1)))
                                                   : (warp == 0 ? 13 : (warp == 8 ? 14 : (warp == 15 ? 15 : -1)));
                        if (code >= 0) p7_ev(uint32_t(code), uint32_t(staged));
                    }
                    if (++s == kStages) { s = 0; ph ^= 1; }
                }
                __syncwarp();  // every lane has read the group before it is released
                if (lane == 0) mbar_arrive1(&rempty[g]);
                if (++g == RG) { g = 0; gph ^= 1; }
            }
        }
    } else {
        // ---- epilogue: warps 16-23, lane quarter lq = warp & 3, chunk parity h ----
        const int lq = warp & 3, h = (warp - kP7EpiW0) >> 2;
        uint32_t it = 0;
        for (uint32_t t = cid; t < NT; t += ncl, ++it) {
            P7Tile T;
            if (!p7_tile<NN>(t, probs, GX, GY, T)) { --it; continue; }
            const TcGemmArgs& P = T.Q->P;
            const uint32_t buf = it % NACC;
            const int nvalid = int(min(size_t(kN), P.n - T.i0));
            // this lane quarter's 32 output columns: one 32-bit half of a word-column
            const size_t col = T.c0 + size_t(kP7MH) * rank + size_t(32 * lq);
            uint32_t* cbase = reinterpret_cast<uint32_t*>(P.C + (col / 64) * P.sc + T.i0) + ((col / 32) & 1);
            // C ^= A*B: this tile's C words are loaded before the accumulator is ready
            // (the tile owns them), so the read is off the epilogue's critical path
            constexpr int kCh = kN / 16 / 2;  // chunks per warp
            uint32_t pre[kCh];
#pragma unroll
            for (int c = 0; c < kCh; ++c) {
                const int r = 16 * (h + 2 * c) + lane;
                pre[c] = (P.acc && lane < 16 && r < nvalid) ? cbase[2 * size_t(r)] : 0u;
            }
            mbar_wait1(&acc_full[buf], (it / NACC) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
            for (int c = 0; c < kCh; ++c) {
                const int ch = h + 2 * c;
                uint32_t v[16];
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
                    "%11, %12, %13, %14, %15}, [%16];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                      "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
                      "=r"(v[14]), "=r"(v[15])
                    : "r"(tmem + (uint32_t(32 * lq) << 16) + buf * G::AccCol + uint32_t(16 * ch)));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                uint32_t mine = 0;
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    const uint32_t par = __float_as_uint(__uint_as_float(v[q]) + 8388608.0f) & 1u;
                    const uint32_t bits = __ballot_sync(0xffffffffu, par);
                    if (lane == q) mine = bits;
                }
                const int r = 16 * ch + lane;
                if (lane < 16 && r < nvalid) cbase[2 * size_t(r)] = mine ^ pre[c];
            }
            // accumulator drained: the leader may start a later tile in it
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) {
                if (rank == 0) mbar_arrive1(&acc_empty[buf]);
                else arrive_in(&acc_empty[buf], 0);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync_all();  // the pair's MMAs and TMEM reads are finished
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
}

int sm_count7() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

using Tc7Fn = void (*)(const Tc7Prob*, uint32_t, uint32_t, uint32_t);
struct Tc7Cfg {
    Tc7Fn fn = nullptr;
    int nn = 0;
    size_t smem = 0;
};

template <int NN, int NACC, int STG, int KPS, int RG, int MODE>
Tc7Cfg make7() {
    Tc7Cfg c;
    // MODE 9: the MMA thread polls `full` with test_wait instead of try_wait
    if (MODE == 9) c.fn = k_gemm_tc7<NN, NACC, STG, KPS, RG, 0, true>;
    else if (MODE == 11) c.fn = k_gemm_tc7<NN, NACC, STG, KPS, RG, 0, false, false>;
    else c.fn = k_gemm_tc7<NN, NACC, STG, KPS, RG, MODE>;
    c.nn = NN;
    c.smem = P7<NN, NACC, STG, KPS, RG>::Smem;
    if (cudaFuncSetAttribute(c.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(c.smem)) != cudaSuccess)
        c.fn = nullptr;
    return c;
}

// F2GPU_TC7 selects the geometry (0 = off): N x accumulators x stages x k-blocks/stage
//   1 (default): 256 x 1 x 3 x 8     2: 256 x 1 x 7 x 4     3: 192 x 2 x 3 x 4
//   4: 160 x 2 x 5 x 4               5: 224 x 2 x 3 x 2
// Measured (one B200, 16384^3 / 8192^3 / decomposition 65536^2): 1: 1697 us / 251 us /
// 58.2 ms; 2: 2006 / 283 us; 3: 2595 / 356 us; k_gemm_tc3 (F2GPU_TC7=0): 1839 / 271 us / 61.6 ms
// F2GPU_TC7_MODE: diagnostics (see k_gemm_tc7)
const Tc7Cfg& tc7_cfg() {
    static const Tc7Cfg cfg = [] {
        const int v = int(options().tc7);
        const int mode = int(options().tc7_mode);
        if (v == 0) return Tc7Cfg{};
#define F2_TC7_PICK(NN, NACC, STG, KPS, RG)                               \
    switch (mode) {                                                       \
        case 10: return make7<NN, NACC, STG, KPS, RG, 10>();              \
        case 11: return make7<NN, NACC, STG, KPS, RG, 11>();              \
        case 1: return make7<NN, NACC, STG, KPS, RG, 1>();                \
        case 7: return make7<NN, NACC, STG, KPS, RG, 7>();                \
        case 3: return make7<NN, NACC, STG, KPS, RG, 3>();                \
        case 8: return make7<NN, NACC, STG, KPS, RG, 8>();                \
        case 9: return make7<NN, NACC, STG, KPS, RG, 9>();                \
        case 2: return make7<NN, NACC, STG, KPS, RG, 2>();                \
        default: return make7<NN, NACC, STG, KPS, RG, 0>();               \
    }
        if (v == 2) { F2_TC7_PICK(256, 1, 7, 4, 6) }
        if (v == 3) { F2_TC7_PICK(192, 2, 3, 4, 6) }
        if (v == 4) { F2_TC7_PICK(160, 2, 5, 4, 6) }
        if (v == 5) { F2_TC7_PICK(224, 2, 3, 2, 6) }
        if (v == 6) { F2_TC7_PICK(128, 2, 3, 8, 6) }
        if (v == 7) { F2_TC7_PICK(160, 2, 2, 8, 6) }
        F2_TC7_PICK(256, 1, 3, 8, 6)
#undef F2_TC7_PICK
    }();
    return cfg;
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encoder() {
    static EncodeFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return EncodeFn(nullptr);
        return reinterpret_cast<EncodeFn>(p);
    }();
    return fn;
}

bool tc7_ready() { return tc7_cfg().fn != nullptr && encoder() != nullptr; }

bool tc7_args_ok(const TcGemmArgs& p) {
    return p.n > 0 && p.k > 0 && p.m > 0 && p.m % kP7M == 0 && p.sbt % 2 == 0 && p.sa % 2 == 0 &&
           reinterpret_cast<uintptr_t>(p.A) % 16 == 0 && reinterpret_cast<uintptr_t>(p.BT) % 16 == 0 &&
           p.n < (size_t(1) << 31) && p.m < (size_t(1) << 31);
}

// 2-D map over a word-column-major operand: dim0 = rows (contiguous words), dim1 =
// k-blocks (stride words apart); box = `box_rows` x 8 k-blocks, OOB zero-filled
bool encode(CUtensorMap* out, const uint64_t* base, size_t rows, size_t kb, size_t stride, uint32_t box_rows) {
    const cuuint64_t dims[2] = {cuuint64_t(rows), cuuint64_t(kb)};
    const cuuint64_t strides[1] = {cuuint64_t(stride * 8)};
    const cuuint32_t box[2] = {box_rows, uint32_t(kP7Grp)};
    const cuuint32_t es[2] = {1, 1};
    return encoder()(out, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<uint64_t*>(base), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Device copies of the problem descriptors (tensor maps + arguments), cached by the
// problem list: a repeated product (the same operands and shapes, e.g. every step of a
// benchmark or a replayed decomposition) reuses its descriptors instead of encoding
// them again and copying them in-stream before the kernel (a pageable H2D copy per
// launch).  A descriptor only holds addresses and shapes, so a stale entry is never
// wrong for a list of identical bytes.  Bounded; the oldest entries are evicted once
// the device is idle for them (cudaFree synchronises).
struct Tc7Cache {
    struct Entry {
        std::vector<TcGemmArgs> key;
        Tc7Prob* d = nullptr;
        uint64_t used = 0;
        cudaStream_t origin = nullptr;  // the stream that copied the descriptors ...
        cudaEvent_t ready = nullptr;    // ... and the copy's completion, for other streams
    };
    std::vector<Entry> e;
    uint64_t tick = 0;
    static constexpr size_t kMax = 512;
};
Tc7Cache& tc7_cache() {
    static Tc7Cache c;
    return c;
}
bool same_args(const TcGemmArgs& a, const TcGemmArgs& b) {
    return a.A == b.A && a.sa == b.sa && a.n == b.n && a.BT == b.BT && a.sbt == b.sbt && a.C == b.C && a.sc == b.sc &&
           a.k == b.k && a.m == b.m && a.acc == b.acc;
}

cudaError_t launch7(const TcGemmArgs* h_probs, int nprob, cudaStream_t s) {
    const Tc7Cfg& c = tc7_cfg();
    size_t mx = 0, nx = 0;
    for (int i = 0; i < nprob; ++i) {
        const TcGemmArgs& p = h_probs[i];
        if (!tc7_args_ok(p)) return cudaErrorInvalidValue;
        mx = std::max(mx, p.m);
        nx = std::max(nx, p.n);
    }
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cap) != cudaSuccess) return cudaErrorInvalidValue;
    if (cap != cudaStreamCaptureStatusNone) {  // inside a capture: stream-ordered allocation, no cache
        std::vector<Tc7Prob> q(static_cast<size_t>(nprob));
        for (int i = 0; i < nprob; ++i) {
            const TcGemmArgs& p = h_probs[i];
            const size_t KB = (p.k + 63) / 64;
            if (!encode(&q[i].mbt, p.BT, p.m, KB, p.sbt, kP7MH) ||
                !encode(&q[i].ma, p.A, p.n, KB, p.sa, uint32_t(c.nn / 2)))
                return cudaErrorInvalidValue;
            q[i].P = p;
        }
        Tc7Prob* d = nullptr;
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&d), q.size() * sizeof(Tc7Prob), s);
        if (e != cudaSuccess) return e;
        e = cudaMemcpyAsync(d, q.data(), q.size() * sizeof(Tc7Prob), cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return e;
        const uint32_t GX = uint32_t(mx / kP7M), GY = uint32_t((nx + c.nn - 1) / c.nn);
        const uint32_t NT = GX * GY * uint32_t(nprob);
        const uint32_t clusters = std::min<uint32_t>(NT, uint32_t(sm_count7() / 2));
        c.fn<<<2 * clusters, kP7Threads, c.smem, s>>>(d, GX, GY, NT);
        e = cudaGetLastError();
        cudaFreeAsync(d, s);
        return e;
    }
    Tc7Cache& cache = tc7_cache();
    Tc7Prob* d = nullptr;
    for (auto& en : cache.e) {
        if (en.key.size() != size_t(nprob)) continue;
        bool eq = true;
        for (int i = 0; i < nprob && eq; ++i) eq = same_args(en.key[size_t(i)], h_probs[i]);
        if (eq) {
            d = en.d;
            en.used = ++cache.tick;
            if (s != en.origin && cudaStreamWaitEvent(s, en.ready, 0) != cudaSuccess) return cudaErrorInvalidValue;
            break;
        }
    }
    cudaError_t e = cudaSuccess;
    if (!d) {
        std::vector<Tc7Prob> q(static_cast<size_t>(nprob));
        for (int i = 0; i < nprob; ++i) {
            const TcGemmArgs& p = h_probs[i];
            const size_t KB = (p.k + 63) / 64;
            if (!encode(&q[i].mbt, p.BT, p.m, KB, p.sbt, kP7MH) ||
                !encode(&q[i].ma, p.A, p.n, KB, p.sa, uint32_t(c.nn / 2)))
                return cudaErrorInvalidValue;
            q[i].P = p;
        }
        if (cache.e.size() >= Tc7Cache::kMax) {  // evict the least recently used entry
            size_t v = 0;
            for (size_t i = 1; i < cache.e.size(); ++i)
                if (cache.e[i].used < cache.e[v].used) v = i;
            cudaFree(cache.e[v].d);  // synchronising: no launch still reads it
            cudaEventDestroy(cache.e[v].ready);
            cache.e.erase(cache.e.begin() + long(v));
        }
        e = cudaMalloc(reinterpret_cast<void**>(&d), q.size() * sizeof(Tc7Prob));
        if (e != cudaSuccess) return e;
        // pageable source: staged before the call returns; ordered before the launch
        e = cudaMemcpyAsync(d, q.data(), q.size() * sizeof(Tc7Prob), cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) { cudaFree(d); return e; }
        cudaEvent_t ev = nullptr;
        if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) return e;
        if ((e = cudaEventRecord(ev, s)) != cudaSuccess) return e;
        cache.e.push_back({std::vector<TcGemmArgs>(h_probs, h_probs + nprob), d, ++cache.tick, s, ev});
    }
    const uint32_t GX = uint32_t(mx / kP7M), GY = uint32_t((nx + c.nn - 1) / c.nn);
    const uint32_t NT = GX * GY * uint32_t(nprob);
    const uint32_t clusters = std::min<uint32_t>(NT, uint32_t(sm_count7() / 2));
    c.fn<<<2 * clusters, kP7Threads, c.smem, s>>>(d, GX, GY, NT);
    return cudaGetLastError();
}

}  // namespace

bool gemm_tc7_enabled() { return tc7_ready(); }

int tc7_trace_read(unsigned long long* out, int cap) {
    const int n = cap < 8192 ? cap : 8192;
    cudaMemcpyFromSymbol(out, g_p7_trace, size_t(n) * 8);
    return n;
}

void tc7_prof_read(unsigned long long* out16, bool reset) {
    cudaMemcpyFromSymbol(out16, g_p7_prof, 16 * sizeof(unsigned long long));
    if (reset) {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbol(g_p7_prof, z, sizeof z);
    }
}

cudaError_t launch_gemm_tc7(const TcGemmArgs& p, cudaStream_t s) {
    if (!tc7_ready()) return cudaErrorInvalidValue;
    return launch7(&p, 1, s);
}

cudaError_t launch_gemm_tc7_batched(const TcGemmArgs* h_probs, const TcGemmArgs*, int nprob, cudaStream_t s) {
    if (!tc7_ready() || nprob <= 0) return cudaErrorInvalidValue;
    return launch7(h_probs, nprob, s);
}

}  // namespace f2
