// tc_leaf.cu — the evaluated alternative GEMM leaf (north_star): GF(2) products
// on the 5th-generation tensor cores.
//
// sm_100a has no binary (b1) MMA: mma.sync .b1 is emulated with IMMA and tcgen05
// has no b1 kind (SURVEY Probe P6).  The leaf therefore expands bits to 0/1
// bytes and runs tcgen05.mma.cta_group::1.kind::i8 with s32 accumulation in
// TMEM; the parity of each accumulator is the GF(2) result.
//
// Transposed formulation D^T = B^T * A^T: the MMA's M dimension (TMEM lanes) is
// the output COLUMN, N (TMEM columns) the output ROW.  After tcgen05.ld each
// thread holds one output column for 32 consecutive rows, so one __ballot_sync
// of the accumulator LSBs yields 32 packed output bits of one row: the epilogue
// costs two instructions per 32 output bits.
//
// Tile: 128 output columns x 256 output rows per CTA, k-blocks of 64 bits
// (two K=32 MMAs), operands expanded in registers into a double-buffered
// canonical K-major no-swizzle layout ((8,n),2):((16B,SBO),LBO) with LBO=128 B,
// SBO=512 B, MMA completion tracked with tcgen05.commit -> mbarrier.
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "kernels.cuh"
#include "options.h"
#include "tc_common.cuh"

namespace f2 {

#if F2GPU_EXPERIMENTAL  // evaluated and rejected variants: built only with F2GPU_EXPERIMENTAL=1 (build.py)
namespace {

constexpr int kTcThreads = 256;  // 8 warps: expansion; thread 0 issues MMAs; warps 0-3 epilogue
constexpr int kTcM = 128;        // output columns per CTA (TMEM lanes)
constexpr int kTcN = 256;        // output rows per CTA (TMEM columns)
constexpr int kTcABytes = kTcM * 64;  // B^T tile: 128 x 64 bytes
constexpr int kTcBBytes = kTcN * 64;  // A^T tile: 256 x 64 bytes
constexpr int kTcStage = kTcABytes + kTcBBytes;
constexpr size_t kTcSmem = 2 * size_t(kTcStage) + 64;

// 8 bits -> 8 bytes of 0/1 (byte j = bit j)
__device__ __forceinline__ uint64_t expand8(uint32_t x) {
    uint64_t y = (uint64_t(x & 0xFFu) * 0x0101010101010101ull) & 0x8040201008040201ull;
    return ((y + 0x7F7F7F7F7F7F7F7Full) >> 7) & 0x0101010101010101ull;
}

// 4 bits -> 4 bytes of 0/1: the shifted copies x, x<<7, x<<14, x<<21 do not
// overlap, so one multiply places bit i at bit 8i
__device__ __forceinline__ uint32_t expand4(uint32_t x) { return ((x & 0xFu) * 0x00204081u) & 0x01010101u; }

// store the 64 0/1 bytes of word w as row r of a K-major tile
__device__ __forceinline__ void store_row(unsigned char* tile, int r, uint64_t w) {
    const uint32_t lo = uint32_t(w), hi = uint32_t(w >> 32);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const uint32_t x = (c < 2) ? (lo >> (16 * c)) : (hi >> (16 * (c - 2)));
        uint4 v;
        v.x = expand4(x);
        v.y = expand4(x >> 4);
        v.z = expand4(x >> 8);
        v.w = expand4(x >> 12);
        *reinterpret_cast<uint4*>(tile + kmaj_off(r, c)) = v;
    }
}

// kind::i8, A=u8, B=u8, D=s32, both K-major, M=128, N=256
constexpr uint32_t kIdesc = (2u << 4) | (0u << 7) | (0u << 10) | (uint32_t(kTcN >> 3) << 17) |
                            (uint32_t(kTcM >> 4) << 24);

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
    const uint32_t z = 0;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %5, %5, %5}, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(kIdesc), "r"(acc), "r"(z));
}

}  // namespace

// C (n x m) = A (n x k) * B (k x m) over GF(2); n % 256 == 0, m % 128 == 0, k % 64 == 0.
// acc != 0: C ^= A*B.
__global__ void __launch_bounds__(kTcThreads, 1)
    k_gemm_tc(const uint64_t* __restrict__ A, size_t sa, const uint64_t* __restrict__ B, size_t sb,
              uint64_t* __restrict__ C, size_t sc, size_t n, size_t k, size_t m, int acc) {
    extern __shared__ __align__(1024) unsigned char smem[];
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + 2 * kTcStage);  // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mbar + 2);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const size_t c0 = size_t(blockIdx.x) * kTcM;  // output column base
    const size_t i0 = size_t(blockIdx.y) * kTcN;  // output row base
    const size_t q0 = c0 / 64;
    const size_t KB = k / 64;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         sm_u32(tmem_slot)),
                     "r"(uint32_t(kTcN)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        mbar_init_n(&mbar[0], 1);
        mbar_init_n(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    uint32_t ph[2] = {0, 0};
    // operand words of the NEXT k-block are prefetched into registers while the
    // current one is expanded (the L2 latency is off the critical path)
    const bool bt_warp = warp < 2;                 // warps 0,1: B^T (transpose + expand)
    const int ar0 = tid - 64, ar1 = tid + 128;     // warps 2..7: A^T rows (1-2 per thread)
    const bool has_ar1 = !bt_warp && ar1 < kTcN;
    uint64_t pa0 = 0, pa1 = 0, pb0 = 0, pb1 = 0;
    auto fetch = [&](size_t kb) {
        if (bt_warp) {
            const uint64_t* bp = B + (q0 + warp) * sb + kb * 64;
            pb0 = bp[lane];
            pb1 = bp[lane + 32];
        } else {
            pa0 = A[kb * sa + i0 + ar0];
            if (has_ar1) pa1 = A[kb * sa + i0 + ar1];
        }
    };
    fetch(0);
    for (size_t kb = 0; kb < KB; ++kb) {
        const int s = int(kb & 1);
        unsigned char* ta = smem + s * kTcStage;  // B^T tile (MMA A operand)
        unsigned char* tb = ta + kTcABytes;       // A^T tile (MMA B operand)
        const uint64_t a0 = pa0, a1 = pa1;
        uint64_t x0 = pb0, x1 = pb1;
        if (kb + 1 < KB) fetch(kb + 1);
        if (kb >= 2) {  // the MMA that last read this stage has completed
            mbar_wait1(&mbar[s], ph[s]);
            ph[s] ^= 1;
        }
        if (!bt_warp) {
            store_row(tb, ar0, a0);
            if (has_ar1) store_row(tb, ar1, a1);
        } else {
            // B^T: transpose the 64x64 bit tile of word-column q0+warp (rows k -> columns)
            {   // stage 32 (in-lane)
                const uint64_t t = ((x0 >> 32) ^ x1) & 0x00000000FFFFFFFFull;
                x1 ^= t;
                x0 ^= t << 32;
            }
            const uint64_t masks[5] = {0x0000FFFF0000FFFFull, 0x00FF00FF00FF00FFull,
                                       0x0F0F0F0F0F0F0F0Full, 0x3333333333333333ull,
                                       0x5555555555555555ull};
#pragma unroll
            for (int st = 0; st < 5; ++st) {
                const int j = 16 >> st;
                const uint64_t msk = masks[st];
                const uint64_t y0 = __shfl_xor_sync(0xffffffffu, x0, j);
                const uint64_t y1 = __shfl_xor_sync(0xffffffffu, x1, j);
                if (!(lane & j)) {
                    x0 ^= (((x0 >> j) ^ y0) & msk) << j;
                    x1 ^= (((x1 >> j) ^ y1) & msk) << j;
                } else {
                    x0 ^= ((y0 >> j) ^ x0) & msk;
                    x1 ^= ((y1 >> j) ^ x1) & msk;
                }
            }
            store_row(ta, 64 * warp + lane, x0);       // output column c0 + 64w + lane
            store_row(ta, 64 * warp + lane + 32, x1);  // output column c0 + 64w + lane + 32
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t sa_ = sm_u32(ta), sb_ = sm_u32(tb);
            mma_i8(tmem, umma_desc(sa_), umma_desc(sb_), kb > 0 ? 1u : 0u);
            mma_i8(tmem, umma_desc(sa_ + kKHalf), umma_desc(sb_ + kKHalf), 1u);
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             sm_u32(&mbar[s]))
                         : "memory");
        }
    }
    // wait for the last MMA (tcgen05.commit tracks all prior MMAs of this thread)
    {
        const int s = int((KB - 1) & 1);
        mbar_wait1(&mbar[s], ph[s]);
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    // epilogue: warp w (0..3) owns TMEM lanes 32w..32w+31 = output columns c0+32w+lane
    const size_t q = q0 + ((warp & 3) >> 1);
    uint32_t* crow = reinterpret_cast<uint32_t*>(C + q * sc + i0) + (warp & 1);
#pragma unroll 1
    for (int chunk = 0; chunk < (warp < 4 ? kTcN / 32 : 0); ++chunk) {
        uint32_t v[32];
        const uint32_t taddr = tmem + (uint32_t(32 * warp) << 16) + uint32_t(32 * chunk);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
            "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
            "%28, %29, %30, %31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
              "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
              "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
              "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
              "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        uint32_t mine = 0;
#pragma unroll
        for (int r = 0; r < 32; ++r) {
            const uint32_t bits = __ballot_sync(0xffffffffu, v[r] & 1u);
            if (lane == r) mine = bits;
        }
        const size_t row = size_t(32 * chunk + lane);
        uint32_t* dst = crow + 2 * row;  // 32-bit half of word (i0+row, q)
        if (acc) mine ^= *dst;
        *dst = mine;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(uint32_t(kTcN)));
}

// ---- v2: 256x256 output tiles, warp-specialised, pre-transposed B ----
// B is transposed once beforehand (B^T: m x k, one pass over B), so both
// operands arrive as "rows of 64 k-bits": word (r, kb) at X[kb * s + r].  Per
// k-block the load warp bulk-copies 256 B^T words + 256 A words (4 KB) into an
// 8-deep raw ring; 16 expansion warps turn one word each into a 64-byte 0/1
// row of the SWIZZLE_64B K-major tiles; the MMA warp issues 4 x (M=128, N=256,
// K=32) int8 MMAs into two TMEM accumulators (all 512 columns) and commits the
// stage release.  The k order inside a k-block is permuted identically for both
// operands ((x >> t) & 0x01010101 spreads bits t, t+8, t+16, t+24 of a 32-bit
// half into one 4-byte word), which a dot product does not see and which costs
// two instructions per 4 output bytes.
constexpr int kT2Exp = 512;                  // expansion threads (warps 0-15)
constexpr int kT2Mma = kT2Exp / 32;          // warp 16: MMA issuer
constexpr int kT2Load = kT2Mma + 1;          // warp 17: bulk loads
constexpr int kT2Threads = kT2Exp + 64;
constexpr int kT2Cols = 256;                 // output columns per CTA (2 x M=128)
constexpr int kT2Rows = 256;                 // output rows per CTA (N=256)
constexpr int kT2ABytes = kT2Cols * 64;      // expanded B^T tile (MMA A operand)
constexpr int kT2BBytes = kT2Rows * 64;      // expanded A^T tile (MMA B operand)
constexpr int kT2Slot = kT2ABytes + kT2BBytes;  // one expanded k-block
constexpr int kT2Kps = 2;                        // k-blocks per pipeline stage
constexpr int kT2Stage = kT2Kps * kT2Slot;
constexpr int kT2Stages = 3;
constexpr int kT2RawBytes = (kT2Rows + kT2Cols) * 8;  // packed words of one k-block
constexpr int kT2Raw = 4;
constexpr size_t kT2Smem = size_t(kT2Stages) * kT2Stage + size_t(kT2Raw) * kT2RawBytes + 256;

// 64 bits -> 64 bytes of 0/1 in the permuted k order, row r of a K-major tile
__device__ __forceinline__ void store_row_perm(unsigned char* tile, int r, uint64_t w) {
    const uint32_t h[2] = {uint32_t(w), uint32_t(w >> 32)};
    constexpr uint32_t M = 0x01010101u;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const uint32_t x = h[c >> 1] >> (4 * (c & 1));
        uint4 v;
        v.x = x & M;
        v.y = (x >> 1) & M;
        v.z = (x >> 2) & M;
        v.w = (x >> 3) & M;
        *reinterpret_cast<uint4*>(tile + kmaj_off(r, c)) = v;
    }
}

// MODE (diagnostic, F2GPU_TC_MODE): 0 normal; 1 expansion warps skip the
// expanded stores (MMA-bound rate); 2 the MMA warp skips the MMAs (expansion rate);
// 3 = 2 without the proxy fence; 4 = full kernel without the proxy fence (timing only)
template <int MODE>
__global__ void __launch_bounds__(kT2Threads, 1)
    k_gemm_tc2(const uint64_t* __restrict__ A, size_t sa, const uint64_t* __restrict__ BT, size_t sbt,
               uint64_t* __restrict__ C, size_t sc, size_t k, int acc) {
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char* raw = smem + size_t(kT2Stages) * kT2Stage;
    uint64_t* full = reinterpret_cast<uint64_t*>(raw + size_t(kT2Raw) * kT2RawBytes);
    uint64_t* empty = full + kT2Stages;
    uint64_t* rfull = empty + kT2Stages;
    uint64_t* rempty = rfull + kT2Raw;
    uint64_t* done = rempty + kT2Raw;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const size_t c0 = size_t(blockIdx.x) * kT2Cols;
    const size_t i0 = size_t(blockIdx.y) * kT2Rows;
    const size_t KB = k / 64;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         sm_u32(tmem_slot)),
                     "r"(512u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int s = 0; s < kT2Stages; ++s) {
            mbar_init_n(&full[s], kT2Exp / 32);  // one arrive per expansion warp
            mbar_init_n(&empty[s], 1);
        }
        for (int s = 0; s < kT2Raw; ++s) {
            mbar_init_n(&rfull[s], 1);
            mbar_init_n(&rempty[s], kT2Exp / 32);
        }
        mbar_init_n(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    if (warp == kT2Load) {
        // ===== load warp: raw operand words, kT2Raw k-blocks ahead =====
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (size_t kb = 0; kb < KB; ++kb) {
                if (kb >= size_t(kT2Raw)) mbar_wait1(&rempty[s], ph ^ 1);
                unsigned char* r = raw + size_t(s) * kT2RawBytes;
                mbar_expect(&rfull[s], kT2RawBytes);
                bulk_g2s(r, BT + kb * sbt + c0, kT2Cols * 8, &rfull[s]);
                bulk_g2s(r + kT2Cols * 8, A + kb * sa + i0, kT2Rows * 8, &rfull[s]);
                if (++s == kT2Raw) { s = 0; ph ^= 1; }
            }
        }
        __syncwarp();
    } else if (warp == kT2Mma) {
        // ===== MMA issuer =====
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (size_t kb = 0; kb < KB; kb += kT2Kps) {
                mbar_wait1(&full[s], ph);
                asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
                for (int j = 0; j < kT2Kps; ++j) {
                    if (kb + j >= KB) break;
                    const uint32_t ta = sm_u32(smem + size_t(s) * kT2Stage + j * kT2Slot);
                    const uint32_t tb = ta + kT2ABytes;
                    const uint32_t a0 = kb + j > 0 ? 1u : 0u;
                    if (MODE != 2 && MODE != 3) {
                        mma_i8(tmem, umma_desc(ta), umma_desc(tb), a0);
                        mma_i8(tmem, umma_desc(ta + kKHalf), umma_desc(tb + kKHalf), 1u);
                        mma_i8(tmem + 256, umma_desc(ta + 128 * 64), umma_desc(tb), a0);
                        mma_i8(tmem + 256, umma_desc(ta + 128 * 64 + kKHalf), umma_desc(tb + kKHalf), 1u);
                    }
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 sm_u32(&empty[s]))
                             : "memory");
                if (++s == kT2Stages) { s = 0; ph ^= 1; }
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             sm_u32(done))
                         : "memory");
        }
        __syncwarp();
    } else {
        // ===== expansion warps 0-15: thread t expands raw word t =====
        // t < 256: B^T row t (output column c0 + t); t >= 256: A^T row t - 256
        const int region = tid < kT2Cols ? 0 : kT2ABytes;
        const int r = tid & 255;
        int s = 0, rs = 0;
        uint32_t ph = 0, rph = 0;
        for (size_t kb = 0, st = 0; kb < KB; kb += kT2Kps, ++st) {
            if (st >= size_t(kT2Stages)) mbar_wait1(&empty[s], ph ^ 1);
#pragma unroll
            for (int j = 0; j < kT2Kps; ++j) {
                if (kb + j >= KB) break;
                mbar_wait1(&rfull[rs], rph);
                const uint64_t x = reinterpret_cast<const uint64_t*>(raw + size_t(rs) * kT2RawBytes)[tid];
                unsigned char* tile = smem + size_t(s) * kT2Stage + j * kT2Slot + region;
                if (MODE == 1) {
                    if (x == 0x123456789ull) tile[r] = 1;  // keep the load alive
                } else {
                    store_row_perm(tile, r, x);
                }
                // the raw slot is released only after x was consumed by the stores
                // above: an arrive right after the LDS can overtake it (the mbarrier
                // unit is not ordered behind outstanding shared loads) and let the
                // next bulk load overwrite a word not yet read
                __syncwarp();
                if (lane == 0) mbar_arrive1(&rempty[rs]);
                if (++rs == kT2Raw) { rs = 0; rph ^= 1; }
            }
            if (MODE < 3) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive1(&full[s]);
            if (++s == kT2Stages) { s = 0; ph ^= 1; }
        }
        // ===== epilogue: warp w -> accumulator (w>>2)&1, TMEM lanes 32(w&3).., row half w>>3 =====
        mbar_wait1(done, 0);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const int accn = (warp >> 2) & 1, lq = warp & 3, rh = warp >> 3;
        const size_t col = c0 + size_t(accn) * 128 + size_t(lq) * 32;  // first output column
        uint32_t* crow = reinterpret_cast<uint32_t*>(C + (col / 64) * sc + i0) + ((col / 32) & 1);
#pragma unroll 1
        for (int chunk = 4 * rh; chunk < 4 * rh + 4; ++chunk) {
            uint32_t v[32];
            const uint32_t taddr = tmem + (uint32_t(32 * lq) << 16) + uint32_t(256 * accn + 32 * chunk);
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
                "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
                "%28, %29, %30, %31}, [%32];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                  "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
                  "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
                  "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
                  "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
                  "=r"(v[31])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            uint32_t mine = 0;
#pragma unroll
            for (int q = 0; q < 32; ++q) {
                const uint32_t bits = __ballot_sync(0xffffffffu, v[q] & 1u);
                if (lane == q) mine = bits;
            }
            uint32_t* dst = crow + 2 * size_t(32 * chunk + lane);
            if (acc) mine ^= *dst;
            *dst = mine;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
}

#endif
// ---- v3: block-scaled FP4 (kind::mxf4) on the same warp-specialised pipeline ----
// A bit becomes the E2M1 nibble 0x2 (= 1.0) or 0x0, two elements per byte, so a
// 64-bit k-block is one 32-byte K=64 row slice: half the expansion stores and
// half the operand reads of the int8 leaf, at twice the int8 MMA rate.  The
// E8M0 scale factors are all 1.0: 32 TMEM columns are filled with 0x7F bytes,
// so the result does not depend on the scale-factor layout.  Accumulators are
// f32 (exact: every sum is an integer <= k < 2^23); parity = LSB of v + 2^23.
// TMEM: two M=128 x N=240 accumulators (480 columns) + the 32 scale columns.
// Output rows are tiled by 240 (ragged last tile); B is pre-transposed.
constexpr int kT3Exp = 512;                 // expansion threads (warps 0-15)
constexpr int kT3Mma = kT3Exp / 32;         // warp 16
constexpr int kT3Load = kT3Mma + 1;         // warp 17
constexpr int kT3Threads = kT3Exp + 64;
constexpr int kT3Cols = 256;                // output columns per CTA (2 x M=128)
constexpr int kT3Rows = 240;                // output rows per CTA (N)
constexpr int kT3ABytes = kT3Cols * 64;     // B^T slot: 2 k-blocks x 32 B per row
constexpr int kT3BBytes = kT3Rows * 64;     // A^T slot
constexpr int kT3Slot = kT3ABytes + kT3BBytes;  // 2 k-blocks
constexpr int kT3Slots = 2;                 // slots per stage -> 4 k-blocks per stage
constexpr int kT3Kps = 2 * kT3Slots;
constexpr int kT3Stage = kT3Slots * kT3Slot;
constexpr int kT3Stages = 3;
constexpr int kT3RawWords = kT3Cols + kT3Rows;
constexpr int kT3RawBytes = kT3RawWords * 8;
constexpr int kT3Raw = 4;  // (an 8-deep ring measured no faster; per-thread __ldg feeds 8 k-blocks ahead
                           //  instead of the bulk copies: 16384^3 2.66 vs 1.85 ms -- the L1/shared
                           //  data path is the limit and global loads use it too, bulk copies do not)
constexpr uint32_t kT3SfCol = 480;
constexpr size_t kT3Smem = size_t(kT3Stages) * kT3Stage + size_t(kT3Raw) * kT3RawBytes + 256;
constexpr uint32_t kIdescF4 = idesc_f4(128, kT3Rows);

__device__ __forceinline__ void ld_shared_u64(uint64_t& v, const void* p) { v = *reinterpret_cast<const uint64_t*>(p); }

#ifdef TC3_PROFILE
__device__ long long g_tc3_prof[8];
#endif
template <int MODE>
__global__ void __launch_bounds__(kT3Threads, 1)
    k_gemm_tc3(TcGemmArgs one, const TcGemmArgs* __restrict__ probs) {
    // one problem per launch, or a batch (blockIdx.z = problem; Strassen leaves)
#ifdef TC3_PROFILE
    const bool prof = blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0;
    if (prof && threadIdx.x == 0) g_tc3_prof[0] = clock64();
#endif
    const TcGemmArgs P = probs ? probs[blockIdx.z] : one;
    if (size_t(blockIdx.x) * kT3Cols >= P.m || size_t(blockIdx.y) * kT3Rows >= P.n) return;
    const uint64_t* __restrict__ A = P.A;
    const uint64_t* __restrict__ BT = P.BT;
    uint64_t* __restrict__ C = P.C;
    const size_t sa = P.sa, n = P.n, sbt = P.sbt, sc = P.sc, k = P.k;
    const int acc = P.acc;
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char* raw = smem + size_t(kT3Stages) * kT3Stage;
    uint64_t* full = reinterpret_cast<uint64_t*>(raw + size_t(kT3Raw) * kT3RawBytes);
    uint64_t* empty = full + kT3Stages;
    uint64_t* rfull = empty + kT3Stages;
    uint64_t* rempty = rfull + kT3Raw;
    uint64_t* done = rempty + kT3Raw;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const size_t c0 = size_t(blockIdx.x) * kT3Cols;
    const size_t i0 = size_t(blockIdx.y) * kT3Rows;
    const int nvalid = int(min(size_t(kT3Rows), n - i0));
    const size_t KB = (k + 63) / 64;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         sm_u32(tmem_slot)),
                     "r"(512u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int s = 0; s < kT3Stages; ++s) {
            mbar_init_n(&full[s], kT3Exp / 32);
            mbar_init_n(&empty[s], 1);
        }
        for (int s = 0; s < kT3Raw; ++s) {
            mbar_init_n(&rfull[s], 1);
            mbar_init_n(&rempty[s], kT3Exp / 32);
        }
        mbar_init_n(done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;
    if (warp < 4) {  // scale factors: every byte of columns 480..511 = E8M0 1.0
        const uint32_t one = 0x7F7F7F7Fu;
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, "
            "%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(
                tmem + (uint32_t(32 * warp) << 16) + kT3SfCol),
            "r"(one)
            : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
#ifdef TC3_PROFILE
    if (prof && threadIdx.x == 0) g_tc3_prof[1] = clock64();
#endif

    if (warp == kT3Load) {
        if (lane == 0) {
            // rows past n: the bulk copy moves an even number of rows (16-byte
            // granule); an odd last row is stored by this thread before the arrive
            const int nb = nvalid & ~1;
            int s = 0;
            uint32_t ph = 0;
            for (size_t kb = 0; kb < KB; ++kb) {
                if (kb >= size_t(kT3Raw)) mbar_wait1(&rempty[s], ph ^ 1);
                unsigned char* r = raw + size_t(s) * kT3RawBytes;
                if (nvalid & 1)
                    reinterpret_cast<uint64_t*>(r)[kT3Cols + nb] = A[kb * sa + i0 + nb];
                mbar_expect(&rfull[s], uint32_t(kT3Cols + nb) * 8);
                bulk_g2s(r, BT + kb * sbt + c0, kT3Cols * 8, &rfull[s]);
                if (nb) bulk_g2s(r + kT3Cols * 8, A + kb * sa + i0, uint32_t(nb) * 8, &rfull[s]);
                if (++s == kT3Raw) { s = 0; ph ^= 1; }
            }
        }
        __syncwarp();
    } else if (warp == kT3Mma) {
        if (lane == 0) {
            const uint32_t tsf = tmem + kT3SfCol;
            int s = 0;
            uint32_t ph = 0;
            for (size_t kb = 0; kb < KB; kb += kT3Kps) {
                mbar_wait1(&full[s], ph);
                asm volatile("tcgen05.fence::after_thread_sync;");
#ifdef TC3_PROFILE
                if (prof && kb == 0) g_tc3_prof[2] = clock64();
#endif
#pragma unroll
                for (int j = 0; j < kT3Kps; ++j) {
                    if (kb + j >= KB) break;
                    const uint32_t ta = sm_u32(smem + size_t(s) * kT3Stage + (j >> 1) * kT3Slot) + (j & 1) * 32;
                    const uint32_t tb = ta + kT3ABytes;
                    const uint32_t a0 = kb + j > 0 ? 1u : 0u;
                    if (MODE != 2) {
                        mma_f4(tmem, umma_desc(ta), umma_desc(tb), kIdescF4, a0, tsf);
                        mma_f4(tmem + kT3Rows, umma_desc(ta + 128 * 64), umma_desc(tb), kIdescF4, a0, tsf);
                    }
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 sm_u32(&empty[s]))
                             : "memory");
                if (++s == kT3Stages) { s = 0; ph ^= 1; }
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             sm_u32(done))
                         : "memory");
#ifdef TC3_PROFILE
            if (prof) g_tc3_prof[3] = clock64();
#endif
        }
        __syncwarp();
    } else {
        // thread t < 256: B^T row t; 256 <= t < 496: A^T row t - 256 (zero past n)
        const bool active = tid < kT3RawWords;
        const int region = tid < kT3Cols ? 0 : kT3ABytes;
        const int r = tid < kT3Cols ? tid : tid - kT3Cols;
        const bool live = active && (tid < kT3Cols || r < nvalid);
        int s = 0, rs = 0;
        uint32_t ph = 0, rph = 0;
        for (size_t kb = 0, st = 0; kb < KB; kb += kT3Kps, ++st) {
            if (st >= size_t(kT3Stages)) mbar_wait1(&empty[s], ph ^ 1);
#pragma unroll
            for (int j = 0; j < kT3Kps; ++j) {
                if (kb + j >= KB) break;
                mbar_wait1(&rfull[rs], rph);
                uint64_t x = 0;
                if (live) ld_shared_u64(x, raw + size_t(rs) * kT3RawBytes + size_t(tid) * 8);
                if (active) {
                    unsigned char* tile = smem + size_t(s) * kT3Stage + (j >> 1) * kT3Slot + region;
                    if (MODE == 1) {
                        if (x == 0x123456789ull) tile[r] = 1;
                    } else {
                        store_row_f4(tile, r, j & 1, x);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive1(&rempty[rs]);
                if (++rs == kT3Raw) { rs = 0; rph ^= 1; }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive1(&full[s]);
            if (++s == kT3Stages) { s = 0; ph ^= 1; }
        }
        // epilogue: lane quarter lq = w & 3; 16-column chunks c = (w >> 2) + 4i of the
        // 2 x 15 chunks; a ballot per row packs the 32 output columns of the quarter.
        // C ^= A*B: this tile's C words are loaded before the accumulator is ready
        // (the CTA owns them), so the read-modify-write is off the chunk chain
        constexpr int kChunks = 2 * (kT3Rows / 16), kPerWarp = (kChunks + 3) / 4;
        const int lq = warp & 3;
        uint32_t* dsts[kPerWarp];
        uint32_t pre[kPerWarp];
#pragma unroll
        for (int it = 0; it < kPerWarp; ++it) {
            const int ch = (warp >> 2) + 4 * it;
            const int accn = ch / (kT3Rows / 16), cc = ch % (kT3Rows / 16);
            const int row = 16 * cc + lane;
            const size_t col = c0 + size_t(accn) * 128 + size_t(lq) * 32;
            const bool mine_row = ch < kChunks && lane < 16 && row < nvalid;
            dsts[it] = mine_row ? reinterpret_cast<uint32_t*>(C + (col / 64) * sc + i0 + row) + ((col / 32) & 1)
                                : nullptr;
            pre[it] = (acc && mine_row) ? *dsts[it] : 0u;
        }
        mbar_wait1(done, 0);
        asm volatile("tcgen05.fence::after_thread_sync;");
#ifdef TC3_PROFILE
        if (prof && threadIdx.x == 0) g_tc3_prof[4] = clock64();
#endif
#pragma unroll
        for (int it = 0; it < kPerWarp; ++it) {
            const int ch = (warp >> 2) + 4 * it;
            if (ch >= kChunks) break;
            const int accn = ch / (kT3Rows / 16), cc = ch % (kT3Rows / 16);
            uint32_t v[16];
            const uint32_t taddr = tmem + (uint32_t(32 * lq) << 16) + uint32_t(kT3Rows * accn + 16 * cc);
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
                "%11, %12, %13, %14, %15}, [%16];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                  "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
                  "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (MODE == 3) {  // debug: raw accumulators of the first tile, [column][row] f32
                if (blockIdx.x == 0 && blockIdx.y == 0) {
                    uint32_t* dump = reinterpret_cast<uint32_t*>(C);
                    const int colx = accn * 128 + lq * 32 + lane;
#pragma unroll
                    for (int q = 0; q < 16; ++q) dump[colx * kT3Rows + 16 * cc + q] = v[q];
                }
                continue;
            }
            uint32_t mine = 0;
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const uint32_t par = __float_as_uint(__uint_as_float(v[q]) + 8388608.0f) & 1u;
                const uint32_t bits = __ballot_sync(0xffffffffu, par);
                if (lane == q) mine = bits;
            }
            if (dsts[it]) *dsts[it] = mine ^ pre[it];
        }
    }
#ifdef TC3_PROFILE
    if (prof && threadIdx.x == 0) g_tc3_prof[5] = clock64();
#endif
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
#ifdef TC3_PROFILE
    if (prof && threadIdx.x == 0) g_tc3_prof[6] = clock64();
#endif
}

#if F2GPU_EXPERIMENTAL  // evaluated and rejected variants: built only with F2GPU_EXPERIMENTAL=1 (build.py)
// ---------------------------------------------------------------------------
// k_gemm_tc5: the fp4 leaf as a PERSISTENT kernel.  k_gemm_tc3 runs one 256x240
// tile per CTA and pays ~7 us per tile of setup, load latency and epilogue (a
// k-scan on 1480 tiles: 7.3 us per wave at k = 64, +3.5 us per 1024 bits), which
// is most of the time of the short-k products in the TRSM recursion.  Here one
// CTA per SM loops over the tiles: TMEM is allocated and the scale-factor
// columns written once, the raw and stage rings run on across tiles (the load
// warp prefetches the next tile's words during the epilogue), and the MMA warp
// waits on an accumulator-empty barrier that the epilogue warps arrive on once
// they have read the previous tile's accumulators out of TMEM.
// Tile t of the launch's linear tile space: z = t / (GX*GY) (the batched
// problem), by = row tile, bx = column tile; tiles outside a problem skipped.
// ---------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(kT3Threads, 1)
    k_gemm_tc5(TcGemmArgs one, const TcGemmArgs* __restrict__ probs, uint32_t GX, uint32_t GY, uint32_t NT) {
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char* raw = smem + size_t(kT3Stages) * kT3Stage;
    uint64_t* full = reinterpret_cast<uint64_t*>(raw + size_t(kT3Raw) * kT3RawBytes);
    uint64_t* empty = full + kT3Stages;
    uint64_t* rfull = empty + kT3Stages;
    uint64_t* rempty = rfull + kT3Raw;
    uint64_t* done = rempty + kT3Raw;
    uint64_t* acc_empty = done + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    auto tile_of = [&](uint32_t t, TcGemmArgs& P, size_t& c0, size_t& i0) -> bool {
        const uint32_t per = GX * GY;
        const uint32_t z = t / per, rem = t - z * per, by = rem / GX, bx = rem - by * GX;
        P = probs ? probs[z] : one;
        c0 = size_t(bx) * kT3Cols;
        i0 = size_t(by) * kT3Rows;
        return c0 < P.m && i0 < P.n;
    };

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         sm_u32(tmem_slot)),
                     "r"(512u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int s = 0; s < kT3Stages; ++s) {
            mbar_init_n(&full[s], kT3Exp / 32);
            mbar_init_n(&empty[s], 1);
        }
        for (int s = 0; s < kT3Raw; ++s) {
            mbar_init_n(&rfull[s], 1);
            mbar_init_n(&rempty[s], kT3Exp / 32);
        }
        mbar_init_n(done, 1);
        mbar_init_n(acc_empty, kT3Exp / 32);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;
    if (warp < 4) {  // scale factors: every byte of columns 480..511 = E8M0 1.0
        const uint32_t onev = 0x7F7F7F7Fu;
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, "
            "%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(
                tmem + (uint32_t(32 * warp) << 16) + kT3SfCol),
            "r"(onev)
            : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");

    if (warp == kT3Load) {
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            size_t issued = 0;
            for (uint32_t t = blockIdx.x; t < NT; t += gridDim.x) {
                TcGemmArgs P;
                size_t c0, i0;
                if (!tile_of(t, P, c0, i0)) continue;
                const int nvalid = int(min(size_t(kT3Rows), P.n - i0));
                const size_t KB = (P.k + 63) / 64;
                // rows past n: the bulk copy moves an even number of rows (16-byte
                // granule); an odd last row is stored by this thread before the arrive
                const int nb = nvalid & ~1;
                for (size_t kb = 0; kb < KB; ++kb, ++issued) {
                    if (issued >= size_t(kT3Raw)) mbar_wait1(&rempty[s], ph ^ 1);
                    unsigned char* r = raw + size_t(s) * kT3RawBytes;
                    if (nvalid & 1)
                        reinterpret_cast<uint64_t*>(r)[kT3Cols + nb] = P.A[kb * P.sa + i0 + nb];
                    mbar_expect(&rfull[s], uint32_t(kT3Cols + nb) * 8);
                    bulk_g2s(r, P.BT + kb * P.sbt + c0, kT3Cols * 8, &rfull[s]);
                    if (nb) bulk_g2s(r + kT3Cols * 8, P.A + kb * P.sa + i0, uint32_t(nb) * 8, &rfull[s]);
                    if (++s == kT3Raw) { s = 0; ph ^= 1; }
                }
            }
        }
        __syncwarp();
    } else if (warp == kT3Mma) {
        if (lane == 0) {
            const uint32_t tsf = tmem + kT3SfCol;
            int s = 0;
            uint32_t ph = 0;
            uint32_t it = 0;
            for (uint32_t t = blockIdx.x; t < NT; t += gridDim.x) {
                TcGemmArgs P;
                size_t c0, i0;
                if (!tile_of(t, P, c0, i0)) continue;
                const size_t KB = (P.k + 63) / 64;
                if (it > 0) {  // the epilogue has read the previous tile's accumulators
                    mbar_wait1(acc_empty, (it - 1) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                }
                for (size_t kb = 0; kb < KB; kb += kT3Kps) {
                    mbar_wait1(&full[s], ph);
                    asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
                    for (int j = 0; j < kT3Kps; ++j) {
                        if (kb + j >= KB) break;
                        const uint32_t ta =
                            sm_u32(smem + size_t(s) * kT3Stage + (j >> 1) * kT3Slot) + (j & 1) * 32;
                        const uint32_t tb = ta + kT3ABytes;
                        const uint32_t a0 = kb + j > 0 ? 1u : 0u;
                        if (MODE != 2) {
                            mma_f4(tmem, umma_desc(ta), umma_desc(tb), kIdescF4, a0, tsf);
                            mma_f4(tmem + kT3Rows, umma_desc(ta + 128 * 64), umma_desc(tb), kIdescF4, a0, tsf);
                        }
                    }
                    asm volatile(
                        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                            sm_u32(&empty[s]))
                        : "memory");
                    if (++s == kT3Stages) { s = 0; ph ^= 1; }
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 sm_u32(done))
                             : "memory");
                ++it;
            }
        }
        __syncwarp();
    } else {
        // thread t < 256: B^T row t; 256 <= t < 496: A^T row t - 256 (zero past n)
        const bool active = tid < kT3RawWords;
        const int region = tid < kT3Cols ? 0 : kT3ABytes;
        const int r = tid < kT3Cols ? tid : tid - kT3Cols;
        int s = 0, rs = 0;
        uint32_t ph = 0, rph = 0;
        size_t staged = 0;
        uint32_t it = 0;
        for (uint32_t t = blockIdx.x; t < NT; t += gridDim.x) {
            TcGemmArgs P;
            size_t c0, i0;
            if (!tile_of(t, P, c0, i0)) continue;
            const int nvalid = int(min(size_t(kT3Rows), P.n - i0));
            const size_t KB = (P.k + 63) / 64;
            const bool live = active && (tid < kT3Cols || r < nvalid);
            for (size_t kb = 0; kb < KB; kb += kT3Kps, ++staged) {
                if (staged >= size_t(kT3Stages)) mbar_wait1(&empty[s], ph ^ 1);
#pragma unroll
                for (int j = 0; j < kT3Kps; ++j) {
                    if (kb + j >= KB) break;
                    mbar_wait1(&rfull[rs], rph);
                    uint64_t x = 0;
                    if (live) ld_shared_u64(x, raw + size_t(rs) * kT3RawBytes + size_t(tid) * 8);
                    if (active) {
                        unsigned char* tile = smem + size_t(s) * kT3Stage + (j >> 1) * kT3Slot + region;
                        if (MODE == 1) {
                            if (x == 0x123456789ull) tile[r] = 1;
                        } else {
                            store_row_f4(tile, r, j & 1, x);
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive1(&rempty[rs]);
                    if (++rs == kT3Raw) { rs = 0; rph ^= 1; }
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive1(&full[s]);
                if (++s == kT3Stages) { s = 0; ph ^= 1; }
            }
            // epilogue: lane quarter lq = w & 3; 16-column chunks c = (w >> 2) + 4i of the
            // 2 x 15 chunks; a ballot per row packs the 32 output columns of the quarter.
            // C ^= A*B: the tile's C words are loaded before the accumulator is ready
            const int lq = warp & 3;
            uint64_t* __restrict__ C = P.C;
            const size_t sc = P.sc;
            const int acc = P.acc;
            constexpr int kChunks = 2 * (kT3Rows / 16), kPerWarp = (kChunks + 3) / 4;
            uint32_t pre[kPerWarp];
#pragma unroll
            for (int q = 0; q < kPerWarp; ++q) {
                const int ch = (warp >> 2) + 4 * q;
                const int row = 16 * (ch % (kT3Rows / 16)) + lane;
                const size_t col = c0 + size_t(ch / (kT3Rows / 16)) * 128 + size_t(lq) * 32;
                pre[q] = (acc && ch < kChunks && lane < 16 && row < nvalid)
                             ? *(reinterpret_cast<const uint32_t*>(C + (col / 64) * sc + i0 + row) + ((col / 32) & 1))
                             : 0u;
            }
            mbar_wait1(done, it & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
            for (int q = 0; q < kPerWarp; ++q) {
                const int ch = (warp >> 2) + 4 * q;
                if (ch >= kChunks) break;
                const int accn = ch / (kT3Rows / 16), cc = ch % (kT3Rows / 16);
                uint32_t v[16];
                const uint32_t taddr = tmem + (uint32_t(32 * lq) << 16) + uint32_t(kT3Rows * accn + 16 * cc);
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
                    "%11, %12, %13, %14, %15}, [%16];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                      "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
                      "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (MODE == 3) {  // debug: raw accumulators of tile (0, 0), [column][row] f32
                    if (c0 == 0 && i0 == 0) {
                        uint32_t* dump = reinterpret_cast<uint32_t*>(C);
                        const int colx = accn * 128 + lq * 32 + lane;
#pragma unroll
                        for (int q = 0; q < 16; ++q) dump[colx * kT3Rows + 16 * cc + q] = v[q];
                    }
                    continue;
                }
                uint32_t mine = 0;
#pragma unroll
                for (int t = 0; t < 16; ++t) {
                    const uint32_t par = __float_as_uint(__uint_as_float(v[t]) + 8388608.0f) & 1u;
                    const uint32_t bits = __ballot_sync(0xffffffffu, par);
                    if (lane == t) mine = bits;
                }
                const int row = 16 * cc + lane;
                const size_t col = c0 + size_t(accn) * 128 + size_t(lq) * 32;
                if (lane < 16 && row < nvalid) {
                    uint32_t* dst = reinterpret_cast<uint32_t*>(C + (col / 64) * sc + i0 + row) + ((col / 32) & 1);
                    *dst = mine ^ pre[q];
                }
            }
            // accumulators read: the MMA warp may overwrite them with the next tile
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) mbar_arrive1(acc_empty);
            ++it;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
}

// ---------------------------------------------------------------------------
// k_gemm_tc6: persistent fp4 leaf with DOUBLE-BUFFERED accumulators, for short-k
// products.  A 256x240 tile needs all 480 TMEM columns, so the next tile's MMAs
// wait for the epilogue (~6.7k cycles of TMEM reads + ballots per tile, ~40% of a
// k = 1024 tile, tools/micro/tc3_prof.cu).  Here a tile is 128 output columns
// (M = 128, one MMA per k-block) x 240 rows: two accumulators fit (columns 0 and
// 240), four dedicated epilogue warps (one per TMEM lane quarter) drain tile t
// while the MMA warp fills the other buffer with tile t+1.  Per MAC it moves
// ~22% more shared memory than k_gemm_tc3 (the 240 B-side rows are expanded per
// 128 columns instead of per 256), so it is used only for short k.
// Warps 0-11 expand (thread t < 128: B^T row t; 128 <= t < 368: A row t - 128),
// 12-19 epilogue (two warps per TMEM lane quarter, alternate 16-column chunks,
// two TMEM loads in flight), 20 MMA, 21 load.
// ---------------------------------------------------------------------------
constexpr int kT6Cols = 128;                 // output columns per tile (M)
constexpr int kT6Rows = kT3Rows;             // output rows per tile (N = 240)
constexpr int kT6Exp = 384;                  // expansion threads (warps 0-11)
constexpr int kT6Epi = 12;                   // first epilogue warp (12-19: two per TMEM lane quarter)
constexpr int kT6EpiWarps = 8;
constexpr int kT6Mma = 20;
constexpr int kT6Load = 21;
constexpr int kT6Threads = 22 * 32;
constexpr int kT6ABytes = kT6Cols * 64;      // B^T side of a slot: 2 k-blocks x 32 B per row
constexpr int kT6BBytes = kT6Rows * 64;      // A side
constexpr int kT6Slot = kT6ABytes + kT6BBytes;
constexpr int kT6Stage = kT3Slots * kT6Slot;  // 4 k-blocks per stage
constexpr int kT6Stages = 3;
constexpr int kT6RawWords = kT6Cols + kT6Rows;
constexpr int kT6RawBytes = kT6RawWords * 8;
constexpr int kT6Raw = 8;
constexpr size_t kT6Smem = size_t(kT6Stages) * kT6Stage + size_t(kT6Raw) * kT6RawBytes + 256;
static_assert(kT6ABytes % 512 == 0 && kT6BBytes % 512 == 0, "SWIZZLE_64B atoms");

template <int MODE>
__global__ void __launch_bounds__(kT6Threads, 1)
    k_gemm_tc6(TcGemmArgs one, const TcGemmArgs* __restrict__ probs, uint32_t GX, uint32_t GY, uint32_t NT) {
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char* raw = smem + size_t(kT6Stages) * kT6Stage;
    uint64_t* full = reinterpret_cast<uint64_t*>(raw + size_t(kT6Raw) * kT6RawBytes);
    uint64_t* empty = full + kT6Stages;
    uint64_t* rfull = empty + kT6Stages;
    uint64_t* rempty = rfull + kT6Raw;
    uint64_t* acc_full = rempty + kT6Raw;   // [2]
    uint64_t* acc_empty = acc_full + 2;     // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    auto tile_of = [&](uint32_t t, TcGemmArgs& P, size_t& c0, size_t& i0) -> bool {
        const uint32_t per = GX * GY;
        const uint32_t z = t / per, rem = t - z * per, by = rem / GX, bx = rem - by * GX;
        P = probs ? probs[z] : one;
        c0 = size_t(bx) * kT6Cols;
        i0 = size_t(by) * kT6Rows;
        return c0 < P.m && i0 < P.n;
    };

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         sm_u32(tmem_slot)),
                     "r"(512u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int s = 0; s < kT6Stages; ++s) {
            mbar_init_n(&full[s], kT6Exp / 32);
            mbar_init_n(&empty[s], 1);
        }
        for (int s = 0; s < kT6Raw; ++s) {
            mbar_init_n(&rfull[s], 1);
            mbar_init_n(&rempty[s], kT6Exp / 32);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init_n(&acc_full[b], 1);
            mbar_init_n(&acc_empty[b], kT6EpiWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;
    if (warp < 4) {  // scale factors: every byte of columns 480..511 = E8M0 1.0
        const uint32_t onev = 0x7F7F7F7Fu;
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, "
            "%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(
                tmem + (uint32_t(32 * warp) << 16) + kT3SfCol),
            "r"(onev)
            : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");

    if (warp == kT6Load) {
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            size_t issued = 0;
            for (uint32_t t = blockIdx.x; t < NT; t += gridDim.x) {
                TcGemmArgs P;
                size_t c0, i0;
                if (!tile_of(t, P, c0, i0)) continue;
                const int nvalid = int(min(size_t(kT6Rows), P.n - i0));
                const size_t KB = (P.k + 63) / 64;
                const int nb = nvalid & ~1;
                for (size_t kb = 0; kb < KB; ++kb, ++issued) {
                    if (issued >= size_t(kT6Raw)) mbar_wait1(&rempty[s], ph ^ 1);
                    unsigned char* r = raw + size_t(s) * kT6RawBytes;
                    if (nvalid & 1)
                        reinterpret_cast<uint64_t*>(r)[kT6Cols + nb] = P.A[kb * P.sa + i0 + nb];
                    mbar_expect(&rfull[s], uint32_t(kT6Cols + nb) * 8);
                    bulk_g2s(r, P.BT + kb * P.sbt + c0, kT6Cols * 8, &rfull[s]);
                    if (nb) bulk_g2s(r + kT6Cols * 8, P.A + kb * P.sa + i0, uint32_t(nb) * 8, &rfull[s]);
                    if (++s == kT6Raw) { s = 0; ph ^= 1; }
                }
            }
        }
        __syncwarp();
    } else if (warp == kT6Mma) {
        if (lane == 0) {
            const uint32_t tsf = tmem + kT3SfCol;
            int s = 0;
            uint32_t ph = 0;
            uint32_t it = 0;
            for (uint32_t t = blockIdx.x; t < NT; t += gridDim.x) {
                TcGemmArgs P;
                size_t c0, i0;
                if (!tile_of(t, P, c0, i0)) continue;
                const size_t KB = (P.k + 63) / 64;
                const uint32_t b = it & 1;
                if (it >= 2) {  // the epilogue has drained this buffer's previous tile
                    mbar_wait1(&acc_empty[b], ((it >> 1) - 1) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                }
                const uint32_t tacc = tmem + b * uint32_t(kT6Rows);
                for (size_t kb = 0; kb < KB; kb += kT3Kps) {
                    mbar_wait1(&full[s], ph);
                    asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
                    for (int j = 0; j < kT3Kps; ++j) {
                        if (kb + j >= KB) break;
                        const uint32_t ta =
                            sm_u32(smem + size_t(s) * kT6Stage + (j >> 1) * kT6Slot) + (j & 1) * 32;
                        const uint32_t tb = ta + kT6ABytes;
                        const uint32_t a0 = kb + j > 0 ? 1u : 0u;
                        if (MODE != 2) mma_f4(tacc, umma_desc(ta), umma_desc(tb), kIdescF4, a0, tsf);
                    }
                    asm volatile(
                        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                            sm_u32(&empty[s]))
                        : "memory");
                    if (++s == kT6Stages) { s = 0; ph ^= 1; }
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 sm_u32(&acc_full[b]))
                             : "memory");
                ++it;
            }
        }
        __syncwarp();
    } else if (warp >= kT6Epi) {
        // epilogue: this warp's TMEM lane quarter lq = 32 output columns; of the 15
        // chunks of 16 accumulator columns (240 output rows) it takes every other
        // one, two loads in flight; a ballot per row
        const int lq = warp & 3, half = (warp - kT6Epi) >> 2;
        uint32_t it = 0;
        for (uint32_t t = blockIdx.x; t < NT; t += gridDim.x) {
            TcGemmArgs P;
            size_t c0, i0;
            if (!tile_of(t, P, c0, i0)) continue;
            const int nvalid = int(min(size_t(kT6Rows), P.n - i0));
            const uint32_t b = it & 1;
            mbar_wait1(&acc_full[b], (it >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            uint64_t* __restrict__ C = P.C;
            const size_t sc = P.sc;
            const int acc = P.acc;
            const size_t col = c0 + size_t(lq) * 32;
            const uint32_t tq = tmem + (uint32_t(32 * lq) << 16) + b * uint32_t(kT6Rows);
            auto emit = [&](const uint32_t (&v)[16], int cc) {
                uint32_t mine = 0;
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    const uint32_t par = __float_as_uint(__uint_as_float(v[q]) + 8388608.0f) & 1u;
                    const uint32_t bits = __ballot_sync(0xffffffffu, par);
                    if (lane == q) mine = bits;
                }
                const int row = 16 * cc + lane;
                if (lane < 16 && row < nvalid) {
                    uint32_t* dst = reinterpret_cast<uint32_t*>(C + (col / 64) * sc + i0 + row) + ((col / 32) & 1);
                    if (acc) mine ^= *dst;
                    *dst = mine;
                }
            };
#pragma unroll 1
            for (int cc = half; cc < kT6Rows / 16; cc += 4) {  // chunks cc and cc + 2
                const bool two = cc + 2 < kT6Rows / 16;
                uint32_t v[16], w[16];
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
                    "%11, %12, %13, %14, %15}, [%16];"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                      "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
                      "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                    : "r"(tq + uint32_t(16 * cc)));
                if (two)
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
                        "%11, %12, %13, %14, %15}, [%16];"
                        : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
                          "=r"(w[7]), "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]),
                          "=r"(w[13]), "=r"(w[14]), "=r"(w[15])
                        : "r"(tq + uint32_t(16 * (cc + 2))));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (MODE == 3) continue;
                emit(v, cc);
                if (two) emit(w, cc + 2);
            }
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) mbar_arrive1(&acc_empty[b]);
            ++it;
        }
    } else {
        const bool active = tid < kT6RawWords;
        const int region = tid < kT6Cols ? 0 : kT6ABytes;
        const int r = tid < kT6Cols ? tid : tid - kT6Cols;
        int s = 0, rs = 0;
        uint32_t ph = 0, rph = 0;
        size_t staged = 0;
        for (uint32_t t = blockIdx.x; t < NT; t += gridDim.x) {
            TcGemmArgs P;
            size_t c0, i0;
            if (!tile_of(t, P, c0, i0)) continue;
            const int nvalid = int(min(size_t(kT6Rows), P.n - i0));
            const size_t KB = (P.k + 63) / 64;
            const bool live = active && (tid < kT6Cols || r < nvalid);
            for (size_t kb = 0; kb < KB; kb += kT3Kps, ++staged) {
                if (staged >= size_t(kT6Stages)) mbar_wait1(&empty[s], ph ^ 1);
#pragma unroll
                for (int j = 0; j < kT3Kps; ++j) {
                    if (kb + j >= KB) break;
                    mbar_wait1(&rfull[rs], rph);
                    uint64_t x = 0;
                    if (live) ld_shared_u64(x, raw + size_t(rs) * kT6RawBytes + size_t(tid) * 8);
                    if (active) {
                        unsigned char* tile = smem + size_t(s) * kT6Stage + (j >> 1) * kT6Slot + region;
                        store_row_f4(tile, r, j & 1, x);
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive1(&rempty[rs]);
                    if (++rs == kT6Raw) { rs = 0; rph ^= 1; }
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive1(&full[s]);
                if (++s == kT6Stages) { s = 0; ph ^= 1; }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
}

bool gemm_tc_ok(size_t n, size_t k, size_t m) {
    return n > 0 && k > 0 && m > 0 && n % kTcN == 0 && m % kTcM == 0 && k % 64 == 0;
}
bool gemm_tc2_ok(size_t n, size_t k, size_t m) {
    return n > 0 && k > 0 && m > 0 && n % kT2Rows == 0 && m % kT2Cols == 0 && k % 64 == 0;
}

// C (n x m) (^)= A (n x k) * B (k x m) given BT = B^T (m x k, stride sbt)
cudaError_t launch_gemm_tc2(const uint64_t* A, size_t sa, const uint64_t* BT, size_t sbt, uint64_t* C,
                            size_t sc, size_t n, size_t k, size_t m, bool acc, cudaStream_t s) {
    static bool attr = false;
    static int mode = 0;
    if (!attr) {
        for (auto fn : {k_gemm_tc2<0>, k_gemm_tc2<1>, k_gemm_tc2<2>, k_gemm_tc2<3>, k_gemm_tc2<4>}) {
            cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 int(kT2Smem));
            if (e != cudaSuccess) return e;
        }
        mode = int(options().tc_mode);
        attr = true;
    }
    if (!gemm_tc2_ok(n, k, m) || (sbt % 2) || (sa % 2) ||
        (reinterpret_cast<uintptr_t>(A) % 16) || (reinterpret_cast<uintptr_t>(BT) % 16))
        return cudaErrorInvalidValue;
    dim3 grid(unsigned(m / kT2Cols), unsigned(n / kT2Rows));
    auto fn = mode == 1 ? k_gemm_tc2<1> : mode == 2 ? k_gemm_tc2<2> : mode == 3 ? k_gemm_tc2<3>
            : mode == 4 ? k_gemm_tc2<4> : k_gemm_tc2<0>;
    fn<<<grid, kT2Threads, kT2Smem, s>>>(A, sa, BT, sbt, C, sc, k, acc ? 1 : 0);
    return cudaGetLastError();
}

#endif
bool gemm_tc3_ok(size_t n, size_t k, size_t m) { return n > 0 && k > 0 && m > 0 && m % kT3Cols == 0; }

#if F2GPU_EXPERIMENTAL  // evaluated and rejected variants: built only with F2GPU_EXPERIMENTAL=1 (build.py)
// ---- v4: the fp4 leaf on CTA pairs (cta_group::2) ----
// A cluster of 2 CTAs computes a 512-column x 240-row tile with M = 256 MMAs
// issued by the leader: for each of the two accumulators the M = 256 output
// columns are split 128/128 over the pair (each CTA expands its own B^T rows) and
// the N = 240 output rows are split 120/120 (each CTA expands half of the A^T
// rows; the MMA reads the other half from the peer's shared memory).  Per SM and
// k-block that is 376 expanded rows and 15.5 KB of operand reads instead of 496
// rows and 23 KB -- the single-CTA leaf is shared-memory-bandwidth-bound (LSU +
// tensor-core wavefronts ~95%, profiles/r1_tc3_summary.txt).  Each CTA's TMEM
// holds its 128 M-rows x 240 columns per accumulator; the epilogue is unchanged.
constexpr int kT4Exp = 384;                 // expansion threads (warps 0-11)
constexpr int kT4Mma = kT4Exp / 32;         // warp 12 (leader CTA issues)
constexpr int kT4Load = kT4Mma + 1;         // warp 13
constexpr int kT4Threads = kT4Exp + 64;
constexpr int kT4Cols = 512;                // output columns per pair (2 accumulators x M = 256)
constexpr int kT4ARows = 256;               // B^T rows expanded per CTA (2 x 128)
constexpr int kT4Rows = 240;                // output rows per pair (N)
constexpr int kT4BRows = kT4Rows / 2;       // A^T rows expanded per CTA
constexpr int kT4ABytes = kT4ARows * 64;    // per 2-k-block slot
constexpr int kT4BBytes = kT4BRows * 64;
constexpr int kT4Slot = 24 * 1024;          // A (16 KB) + B (7.5 KB), padded to 1 KB
constexpr int kT4Slots = 2;                 // 4 k-blocks per stage
constexpr int kT4Kps = 2 * kT4Slots;
constexpr int kT4Stage = kT4Slots * kT4Slot;
constexpr int kT4Stages = 4;
constexpr int kT4RawWords = kT4ARows + kT4BRows;
constexpr int kT4RawBytes = 3072;           // 376 words, padded
constexpr int kT4Raw = 4;
constexpr uint32_t kT4SfCol = 480;
constexpr size_t kT4Smem = size_t(kT4Stages) * kT4Stage + size_t(kT4Raw) * kT4RawBytes + 512;
constexpr uint32_t kIdescF4Pair = idesc_f4(256, kT4Rows);

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kT4Threads, 1)
    k_gemm_tc4(TcGemmArgs one, const TcGemmArgs* __restrict__ probs) {
    const TcGemmArgs P = probs ? probs[blockIdx.z] : one;
    const uint32_t rank = cluster_rank();
    const size_t pc0 = size_t(blockIdx.x >> 1) * kT4Cols;   // pair's first output column
    const size_t i0 = size_t(blockIdx.y) * kT4Rows;
    if (pc0 >= P.m || i0 >= P.n) return;  // uniform over the pair
    const uint64_t* __restrict__ A = P.A;
    const uint64_t* __restrict__ BT = P.BT;
    uint64_t* __restrict__ C = P.C;
    const size_t sa = P.sa, n = P.n, sbt = P.sbt, sc = P.sc, k = P.k;
    const int acc = P.acc;
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char* raw = smem + size_t(kT4Stages) * kT4Stage;
    uint64_t* full = reinterpret_cast<uint64_t*>(raw + size_t(kT4Raw) * kT4RawBytes);
    uint64_t* empty = full + kT4Stages;
    uint64_t* rfull = empty + kT4Stages;
    uint64_t* rempty = rfull + kT4Raw;
    uint64_t* done = rempty + kT4Raw;
    uint64_t* pfull = done + 1;  // leader: the peer's stage s is expanded (forwarded)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pfull + kT4Stages);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // this CTA's A^T rows: i0 + 120*rank .. (zero past n)
    const size_t bi0 = i0 + size_t(kT4BRows) * rank;
    const int bvalid = bi0 >= n ? 0 : int(min(size_t(kT4BRows), n - bi0));
    const int nvalid = int(min(size_t(kT4Rows), n - i0));  // output rows of the pair tile
    const size_t KB = (k + 63) / 64;

    if (tid == 0) {
        for (int s = 0; s < kT4Stages; ++s) {
            mbar_init_n(&full[s], kT4Exp / 32);  // this CTA's expansion warps
            mbar_init_n(&empty[s], 1);
            mbar_init_n(&pfull[s], 1);
        }
        for (int s = 0; s < kT4Raw; ++s) {
            mbar_init_n(&rfull[s], 1);
            mbar_init_n(&rempty[s], kT4Exp / 32);
        }
        mbar_init_n(done, 1);
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
    if (warp < 4) {  // scale factors: every byte of columns 480..511 = E8M0 1.0
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, "
            "%1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1, %1};" ::"r"(
                tmem + (uint32_t(32 * warp) << 16) + kT4SfCol),
            "r"(0x7F7F7F7Fu)
            : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync_all();  // both CTAs: barriers initialised, TMEM allocated, scales set
    asm volatile("tcgen05.fence::after_thread_sync;");

    if (warp == kT4Load) {
        if (lane == 0) {
            const int nb = bvalid & ~1;
            const size_t ca = pc0 + size_t(128) * rank, cb = ca + 256;  // B^T rows of acc 0 / acc 1
            int s = 0;
            uint32_t ph = 0;
            for (size_t kb = 0; kb < KB; ++kb) {
                if (kb >= size_t(kT4Raw)) mbar_wait1(&rempty[s], ph ^ 1);
                uint64_t* r = reinterpret_cast<uint64_t*>(raw + size_t(s) * kT4RawBytes);
                if (bvalid & 1) r[kT4ARows + nb] = A[kb * sa + bi0 + nb];
                mbar_expect(&rfull[s], uint32_t(kT4ARows + nb) * 8);
                bulk_g2s(r, BT + kb * sbt + ca, 128 * 8, &rfull[s]);
                bulk_g2s(r + 128, BT + kb * sbt + cb, 128 * 8, &rfull[s]);
                if (nb) bulk_g2s(r + kT4ARows, A + kb * sa + bi0, uint32_t(nb) * 8, &rfull[s]);
                if (++s == kT4Raw) { s = 0; ph ^= 1; }
            }
        }
        __syncwarp();
    } else if (warp == kT4Mma) {
        if (lane == 0 && rank == 1) {
            // peer: forward each locally completed stage to the leader with one
            // cluster-scope release (the expansion warps only arrive CTA-locally)
            const uint32_t pfull_leader = mapa_shared(pfull, 0);
            int s = 0;
            uint32_t ph = 0;
            for (size_t kb = 0; kb < KB; kb += kT4Kps) {
                mbar_wait1(&full[s], ph);
                mbar_arrive_cluster(pfull_leader + uint32_t(s) * 8);
                if (++s == kT4Stages) { s = 0; ph ^= 1; }
            }
        }
        if (lane == 0 && rank == 0) {
            const uint32_t tsf = tmem + kT4SfCol;
            int s = 0;
            uint32_t ph = 0;
            for (size_t kb = 0; kb < KB; kb += kT4Kps) {
                mbar_wait1(&full[s], ph);
                mbar_wait1(&pfull[s], ph);
                asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
                for (int j = 0; j < kT4Kps; ++j) {
                    if (kb + j >= KB) break;
                    const uint32_t ta = sm_u32(smem + size_t(s) * kT4Stage + (j >> 1) * kT4Slot) + (j & 1) * 32;
                    const uint32_t tb = ta + kT4ABytes;
                    const uint32_t a0 = kb + j > 0 ? 1u : 0u;
                    mma_f4_pair(tmem, umma_desc(ta), umma_desc(tb), kIdescF4Pair, a0, tsf);
                    mma_f4_pair(tmem + kT4Rows, umma_desc(ta + 128 * 64), umma_desc(tb), kIdescF4Pair, a0, tsf);
                }
                tc_commit_pair(&empty[s], 0x3);
                if (++s == kT4Stages) { s = 0; ph ^= 1; }
            }
            tc_commit_pair(done, 0x3);
        }
        __syncwarp();
    } else {
        // thread t < 256: B^T row t (acc t / 128); 256 <= t < 376: A^T row t - 256
        const bool active = tid < kT4RawWords;
        const int region = tid < kT4ARows ? 0 : kT4ABytes;
        const int r = tid < kT4ARows ? tid : tid - kT4ARows;
        const bool live = active && (tid < kT4ARows || r < bvalid);
        int s = 0, rs = 0;
        uint32_t ph = 0, rph = 0;
        for (size_t kb = 0, st = 0; kb < KB; kb += kT4Kps, ++st) {
            if (st >= size_t(kT4Stages)) mbar_wait1(&empty[s], ph ^ 1);
#pragma unroll
            for (int j = 0; j < kT4Kps; ++j) {
                if (kb + j >= KB) break;
                mbar_wait1(&rfull[rs], rph);
                uint64_t x = 0;
                if (live) x = reinterpret_cast<const uint64_t*>(raw + size_t(rs) * kT4RawBytes)[tid];
                if (active) store_row_f4(smem + size_t(s) * kT4Stage + (j >> 1) * kT4Slot + region, r, j & 1, x);
                __syncwarp();  // x consumed by every lane before the raw slot is released
                if (lane == 0) mbar_arrive1(&rempty[rs]);
                if (++rs == kT4Raw) { rs = 0; rph ^= 1; }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive1(&full[s]);
            if (++s == kT4Stages) { s = 0; ph ^= 1; }
        }
        // epilogue: lane quarter lq = w & 3; 16-column chunks (acc, cc) = (w >> 2) + 3i
        // of 2 x 15; this CTA's output columns are pc0 + 256 acc + 128 rank + 32 lq + lane
        mbar_wait1(done, 0);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const int lq = warp & 3;
#pragma unroll 1
        for (int ch = warp >> 2; ch < 2 * (kT4Rows / 16); ch += kT4Exp / 128) {
            const int accn = ch / (kT4Rows / 16), cc = ch % (kT4Rows / 16);
            uint32_t v[16];
            const uint32_t taddr = tmem + (uint32_t(32 * lq) << 16) + uint32_t(kT4Rows * accn + 16 * cc);
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
                "%11, %12, %13, %14, %15}, [%16];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                  "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
                  "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            uint32_t mine = 0;
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const uint32_t par = __float_as_uint(__uint_as_float(v[q]) + 8388608.0f) & 1u;
                const uint32_t bits = __ballot_sync(0xffffffffu, par);
                if (lane == q) mine = bits;
            }
            const int row = 16 * cc + lane;
            const size_t col = pc0 + size_t(accn) * 256 + size_t(128) * rank + size_t(lq) * 32;
            if (lane < 16 && row < nvalid) {
                uint32_t* dst = reinterpret_cast<uint32_t*>(C + (col / 64) * sc + i0 + row) + ((col / 32) & 1);
                if (acc) mine ^= *dst;
                *dst = mine;
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync_all();  // the pair's MMAs and TMEM reads are finished
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
}

#endif
namespace {
#if F2GPU_EXPERIMENTAL  // evaluated and rejected variants: built only with F2GPU_EXPERIMENTAL=1 (build.py)
using Tc5Fn = void (*)(TcGemmArgs, const TcGemmArgs*, uint32_t, uint32_t, uint32_t);
Tc5Fn tc5_fn() {
    static Tc5Fn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        // opt-in: at 65536^2 it measured no faster (64.66-64.71 ms for k <= 1024..4096
        // vs 64.71 without), and its main loop is ~9% slower at large k
        if (options().tc_persist != 1) return nullptr;
        for (auto f : {k_gemm_tc5<0>, k_gemm_tc5<1>, k_gemm_tc5<2>, k_gemm_tc5<3>})
            if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kT3Smem)) != cudaSuccess)
                return nullptr;
        const int mode = int(options().tc_mode);
        fn = mode == 1 ? k_gemm_tc5<1> : mode == 2 ? k_gemm_tc5<2> : mode == 3 ? k_gemm_tc5<3> : k_gemm_tc5<0>;
    }
    return fn;
}
using Tc6Fn = void (*)(TcGemmArgs, const TcGemmArgs*, uint32_t, uint32_t, uint32_t);
// F2GPU_TC6_MAXK: short-k products on the double-buffered leaf (default 0 = off).
// Measured: its epilogue overlaps (3.4 us per 128-column tile at k = 64 vs 5.3 us
// per 256-column-equivalent for k_gemm_tc3), but its main loop is ~2x slower per
// MAC, so at k = 1024 it only ties and at k >= 2048 it loses; the decomposition
// showed no gain (64.08 vs 64.13 ms at k <= 1024).
size_t tc6_max_k() {
    static const size_t v = [] {
        return size_t(std::max<long long>(0, options().tc6_maxk));
    }();
    return v;
}
Tc6Fn tc6_fn() {
    static Tc6Fn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        if (tc6_max_k() == 0) return nullptr;
        for (auto f : {k_gemm_tc6<0>, k_gemm_tc6<2>})
            if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kT6Smem)) != cudaSuccess)
                return nullptr;
        fn = options().tc_mode == 2 ? k_gemm_tc6<2> : k_gemm_tc6<0>;
    }
    return fn;
}
size_t tc5_max_k() {  // F2GPU_TC5_MAXK (default 2048)
    static const size_t v = [] {
        return size_t(std::max<long long>(0, options().tc5_maxk));
    }();
    return v;
}
#endif
#if F2GPU_EXPERIMENTAL
int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}
#endif
using Tc3Fn = void (*)(TcGemmArgs, const TcGemmArgs*);
Tc3Fn tc3_fn() {
    static Tc3Fn fn = nullptr;
    if (!fn) {
        for (auto f : {k_gemm_tc3<0>, k_gemm_tc3<1>, k_gemm_tc3<2>, k_gemm_tc3<3>})
            if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kT3Smem)) != cudaSuccess)
                return nullptr;
        const int mode = int(options().tc_mode);
        fn = mode == 1 ? k_gemm_tc3<1> : mode == 2 ? k_gemm_tc3<2> : mode == 3 ? k_gemm_tc3<3> : k_gemm_tc3<0>;
    }
    return fn;
}
#if F2GPU_EXPERIMENTAL  // evaluated and rejected variants: built only with F2GPU_EXPERIMENTAL=1 (build.py)
// the pair kernel is opt-in (F2GPU_TC_PAIR=1) for products whose width is a
// multiple of 512.  Measured at 16384^3: 1.85 ms vs 1.86 ms for the single-CTA
// kernel -- it takes the shared-memory pipe from ~95% to ~64% busy, but the raw-
// operand feed (and with deeper raw rings, 1.99 ms) then limits it, so the
// simpler single-CTA kernel stays the default.
bool tc4_use(size_t m) {
    static const int on = [] {
        if (options().tc_pair != 1) return 0;
        return cudaFuncSetAttribute(k_gemm_tc4, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kT4Smem)) ==
                       cudaSuccess
                   ? 1
                   : 0;
    }();
    return on && m % kT4Cols == 0;
}
#endif
bool tc3_args_ok(const TcGemmArgs& p) {
    return gemm_tc3_ok(p.n, p.k, p.m) && p.sbt % 2 == 0 && p.sa % 2 == 0 &&
           reinterpret_cast<uintptr_t>(p.A) % 16 == 0 && reinterpret_cast<uintptr_t>(p.BT) % 16 == 0;
}
}  // namespace

// fp4 leaf: C (n x m) (^)= A (n x k) * B (k x m) given BT = B^T (m x k, stride sbt,
// bits past k zero); n and k arbitrary, m % 256 == 0
cudaError_t launch_gemm_tc3(const uint64_t* A, size_t sa, size_t n, const uint64_t* BT, size_t sbt,
                            uint64_t* C, size_t sc, size_t k, size_t m, bool acc, cudaStream_t s) {
    Tc3Fn fn = tc3_fn();
    if (!fn) return cudaErrorInvalidValue;
    const TcGemmArgs p{A, sa, n, BT, sbt, C, sc, k, m, acc ? 1 : 0};
    if (!tc3_args_ok(p)) return cudaErrorInvalidValue;
    if (gemm_tc7_enabled()) return launch_gemm_tc7(p, s);
#if F2GPU_EXPERIMENTAL
    if (tc4_use(m)) {
        dim3 grid4(unsigned(2 * (m / kT4Cols)), unsigned((n + kT4Rows - 1) / kT4Rows));
        k_gemm_tc4<<<grid4, kT4Threads, kT4Smem, s>>>(p, nullptr);
        return cudaGetLastError();
    }
    if (Tc6Fn f6 = tc6_fn(); f6 && k <= tc6_max_k()) {
        const uint32_t GX6 = uint32_t(m / kT6Cols), GY6 = uint32_t((n + kT6Rows - 1) / kT6Rows), NT = GX6 * GY6;
        f6<<<std::min<uint32_t>(NT, uint32_t(sm_count())), kT6Threads, kT6Smem, s>>>(p, nullptr, GX6, GY6, NT);
        return cudaGetLastError();
    }
    const uint32_t GX = uint32_t(m / kT3Cols), GY = uint32_t((n + kT3Rows - 1) / kT3Rows);
    // the persistent kernel hides the per-tile setup and load latency (~1.3 us of
    // ~7) but its main loop measured ~9% slower at large k: short-k products only
    if (Tc5Fn f5 = tc5_fn(); f5 && k <= tc5_max_k()) {
        const uint32_t NT = GX * GY;
        f5<<<std::min<uint32_t>(NT, uint32_t(sm_count())), kT3Threads, kT3Smem, s>>>(p, nullptr, GX, GY, NT);
        return cudaGetLastError();
    }
#else
    const uint32_t GX = uint32_t(m / kT3Cols), GY = uint32_t((n + kT3Rows - 1) / kT3Rows);
#endif
    dim3 grid(GX, GY);
    fn<<<grid, kT3Threads, kT3Smem, s>>>(p, nullptr);
    return cudaGetLastError();
}

// a batch of fp4-leaf problems (host copy h_probs, device copy d_probs), one launch
cudaError_t launch_gemm_tc3_batched(const TcGemmArgs* h_probs, const TcGemmArgs* d_probs, int nprob,
                                    cudaStream_t s) {
    Tc3Fn fn = tc3_fn();
    if (!fn || nprob <= 0 || nprob > 65535) return cudaErrorInvalidValue;
    size_t mx = 0, nx = 0;
    for (int i = 0; i < nprob; ++i) {
        if (!tc3_args_ok(h_probs[i])) return cudaErrorInvalidValue;
        mx = std::max(mx, h_probs[i].m);
        nx = std::max(nx, h_probs[i].n);
    }
    if (gemm_tc7_enabled()) return launch_gemm_tc7_batched(h_probs, d_probs, nprob, s);
    const uint32_t GX = uint32_t(mx / kT3Cols), GY = uint32_t((nx + kT3Rows - 1) / kT3Rows);
#if F2GPU_EXPERIMENTAL
    bool all4 = true;
    for (int i = 0; i < nprob; ++i) all4 = all4 && tc4_use(h_probs[i].m);
    if (all4) {
        dim3 grid4(unsigned(2 * (mx / kT4Cols)), unsigned((nx + kT4Rows - 1) / kT4Rows), unsigned(nprob));
        k_gemm_tc4<<<grid4, kT4Threads, kT4Smem, s>>>(TcGemmArgs{}, d_probs);
        return cudaGetLastError();
    }
    size_t kmax = 0;
    for (int i = 0; i < nprob; ++i) kmax = std::max(kmax, h_probs[i].k);
    if (Tc6Fn f6 = tc6_fn(); f6 && kmax <= tc6_max_k()) {
        const uint32_t GX6 = uint32_t(mx / kT6Cols), GY6 = uint32_t((nx + kT6Rows - 1) / kT6Rows);
        const uint32_t NT = GX6 * GY6 * uint32_t(nprob);
        f6<<<std::min<uint32_t>(NT, uint32_t(sm_count())), kT6Threads, kT6Smem, s>>>(TcGemmArgs{}, d_probs, GX6,
                                                                                       GY6, NT);
        return cudaGetLastError();
    }
    if (Tc5Fn f5 = tc5_fn(); f5 && kmax <= tc5_max_k()) {
        const uint32_t NT = GX * GY * uint32_t(nprob);
        f5<<<std::min<uint32_t>(NT, uint32_t(sm_count())), kT3Threads, kT3Smem, s>>>(TcGemmArgs{}, d_probs, GX, GY,
                                                                                       NT);
        return cudaGetLastError();
    }
#endif
    dim3 grid(GX, GY, unsigned(nprob));
    fn<<<grid, kT3Threads, kT3Smem, s>>>(TcGemmArgs{}, d_probs);
    return cudaGetLastError();
}

#if F2GPU_EXPERIMENTAL  // evaluated and rejected variants: built only with F2GPU_EXPERIMENTAL=1 (build.py)
cudaError_t launch_gemm_tc(const uint64_t* A, size_t sa, const uint64_t* B, size_t sb, uint64_t* C,
                           size_t sc, size_t n, size_t k, size_t m, bool acc, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_gemm_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(kTcSmem));
        if (e != cudaSuccess) return e;
        attr = true;
    }
    if (!gemm_tc_ok(n, k, m)) return cudaErrorInvalidValue;
    dim3 grid(unsigned(m / kTcM), unsigned(n / kTcN));
    k_gemm_tc<<<grid, kTcThreads, kTcSmem, s>>>(A, sa, B, sb, C, sc, n, k, m, acc ? 1 : 0);
    return cudaGetLastError();
}

#endif

}  // namespace f2
