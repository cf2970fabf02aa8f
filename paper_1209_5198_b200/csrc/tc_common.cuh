// tc_common.cuh -- shared tcgen05 / mbarrier / bulk-copy helpers of the
// tensor-core kernels (tc_leaf.cu, tc_update.cu).
#pragma once
#include <cstdint>

namespace f2 {

static __device__ __forceinline__ uint32_t sm_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// canonical K-major SWIZZLE_64B offset of (row r, 16-byte k-chunk c) in a tile:
// 8-row atoms of 64-byte rows (SBO = 512 B), chunk index XOR-ed with address
// bits [7,9) = (r >> 1) & 3 (Swizzle<2,4,3>).  Tiles start 1024-byte aligned.
static __device__ __forceinline__ uint32_t kmaj_off(int r, int c) {
    return uint32_t((r >> 3) * 512 + (r & 7) * 64 + ((c ^ ((r >> 1) & 3)) * 16));
}

// smem matrix descriptor for a SWIZZLE_64B K-major tile; a K step inside the
// 64-byte row advances the start address (32 B per int8 K=32 / fp4 K=64 step)
static __device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFF);  // start address
    d |= uint64_t(1) << 16;                // LBO (unused for swizzled K-major)
    d |= uint64_t(512 >> 4) << 32;         // SBO: next 8-row atom
    d |= uint64_t(1) << 46;                // version (Blackwell)
    d |= uint64_t(4) << 61;                // SWIZZLE_64B
    return d;
}
constexpr uint32_t kKHalf = 32u;

// instruction descriptor of kind::mxf4 (E2M1 x E2M1, E8M0 scales, K=64), M x N
__host__ __device__ constexpr uint32_t idesc_f4(int M, int N) {
    return (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (1u << 23) | (uint32_t(M >> 4) << 24);
}
static __device__ __forceinline__ void mma_f4(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                              uint32_t acc, uint32_t tsf) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%5], [%5], p;\n\t}\n" ::"r"(
            tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(tsf));
}
// separate A / B scale-factor TMEM addresses
static __device__ __forceinline__ void mma_f4_sf(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                                 uint32_t acc, uint32_t tsfa, uint32_t tsfb) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%5], [%6], p;\n\t}\n" ::"r"(
            tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(tsfa), "r"(tsfb));
}
// CTA-pair (cta_group::2) variants: issued by the leader CTA of a 2-CTA cluster;
// A (M = 256) is split by rows over the pair, B by N halves, each CTA's TMEM
// receives the D rows of its own M half
static __device__ __forceinline__ void mma_f4_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                                   uint32_t acc, uint32_t tsf) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%5], [%5], p;\n\t}\n" ::"r"(
            tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc), "r"(tsf));
}
// arrive on the barrier at the same shared offset in every CTA of mask
static __device__ __forceinline__ void tc_commit_pair(uint64_t* bar, uint16_t mask) {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     sm_u32(bar)),
                 "h"(mask)
                 : "memory");
}
static __device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// shared::cluster address of `p` (a shared::cta address in this CTA) in CTA `rank`
static __device__ __forceinline__ uint32_t mapa_shared(const void* p, uint32_t rank) {
    uint32_t a;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(sm_u32(p)), "r"(rank));
    return a;
}
static __device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
static __device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
static __device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sm_u32(bar))
                 : "memory");
}

// 64 bits -> 64 E2M1 nibbles (0x2 = 1.0 / 0x0), k-block j (32 bytes) of row r
// of a 64-byte-row K-major tile.  The k order inside the block is permuted the
// same way for both operands (nibble q of word t <- bit 4q + t).
static __device__ __forceinline__ void store_row_f4(unsigned char* tile, int r, int j, uint64_t w) {
    constexpr uint32_t M = 0x22222222u;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const uint32_t x = uint32_t(w >> (32 * h));
        uint4 v;
        v.x = (x << 1) & M;
        v.y = x & M;
        v.z = (x >> 1) & M;
        v.w = (x >> 2) & M;
        *reinterpret_cast<uint4*>(tile + kmaj_off(r, 2 * j + h)) = v;
    }
}

static __device__ __forceinline__ void mbar_init_n(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sm_u32(b)), "r"(n));
}
static __device__ __forceinline__ void mbar_wait1(uint64_t* b, uint32_t ph) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "L_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra L_%=;\n}" ::"r"(sm_u32(b)),
        "r"(ph)
        : "memory");
}
static __device__ __forceinline__ void mbar_arrive1(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sm_u32(b)) : "memory");
}
static __device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_u32(b)), "r"(bytes)
                 : "memory");
}
static __device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            sm_u32(dst)),
        "l"(src), "r"(bytes), "r"(sm_u32(bar))
        : "memory");
}
// global[dst] ^= smem[src] (bytes % 16 == 0), tracked by the bulk-group counter
static __device__ __forceinline__ void bulk_xor_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.xor.b64 [%0], [%1], %2;" ::"l"(dst),
                 "r"(sm_u32(src)), "r"(bytes)
                 : "memory");
}
static __device__ __forceinline__ void bulk_commit_group() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
static __device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
static __device__ __forceinline__ void bulk_wait() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

}  // namespace f2
