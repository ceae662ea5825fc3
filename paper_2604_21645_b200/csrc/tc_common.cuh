// tc_common.cuh -- tcgen05 / TMEM / bulk-copy helpers and the K-major
// no-swizzle UMMA operand layout shared by the tensor-core kernels that stream
// pre-split TF32 hi/lo operands (umma_big.cu).
#pragma once

#include "kernels.cuh"

namespace pqg {
namespace tc {

constexpr int kR = 128;             // rows per tile (MMA M)
constexpr int kN = 256;             // centroids per N block (MMA N)
#ifndef PQG_BIG_KC
#define PQG_BIG_KC 16
#endif
#ifndef PQG_BIG_STAGES
#define PQG_BIG_STAGES 4
#endif
// r2e: 16-element K chunks (48 KB stages) in a 4-deep ring instead of 32 (96
// KB) x 2: the producer keeps four bulk copies in flight, and the constant
// columns' chunk is 16 wide (d = 128: 9 chunks = 144 K instead of 160)
constexpr int kKC = PQG_BIG_KC;     // K elements per chunk
constexpr int kBigStages = PQG_BIG_STAGES;
constexpr uint32_t kSBO = (kKC / 4) * 128;  // 1024 B between 8-row groups
constexpr uint32_t kAChunk = kR * kKC * 4;   // 16 KB per half
constexpr uint32_t kBChunk = kN * kKC * 4;   // 32 KB per half
constexpr uint32_t kStage = 2 * kAChunk + 2 * kBChunk;  // 96 KB

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
           (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46);
}
__host__ __device__ constexpr uint32_t idesc_tf32(uint32_t M, uint32_t N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                 :: "r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bar_init(uint64_t* bar, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile("{\n\t.reg .pred done;\nW_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
                 "@!done bra W_%=;\n\t}\n" :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
          "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
          "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ float tf32_hi(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}
__device__ __forceinline__ uint32_t il_off(uint32_t row, uint32_t k) {  // within one K chunk
    return (row >> 3) * kSBO + (k >> 2) * 128u + (row & 7u) * 16u + (k & 3u) * 4u;
}

// E bound of the 3xTF32 screen (see umma.cu tc_error_bound): 2 ulps of the
// accumulator magnitude per MMA instruction plus split residuals, doubled.
__device__ __forceinline__ float big_error_bound(float S, uint32_t kchunks) {
    const float n_mma = float(3 * (kKC / 8) * kchunks);
    return 2.f * (2.f * n_mma + 8.f) * kU * S + 1e-30f;
}

}  // namespace tc
}  // namespace pqg
