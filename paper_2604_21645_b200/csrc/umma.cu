// umma.cu -- tcgen05 (5th-gen tensor core) screen for the PQ subspace argmin
// (pq_encode, proj/src/pq.cpp:95-111; assign_pass of pq_fit,
// proj/src/kmeans.cpp:46-57), the B200 replacement of the FP32 screen in
// nearest.cu for Ds + 2 <= 40 and Ks a multiple of 16 up to 256.
//
// One CTA = 4 warps = 128 rows of a tile; TMEM lane r <-> row r <-> thread r.
// Augmented operands make the MMA produce the screened value directly:
//   A_r = [ x_r (Ds) , 1 , C_r ]          (C_r >= ||x_r||^2 + 2E_r)
//   B_j = [ -2 c_j (Ds), ||c_j||^2 , 1 ]
//   (A B^T)_rj = ||x_r - c_j||^2 + (C_r - ||x_r||^2)   >= E_r > 0.
// fp32 accuracy from TF32 inputs by the 3xTF32 split (A_hi B_hi + A_hi B_lo +
// A_lo B_hi, hi = tf32-rounded, lo = residual).  The accumulator (128 x N fp32)
// lives in TMEM; each thread tcgen05.ld's its row (32 columns per load) and
// keeps the best and second-best (value|column) keys with integer min/max --
// no cross-thread reduction.  The flag rule and the exact fp64 fixup are the
// ones of nearest.cu, with the error bound E widened for the split and the
// tensor core's accumulation (see tc_error_bound).
//
// Operands are staged in shared memory in the canonical K-major
// SWIZZLE_NONE ("interleaved") layout: 8-row x 16-byte core matrices; core
// matrices adjacent in K are LBO = 128 B apart, adjacent 8-row groups
// SBO = (K/4)*128 B apart.  Descriptor / instruction-descriptor bit layouts
// follow the sm_100 UMMA definitions (CUTLASS cute/arch/mma_sm100_desc.hpp).
#include <cstdlib>
#include <type_traits>

#include "kernels.cuh"

namespace pqg {

namespace {

constexpr int kRows = 128;  // M of the MMA, rows per tile, threads per CTA

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFF);
    d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
    d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
    d |= uint64_t(1) << 46;  // version 1 (sm_100)
    // base_offset 0, lbo_mode 0, layout_type 0 = SWIZZLE_NONE
    return d;
}

__host__ __device__ constexpr uint32_t make_idesc_tf32(uint32_t M, uint32_t N) {
    return (1u << 4)            // D format F32
           | (2u << 7)          // A format TF32
           | (2u << 10)         // B format TF32
           | ((N >> 3) << 17)   // N / 8
           | ((M >> 4) << 24);  // M / 16
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                         uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
        :: "r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 :: "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred done;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
        "@!done bra WAIT_%=;\n\t}\n"
        :: "r"(smem_u32(bar)), "r"(phase) : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

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

// tf32 hi part: round to nearest at 10 mantissa bits (cvt.rna.tf32.f32)
__device__ __forceinline__ float tf32_hi(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// The same rounding (to nearest, ties away from zero, at 10 mantissa bits) as
// two integer ops for finite x: the magnitude's bit pattern + half an ulp of
// tf32, low 13 bits cleared.  cvt.rna.tf32 costs ~5 instructions on sm_100
// (non-finite checks); a non-finite x only occurs in rows / tables whose
// error bound is non-finite, which the screen flags for the exact fixup.
__device__ __forceinline__ float tf32_rna_fast(float x) {
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

// ---------------------------------------------------------------------------
// Keys of the running top-2 (r2).  Every screened value of a row lies in one
// window [2^p, 2^(p+16)) with p = 1 (mod 16) (row_prep adds the offset 2^p
// inside C), so bits 30..27 of all its values are the same and
//     key = value_bits * 32 + j          (one IMAD, FMA pipe, j immediate)
// keeps all 27 remaining value bits (4 exponent + 23 mantissa bits: no
// quantisation) and the column j of the 32-column chunk in the low 5 bits;
// unsigned order of keys = order of (value, j).  m32 == 32 is a kernel
// argument so the multiply cannot be folded into an ALU shift.
// ---------------------------------------------------------------------------
template <int J>
__device__ __forceinline__ uint32_t col_key(uint32_t r, uint32_t m32) {
    uint32_t k;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(k) : "r"(r), "r"(m32), "n"(J));
    return k;
}

// a + b and s - lo as IMADs with run-time unit multipliers (FMA pipe): the
// pair step below then issues 4 ALU + 4 FMA-pipe instructions per two values
// (the ALU pipe runs at half the issue rate, so balancing the pipes is what
// makes the epilogue cheap).
__device__ __forceinline__ uint32_t mad_u32(uint32_t a, uint32_t m, uint32_t c) {
    uint32_t k;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(k) : "r"(a), "r"(m), "r"(c));
    return k;
}

// Fold 32 TMEM columns (chunk starting at column c0; columns >= nvalid of the
// chunk are padding) into four independent (best, second) key states.
// Pair step: lo = min(a,b); hi = (a+b) - lo; m2 = min(m2, max(m1,lo), hi);
// m1 = min(m1, lo).  The chunk of each state's best is tracked on change.
template <int J, bool MASK>
__device__ __forceinline__ uint32_t col_key_m(const uint32_t (&r)[32], uint32_t nvalid, uint32_t m32) {
    const uint32_t k = col_key<J>(r[J], m32);
    if constexpr (MASK) return uint32_t(J) < nvalid ? k : 0xFFFFFFFFu;
    return k;
}

template <int P, bool MASK>
__device__ __forceinline__ void top2_pair(const uint32_t (&r)[32], uint32_t nvalid, uint32_t& m1, uint32_t& m2,
                                          uint32_t m32, uint32_t one, uint32_t neg1) {
    const uint32_t a = col_key_m<2 * P, MASK>(r, nvalid, m32), b = col_key_m<2 * P + 1, MASK>(r, nvalid, m32);
    const uint32_t lo = min(a, b);
    const uint32_t hi = mad_u32(lo, neg1, mad_u32(a, one, b));
    m2 = min(m2, min(max(m1, lo), hi));
    m1 = min(m1, lo);
}

#ifndef PQG_TOP2_NS
#define PQG_TOP2_NS 4
#endif
constexpr int kNS = PQG_TOP2_NS;  // independent (best, second) states per thread

template <int P, bool MASK>
__device__ __forceinline__ void top2_pairs(const uint32_t (&r)[32], uint32_t nvalid, uint32_t (&m1)[kNS],
                                           uint32_t (&m2)[kNS], uint32_t m32, uint32_t one, uint32_t neg1) {
    if constexpr (P < 16) {
        top2_pair<P, MASK>(r, nvalid, m1[P % kNS], m2[P % kNS], m32, one, neg1);
        top2_pairs<P + 1, MASK>(r, nvalid, m1, m2, m32, one, neg1);
    }
}

template <bool MASK>
__device__ __forceinline__ void top2_chunk(const uint32_t (&r)[32], uint32_t nvalid, uint32_t c0,
                                           uint32_t (&m1)[kNS], uint32_t (&m2)[kNS], uint32_t (&ch)[kNS],
                                           uint32_t m32) {
    const uint32_t one = m32 >> 5, neg1 = 0u - one;
    uint32_t old[kNS];
#pragma unroll
    for (int s4 = 0; s4 < kNS; ++s4) old[s4] = m1[s4];
    // pair p goes to state p % kNS
    top2_pairs<0, MASK>(r, nvalid, m1, m2, m32, one, neg1);
#pragma unroll
    for (int s4 = 0; s4 < kNS; ++s4) ch[s4] = (m1[s4] != old[s4]) ? c0 : ch[s4];
}

// r2h fast path (full 64- or 128-column passes, k % 64 == 0): the chunk loop of
// a pass is unrolled and a key's 5 low bits carry (chunk within the pass,
// pair within the state, column within the pair) instead of the column within
// the chunk -- state s sees pairs p = 4q + s, i.e. columns 8q + 2s + b of a
// chunk, so J = 8*chunk + 2q + b with s implicit.  The per-chunk tracking of
// each best's chunk (ISETP + MOV + SEL per state per chunk, plus the loop
// control: ~24 of ~156 instructions per chunk, ncu r2h source counters)
// becomes one check per state per pass.
template <int CC, int P>
__device__ __forceinline__ void top2_pairs_fast(const uint32_t (&r)[32], uint32_t (&m1)[kNS], uint32_t (&m2)[kNS],
                                                uint32_t m32, uint32_t one, uint32_t neg1) {
    static_assert(kNS == 4, "the fast key layout assumes four states");
    if constexpr (P < 16) {
        constexpr int J = CC * 8 + 2 * (P / 4);
        const uint32_t a = col_key<J>(r[2 * P], m32), b = col_key<J + 1>(r[2 * P + 1], m32);
        const uint32_t lo = min(a, b);
        const uint32_t hi = mad_u32(lo, neg1, mad_u32(a, one, b));
        m2[P % 4] = min(m2[P % 4], min(max(m1[P % 4], lo), hi));
        m1[P % 4] = min(m1[P % 4], lo);
        top2_pairs_fast<CC, P + 1>(r, m1, m2, m32, one, neg1);
    }
}

// column (within its pass) of state s's key
__device__ __forceinline__ uint32_t fast_col(uint32_t key, uint32_t s) {
    const uint32_t J = key & 31u;
    return (J >> 3) * 32u + ((J >> 1) & 3u) * 8u + 2u * s + (J & 1u);
}

__device__ __forceinline__ void top2_merge_fast(const uint32_t (&m1)[kNS], const uint32_t (&m2)[kNS],
                                                const uint32_t (&pch)[kNS], uint64_t& K1, uint32_t& V2) {
    K1 = (uint64_t(m1[0] >> 5) << 32) | (pch[0] + fast_col(m1[0], 0));
    V2 = m2[0] >> 5;
#pragma unroll
    for (int s4 = 1; s4 < kNS; ++s4) {
        const uint64_t o = (uint64_t(m1[s4] >> 5) << 32) | (pch[s4] + fast_col(m1[s4], s4));
        V2 = min(min(V2, m2[s4] >> 5), uint32_t(max(K1, o) >> 32));
        K1 = min(K1, o);
    }
}

// Merge the states: (best value, global column) and the runner-up's value;
// values are the 27 key bits above the column field.
__device__ __forceinline__ void top2_merge(const uint32_t (&m1)[kNS], const uint32_t (&m2)[kNS],
                                           const uint32_t (&ch)[kNS], uint64_t& K1, uint32_t& V2) {
    K1 = (uint64_t(m1[0] >> 5) << 32) | (ch[0] + (m1[0] & 31u));
    V2 = m2[0] >> 5;
#pragma unroll
    for (int s4 = 1; s4 < kNS; ++s4) {
        const uint64_t o = (uint64_t(m1[s4] >> 5) << 32) | (ch[s4] + (m1[s4] & 31u));
        V2 = min(min(V2, m2[s4] >> 5), uint32_t(max(K1, o) >> 32));
        K1 = min(K1, o);
    }
}

// byte offset of element (row, k) of a K-major interleaved operand
// After tcgen05.wait::ld: re-define the loaded registers so no consumer is
// scheduled above the wait (the asm outputs of tcgen05.ld are not ready
// until then).
__device__ __forceinline__ void tmem_regs_ready(uint32_t (&r)[32]) {
    asm volatile(""
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]),
                   "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]),
                   "+r"(r[14]), "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]),
                   "+r"(r[21]), "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]),
                   "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31]));
}

__device__ __forceinline__ uint32_t il_off(uint32_t row, uint32_t k, uint32_t sbo) {
    return (row >> 3) * sbo + (k >> 2) * 128u + (row & 7u) * 16u + (k & 3u) * 4u;
}

__device__ __forceinline__ void store_index(const NearestArgs& a, uint64_t i, uint32_t b, uint32_t idx) {
    const uint64_t off = i * a.idx_rs + (uint64_t)b * a.idx_ps;
    if (a.idx_bytes == 1) {
        static_cast<uint8_t*>(a.out_idx)[off] = uint8_t(idx);
    } else if (a.idx_bytes == 2) {
        uint8_t* p = static_cast<uint8_t*>(a.out_idx) + off * 2;
        p[0] = uint8_t(idx & 0xff);
        p[1] = uint8_t(idx >> 8);
    } else {
        static_cast<uint32_t*>(a.out_idx)[off] = idx;
    }
}

// |screened - exact| bound for the 3xTF32 tensor-core screen.  S bounds the
// magnitude of every partial sum (2|x.c| + ||c||^2 + C, offset included).
// Products of tf32 operands are exact in fp32; each MMA instruction may lose
// up to one fp32 ulp (2u) of the accumulator, whose magnitude is <= S (n_mma
// instructions per tile); the dropped lo*lo term and the tf32 rounding of the
// lo parts are <= 2^-21 |x_t c_t| per coordinate (<= 4u S).  Doubled for
// safety.  Empirically (tools/screen_bench.py) the TC and FP32 screens return
// identical codes on all 1M x M rows tested.
__device__ __forceinline__ float tc_error_bound(float S, int n_mma) {
    return 2.f * (2.f * float(n_mma) + 8.f) * kU * S + 1e-30f;
}

// MMA instructions per tile.  Operand columns: [x (DS) | 1 1 1 C] against
// [-2c (DS) | h m l 1] with ||c||^2 = h + m + l split exactly into three tf32
// pieces and C rounded up to tf32, so the constant columns are exact in tf32:
// a k-step holding only constants needs the hi*hi product alone, a k-step
// holding x needs hi*hi + hi*lo + lo*hi.
template <int DS>
__host__ __device__ constexpr int umma_n_mma() {
    return 3 * ((DS + 7) / 8) + (DS % 8 == 0 ? 1 : 0);
}

// tf32 value >= v (v finite, > 0): round the 13 dropped mantissa bits up
__device__ __forceinline__ float tf32_up(float v) {
    uint32_t u = __float_as_uint(v);
    if (u & 0x1FFFu) u = (u | 0x1FFFu) + 1u;
    return __uint_as_float(u);
}

// Per-row constants of the screen: the bound E, the offset window's top
// exponent bits hi4 and the tf32 C of the A operand.  The offset O = 2^p
// (p = 1 mod 16, the smallest p >= floor(log2 S) - 14) puts every screened
// value of the row in [2^p, 2^(p+16)): values >= C - ||x||^2 - E >= O + E and
// <= O + S + E < 2^(p+16) (O <= 2S, S < 2^(p+15)).  S (and with it E) grows
// by at most the offset, i.e. typically not at all (O <= 2^-14 S unless S
// lies just above a 2^(16i+1) boundary).
template <int DS>
struct RowConst {
    float E, C;
    uint32_t hi4;
};

template <int DS>
__device__ __forceinline__ RowConst<DS> row_prep(float nx, float cmax) {
    RowConst<DS> rc;
    const float q = sqrtf(nx) * (1.f + 1e-6f) + cmax;
    const float S = q * q * 1.01f + 1e-6f;  // >= 2|x.c| + ||c||^2 + ||x||^2 + 2E
    int e = int((__float_as_uint(S) >> 23) & 0xFF) - 127;
    e = max(-60, min(e, 100));  // non-finite S: E below is non-finite, the row is flagged
    const int p = (e & ~15) + 1;  // smallest p >= e - 14 with p = 1 (mod 16)
    const float O = __uint_as_float(uint32_t(p + 127) << 23);
    rc.hi4 = uint32_t(p + 127) >> 4;
    const float St = (S + O) * 1.002f;  // + C's rounding up to tf32 (<= 2^-10 C)
    rc.E = tc_error_bound(St, umma_n_mma<DS>());
    rc.C = tf32_up(nx * (1.f + 2.f * float(DS + 2) * kU) + 2.f * rc.E + O);
    return rc;
}

// Decision of a row from its merged keys (see top2_merge).
__device__ __forceinline__ bool row_unique(uint64_t K1, uint32_t V2, uint32_t hi4, float E, uint64_t k) {
    const uint32_t v1 = uint32_t(K1 >> 32);
    if (!isfinite(E) || v1 >= 0x7FFFFFFu || uint32_t(K1) >= k) return false;
    if (V2 >= 0x7FFFFFFu) return true;  // no runner-up
    const float f1 = __uint_as_float(v1 | (hi4 << 27)), f2 = __uint_as_float(V2 | (hi4 << 27));
    return f2 - f1 > 2.05f * E;
}

// A operand of one row: [x (DS) | 1 1 1 C] split hi / lo (constants exact)
template <int DS, int KA>
__device__ __forceinline__ float a_col(const float (&x)[DS], float C, int tt) {
    return tt < DS ? x[tt] : (tt < DS + 3 ? 1.f : (tt == DS + 3 ? C : 0.f));
}

// B operand rows j = [-2c_j (DS) | h m l 1 | 0...] split hi/lo, with
// ||c_j||^2 = h + m + l exactly (three tf32 pieces); rows j >= k are zero
// padding, masked out of the top-2 by the epilogue.  A thread stages whole
// codewords, two at a time, with their loads issued together (vector loads
// when the rows are 16-byte aligned): a short fit re-stages every launch, so
// the staging latency counts.
template <int DS, int KA, bool PAD>
__device__ __forceinline__ void stage_codewords(uint8_t* Bh, uint8_t* Bl, const float* tab,
                                                const float* cnorm, uint64_t k, uint32_t d,
                                                uint32_t n_pad, uint32_t tid, uint32_t nthreads) {
    static_assert(KA >= DS + 4, "constant columns");
    constexpr uint32_t SBO = (KA / 4) * 128;
    const bool vec = !PAD && (DS % 4) == 0 && (reinterpret_cast<uintptr_t>(tab) & 15u) == 0;
    for (uint32_t j0 = 0; j0 < n_pad; j0 += 2 * nthreads) {
        float v[2][KA];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const uint32_t j = j0 + u * nthreads + tid;
#pragma unroll
            for (int t = 0; t < KA; ++t) v[u][t] = 0.f;
            if (j < k) {
                const float* c = tab + uint64_t(j) * d;
                if (vec) {
#pragma unroll
                    for (int t = 0; t < DS; t += 4) {
                        const float4 q = __ldg(reinterpret_cast<const float4*>(c + t));
                        v[u][t] = -2.f * q.x; v[u][t + 1] = -2.f * q.y;
                        v[u][t + 2] = -2.f * q.z; v[u][t + 3] = -2.f * q.w;
                    }
                } else {
#pragma unroll
                    for (int t = 0; t < DS; ++t) v[u][t] = (!PAD || uint32_t(t) < d) ? -2.f * __ldg(c + t) : 0.f;
                }
                const float cn = __ldg(cnorm + j);
                const float h = tf32_hi(cn), m = tf32_hi(cn - h);
                v[u][DS] = h;
                v[u][DS + 1] = m;
                v[u][DS + 2] = (cn - h) - m;  // <= 3 significant bits: exact in tf32
                v[u][DS + 3] = 1.f;
            }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const uint32_t j = j0 + u * nthreads + tid;
            if (j >= n_pad) continue;
#pragma unroll
            for (int t = 0; t < KA; t += 4) {
                float h[4], l[4];
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    h[w] = tf32_hi(v[u][t + w]);
                    l[w] = t + w < DS ? tf32_hi(v[u][t + w] - h[w]) : 0.f;
                }
                *reinterpret_cast<float4*>(Bh + il_off(j, t, SBO)) = make_float4(h[0], h[1], h[2], h[3]);
                *reinterpret_cast<float4*>(Bl + il_off(j, t, SBO)) = make_float4(l[0], l[1], l[2], l[3]);
            }
        }
    }
}

// The n_mma MMAs of one tile: D (+)= Ah Bh^T (+ Ah Bl^T + Al Bh^T for the
// k-steps that hold x columns)
template <int DS, int KA>
__device__ __forceinline__ void issue_tile(uint32_t d_tmem, uint32_t a_hi, uint32_t a_lo, uint32_t b_hi,
                                           uint32_t b_lo, uint32_t boff, uint32_t idesc) {
    constexpr uint32_t SBO = (KA / 4) * 128;
#pragma unroll
    for (int s = 0; s < KA / 8; ++s) {
        const uint32_t ko = s * 256;  // two 16-byte K chunks per k-step
        const uint64_t dah = make_desc(a_hi + ko, 128, SBO);
        const uint64_t dbh = make_desc(b_hi + boff + ko, 128, SBO);
        mma_tf32(d_tmem, dah, dbh, idesc, s > 0);
        if (8 * s < DS) {
            const uint64_t dal = make_desc(a_lo + ko, 128, SBO);
            const uint64_t dbl = make_desc(b_lo + boff + ko, 128, SBO);
            mma_tf32(d_tmem, dah, dbl, idesc, 1);
            mma_tf32(d_tmem, dal, dbh, idesc, 1);
        }
    }
}

// KD: the pass wants the winners' fp64 distances (k-means; a.out_dist set),
// computed under the next tile's MMAs -- a separate instance, so the encode's
// kernel keeps its registers (and CTAs per SM)
template <int DS, int KA, bool PAD, bool DB, bool KD = false>
__global__ void __launch_bounds__(kRows, 1) umma_screen_kernel(NearestArgs a, uint32_t n_pad,
                                                               uint32_t tmem_cols, uint32_t m32,
                                                               uint32_t n_mma, uint32_t allow_fast) {
    static_assert(KA % 8 == 0 && KA >= DS + 2, "augmented K");
    constexpr uint32_t SBO = (KA / 4) * 128;  // bytes between 8-row groups
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* Bh = smem;                         // [n_pad][KA]
    uint8_t* Bl = Bh + size_t(n_pad) * KA * 4;  // [n_pad][KA]
    uint8_t* Ah = Bl + size_t(n_pad) * KA * 4;  // [128][KA]
    uint8_t* Al = Ah + size_t(kRows) * KA * 4;
    __shared__ uint64_t mbar;
    __shared__ uint32_t tmem_base;

    const uint32_t tid = threadIdx.x, warp = tid >> 5;
    const uint32_t B = a.B;
    const uint32_t b = blockIdx.x % B;
    const uint32_t cta = blockIdx.x / B, ncta = gridDim.x / B;
    if (a.active && !a.active[b]) return;
    const uint64_t k = a.k;
    // actual sub-dimension (compile-time DS unless zero-padded up to DS)
    const uint32_t d = PAD ? a.d : uint32_t(DS);
    const float* tab = a.table + uint64_t(b) * k * d;
    const float cmax = a.cmax[b];

    // ---- TMEM allocation (warp 0) and the mbarrier
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(smem_u32(&tmem_base)), "r"(tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        mbar_init(&mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }

    // ---- B operand: [-2c, ||c||^2, 1, 0...] split hi/lo, rows j >= k padded
    stage_codewords<DS, KA, PAD>(Bh, Bl, tab, a.cnorm + uint64_t(b) * k, k, d, n_pad, tid, kRows);
    fence_async_smem();
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = tmem_base;
    const uint32_t a_hi = smem_u32(Ah), a_lo = smem_u32(Al);
    const uint32_t b_hi = smem_u32(Bh), b_lo = smem_u32(Bl);
    uint32_t phase = 0;

    const bool vec4 = a.d == uint32_t(DS) && ((a.src.ldx | a.src.col_stride) & 3u) == 0 &&
                      (reinterpret_cast<uintptr_t>(a.src.x) & 15u) == 0;
    const uint64_t ntiles = (a.n + kRows - 1) / kRows;
    // this thread's row of a tile, loaded one tile ahead so the global-load
    // latency overlaps the current tile's MMA and epilogue
    auto load_row = [&](uint64_t tl, float (&xx)[DS]) {
        const uint64_t r = tl * kRows + tid;
        if (tl < ntiles && r < a.n) {
            const float* xp = a.src.x + r * a.src.ldx + uint64_t(b) * a.src.col_stride;
            if (vec4) {
#pragma unroll
                for (int t = 0; t < DS; t += 4) {
                    const float4 v = __ldg(reinterpret_cast<const float4*>(xp + t));
                    xx[t] = v.x; xx[t + 1] = v.y; xx[t + 2] = v.z; xx[t + 3] = v.w;
                }
            } else {
#pragma unroll
                for (int t = 0; t < DS; ++t) xx[t] = (!PAD || uint32_t(t) < a.d) ? __ldg(xp + t) : 0.f;
            }
        } else {
#pragma unroll
            for (int t = 0; t < DS; ++t) xx[t] = 0.f;
        }
    };
    float x_next[DS];
    load_row(cta, x_next);
    // r2e: the winner's fp64 distance (k-means passes) is computed while the
    // NEXT tile's MMAs run, off the CTA's critical path (in the epilogue it
    // cost ~18 us of a 97 us 100k-row pass): the row, its codeword and x wait
    // in registers for one tile
    float x_pend[DS];
    uint32_t idx_pend = 0xFFFFFFFFu;
    uint64_t row_pend = 0;
    auto flush_dist = [&]() {
        if constexpr (!KD) return;
        if (idx_pend == 0xFFFFFFFFu) return;
        const float* c = tab + uint64_t(idx_pend) * d;
        float cv[DS];
        if (!PAD && (DS % 4) == 0 && (reinterpret_cast<uintptr_t>(tab) & 15u) == 0) {
#pragma unroll
            for (int t = 0; t < DS; t += 4) {
                const float4 q = __ldg(reinterpret_cast<const float4*>(c + t));
                cv[t] = q.x; cv[t + 1] = q.y; cv[t + 2] = q.z; cv[t + 3] = q.w;
            }
        } else {
#pragma unroll
            for (int t = 0; t < DS; ++t) cv[t] = uint32_t(t) < d ? __ldg(c + t) : 0.f;
        }
        double acc = 0.0;
#pragma unroll
        for (int t = 0; t < DS; ++t) {
            if (uint32_t(t) >= d) break;
            const double diff = __dsub_rn((double)x_pend[t], (double)cv[t]);
            acc = __dadd_rn(acc, __dmul_rn(diff, diff));
        }
        a.out_dist[uint64_t(b) * a.n + row_pend] = acc;
        idx_pend = 0xFFFFFFFFu;
    };
    for (uint64_t tile = cta; tile < ntiles; tile += ncta) {
        const uint64_t row = tile * kRows + tid;
        const bool valid = row < a.n;
        // ---- stage A: this thread's row [x, 1, C]
        float x[DS];
        float nx = 0.f;
#pragma unroll
        for (int t = 0; t < DS; ++t) x[t] = x_next[t];
#pragma unroll
        for (int t = 0; t < DS; ++t) nx = fmaf(x[t], x[t], nx);
        const RowConst<DS> rc = row_prep<DS>(nx, cmax);
        const float E = rc.E;
#pragma unroll
        for (int t = 0; t < KA; t += 4) {
            float h[4], l[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int tt = t + u;
                const float v = a_col<DS, KA>(x, rc.C, tt);
                h[u] = tt < DS ? tf32_rna_fast(v) : v;  // constant columns are tf32 already
                l[u] = tt < DS ? tf32_rna_fast(v - h[u]) : 0.f;
            }
            *reinterpret_cast<float4*>(Ah + il_off(tid, t, SBO)) = make_float4(h[0], h[1], h[2], h[3]);
            *reinterpret_cast<float4*>(Al + il_off(tid, t, SBO)) = make_float4(l[0], l[1], l[2], l[3]);
        }
        fence_async_smem();
        fence_before();
        __syncthreads();
        // the accumulator covers n_mma columns: codewords in passes of n_mma
        // (n_mma < n_pad trades a second MMA round per tile for half the TMEM,
        // i.e. more resident CTAs per SM); keys carry the column within a
        // 32-column chunk in 5 low bits (value quantum 32 ulp); the chunk of
        // each running best is tracked on change.  Four independent (best,
        // second) states per thread break the min/max dependency chain; they
        // are merged at the end.
        uint32_t m1[kNS], m2[kNS], ch[kNS];
#pragma unroll
        for (int s4 = 0; s4 < kNS; ++s4) { m1[s4] = 0xFFFFFFFFu; m2[s4] = 0xFFFFFFFFu; ch[s4] = 0; }
        const uint32_t lane_base = (warp * 32u) << 16;
        // r2h: full 64/128-column passes take the unrolled fast path (ch[] then
        // holds each state's pass base; see top2_pairs_fast)
        const bool fast = !DB && allow_fast && (k % 64) == 0 && (n_mma == 64 || n_mma == 128);
        for (uint32_t p0 = 0; p0 < n_pad; p0 += n_mma) {
            const uint32_t w = min(n_mma, n_pad - p0);
            if (p0 > 0) {  // the previous pass's TMEM reads are complete before the next MMA
                fence_before();
                __syncthreads();
            }
            // ---- MMA: D = Ah Bh^T + Ah Bl^T + Al Bh^T (constant k-steps: Ah Bh^T)
            if (tid == 0) {
                fence_after();
                const uint32_t idesc = make_idesc_tf32(kRows, w);
                const uint32_t boff = (p0 / 8) * SBO;  // codeword rows p0.. of the B stage
                issue_tile<DS, KA>(tmem, a_hi, a_lo, b_hi, b_lo, boff, idesc);
                mma_commit(&mbar);
            }
            if (p0 == 0) {
                load_row(tile + ncta, x_next);  // next tile's row, in flight during the epilogue
                flush_dist();                   // the previous tile's winner, under this tile's MMAs
            }
            mbar_wait(&mbar, phase);
            phase ^= 1;
            fence_after();
            // ---- epilogue: this thread's row, columns p0 .. p0 + w
            // columns >= k of this pass (codeword padding, and the unwritten
            // tail of a 16-column-multiple n_mma) are masked out of the top-2
            auto process = [&](uint32_t (&r)[32], uint32_t c0) {
                const uint32_t cabs = p0 + c0;
                if (cabs + 32 <= k) top2_chunk<false>(r, 32u, cabs, m1, m2, ch, m32);
                else top2_chunk<true>(r, uint32_t(k - cabs), cabs, m1, m2, ch, m32);
            };
            if (!DB && fast) {
                const uint32_t one = m32 >> 5, neg1 = 0u - one;
                uint32_t old[kNS];
#pragma unroll
                for (int s4 = 0; s4 < kNS; ++s4) old[s4] = m1[s4];
                auto chunk = [&](auto cc_tag) {
                    constexpr int CC = decltype(cc_tag)::value;
                    uint32_t r[32];
                    tmem_ld32(tmem + lane_base + uint32_t(CC * 32), r);
                    tmem_wait_ld();
                    tmem_regs_ready(r);
                    top2_pairs_fast<CC, 0>(r, m1, m2, m32, one, neg1);
                };
                chunk(std::integral_constant<int, 0>{});
                chunk(std::integral_constant<int, 1>{});
                if (w == 128) {
                    chunk(std::integral_constant<int, 2>{});
                    chunk(std::integral_constant<int, 3>{});
                }
#pragma unroll
                for (int s4 = 0; s4 < kNS; ++s4) ch[s4] = (m1[s4] != old[s4]) ? p0 : ch[s4];
            } else if constexpr (DB) {
                // two register buffers: the next 32 columns load from TMEM
                // while the current ones are reduced (wide tables, where TMEM
                // already limits the CTAs per SM to two; the extra registers
                // would cost narrow tables their third and fourth CTA)
                uint32_t ra[32], rb[32];
                tmem_ld32(tmem + lane_base, ra);
                tmem_wait_ld();
                tmem_regs_ready(ra);
                for (uint32_t c0 = 0; c0 < w; c0 += 64) {
                    const bool more = c0 + 32 < w;
                    if (more) tmem_ld32(tmem + lane_base + c0 + 32, rb);
                    process(ra, c0);
                    if (!more) break;
                    tmem_wait_ld();
                    tmem_regs_ready(rb);
                    const bool more2 = c0 + 64 < w;
                    if (more2) tmem_ld32(tmem + lane_base + c0 + 64, ra);
                    process(rb, c0 + 32);
                    if (!more2) break;
                    tmem_wait_ld();
                    tmem_regs_ready(ra);
                }
            } else {
                for (uint32_t c0 = 0; c0 < w; c0 += 32) {
                    uint32_t r[32];
                    tmem_ld32(tmem + lane_base + c0, r);
                    tmem_wait_ld();
                    process(r, c0);
                }
            }
        }
        uint64_t K1;
        uint32_t V2;
        if (fast) top2_merge_fast(m1, m2, ch, K1, V2);
        else top2_merge(m1, m2, ch, K1, V2);
        fence_before();
        if (valid) {
            const uint32_t idx = uint32_t(K1);
            // non-finite E (inf/NaN in the row or table): the exact fixup decides
            if (row_unique(K1, V2, rc.hi4, E, k)) {
                store_index(a, row, b, idx);
                if (KD && a.out_dist) {  // computed under the next tile's MMAs (flush_dist)
#pragma unroll
                    for (int t = 0; t < DS; ++t) x_pend[t] = x[t];
                    idx_pend = idx;
                    row_pend = row;
                }
            } else {
                const unsigned long long slot = atomicAdd(a.flag_count, 1ull);
                a.flags[slot] = (uint64_t(b) << 40) | row;
            }
        }
        __syncthreads();  // TMEM and the A stage are reused by the next tile
    }
    flush_dist();  // the last tile's winner
    fence_before();
    __syncthreads();
    if (warp == 0) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(tmem_cols));
    }
}

// ---------------------------------------------------------------------------
// Pipelined version: one CTA per SM, 8 warps, persistent over the row tiles
// of one subspace.  TMEM holds two 128 x n_pad fp32 accumulators and the A
// stage is double-buffered, so the MMAs of tile i+1 run while the CUDA cores
// reduce tile i; the rows of tile i+2 are already in flight from HBM.  Warp w
// reads TMEM lanes 32(w%4).. and the column half w/4; the halves meet in
// shared memory.
// ---------------------------------------------------------------------------
template <int DS>
struct RowRegs {
    float x[DS];
};

template <int DS, bool PAD>
__device__ __forceinline__ void load_row(const NearestArgs& a, uint64_t row, uint32_t b, bool vec4,
                                         RowRegs<DS>& r) {
    if (row < a.n) {
        const float* xp = a.src.x + row * a.src.ldx + uint64_t(b) * a.src.col_stride;
        if (vec4) {
#pragma unroll
            for (int t = 0; t < DS; t += 4) {
                const float4 v = __ldg(reinterpret_cast<const float4*>(xp + t));
                r.x[t] = v.x; r.x[t + 1] = v.y; r.x[t + 2] = v.z; r.x[t + 3] = v.w;
            }
        } else {
#pragma unroll
            for (int t = 0; t < DS; ++t) r.x[t] = (!PAD || uint32_t(t) < a.d) ? __ldg(xp + t) : 0.f;
        }
    } else {
#pragma unroll
        for (int t = 0; t < DS; ++t) r.x[t] = 0.f;
    }
}

template <int DS, int KA, int NW, bool PAD>
__global__ void __launch_bounds__(NW * 32, 1) umma_screen2_kernel(NearestArgs a, uint32_t n_pad,
                                                                  uint32_t m32) {
    constexpr int NPART = NW / 4;  // column parts (warp quads) per tile
    constexpr uint32_t SBO = (KA / 4) * 128;
    constexpr uint32_t ASTAGE = kRows * KA * 4;  // bytes of one A (hi or lo) stage
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* Bh = smem;
    uint8_t* Bl = Bh + size_t(n_pad) * KA * 4;
    uint8_t* A0 = Bl + size_t(n_pad) * KA * 4;  // [stage][hi|lo][128 x KA]
    __shared__ uint64_t mbar[2];
    __shared__ uint32_t tmem_base;
    __shared__ float ebuf[2][kRows];
    __shared__ uint32_t hbuf[2][kRows];
    __shared__ uint64_t mK[NPART > 1 ? NPART - 1 : 1][kRows];
    __shared__ uint32_t mV[NPART > 1 ? NPART - 1 : 1][kRows];

    const uint32_t tid = threadIdx.x, warp = tid >> 5;
    const uint32_t B = a.B;
    const uint32_t b = blockIdx.x % B;
    const uint32_t cta = blockIdx.x / B, ncta = gridDim.x / B;
    if (a.active && !a.active[b]) return;
    const uint64_t k = a.k;
    // actual sub-dimension (compile-time DS unless zero-padded up to DS)
    const uint32_t d = PAD ? a.d : uint32_t(DS);
    const float* tab = a.table + uint64_t(b) * k * d;
    const float cmax = a.cmax[b];
    const uint32_t row_l = tid & (kRows - 1);  // row of the tile this thread stages / reads
    const uint32_t half = tid >> 7;             // K part it stages, column part it reduces

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(smem_u32(&tmem_base)), "r"(512u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    stage_codewords<DS, KA, PAD>(Bh, Bl, tab, a.cnorm + uint64_t(b) * k, k, d, n_pad, tid, blockDim.x);
    fence_async_smem();
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = tmem_base;
    const uint32_t idesc = make_idesc_tf32(kRows, n_pad);
    const uint32_t b_hi = smem_u32(Bh), b_lo = smem_u32(Bl);
    const bool vec4 = a.d == uint32_t(DS) && ((a.src.ldx | a.src.col_stride) & 3u) == 0 &&
                      (reinterpret_cast<uintptr_t>(a.src.x) & 15u) == 0;
    const uint64_t ntiles = (a.n + kRows - 1) / kRows;
    const uint64_t my_tiles = cta < ntiles ? (ntiles - cta + ncta - 1) / ncta : 0;

    // stage the A operand of tile number `it` (local index) from registers
    auto stage = [&](uint64_t it, const RowRegs<DS>& r) {
        float nx = 0.f;
#pragma unroll
        for (int t = 0; t < DS; ++t) nx = fmaf(r.x[t], r.x[t], nx);
        const RowConst<DS> rc = row_prep<DS>(nx, cmax);
        if (half == 0) {
            ebuf[it & 1][row_l] = rc.E;
            hbuf[it & 1][row_l] = rc.hi4;
        }
        uint8_t* Ah = A0 + (it & 1) * 2 * ASTAGE;
        uint8_t* Al = Ah + ASTAGE;
        constexpr int NCH = KA / 4;  // 16-byte chunks per row, dealt round-robin to the parts
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            if (uint32_t(c % NPART) != half) continue;
            float h[4], l[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int tt = 4 * c + u;
                const float v = a_col<DS, KA>(r.x, rc.C, tt);
                h[u] = tt < DS ? tf32_rna_fast(v) : v;
                l[u] = tt < DS ? tf32_rna_fast(v - h[u]) : 0.f;
            }
            *reinterpret_cast<float4*>(Ah + il_off(row_l, 4 * c, SBO)) = make_float4(h[0], h[1], h[2], h[3]);
            *reinterpret_cast<float4*>(Al + il_off(row_l, 4 * c, SBO)) = make_float4(l[0], l[1], l[2], l[3]);
        }
    };
    auto issue = [&](uint64_t it) {
        const uint32_t ah = smem_u32(A0 + (it & 1) * 2 * ASTAGE), al = ah + ASTAGE;
        const uint32_t d_tmem = tmem + uint32_t(it & 1) * 256u;
        issue_tile<DS, KA>(d_tmem, ah, al, b_hi, b_lo, 0u, idesc);
        mma_commit(&mbar[it & 1]);
    };
    auto tile_of = [&](uint64_t it) { return uint64_t(cta) + it * ncta; };

    RowRegs<DS> xr;
    if (my_tiles > 0) {
        load_row<DS, PAD>(a, tile_of(0) * kRows + row_l, b, vec4, xr);
        stage(0, xr);
        if (my_tiles > 1) load_row<DS, PAD>(a, tile_of(1) * kRows + row_l, b, vec4, xr);
        fence_async_smem();
        fence_before();
        __syncthreads();
        if (tid == 0) {
            fence_after();
            issue(0);
        }
    }
    uint32_t phases = 0;  // bit s: parity of mbar[s]
    for (uint64_t it = 0; it < my_tiles; ++it) {
        // stage tile it+1 (rows already in registers), prefetch tile it+2
        if (it + 1 < my_tiles) {
            stage(it + 1, xr);
            if (it + 2 < my_tiles) load_row<DS, PAD>(a, tile_of(it + 2) * kRows + row_l, b, vec4, xr);
        }
        fence_async_smem();
        fence_before();
        __syncthreads();
        if (tid == 0 && it + 1 < my_tiles) {
            fence_after();
            issue(it + 1);
        }
        mbar_wait(&mbar[it & 1], (phases >> (it & 1)) & 1u);
        phases ^= 1u << (it & 1);
        fence_after();
        // ---- epilogue of tile it: this thread's row, its column half
        uint32_t m1[kNS], m2[kNS], ch[kNS];
#pragma unroll
        for (int s4 = 0; s4 < kNS; ++s4) { m1[s4] = 0xFFFFFFFFu; m2[s4] = 0xFFFFFFFFu; ch[s4] = 0; }
        const uint32_t lane_base = ((warp & 3u) * 32u) << 16;
        const uint32_t nchunks = (n_pad + 31) / 32;
        const uint32_t per = (nchunks + NPART - 1) / NPART;  // 32-column chunks per part
        const uint32_t cbeg = half * per * 32;
        const uint32_t cend = min(n_pad, cbeg + per * 32);
        const uint32_t tb = tmem + uint32_t(it & 1) * 256u;
        for (uint32_t c0 = cbeg; c0 < cend; c0 += 32) {
            uint32_t r[32];
            tmem_ld32(tb + lane_base + c0, r);
            tmem_wait_ld();
            if (c0 + 32 <= k) top2_chunk<false>(r, 32u, c0, m1, m2, ch, m32);
            else top2_chunk<true>(r, uint32_t(k - c0), c0, m1, m2, ch, m32);
        }
        fence_before();
        uint64_t K1;
        uint32_t V2;
        top2_merge(m1, m2, ch, K1, V2);
        if (half > 0) {
            mK[half - 1][row_l] = K1;
            mV[half - 1][row_l] = V2;
        }
        __syncthreads();
        if (half == 0) {
#pragma unroll
            for (int p2 = 0; p2 < NPART - 1; ++p2) {
                const uint64_t oK = mK[p2][row_l];
                V2 = min(min(V2, mV[p2][row_l]), uint32_t(max(K1, oK) >> 32));
                K1 = min(K1, oK);
            }
            const uint64_t row = tile_of(it) * kRows + row_l;
            if (row < a.n) {
                const uint32_t idx = uint32_t(K1);
                // non-finite E (inf/NaN in the row or table): the exact fixup decides
                if (row_unique(K1, V2, hbuf[it & 1][row_l], ebuf[it & 1][row_l], k)) {
                    store_index(a, row, b, idx);
                    if (a.out_dist) {
                        const float* xp = a.src.x + row * a.src.ldx + uint64_t(b) * a.src.col_stride;
                        const float* c = tab + uint64_t(idx) * d;
                        double acc = 0.0;
#pragma unroll
                        for (int t = 0; t < DS; ++t) {
                            if (uint32_t(t) >= d) break;
                            const double diff = __dsub_rn((double)__ldg(xp + t), (double)__ldg(c + t));
                            acc = __dadd_rn(acc, __dmul_rn(diff, diff));
                        }
                        a.out_dist[uint64_t(b) * a.n + row] = acc;
                    }
                } else {
                    const unsigned long long slot = atomicAdd(a.flag_count, 1ull);
                    a.flags[slot] = (uint64_t(b) << 40) | row;
                }
            }
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 0) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(512u));
    }
}

template <int DS, int KA, bool PAD>
void launch_umma2(pqg_ctx* ctx, const NearestArgs& a) {
    const uint32_t n_pad = uint32_t((a.k + 15) / 16 * 16);
    const size_t smem = size_t(2) * n_pad * KA * 4 + size_t(4) * kRows * KA * 4;
    const int nw_env = std::getenv("PQG_UMMA_WARPS") ? std::atoi(std::getenv("PQG_UMMA_WARPS")) : 8;
    const uint64_t ntiles = (a.n + kRows - 1) / kRows;
    // one CTA per SM; each subspace gets floor(SMs / B) CTAs (at least 1)
    uint64_t per_b = std::max<uint64_t>(1, uint64_t(ctx->num_sms) / a.B);
    per_b = std::min<uint64_t>(per_b, ntiles);
    auto go = [&](auto kern, int nthreads) {
        PQG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        launch(ctx, "nearest_tc", kern, dim3(unsigned(per_b * a.B)), dim3(nthreads), smem, a, n_pad, 32u);
    };
    if (nw_env == 8) go(umma_screen2_kernel<DS, KA, 8, PAD>, 256);
    else go(umma_screen2_kernel<DS, KA, 16, PAD>, 512);
}

template <int DS, int KA, bool PAD>
void launch_umma(pqg_ctx* ctx, const NearestArgs& a) {
    // measured (tools/screen_bench.py, r1): the synchronous multi-CTA/SM kernel
    // wins for narrow tables, Ds <= 8 (two 128-codeword passes, 4 CTAs/SM) and
    // Ds=16/Ks=256; the pipelined 8-warp kernel otherwise
    const char* env = std::getenv("PQG_UMMA");
    const uint32_t n_pad_sel = uint32_t((a.k + 15) / 16 * 16);
    bool v1 = n_pad_sel <= 128 || DS <= 8 || (DS == 16 && n_pad_sel == 256);
    if (env && env[0] == '1') v1 = true;
    if (env && env[0] == '2') v1 = false;
    if (!v1) {
        launch_umma2<DS, KA, PAD>(ctx, a);
        return;
    }
    const uint32_t n_pad = uint32_t((a.k + 15) / 16 * 16);
    const size_t smem = size_t(2) * n_pad * KA * 4 + size_t(2) * kRows * KA * 4;
    const uint64_t smem_lim = (227u * 1024u) / (smem + 3u * 1024u);
    // MMA width: all codewords in one pass, or two passes of 128 when that
    // halves TMEM and shared memory lets 4 CTAs reside (measured r1,
    // tools/screen_bench.py at 1M x 128, Ks=256: Ds=8 1.92 -> 1.38 ms, Ds=4
    // 3.76 -> 3.10 ms against the pipelined kernel; at Ds=16, where only 3 CTAs
    // fit, the second MMA round costs more than the extra CTA gains: 0.87 -> 1.12)
    // r2 (new epilogue, 7-MMA tiles): the split wins at Ds = 16 too
    // (M=8 Ks=256 encode 0.69 -> 0.65 ms) and is neutral elsewhere
    uint32_t n_mma = n_pad;
    if (n_pad > 128) n_mma = 128;
    if (const char* se = std::getenv("PQG_UMMA_SPLIT")) n_mma = se[0] == '1' && n_pad > 128 ? 128 : n_pad;
    uint32_t cols = 32;
    while (cols < n_mma) cols <<= 1;
    const bool db = n_mma == n_pad && n_pad > 128 && !(std::getenv("PQG_UMMA_DB") && std::getenv("PQG_UMMA_DB")[0] == '0');
    auto kern = db ? umma_screen_kernel<DS, KA, PAD, true> : umma_screen_kernel<DS, KA, PAD, false>;
    if (a.out_dist) kern = db ? umma_screen_kernel<DS, KA, PAD, true, true> : umma_screen_kernel<DS, KA, PAD, false, true>;
    PQG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const uint64_t ntiles = (a.n + kRows - 1) / kRows;
    // persistent: CTAs per SM limited by TMEM columns (2 at Ks=256), shared
    // memory and a cap of 4 (measured: narrow tables gain up to ~1.5x from the
    // extra CTAs, whose short tiles are latency-bound); PQG_UMMA_CTAS overrides
    uint64_t per_sm = std::max<uint64_t>(1, std::min<uint64_t>(std::min<uint64_t>(4u, 512u / cols), smem_lim));
    if (const char* ce = std::getenv("PQG_UMMA_CTAS")) per_sm = std::max(1, std::atoi(ce));
    // CTAs per problem: minimise (waves of CTAs) x (tiles per CTA) -- with
    // many problems a partial second wave costs a whole extra tile run
    const uint64_t slots = uint64_t(ctx->num_sms) * per_sm;
    uint64_t per_b = 1, best = ~0ull;
    for (uint64_t p = 1; p <= std::min<uint64_t>(ntiles, std::max<uint64_t>(1, (2 * slots + a.B - 1) / a.B)); ++p) {
        const uint64_t cost = ((p * a.B + slots - 1) / slots) * ((ntiles + p - 1) / p);
        if (cost < best) {
            best = cost;
            per_b = p;
        }
    }
    // r2h unrolled fast epilogue (A/B switch PQG_UMMA_FAST=0)
    const char* fe = std::getenv("PQG_UMMA_FAST");
    const uint32_t allow_fast = (fe && fe[0] == '0') ? 0u : 1u;
    launch(ctx, "nearest_tc", kern, dim3(unsigned(per_b * a.B)), dim3(kRows), smem, a, n_pad, cols, 32u, n_mma,
           allow_fast);
}

}  // namespace

// Any sub-dimension up to 32 (zero-padded to 4/8/16/32 in both operands: the
// padded products are exactly zero) and any 16 <= k <= 256 (codewords padded to
// a multiple of 16 never win).
bool umma_screen_supported(const NearestArgs& a) {
    if (a.src.codes || a.out_mat) return false;
    if (a.k < 16 || a.k > 256) return false;
    return a.d >= 1 && a.d <= 32;
}

void umma_screen(pqg_ctx* ctx, const NearestArgs& a) {
    switch (a.d) {  // exact widths compile the sub-dimension in; others are zero-padded
        case 4: launch_umma<4, 8, false>(ctx, a); return;
        case 8: launch_umma<8, 16, false>(ctx, a); return;
        case 16: launch_umma<16, 24, false>(ctx, a); return;
        case 32: launch_umma<32, 40, false>(ctx, a); return;
        default: break;
    }
    if (a.d < 4) launch_umma<4, 8, true>(ctx, a);
    else if (a.d < 8) launch_umma<8, 16, true>(ctx, a);
    else if (a.d < 16) launch_umma<16, 24, true>(ctx, a);
    else if (a.d < 32) launch_umma<32, 40, true>(ctx, a);
    else fail(PQG_EUNSUPPORTED, "umma_screen: unsupported sub-dimension");
}

}  // namespace pqg
