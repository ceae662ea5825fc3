// umma_big.cu -- tcgen05 GEMM-argmin for the coarse quantizer: many rows
// against many centroids in full dimension (assign_items / probe_order /
// coarse kmeans_fit: proj/src/ivf.cpp:36-49, :91-101, proj/src/kmeans.cpp:46-57),
// e.g. 1M x 128 rows against nlist = 1024..16384 centroids.
//
// Operands are prepared once per call in global memory, already split into
// TF32 hi/lo halves and laid out in the canonical K-major no-swizzle UMMA
// layout, so the main kernel only moves bytes:
//   A (rows)      : [row tile of 128][K chunk of 32][hi|lo][16 KB]
//   B (centroids) : [N block of 256][K chunk of 32][hi|lo][32 KB]
// with the augmented rows A_r = [x_r, 1, C_r, 0..], B_j = [-2c_j, ||c_j||^2, 1, 0..]
// (see umma.cu), so the MMA accumulates the screened value directly.
//
// Main kernel: persistent, one CTA per SM, 6 warps.
//   warp 0     producer: cp.async.bulk of the A and B chunks of each
//              (row tile, N block, K chunk) into a 2-stage smem ring
//              (mbarrier complete_tx)
//   warp 1     MMA issuer: 4 k-steps x 3 (3xTF32) tcgen05.mma per chunk into
//              one of two TMEM accumulators (128 x 256 fp32 each)
//   warps 2-5  epilogue: thread = row = TMEM lane; tcgen05.ld 32 columns at a
//              time; keep the 4 smallest (value, column) per row across all N
//              blocks; at the end of the row tile resolve the winner:
//              every centroid within 2E of the best is among the top 4 unless
//              the 4th is itself inside the band, so <= 3 candidates are
//              re-scored in the reference's exact fp64 arithmetic in-kernel
//              and only rows with >= 4 candidates in the band go to the
//              global fixup.  MAT mode instead writes the screened matrix.
#include <cstdlib>
#include <cstring>

#include "tc_common.cuh"

namespace pqg {

namespace {

using namespace tc;

__device__ __forceinline__ float row_x(const RowSrc& s, uint64_t i, uint32_t t) {
    if (s.codes) {
        const uint32_t m = t / s.dds, tt = t - m * s.dds;
        const uint8_t* p = s.codes + (i * s.dM + m) * s.dw;
        uint32_t code = s.dw == 1 ? uint32_t(p[0]) : (uint32_t(p[0]) | (uint32_t(p[1]) << 8));
        if (code >= s.dks) code = s.dks - 1;
        return __ldg(s.dtab + ((uint64_t)m * s.dks + code) * s.dds + tt);
    }
    return __ldg(s.x + i * s.ldx + t);
}


// ---- operand preparation ---------------------------------------------------
// A_r = [x_r, 1, C_r, 0...], split hi/lo, interleaved.  C_r = ||x_r||^2 (+ 2E
// margin in matrix mode, whose consumer orders values as unsigned bits); the
// argmin epilogue compares floats and recomputes E from the stored ||x_r||^2
// and the current max ||c||.  Two passes: the row norms (thread per row, the
// same sequential fmaf order as before), then one thread per (row, K chunk,
// 4-element group) with a warp covering 8 rows x 4 groups, so the x reads use
// whole sectors and every interleaved 128-byte core-matrix line is written by
// one warp instruction.
__global__ void row_norms_kernel(RowSrc src, uint64_t n, uint32_t d, float* nxrow) {
    // a warp per row, coalesced loads, tree-reduced: ||x||^2 only feeds C_r
    // and the error bound E_r, whose margins cover any summation order (the
    // split and the epilogue read the same stored value)
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t w0 = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    const bool vec = !src.codes && (d & 3u) == 0 && (src.ldx & 3u) == 0 &&
                     (reinterpret_cast<uintptr_t>(src.x) & 15u) == 0;
    for (uint64_t r = w0; r < n; r += nw) {
        float nx = 0.f;
        if (vec) {
            const float4* xp = reinterpret_cast<const float4*>(src.x + r * src.ldx);
            for (uint32_t t4 = lane; t4 < d / 4; t4 += 32) {
                const float4 v = __ldg(xp + t4);
                nx = fmaf(v.x, v.x, nx);
                nx = fmaf(v.y, v.y, nx);
                nx = fmaf(v.z, v.z, nx);
                nx = fmaf(v.w, v.w, nx);
            }
        } else {
            for (uint32_t t = lane; t < d; t += 32) {
                const float v = row_x(src, r, t);
                nx = fmaf(v, v, nx);
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) nx += __shfl_xor_sync(0xffffffffu, nx, off);
        if (lane == 0) nxrow[r] = nx;
    }
}

// element group g -> (row within the tile, K chunk, group of 4 within the chunk)
struct SplitIdx {
    uint64_t tile;
    uint32_t rl, kc, k4;
};
__device__ __forceinline__ SplitIdx split_idx(uint64_t g, uint32_t rows, uint32_t kchunks) {
    SplitIdx s;
    const uint32_t lo = uint32_t(g & 7u);
    constexpr uint32_t KG = kKC / 4;  // groups of 4 K elements per chunk
    s.k4 = uint32_t((g >> 3) % KG) * 4u;
    const uint64_t rest = (g >> 3) / KG;
    const uint32_t hi = uint32_t(rest % (rows / 8));
    const uint64_t rest2 = rest / (rows / 8);
    s.kc = uint32_t(rest2 % kchunks);
    s.tile = rest2 / kchunks;
    s.rl = hi * 8 + lo;
    return s;
}

__global__ void split_rows_kernel(RowSrc src, uint64_t n, uint32_t d, uint32_t kchunks,
                                  const float* cmax_p, int margin, uint8_t* A, const float* nxrow) {
    const float cmax = *cmax_p;
    const uint64_t total = (n + kR - 1) / kR * kR * kchunks * (kKC / 4);
    for (uint64_t g = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < total;
         g += uint64_t(gridDim.x) * blockDim.x) {
        const SplitIdx ix = split_idx(g, kR, kchunks);
        const uint64_t r = ix.tile * kR + ix.rl;
        const bool valid = r < n;
        const float nx = valid ? nxrow[r] : 0.f;
        const float q = sqrtf(nx) * (1.f + 1e-6f) + cmax;
        const float S = q * q * 1.01f + 1e-6f;
        const float E = big_error_bound(S, kchunks);
        const float C = margin ? nx * (1.f + 2.f * float(d + 2) * kU) + 2.f * E : nx;
        uint8_t* blk = A + (ix.tile * kchunks + ix.kc) * (2 * kAChunk);
        float h[4], l[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t t = ix.kc * kKC + ix.k4 + u;
            float v = 0.f;
            if (valid) v = t < d ? row_x(src, r, t) : (t == d ? 1.f : (t == d + 1 ? C : 0.f));
            h[u] = tf32_hi(v);
            l[u] = tf32_hi(v - h[u]);
        }
        *reinterpret_cast<float4*>(blk + il_off(ix.rl, ix.k4)) = make_float4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<float4*>(blk + kAChunk + il_off(ix.rl, ix.k4)) = make_float4(l[0], l[1], l[2], l[3]);
    }
}

// B_j = [-2c_j, ||c_j||^2, 1, 0...]; padded rows never win.  Same thread
// layout as split_rows_kernel over 256-row blocks.
__global__ void split_table_kernel(const float* table, const float* cnorm, uint64_t k, uint32_t d,
                                   uint32_t kchunks, uint64_t k_pad, uint8_t* Bm) {
    const uint64_t total = k_pad * kchunks * (kKC / 4);
    for (uint64_t g = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < total;
         g += uint64_t(gridDim.x) * blockDim.x) {
        const SplitIdx ix = split_idx(g, kN, kchunks);
        const uint64_t j = ix.tile * kN + ix.rl;
        uint8_t* blk = Bm + (ix.tile * kchunks + ix.kc) * (2 * kBChunk);
        float h[4], l[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t t = ix.kc * kKC + ix.k4 + u;
            float v = 0.f;
            if (j < k) {
                if (t < d) v = -2.f * __ldg(table + j * d + t);
                else if (t == d) v = __ldg(cnorm + j);
                else if (t == d + 1) v = 1.f;
            } else if (t == d) {
                v = 3.0e38f;
            }
            h[u] = tf32_hi(v);
            l[u] = tf32_hi(v - h[u]);
        }
        *reinterpret_cast<float4*>(blk + il_off(ix.rl, ix.k4)) = make_float4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<float4*>(blk + kBChunk + il_off(ix.rl, ix.k4)) = make_float4(l[0], l[1], l[2], l[3]);
    }
}

__device__ __forceinline__ void store_index(const NearestArgs& a, uint64_t i, uint32_t idx) {
    const uint64_t off = i * a.idx_rs;
    if (a.idx_bytes == 1) static_cast<uint8_t*>(a.out_idx)[off] = uint8_t(idx);
    else if (a.idx_bytes == 2) {
        uint8_t* p = static_cast<uint8_t*>(a.out_idx) + off * 2;
        p[0] = uint8_t(idx & 0xff);
        p[1] = uint8_t(idx >> 8);
    } else static_cast<uint32_t*>(a.out_idx)[off] = idx;
}

__device__ __forceinline__ double exact_row_dist(const NearestArgs& a, uint64_t row, uint32_t j) {
    const float* c = a.table + uint64_t(j) * a.d;
    double acc = 0.0;
    for (uint32_t t = 0; t < a.d; ++t) {
        const double diff = __dsub_rn((double)row_x(a.src, row, t), (double)__ldg(c + t));
        acc = __dadd_rn(acc, __dmul_rn(diff, diff));
    }
    return acc;
}

// ---- main kernel -----------------------------------------------------------
template <bool MAT>
__global__ void __launch_bounds__(192, 1) big_kernel(NearestArgs a, const uint8_t* __restrict__ A,
                                                     const uint8_t* __restrict__ Bm,
                                                     const float* __restrict__ nxrow,
                                                     uint32_t kchunks, uint32_t nblocks,
                                                     uint64_t row_base) {
    if (a.active && !a.active[0]) return;
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t full[kBigStages], empty[kBigStages], tfull[2], tempty[2];
    __shared__ uint32_t tmem_base;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t ntiles = (a.n + kR - 1) / kR;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(smem_u32(&tmem_base)), "r"(512u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 32) {
        for (int s = 0; s < kBigStages; ++s) {
            bar_init(&full[s], 1);
            bar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            bar_init(&tfull[s], 1);
            bar_init(&tempty[s], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = tmem_base;

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            uint32_t q = 0;
            for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                for (uint32_t nb = 0; nb < nblocks; ++nb) {
                    for (uint32_t kc = 0; kc < kchunks; ++kc, ++q) {
                        const uint32_t s = q % kBigStages, ph = (q / kBigStages) & 1;
                        bar_wait(&empty[s], ph ^ 1);
                        uint8_t* st = smem + s * kStage;
                        bar_expect_tx(&full[s], kStage);
                        bulk_g2s(st, A + (tile * kchunks + kc) * (2 * kAChunk), 2 * kAChunk, &full[s]);
                        bulk_g2s(st + 2 * kAChunk, Bm + (uint64_t(nb) * kchunks + kc) * (2 * kBChunk),
                                 2 * kBChunk, &full[s]);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t idesc = idesc_tf32(kR, kN);
            uint32_t q = 0, u = 0;
            for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                for (uint32_t nb = 0; nb < nblocks; ++nb, ++u) {
                    const uint32_t buf = u & 1, tph = (u >> 1) & 1;
                    bar_wait(&tempty[buf], tph ^ 1);
                    fence_after();
                    const uint32_t d_tmem = tmem + buf * 256u;
                    for (uint32_t kc = 0; kc < kchunks; ++kc, ++q) {
                        const uint32_t s = q % kBigStages, ph = (q / kBigStages) & 1;
                        bar_wait(&full[s], ph);
                        fence_after();
                        const uint32_t base = smem_u32(smem + s * kStage);
                        const uint32_t ah = base, al = base + kAChunk;
                        const uint32_t bh = base + 2 * kAChunk, bl = bh + kBChunk;
#pragma unroll
                        for (int k4 = 0; k4 < kKC / 8; ++k4) {
                            const uint32_t ko = k4 * 256;
                            const uint64_t dah = make_desc(ah + ko, 128, kSBO);
                            const uint64_t dal = make_desc(al + ko, 128, kSBO);
                            const uint64_t dbh = make_desc(bh + ko, 128, kSBO);
                            const uint64_t dbl = make_desc(bl + ko, 128, kSBO);
                            mma_tf32(d_tmem, dah, dbh, idesc, (kc | k4) != 0);
                            mma_tf32(d_tmem, dah, dbl, idesc, 1);
                            mma_tf32(d_tmem, dal, dbh, idesc, 1);
                        }
                        commit(&empty[s]);  // smem stage free once these MMAs are done
                    }
                    commit(&tfull[buf]);  // accumulator ready for the epilogue
                }
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const uint32_t quarter = warp & 3u;  // TMEM lane quarter of this warp
        const uint32_t rl = quarter * 32 + lane;
        const uint32_t lane_base = (quarter * 32u) << 16;
        uint32_t u = 0;
        for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const uint64_t row = tile * kR + rl;
            float tv[4];
            uint32_t ti[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) { tv[i] = __int_as_float(0x7f800000); ti[i] = 0xFFFFFFFFu; }
            for (uint32_t nb = 0; nb < nblocks; ++nb, ++u) {
                const uint32_t buf = u & 1, tph = (u >> 1) & 1;
                bar_wait(&tfull[buf], tph);
                fence_after();
                const uint32_t tb = tmem + buf * 256u + lane_base;
                for (uint32_t c0 = 0; c0 < uint32_t(kN); c0 += 32) {
                    uint32_t r[32];
                    tmem_ld32(tb + c0, r);
                    tmem_wait_ld();
                    const uint32_t col0 = nb * kN + c0;
                    if constexpr (MAT) {
                        if (row < a.n) {
                            float* o = a.out_mat + row * a.ld_mat + col0;
                            if (col0 + 32 <= a.k && ((reinterpret_cast<uintptr_t>(o) & 15u) == 0)) {
                                // the row's 128-byte chunk as eight 16-byte stores
#pragma unroll
                                for (int j = 0; j < 32; j += 4)
                                    *reinterpret_cast<float4*>(o + j) =
                                        make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                                    __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
                            } else {
#pragma unroll
                                for (int j = 0; j < 32; ++j)
                                    if (col0 + j < a.k) o[j] = __uint_as_float(r[j]);
                            }
                        }
                    } else {
                        // r2e: the chunk's minimum first; a warp whose lanes all
                        // hold a 4th best below it skips the chunk.  Otherwise each
                        // value is offered to the lanes' top 4 with a warp-uniform
                        // vote and a branch-free insertion (the per-lane nested
                        // branches diverged on every value: the epilogue, not the
                        // MMAs, bound this kernel -- 18.5 ms against 7.5 without it;
                        // now 16.1).  Strict '<' at every level as before; NaN
                        // never enters.
                        float cm[16];
#pragma unroll
                        for (int j = 0; j < 16; ++j) cm[j] = fminf(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1]));
#pragma unroll
                        for (int w2 = 8; w2 >= 1; w2 >>= 1)
#pragma unroll
                            for (int j = 0; j < w2; ++j) cm[j] = fminf(cm[j], cm[j + w2]);
                        if (__any_sync(0xffffffffu, cm[0] < tv[3])) {
#pragma unroll
                            for (int j = 0; j < 32; ++j) {
                                const float v = __uint_as_float(r[j]);
                                const bool p3 = v < tv[3];
                                if (__any_sync(0xffffffffu, p3)) {
                                    const uint32_t c = col0 + j;
                                    const bool p2 = v < tv[2], p1 = v < tv[1], p0 = v < tv[0];
                                    const float o0 = tv[0], o1 = tv[1], o2 = tv[2];
                                    const uint32_t i0 = ti[0], i1 = ti[1], i2 = ti[2];
                                    tv[3] = p2 ? o2 : (p3 ? v : tv[3]);
                                    ti[3] = p2 ? i2 : (p3 ? c : ti[3]);
                                    tv[2] = p1 ? o1 : (p2 ? v : o2);
                                    ti[2] = p1 ? i1 : (p2 ? c : i2);
                                    tv[1] = p0 ? o0 : (p1 ? v : o1);
                                    ti[1] = p0 ? i0 : (p1 ? c : i1);
                                    tv[0] = p0 ? v : o0;
                                    ti[0] = p0 ? c : i0;
                                }
                            }
                        }
                    }
                }
                fence_before();
                __syncwarp();
                if (lane == 0) bar_arrive(&tempty[buf]);
            }
            if (row < a.n) {
                const float q = sqrtf(nxrow[row]) * (1.f + 1e-6f) + *a.cmax;
                const float E = big_error_bound(q * q * 1.01f + 1e-6f, kchunks);
                if constexpr (MAT) {
                    if (a.row_err) a.row_err[row] = E;
                } else {
                    const float band0 = tv[0] + 2.05f * E;
                    const float band = band0 + 4.f * kU * fabsf(band0);
                    if (tv[3] > band) {
                        // all possible fp64 winners are among the top 3: re-score exactly
                        double best = __longlong_as_double(0x7ff0000000000000LL);
                        uint32_t bj = 0xFFFFFFFFu;
                        for (int i = 0; i < 3; ++i) {
                            if (ti[i] == 0xFFFFFFFFu || !(tv[i] <= band)) continue;
                            const double dd = exact_row_dist(a, row, ti[i]);
                            if (dd < best || (dd == best && ti[i] < bj)) { best = dd; bj = ti[i]; }
                        }
                        if (bj != 0xFFFFFFFFu) {
                            store_index(a, row, bj);
                            if (a.out_dist) a.out_dist[row] = best;
                        } else {
                            const unsigned long long slot = atomicAdd(a.flag_count, 1ull);
                            a.flags[slot] = row_base + row;
                        }
                    } else {
                        const unsigned long long slot = atomicAdd(a.flag_count, 1ull);
                        a.flags[slot] = row_base + row;
                    }
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

bool umma_big_supported_impl(const NearestArgs& a) {
    if (a.B != 1) return false;  // single problem (coarse) only
    if (a.d < 24) return false;              // small d: the PQ kernels
    if (a.k < 64) return false;
    return true;
}

}  // namespace

bool umma_big_supported(const NearestArgs& a) { return umma_big_supported_impl(a); }

bool umma_big_prepare_rows(pqg_ctx* ctx, NearestArgs& a) {
    const char* mode = std::getenv("PQG_SCREEN");
    if (mode && std::strcmp(mode, "fp32") == 0) return false;
    NearestArgs probe = a;
    probe.active = nullptr;
    if (!umma_big_supported_impl(probe) || a.n > (uint64_t(2) << 20)) return false;
    const uint32_t kchunks = (a.d + 2 + kKC - 1) / kKC;
    const uint64_t ntiles = (a.n + kR - 1) / kR;
    uint8_t* Am = scratch<uint8_t>(ctx, ntiles * kchunks * 2 * kAChunk);
    float* nx = scratch<float>(ctx, a.n);
    launch(ctx, "big_split", row_norms_kernel, dim3(grid1d(a.n * 32, 256, 1u << 20)), dim3(256), 0, a.src,
           a.n, a.d, nx);
    launch(ctx, "big_split", split_rows_kernel, dim3(grid1d(ntiles * kR * kchunks * (kKC / 4), 256, 1u << 20)),
           dim3(256), 0, a.src, a.n, a.d, kchunks, a.cmax, 0, Am, (const float*)nx);
    a.big_rows = Am;
    a.big_nx = nx;
    return true;
}

void umma_big(pqg_ctx* ctx, const NearestArgs& a0) {
    const uint32_t kchunks = (a0.d + 2 + kKC - 1) / kKC;
    const uint32_t nblocks = uint32_t((a0.k + kN - 1) / kN);
    const uint64_t k_pad = uint64_t(nblocks) * kN;
    uint8_t* Bm = scratch<uint8_t>(ctx, uint64_t(nblocks) * kchunks * 2 * kBChunk);
    launch(ctx, "big_split", split_table_kernel, dim3(grid1d(k_pad * kchunks * (kKC / 4), 256, 1u << 20)),
           dim3(256), 0, a0.table, a0.cnorm, a0.k, a0.d, kchunks, k_pad, Bm);
    const size_t smem = size_t(kBigStages) * size_t(kStage);
    PQG_CUDA(cudaFuncSetAttribute(big_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    PQG_CUDA(cudaFuncSetAttribute(big_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    if (a0.big_rows) {  // rows prepared by umma_big_prepare_rows (single chunk)
        const uint64_t ntiles = (a0.n + kR - 1) / kR;
        const unsigned grid = unsigned(std::min<uint64_t>(ntiles, uint64_t(ctx->num_sms)));
        launch(ctx, "nearest_big_tc", big_kernel<false>, dim3(grid), dim3(192), smem, a0, a0.big_rows,
               (const uint8_t*)Bm, a0.big_nx, kchunks, nblocks, uint64_t(0));
        return;
    }
    // rows in chunks so the split operand stays <= ~2.5 GB of scratch
    const uint64_t chunk_rows = uint64_t(2) << 20;
    const auto mark = ctx->arena.mark();
    for (uint64_t r0 = 0; r0 < a0.n; r0 += chunk_rows) {
        ctx->arena.reset_to(mark);
        NearestArgs a = a0;
        a.n = std::min<uint64_t>(chunk_rows, a0.n - r0);
        if (a.src.codes) a.src.codes += r0 * a.src.dM * a.src.dw;
        else a.src.x += r0 * a.src.ldx;
        const uint64_t ntiles = (a.n + kR - 1) / kR;
        uint8_t* Am = scratch<uint8_t>(ctx, ntiles * kchunks * 2 * kAChunk);
        float* nx = scratch<float>(ctx, a.n);
        launch(ctx, "big_split", row_norms_kernel, dim3(grid1d(a.n * 32, 256, 1u << 20)), dim3(256), 0, a.src,
               a.n, a.d, nx);
        launch(ctx, "big_split", split_rows_kernel,
               dim3(grid1d(ntiles * kR * kchunks * (kKC / 4), 256, 1u << 20)), dim3(256), 0, a.src, a.n, a.d,
               kchunks, a.cmax, a.out_mat ? 1 : 0, Am, (const float*)nx);
        const unsigned grid = unsigned(std::min<uint64_t>(ntiles, uint64_t(ctx->num_sms)));
        if (a.out_mat) {
            a.out_mat += r0 * a.ld_mat;
            if (a.row_err) a.row_err += r0;
            launch(ctx, "distance_matrix_tc", big_kernel<true>, dim3(grid), dim3(192), smem, a,
                   (const uint8_t*)Am, (const uint8_t*)Bm, (const float*)nx, kchunks, nblocks, r0);
        } else {
            a.out_idx = static_cast<uint8_t*>(a.out_idx) + r0 * a.idx_rs * uint64_t(a.idx_bytes);
            if (a.out_dist) a.out_dist += r0;
            launch(ctx, "nearest_big_tc", big_kernel<false>, dim3(grid), dim3(192), smem, a,
                   (const uint8_t*)Am, (const uint8_t*)Bm, (const float*)nx, kchunks, nblocks, r0);
        }
    }
}

}  // namespace pqg
