// nearest.cu -- K1/K3/K5: batched nearest-centroid search with an fp32
// tensor-style screen and an exact fp64 fixup.
//
// Replaces the reference's innermost loop nearest_in_table / squared_l2
// (proj/src/kmeans.cpp:11-31), called by assign_pass (:46-57), pq_encode
// (proj/src/pq.cpp:95-111) and assign_items (proj/src/ivf.cpp:36-49).
//
// Screen: per CTA a 128-row tile against 16*TN centroids at a time; every
// thread owns an 8 x TN block of the row-by-centroid distance matrix in
// registers, computed in the expanded form ||c||^2 - 2 x.c + C_row with fp32
// FMAs (x staged in shared memory pre-scaled by -2, which is exact).  C_row
// (>= ||x||^2 plus a margin) makes every screened value non-negative, so a
// value's bit pattern orders like the value and the low 3 bits can carry the
// thread-local column: the running best / second-best are two IMNMX each.
//
// Exactness: E_row bounds |screened - exact| (fp32 rounding of the expanded
// form, (d+4) u (||x|| + max||c||)^2, doubled).  When the second-best lower
// bound exceeds the best upper bound by more than 2 E_row the fp32 winner is
// provably the fp64 winner of the reference (whose own rounding is ~1e-16
// relative).  Otherwise the (row, problem) pair is appended to a flag list
// and the fixup kernel recomputes it exhaustively in the reference's exact
// fp64 arithmetic (strict '<', lowest index on ties).  The result is
// bit-identical to nearest_in_table for every row.
#include <cfloat>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include <cstdio>

#include "kernels.cuh"
#include "tc_common.cuh"
#include "tmap.cuh"

namespace pqg {

namespace {

constexpr int BM = 128;  // rows per CTA
constexpr int TM = 8;    // rows per thread
constexpr int NT = 256;  // threads per CTA (16 column groups x 16 row groups)
constexpr int LDX = BM + 4;
constexpr int BK = 32;   // K chunk of the generic (large-d) variant

__device__ __forceinline__ uint32_t read_code(const uint8_t* p, uint32_t w) {
    return w == 1 ? uint32_t(p[0]) : (uint32_t(p[0]) | (uint32_t(p[1]) << 8));
}

__device__ __forceinline__ float load_x(const RowSrc& s, uint64_t i, uint32_t b, uint32_t t) {
    if (s.codes) {
        const uint32_t m = t / s.dds, tt = t - m * s.dds;
        uint32_t code = read_code(s.codes + (i * s.dM + m) * s.dw, s.dw);
        if (code >= s.dks) code = s.dks - 1;  // validated on the host side path
        return __ldg(s.dtab + ((uint64_t)m * s.dks + code) * s.dds + tt);
    }
    return __ldg(s.x + i * s.ldx + (uint64_t)b * s.col_stride + t);
}

__device__ __forceinline__ void store_index(const NearestArgs& a, uint64_t i, uint32_t b,
                                            uint32_t idx) {
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

__device__ __forceinline__ double exact_dist(const NearestArgs& a, uint64_t i, uint32_t b,
                                             const float* crow) {
    double acc = 0.0;
    for (uint32_t t = 0; t < a.d; ++t) {
        const double diff = __dsub_rn((double)load_x(a.src, i, b, t), (double)__ldg(crow + t));
        acc = __dadd_rn(acc, __dmul_rn(diff, diff));
    }
    return acc;
}

// Column owned by thread tx, slot j, within a 16*TN-wide tile.  TN == 8 is
// split into two 4-wide halves so each float4 shared load of a warp covers
// 256 contiguous bytes.
template <int TN>
__device__ __forceinline__ int col_of(int tx, int j) {
    if constexpr (TN == 8) return j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4);
    else return tx * TN + j;
}

template <int TN>
__device__ __forceinline__ void load_c(const float* Cs_t, int tx, float (&c)[TN]) {
    if constexpr (TN == 8) {
        const float4 u = *reinterpret_cast<const float4*>(Cs_t + tx * 4);
        const float4 v = *reinterpret_cast<const float4*>(Cs_t + 64 + tx * 4);
        c[0] = u.x; c[1] = u.y; c[2] = u.z; c[3] = u.w;
        c[4] = v.x; c[5] = v.y; c[6] = v.z; c[7] = v.w;
    } else if constexpr (TN == 4) {
        const float4 u = *reinterpret_cast<const float4*>(Cs_t + tx * 4);
        c[0] = u.x; c[1] = u.y; c[2] = u.z; c[3] = u.w;
    } else if constexpr (TN == 2) {
        const float2 u = *reinterpret_cast<const float2*>(Cs_t + tx * 2);
        c[0] = u.x; c[1] = u.y;
    } else {
        c[0] = Cs_t[tx];
    }
}

// DP > 0: the whole (padded) dimension fits one chunk and is a compile-time
// constant (PQ subspaces, Ds in {4, 8, 16, 32}); DP == 0: generic d streamed
// in chunks of BK.  MAT: write the screened matrix instead of the argmin.
template <int TN, int DP, bool MAT>
__global__ void __launch_bounds__(NT, 2) nearest_kernel(NearestArgs a) {
    constexpr int BN = 16 * TN;
    constexpr int LDC = BN + 4;
    constexpr int KCH = DP > 0 ? DP : BK;
    extern __shared__ __align__(16) float smem[];
    float* rowC = smem;               // [BM]
    float* rowE = rowC + BM;          // [BM]
    float* Xs = rowE + BM;            // [KCH][LDX], -2 * x
    float* Cs = Xs + KCH * LDX;       // [KCH][LDC]
    float* cn_s = Cs + KCH * LDC;     // [BN]

    // problem index fastest: the B CTAs that read the same rows run together,
    // so each row is fetched from HBM once and served to the others by L2
    const uint32_t b = blockIdx.x % a.B;
    if (a.active && !a.active[b]) return;
    const uint64_t i0 = (uint64_t)(blockIdx.x / a.B) * BM;
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int d = int(a.d);
    const int dp = (d + 3) & ~3;
    const uint64_t k = a.k;
    const float* tab = a.table + (uint64_t)b * k * d;
    const float* cnb = a.cnorm + (uint64_t)b * k;
    const float cmax = a.cmax[b];
    const int rows_here = int(min64(BM, a.n - i0));

    auto load_x_chunk = [&](int t0, int kc) {
        for (int e = tid; e < BM * kc; e += NT) {
            const int r = e / kc, tt = e - r * kc;
            float v = 0.f;
            if (r < rows_here && t0 + tt < d) v = load_x(a.src, i0 + r, b, uint32_t(t0 + tt));
            Xs[tt * LDX + r] = -2.f * v;
        }
    };
    auto load_c_chunk = [&](uint64_t n0, int t0, int kc) {
        for (int e = tid; e < BN * kc; e += NT) {
            const int jj = e / kc, tt = e - jj * kc;
            const uint64_t j = n0 + jj;
            float v = 0.f;
            if (j < k && t0 + tt < d) v = __ldg(tab + j * d + t0 + tt);
            Cs[tt * LDC + jj] = v;
        }
    };

    // ---- row norms -> C_row (offset that keeps screened values >= 0) and E_row
    {
        float s = 0.f;
        if constexpr (DP > 0) {
            load_x_chunk(0, DP);
            __syncthreads();
            if (tid < BM) {
#pragma unroll
                for (int t = 0; t < DP; ++t) {
                    const float v = Xs[t * LDX + tid];
                    s = fmaf(v, v, s);
                }
            }
        } else {
            for (int t0 = 0; t0 < dp; t0 += BK) {
                const int kc = min(BK, dp - t0);
                __syncthreads();
                load_x_chunk(t0, kc);
                __syncthreads();
                if (tid < BM)
                    for (int t = 0; t < kc; ++t) {
                        const float v = Xs[t * LDX + tid];
                        s = fmaf(v, v, s);
                    }
            }
        }
        if (tid < BM) {
            const float nx = 0.25f * s;
            const float q = sqrtf(nx) * (1.f + 1e-6f) + cmax;
            const float E = 2.f * float(d + 4) * kU * q * q + 1e-30f;
            rowE[tid] = E;
            rowC[tid] = nx * (1.f + 2.f * float(d + 2) * kU) + 2.f * E;
            if constexpr (MAT) {
                if (tid < rows_here) a.row_err[i0 + tid] = E;
            }
        }
    }

    uint32_t m1[TM], m2[TM], t1[TM];
#pragma unroll
    for (int i = 0; i < TM; ++i) { m1[i] = 0xFFFFFFFFu; m2[i] = 0xFFFFFFFFu; t1[i] = 0; }

    const uint64_t ntiles = (k + BN - 1) / BN;
    for (uint64_t nt = 0; nt < ntiles; ++nt) {
        const uint64_t n0 = nt * BN;
        float acc[TM][TN];
        __syncthreads();
        for (int jj = tid; jj < BN; jj += NT) {
            const uint64_t j = n0 + jj;
            cn_s[jj] = j < k ? __ldg(cnb + j) : __int_as_float(0x7f800000);
        }
        if constexpr (DP > 0) {
            load_c_chunk(n0, 0, DP);
            __syncthreads();
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) acc[i][j] = cn_s[col_of<TN>(tx, j)] + rowC[ty * 8 + i];
#pragma unroll
            for (int t = 0; t < DP; ++t) {
                const float4 xa = *reinterpret_cast<const float4*>(Xs + t * LDX + ty * 8);
                const float4 xb = *reinterpret_cast<const float4*>(Xs + t * LDX + ty * 8 + 4);
                const float xr[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
                float cr[TN];
                load_c<TN>(Cs + t * LDC, tx, cr);
#pragma unroll
                for (int i = 0; i < TM; ++i)
#pragma unroll
                    for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(xr[i], cr[j], acc[i][j]);
            }
        } else {
            __syncthreads();
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) acc[i][j] = cn_s[col_of<TN>(tx, j)] + rowC[ty * 8 + i];
            for (int t0 = 0; t0 < dp; t0 += BK) {
                const int kc = min(BK, dp - t0);
                __syncthreads();
                load_x_chunk(t0, kc);
                load_c_chunk(n0, t0, kc);
                __syncthreads();
#pragma unroll 4
                for (int t = 0; t < kc; ++t) {
                    const float4 xa = *reinterpret_cast<const float4*>(Xs + t * LDX + ty * 8);
                    const float4 xb = *reinterpret_cast<const float4*>(Xs + t * LDX + ty * 8 + 4);
                    const float xr[8] = {xa.x, xa.y, xa.z, xa.w, xb.x, xb.y, xb.z, xb.w};
                    float cr[TN];
                    load_c<TN>(Cs + t * LDC, tx, cr);
#pragma unroll
                    for (int i = 0; i < TM; ++i)
#pragma unroll
                        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(xr[i], cr[j], acc[i][j]);
                }
            }
        }

        // ---- epilogue of this column tile
        if constexpr (MAT) {
#pragma unroll
            for (int i = 0; i < TM; ++i) {
                const int r = ty * 8 + i;
                if (r >= rows_here) continue;
                float* out = a.out_mat + (i0 + r) * a.ld_mat;
#pragma unroll
                for (int j = 0; j < TN; ++j) {
                    const uint64_t col = n0 + col_of<TN>(tx, j);
                    if (col < k) out[col] = acc[i][j];
                }
            }
        } else {
#pragma unroll
            for (int i = 0; i < TM; ++i) {
                const uint32_t old = m1[i];
#pragma unroll
                for (int j = 0; j < TN; ++j) {
                    const uint32_t key = (__float_as_uint(acc[i][j]) & ~7u) | uint32_t(j);
                    m2[i] = min(m2[i], max(m1[i], key));
                    m1[i] = min(m1[i], key);
                }
                t1[i] = (m1[i] != old) ? uint32_t(nt) : t1[i];
            }
        }
    }
    if constexpr (MAT) return;

    // ---- combine the 16 column groups of each row through shared memory:
    // every thread parks (best key|column, second-best value) of its 8 rows,
    // then one thread per row folds the 16 entries.
    __syncthreads();
    uint64_t* redK = reinterpret_cast<uint64_t*>(smem + 2 * BM);  // [BM][16] (reuses Xs/Cs)
    uint32_t* redV = reinterpret_cast<uint32_t*>(redK + BM * 16);  // [BM][16]
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const uint32_t col = uint32_t(t1[i]) * BN + uint32_t(col_of<TN>(tx, int(m1[i] & 7u)));
        redK[(ty * 8 + i) * 16 + tx] = (uint64_t(m1[i] & ~7u) << 32) | col;
        redV[(ty * 8 + i) * 16 + tx] = m2[i] & ~7u;
    }
    __syncthreads();
    if (tid >= rows_here) return;
    uint64_t K = redK[tid * 16];
    uint32_t V2 = redV[tid * 16];
#pragma unroll
    for (int g = 1; g < 16; ++g) {
        const uint64_t oK = redK[tid * 16 + g];
        const uint32_t oV = redV[tid * 16 + g];
        V2 = min(min(V2, oV), uint32_t(max(K, oK) >> 32));
        K = min(K, oK);
    }
    const uint64_t row = i0 + tid;
    const uint32_t v1hi = uint32_t(K >> 32);
    const uint32_t idx = uint32_t(K);
    const float E = rowE[tid];
    // non-finite E (inf/NaN in the row or table) or best: the exact fixup decides
            const bool unique = isfinite(E) && v1hi < 0x7f800000u && ((V2 >= 0x7f800000u) ||
                        (__uint_as_float(V2) - __uint_as_float(v1hi | 7u) > 2.05f * E));
    if (unique) {
        store_index(a, row, b, idx);
        if (a.out_dist) a.out_dist[(uint64_t)b * a.n + row] = exact_dist(a, row, b, tab + (uint64_t)idx * d);
    } else {
        const unsigned long long slot = atomicAdd(a.flag_count, 1ull);
        a.flags[slot] = (uint64_t(b) << 40) | row;
    }
}

// Exact argmin for flagged (row, problem) pairs, one warp per pair.
// Pass 1: fp32 direct-form distances (relative error <= eps = (d+2)u), warp
// minimum vmin.  A candidate can tie or beat the fp64 winner only if its fp32
// value is <= vmin (1+eps)/(1-eps); pass 2 re-scores exactly those in the
// reference's fp64 arithmetic and takes the (dist, index) minimum -- the
// result of nearest_in_table (strict '<', lowest index on ties).
constexpr int kFixThreads = 256;
constexpr int kFixMaxD = 512;

// Exact resolution of the flagged (row, problem) pairs: one CTA per pair, its
// threads split the k centroids (a single flagged row no longer runs on one
// warp's latency).  Pass 1: fp32 distances, block minimum; pass 2: every
// centroid whose fp32 distance is within the fp32 error of that minimum is
// re-scored in the reference's fp64 arithmetic (kmeans.cpp:11-31), strict '<'
// with the lowest index on ties.
__global__ void __launch_bounds__(kFixThreads, 1) fixup_kernel(NearestArgs a, int tstaged) {
    __shared__ float xs[kFixMaxD];
    extern __shared__ float tsm[];  // tstaged: the problem's table, rows padded to d+1 floats
    uint32_t staged_b = 0xFFFFFFFFu;
    __shared__ float red_f[kFixThreads / 32];
    __shared__ double red_d[kFixThreads / 32];
    __shared__ uint32_t red_j[kFixThreads / 32];
    const unsigned long long cnt = *a.flag_count;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t d = a.d;
    const bool staged = d <= kFixMaxD;
    const float eps = float(d + 2) * kU * 1.01f;
    for (uint64_t f = blockIdx.x; f < cnt; f += gridDim.x) {
        const uint64_t item = a.flags[f];
        const uint32_t b = uint32_t(item >> 40);
        const uint64_t row = item & ((uint64_t(1) << 40) - 1);
        const float* tab = a.table + (uint64_t)b * a.k * d;
        __syncthreads();  // previous item's reductions are consumed
        if (staged)
            for (uint32_t t = threadIdx.x; t < d; t += blockDim.x) xs[t] = load_x(a.src, row, b, t);
        if (tstaged && b != staged_b) {  // coalesced once per problem, not per distance
            const uint64_t kd = a.k * d;
            for (uint64_t e0 = threadIdx.x; e0 < kd; e0 += 8 * blockDim.x) {
                float v[8];  // eight loads in flight per thread (clamped, unpredicated)
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = __ldg(tab + min64(e0 + u * blockDim.x, kd - 1));
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint64_t e = e0 + u * blockDim.x;
                    if (e >= kd) break;
                    const uint64_t j = e / d;
                    tsm[j * (d + 1) + (e - j * d)] = v[u];
                }
            }
            staged_b = b;
        }
        __syncthreads();
        auto xval = [&](uint32_t t) { return staged ? xs[t] : load_x(a.src, row, b, t); };
        auto cval = [&](uint64_t j, uint32_t t) { return tstaged ? tsm[j * (d + 1) + t] : __ldg(tab + j * d + t); };
        auto fdist = [&](uint64_t j) {
            float v = 0.f;
            for (uint32_t t = 0; t < d; ++t) {
                const float df = xval(t) - cval(j, t);
                v = fmaf(df, df, v);
            }
            return v;
        };
        float vmin = __int_as_float(0x7f800000);
        for (uint64_t j = threadIdx.x; j < a.k; j += blockDim.x) vmin = fminf(vmin, fdist(j));
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) vmin = fminf(vmin, __shfl_xor_sync(0xffffffffu, vmin, off));
        if (lane == 0) red_f[wid] = vmin;
        __syncthreads();
        vmin = red_f[0];
        for (int w = 1; w < kFixThreads / 32; ++w) vmin = fminf(vmin, red_f[w]);
        const float thr = vmin * ((1.f + eps) / (1.f - eps)) * (1.f + 4.f * kU) + 1e-37f;
        double best = __longlong_as_double(0x7ff0000000000000LL);
        uint32_t bj = 0xFFFFFFFFu;
        for (uint64_t j = threadIdx.x; j < a.k; j += blockDim.x) {
            const float v = fdist(j);
            if (!(v <= thr) && !(v != v)) continue;  // NaN candidates go to the exact path
            double acc = 0.0;
            for (uint32_t t = 0; t < d; ++t) {
                const double diff = __dsub_rn((double)xval(t), (double)cval(j, t));
                acc = __dadd_rn(acc, __dmul_rn(diff, diff));
            }
            if (acc < best || (acc == best && uint32_t(j) < bj)) { best = acc; bj = uint32_t(j); }
        }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, off);
            const uint32_t oj = __shfl_xor_sync(0xffffffffu, bj, off);
            if (ob < best || (ob == best && oj < bj)) { best = ob; bj = oj; }
        }
        if (lane == 0) {
            red_d[wid] = best;
            red_j[wid] = bj;
        }
        __syncthreads();
        if (threadIdx.x == 0) {  // holds warp 0's result; merge the other warps
            for (int w = 1; w < kFixThreads / 32; ++w)
                if (red_d[w] < best || (red_d[w] == best && red_j[w] < bj)) {
                    best = red_d[w];
                    bj = red_j[w];
                }
            // nearest_in_table starts from (0, d_0) and only a strictly smaller
            // distance replaces it (kmeans.cpp:20-31): a NaN d_0 is never replaced
            // and NaN distances never win
            double d0 = 0.0;  // exact_dist to codeword 0, from the staged copies
            for (uint32_t t = 0; t < d; ++t) {
                const double diff = __dsub_rn((double)xval(t), (double)cval(0, t));
                d0 = __dadd_rn(d0, __dmul_rn(diff, diff));
            }
            if (bj == 0xFFFFFFFFu || d0 != d0) {
                bj = 0;
                best = d0;
            }
            store_index(a, row, b, bj);
            if (a.out_dist) a.out_dist[(uint64_t)b * a.n + row] = best;
        }
    }
}

// Flagged pairs of the PQ subspaces (d = DS in {4, 8, 16, 32}, rows of x and
// the table 16-byte aligned, no decoded-row source): one warp per pair, the
// row in registers, lane j scoring codewords j, j+32, ... from the (L1-
// resident) table with float4 loads; the same fp32 pass / threshold / fp64
// re-score / (0, d_0) rule as fixup_kernel.  Pairs are taken in flag order,
// a warp per pair across the whole GPU -- no per-pair block barriers.
template <int DS>
__global__ void __launch_bounds__(256) fixup_warp_kernel(NearestArgs a) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t gw = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    const unsigned long long cnt = *a.flag_count;
    const uint64_t k = a.k;
    constexpr float eps = float(DS + 2) * kU * 1.01f;
    for (uint64_t f = gw; f < cnt; f += nw) {
        const uint64_t item = __ldcg(a.flags + f);
        const uint32_t b = uint32_t(item >> 40);
        const uint64_t row = item & ((uint64_t(1) << 40) - 1);
        const float* tab = a.table + (uint64_t)b * k * DS;
        float x[DS];
        const float4* xp = reinterpret_cast<const float4*>(a.src.x + row * a.src.ldx + (uint64_t)b * a.src.col_stride);
#pragma unroll
        for (int t = 0; t < DS; t += 4) {
            const float4 v = __ldg(xp + t / 4);
            x[t] = v.x; x[t + 1] = v.y; x[t + 2] = v.z; x[t + 3] = v.w;
        }
        auto fdist = [&](uint64_t j) {
            const float4* c = reinterpret_cast<const float4*>(tab + j * DS);
            float c4[DS];
#pragma unroll
            for (int t = 0; t < DS; t += 4) {
                const float4 v = __ldg(c + t / 4);
                c4[t] = v.x; c4[t + 1] = v.y; c4[t + 2] = v.z; c4[t + 3] = v.w;
            }
            float v = 0.f;
#pragma unroll
            for (int t = 0; t < DS; ++t) {
                const float df = x[t] - c4[t];
                v = fmaf(df, df, v);
            }
            return v;
        };
        // r2e: k <= 256 (PQ codebooks) -- a lane's eight codewords scored with
        // all their loads in flight and kept in registers for the second pass
        // (the per-pair chain of dependent L2 round trips was the kernel)
        constexpr int kPer = 8;
        float vr[kPer];
        const bool small = k <= uint64_t(32 * kPer);
        float vmin = __int_as_float(0x7f800000);
        if (small) {
#pragma unroll
            for (int i = 0; i < kPer; ++i) {
                const uint64_t j = lane + 32u * i;
                vr[i] = j < k ? fdist(j) : __int_as_float(0x7f800000);
            }
#pragma unroll
            for (int i = 0; i < kPer; ++i) vmin = fminf(vmin, vr[i]);
        } else {
            for (uint64_t j = lane; j < k; j += 32) vmin = fminf(vmin, fdist(j));
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) vmin = fminf(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
        const float thr = vmin * ((1.f + eps) / (1.f - eps)) * (1.f + 4.f * kU) + 1e-37f;
        double best = __longlong_as_double(0x7ff0000000000000LL);
        uint32_t bj = 0xFFFFFFFFu;
        for (uint64_t j = lane, i = 0; j < k; j += 32, ++i) {
            float v = 0.f;
            if (small) {
#pragma unroll
                for (int u = 0; u < kPer; ++u)
                    if (uint64_t(u) == i) v = vr[u];
            } else {
                v = fdist(j);
            }
            if (!(v <= thr) && !(v != v)) continue;  // NaN candidates go to the exact path
            const float* c = tab + j * DS;
            double acc = 0.0;
#pragma unroll
            for (int t = 0; t < DS; ++t) {
                const double diff = __dsub_rn((double)x[t], (double)__ldg(c + t));
                acc = __dadd_rn(acc, __dmul_rn(diff, diff));
            }
            if (acc < best || (acc == best && uint32_t(j) < bj)) { best = acc; bj = uint32_t(j); }
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const uint32_t oj = __shfl_xor_sync(0xffffffffu, bj, o);
            if (ob < best || (ob == best && oj < bj)) { best = ob; bj = oj; }
        }
        if (lane == 0) {
            // nearest_in_table starts from (0, d_0), strict '<' (kmeans.cpp:20-31):
            // a NaN d_0 is never replaced and NaN distances never win
            double d0 = 0.0;
#pragma unroll
            for (int t = 0; t < DS; ++t) {
                const double diff = __dsub_rn((double)x[t], (double)__ldg(tab + t));
                d0 = __dadd_rn(d0, __dmul_rn(diff, diff));
            }
            if (bj == 0xFFFFFFFFu || d0 != d0) {
                bj = 0;
                best = d0;
            }
            store_index(a, row, b, bj);
            if (a.out_dist) a.out_dist[(uint64_t)b * a.n + row] = best;
        }
    }
}

// Small tables (Ks <= 16 and Ds in {4, 8, 32}: the narrow-codebook encodes
// and fits): thread per row, the problem's subspaces in one pass, the whole
// codebook in shared memory read as broadcast float4s.  Same screened value
// and bound as nearest_kernel's FP32 screen: acc_j = (C_r + ||c_j||^2) +
// sum_t (-2x_t) c_jt (fma chain), E = 2 (Ds+4) u q^2; a row whose runner-up
// is within 2.05 E of its best goes to the exact fixup.  Measured r1 (1M x
// 128, encode): Ks=16 M=4 2.8 -> 3.6, M=16 2.4 -> 2.7, M=32 1.5 -> 2.0 G
// vectors/s against the tensor-core screen, which re-stages every (row,
// subspace) as a 128-row MMA tile; slower at Ds=16 and at Ks=64.
constexpr int kSmallThreads = 128;
template <int DS>
__global__ void __launch_bounds__(kSmallThreads) small_table_kernel(NearestArgs a) {
    extern __shared__ __align__(16) float st[];  // [B][k][DS] then cnorm [B][k]
    const uint32_t B = a.B;
    const uint64_t k = a.k;
    float* cn_s = st + uint64_t(B) * k * DS;
    for (uint64_t e = threadIdx.x; e < uint64_t(B) * k * DS; e += blockDim.x) st[e] = __ldg(a.table + e);
    for (uint64_t e = threadIdx.x; e < uint64_t(B) * k; e += blockDim.x) cn_s[e] = __ldg(a.cnorm + e);
    __syncthreads();
    constexpr float kE = 2.f * float(DS + 4) * kU;
    for (uint64_t row = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; row < a.n;
         row += uint64_t(gridDim.x) * blockDim.x) {
        for (uint32_t b = 0; b < B; ++b) {
            if (a.active && !a.active[b]) continue;
            float x[DS];
            const float4* xp = reinterpret_cast<const float4*>(a.src.x + row * a.src.ldx + uint64_t(b) * a.src.col_stride);
#pragma unroll
            for (int t = 0; t < DS; t += 4) {
                const float4 v = __ldg(xp + t / 4);
                x[t] = -2.f * v.x; x[t + 1] = -2.f * v.y; x[t + 2] = -2.f * v.z; x[t + 3] = -2.f * v.w;
            }
            float s = 0.f;
#pragma unroll
            for (int t = 0; t < DS; ++t) s = fmaf(x[t], x[t], s);
            const float nx = 0.25f * s;
            const float q = sqrtf(nx) * (1.f + 1e-6f) + a.cmax[b];
            const float E = kE * q * q + 1e-30f;
            const float C = nx * (1.f + 2.f * float(DS + 2) * kU) + 2.f * E;
            const float* tb = st + uint64_t(b) * k * DS;
            const float* cnb = cn_s + uint64_t(b) * k;
            float b1 = __int_as_float(0x7f800000), b2 = b1;
            uint32_t i1 = 0;
#pragma unroll 4
            for (uint32_t j = 0; j < k; ++j) {
                float acc = cnb[j] + C;
                const float4* c4 = reinterpret_cast<const float4*>(tb + uint64_t(j) * DS);
#pragma unroll
                for (int t = 0; t < DS; t += 4) {
                    const float4 c = c4[t / 4];
                    acc = fmaf(x[t], c.x, acc);
                    acc = fmaf(x[t + 1], c.y, acc);
                    acc = fmaf(x[t + 2], c.z, acc);
                    acc = fmaf(x[t + 3], c.w, acc);
                }
                if (acc < b1) {  // strict: the lowest column keeps equal values
                    b2 = b1;
                    b1 = acc;
                    i1 = j;
                } else {
                    b2 = fminf(b2, acc);
                }
            }
            const bool unique = isfinite(E) && b1 < __int_as_float(0x7f800000) &&
                                (!(b2 < __int_as_float(0x7f800000)) || b2 - b1 > 2.05f * E);
            if (unique) {
                store_index(a, row, b, i1);
                if (a.out_dist) {  // -0.5 * (-2x) == x exactly
                    const float* c = tb + uint64_t(i1) * DS;
                    double acc = 0.0;
#pragma unroll
                    for (int t = 0; t < DS; ++t) {
                        const double diff = __dsub_rn((double)(-0.5f * x[t]), (double)c[t]);
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

// Row-blocked screen for narrow codebooks (r2): Ks <= 32, Ds in {4, 8, 16, 32}.
// The whole codebook sits in shared memory.  A warp owns 64-row blocks (lane
// L: rows L and L+32); the rows reach shared memory by 2-D TMA, one box of
// 64 rows x 32 floats (SG = 32/Ds subspaces) at a time, 128-byte swizzled so
// a lane reading its row's 16-byte chunks hits distinct bank groups, double-
// buffered per warp (the next box is in flight while this one is screened:
// per-subspace 16-byte row slices read straight from HBM left the kernel
// latency- and L2-bound).  Per codeword pair a lane reads the two codewords
// once (broadcast LDS.128) for both rows and advances them together with
// packed FFMA2 (the rows in the two halves, the codeword coordinate as the
// scalar operand); keys are value_bits * 32 + j (one IMAD, the per-row offset
// window of the register-resident kernel below), five ALU min/max per
// codeword pair and row.  Bound and fixup hand-off as in small_table_kernel.
constexpr int kRowWarps = 4;
constexpr int kRowRows = 64;  // rows per warp block

template <int DS, int KS, bool PADK>
__global__ void __launch_bounds__(kRowWarps * 32) row_screen_kernel(NearestArgs a, uint32_t m32,
                                                                    const __grid_constant__ CUtensorMap xmap) {
    extern __shared__ __align__(1024) uint8_t smem_rs[];
    constexpr int KP = KS / 2;
    constexpr int SG = 32 / DS;          // subspaces per staged box
    constexpr uint32_t BOX = kRowRows * 128;  // bytes per box
    constexpr float kE = 2.f * float(DS + 4) * kU;
    __shared__ uint64_t bars[kRowWarps][2];
    const uint32_t B = a.B;
    const uint32_t k = uint32_t(a.k);
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint8_t* xbuf = smem_rs + size_t(warp) * 2 * BOX;                                   // [2][64][128 B]
    float* st = reinterpret_cast<float*>(smem_rs + size_t(kRowWarps) * 2 * BOX);      // [B][KS][DS]
    float* cn_s = st + size_t(B) * KS * DS;                                            // [B][KS]
    for (uint32_t e = threadIdx.x; e < B * KS * DS; e += blockDim.x) {
        const uint32_t b = e / (KS * DS), r = e - b * (KS * DS), j = r / DS;
        st[e] = j < k ? __ldg(a.table + (uint64_t(b) * k + j) * DS + (r - j * DS)) : 0.f;
    }
    for (uint32_t e = threadIdx.x; e < B * KS; e += blockDim.x) {
        const uint32_t b = e / KS, j = e - b * KS;
        cn_s[e] = j < k ? __ldg(a.cnorm + uint64_t(b) * k + j) : 0.f;
    }
    if (lane == 0) {
        tc::bar_init(&bars[warp][0], 1);
        tc::bar_init(&bars[warp][1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint64_t nblk = (a.n + kRowRows - 1) / kRowRows;
    const uint32_t ngrp = (B + SG - 1) / SG;
    const uint64_t w0 = uint64_t(blockIdx.x) * kRowWarps + warp, wstep = uint64_t(gridDim.x) * kRowWarps;
    // the warp's sequence of (block, group) boxes; box i goes to buffer i & 1
    auto issue = [&](uint64_t i) {
        const uint64_t blk = w0 + (i / ngrp) * wstep;
        if (blk >= nblk) return;
        const uint32_t g = uint32_t(i % ngrp);
        uint64_t* bar = &bars[warp][i & 1];
        tc::bar_expect_tx(bar, BOX);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
            :: "r"(tc::smem_u32(xbuf + (i & 1) * BOX)), "l"(reinterpret_cast<uint64_t>(&xmap)),
               "r"(int(g * SG * DS)), "r"(int(blk * kRowRows)), "r"(tc::smem_u32(bar)) : "memory");
    };
    if (lane == 0) issue(0);
    for (uint64_t i = 0;; ++i) {
        const uint64_t blk = w0 + (i / ngrp) * wstep;
        if (blk >= nblk) break;
        const uint32_t g = uint32_t(i % ngrp);
        if (lane == 0) issue(i + 1);  // its buffer was released by the __syncwarp of box i - 1
        tc::bar_wait(&bars[warp][i & 1], uint32_t(i >> 1) & 1u);
        const uint8_t* xb = xbuf + (i & 1) * BOX;
        const uint64_t row0 = blk * kRowRows + lane, row1 = row0 + 32;
        const bool on0 = row0 < a.n, on1 = row1 < a.n;
        for (uint32_t sj = 0; sj < SG; ++sj) {
            const uint32_t b = g * SG + sj;
            if (b >= B) break;
            if (a.active && !a.active[b]) continue;
            // the two rows' sub-vectors (swizzled chunks c ^ (row & 7)), as -2x pairs
            float2 xa[DS];
            float nxa = 0.f, nxb = 0.f;
#pragma unroll
            for (int q = 0; q < DS / 4; ++q) {
                const uint32_t c = sj * (DS / 4) + q;
                const float4 u = *reinterpret_cast<const float4*>(xb + lane * 128 + ((c ^ (lane & 7)) << 4));
                const float4 v = *reinterpret_cast<const float4*>(xb + (lane + 32) * 128 + ((c ^ (lane & 7)) << 4));
                const float uu[4] = {-2.f * u.x, -2.f * u.y, -2.f * u.z, -2.f * u.w};
                const float vv[4] = {-2.f * v.x, -2.f * v.y, -2.f * v.z, -2.f * v.w};
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    xa[4 * q + w] = make_float2(uu[w], vv[w]);
                    nxa = fmaf(uu[w], uu[w], nxa);
                    nxb = fmaf(vv[w], vv[w], nxb);
                }
            }
            const float cm = a.cmax[b];
            float E[2], Cc[2];
            uint32_t hi4[2];
#pragma unroll
            for (int i2 = 0; i2 < 2; ++i2) {
                const float nx = 0.25f * (i2 ? nxb : nxa);
                const float S = 2.f * (nx * (1.f + 1e-6f) + cm * cm) + 1e-6f;
                int e = int((__float_as_uint(S) >> 23) & 0xFF) - 127;
                e = max(-60, min(e, 100));
                const int pw = (e & ~15) + 1;  // smallest p >= e - 14 with p = 1 (mod 16)
                const float O = __uint_as_float(uint32_t(pw + 127) << 23);
                hi4[i2] = uint32_t(pw + 127) >> 4;
                E[i2] = kE * (S + O) * 1.001f + 1e-30f;
                Cc[i2] = nx * (1.f + 2.f * float(DS + 2) * kU) + 2.f * E[i2] + O;
            }
            const float2 C2 = make_float2(Cc[0], Cc[1]);
            uint32_t m1[2][2], m2[2][2];
#pragma unroll
            for (int i2 = 0; i2 < 2; ++i2) m1[i2][0] = m1[i2][1] = m2[i2][0] = m2[i2][1] = 0xFFFFFFFFu;
            const float* tb = st + size_t(b) * KS * DS;
            const float* cnb = cn_s + size_t(b) * KS;
#pragma unroll
            for (int p = 0; p < KP; ++p) {
                const float2 cnp = *reinterpret_cast<const float2*>(cnb + 2 * p);
                float2 a0 = __fadd2_rn(C2, make_float2(cnp.x, cnp.x));
                float2 a1 = __fadd2_rn(C2, make_float2(cnp.y, cnp.y));
#pragma unroll
                for (int t = 0; t < DS; t += 4) {
                    const float4 c0 = *reinterpret_cast<const float4*>(tb + (2 * p) * DS + t);
                    const float4 c1 = *reinterpret_cast<const float4*>(tb + (2 * p + 1) * DS + t);
                    const float v0[4] = {c0.x, c0.y, c0.z, c0.w}, v1[4] = {c1.x, c1.y, c1.z, c1.w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        a0 = __ffma2_rn(xa[t + q], make_float2(v0[q], v0[q]), a0);
                        a1 = __ffma2_rn(xa[t + q], make_float2(v1[q], v1[q]), a1);
                    }
                }
                const float r0[2] = {a0.x, a0.y}, r1[2] = {a1.x, a1.y};
#pragma unroll
                for (int i2 = 0; i2 < 2; ++i2) {
                    uint32_t ka, kb;
                    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(ka) : "r"(__float_as_uint(r0[i2])), "r"(m32), "r"(2 * p));
                    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(kb) : "r"(__float_as_uint(r1[i2])), "r"(m32), "r"(2 * p + 1));
                    if constexpr (PADK) {
                        ka = uint32_t(2 * p) < k ? ka : 0xFFFFFFFFu;
                        kb = uint32_t(2 * p + 1) < k ? kb : 0xFFFFFFFFu;
                    }
                    const uint32_t lo = min(ka, kb), hi = max(ka, kb);
                    m2[i2][p & 1] = min(m2[i2][p & 1], min(max(m1[i2][p & 1], lo), hi));
                    m1[i2][p & 1] = min(m1[i2][p & 1], lo);
                }
            }
#pragma unroll
            for (int i2 = 0; i2 < 2; ++i2) {
                const uint64_t row = i2 ? row1 : row0;
                if (!(i2 ? on1 : on0)) continue;
                const uint32_t k1 = min(m1[i2][0], m1[i2][1]);
                const uint32_t k2 = min(min(m2[i2][0], m2[i2][1]), max(m1[i2][0], m1[i2][1]));
                const uint32_t i1 = k1 & 31u;
                bool unique = false;
                if (isfinite(E[i2]) && k1 != 0xFFFFFFFFu) {
                    if (k2 == 0xFFFFFFFFu) {
                        unique = true;
                    } else {
                        const float f1 = __uint_as_float((k1 >> 5) | (hi4[i2] << 27));
                        const float f2 = __uint_as_float((k2 >> 5) | (hi4[i2] << 27));
                        unique = f2 - f1 > 2.05f * E[i2];
                    }
                }
                if (unique && i1 < k) {
                    store_index(a, row, b, i1);
                    if (a.out_dist) {  // -0.5 * (-2x) == x exactly
                        const float* c = tb + i1 * DS;
                        double accd = 0.0;
#pragma unroll
                        for (int t = 0; t < DS; ++t) {
                            const float xv = -0.5f * (i2 ? xa[t].y : xa[t].x);
                            const double diff = __dsub_rn((double)xv, (double)c[t]);
                            accd = __dadd_rn(accd, __dmul_rn(diff, diff));
                        }
                        a.out_dist[uint64_t(b) * a.n + row] = accd;
                    }
                } else {
                    const unsigned long long slot = atomicAdd(a.flag_count, 1ull);
                    a.flags[slot] = (uint64_t(b) << 40) | row;
                }
            }
        }
        __syncwarp();  // every lane is done with buffer i & 1 before box i + 2 lands there
    }
}

bool row_screen_supported(const NearestArgs& a) {
    const char* e = std::getenv("PQG_ROWSCREEN");
    if (e && e[0] == '0') return false;
    // measured r2 (1M x 128 encodes): the register-resident narrow kernel
    // keeps Ds = 4 (M=32 Ks=16: 0.32 vs 0.37 ms); this one wins at Ds >= 8
    // (M=16: 0.26 vs 0.32, M=8: 0.20 vs 0.33 / tcgen05 0.24, M=4: 0.18 vs 0.26)
    if (a.d == 4 && !(e && e[0] == '1')) return false;
    if (a.src.codes || a.sse_part || a.out_mat) return false;
    if (!(a.d == 4 || a.d == 8 || a.d == 16 || a.d == 32) || a.k < 2 || a.k > 32) return false;
    // the TMA box walks the rows' subspace columns: the standard row layout
    if (a.src.col_stride != a.d || a.src.ldx != uint64_t(a.B) * a.d || (a.src.ldx * 4) % 16 != 0 ||
        (reinterpret_cast<uintptr_t>(a.src.x) & 15u) != 0 || a.n >= (uint64_t(1) << 31))
        return false;
    const uint64_t KS = a.k <= 16 ? 16 : 32;
    return uint64_t(a.B) * KS * (a.d + 1) * sizeof(float) + 2ull * kRowWarps * kRowRows * 128 <= 220 * 1024;
}

void row_screen(pqg_ctx* ctx, const NearestArgs& a) {
    const uint32_t KS = a.k <= 16 ? 16 : 32;
    const size_t smem = size_t(2) * kRowWarps * kRowRows * 128 + size_t(a.B) * KS * (a.d + 1) * sizeof(float);
    CUtensorMap xmap;
    if (!encode_rows_map(&xmap, a.src.x, a.n, a.src.ldx, kRowRows, 32, CU_TENSOR_MAP_SWIZZLE_128B))
        fail(PQG_ECUDA, "row_screen: tensor map encoding failed");
    const uint64_t nblk = (a.n + kRowRows - 1) / kRowRows;
    const unsigned grid = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((nblk + kRowWarps - 1) / kRowWarps,
                                                                         uint64_t(ctx->num_sms) * 3)));
    auto go = [&](auto kern) {
        set_smem(kern, smem);
        launch(ctx, "nearest_rows", kern, dim3(grid), dim3(kRowWarps * 32), smem, a, 32u, xmap);
    };
    const bool pad = a.k != KS;
    auto pick = [&](auto ds_tag) {
        constexpr int DS = decltype(ds_tag)::value;
        if (KS == 16) pad ? go(row_screen_kernel<DS, 16, true>) : go(row_screen_kernel<DS, 16, false>);
        else pad ? go(row_screen_kernel<DS, 32, true>) : go(row_screen_kernel<DS, 32, false>);
    };
    if (a.d == 4) pick(std::integral_constant<int, 4>());
    else if (a.d == 8) pick(std::integral_constant<int, 8>());
    else if (a.d == 16) pick(std::integral_constant<int, 16>());
    else pick(std::integral_constant<int, 32>());
}

// Narrow sub-vectors, register-resident codebook (r2): Ds in {4, 8, 16},
// Ks <= 256.  The codebook lives in REGISTERS, split over lanes: lane l owns
// one (subspace s, part g) task -- codewords g*KL .. (g+1)*KL - 1 of subspace
// s, KL*Ds <= 128 floats -- for the whole kernel, so the inner loop reads no
// memory.  A row's M*G tasks are LG consecutive lanes (LG <= 32: a warp covers
// 32/LG rows per step; LG > 32: LG/32 warps share each row), so the x loads of
// a warp step are whole consecutive rows, fully coalesced; the G lanes of a
// (row, subspace) merge their top-2 with shuffles and the group's first lane
// writes the code (consecutive subspaces -> consecutive bytes).
//
// Per codeword pair the lane issues Ds/2... no: Ds packed FFMA2 (two
// codewords per instruction, __ffma2_rn: the FP32 pipe's two-wide form), one
// FADD2 for the start value, one IMAD per key and five ALU min/max for the
// running (best, second): ~(Ds + 6)/2 instructions per (row, codeword) where
// the r1 kernel needed Ds + 6.  Keys are value_bits * 32 + local index (one
// IMAD with an immediate): a per-row offset 2^p inside C puts every screened
// value of the row in [2^p, 2^(p+16)) (p = 1 mod 16; see umma.cu row_prep), so
// the dropped bits 31..27 are constant and the 27 kept value bits are exact.
// Screened value and bound: small_table_kernel's acc_j = (C_r + ||c_j||^2) +
// sum_t (-2x_t) c_jt (fma chain), E = 2 (Ds+4) u S with S >= every partial
// sum's magnitude (offset included); a row whose runner-up is within 2.05 E of
// its best goes to the exact fixup.
constexpr int kNarrowThreads = 256;

template <int J>
__device__ __forceinline__ uint32_t nkey(float v, uint32_t m32) {
    uint32_t k;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(k) : "r"(__float_as_uint(v)), "r"(m32), "n"(J));
    return k;
}

template <int P, int KP, int NS, bool PADK, int DS>
__device__ __forceinline__ void narrow_pairs(const float2 (&cb)[KP][DS], const float2 (&cn)[KP],
                                             const float2 (&xx)[DS], float2 C2, uint32_t (&m1)[NS],
                                             uint32_t (&m2)[NS], uint32_t m32, uint32_t jvalid) {
    if constexpr (P < KP) {
        float2 acc = __fadd2_rn(cn[P], C2);
#pragma unroll
        for (int t = 0; t < DS; ++t) acc = __ffma2_rn(xx[t], cb[P][t], acc);
        uint32_t ka = nkey<2 * P>(acc.x, m32), kb = nkey<2 * P + 1>(acc.y, m32);
        if constexpr (PADK) {  // local codewords >= jvalid are padding
            ka = uint32_t(2 * P) < jvalid ? ka : 0xFFFFFFFFu;
            kb = uint32_t(2 * P + 1) < jvalid ? kb : 0xFFFFFFFFu;
        }
        const uint32_t lo = min(ka, kb), hi = max(ka, kb);
        m2[P % NS] = min(m2[P % NS], min(max(m1[P % NS], lo), hi));
        m1[P % NS] = min(m1[P % NS], lo);
        narrow_pairs<P + 1, KP, NS, PADK, DS>(cb, cn, xx, C2, m1, m2, m32, jvalid);
    }
}

template <int DS, int KS, int G, bool PADK>
__global__ void __launch_bounds__(kNarrowThreads, (KS / G) * DS <= 64 ? 2 : 1) narrow_kernel(NearestArgs a, uint32_t LG, uint32_t RPC,
                                                                uint32_t WR, uint32_t m32) {
    constexpr int KL = KS / G;  // codewords per lane
    constexpr int KP = KL / 2;  // codeword pairs per lane
    constexpr int NS = KP >= 8 ? 4 : (KP >= 4 ? 2 : 1);  // independent top-2 states
    static_assert(KL % 2 == 0 && KL <= 32, "lane codewords");
    constexpr float kE = 2.f * float(DS + 4) * kU;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t gw = uint64_t(blockIdx.x) * (kNarrowThreads / 32) + (threadIdx.x >> 5);
    const uint64_t nwarps = uint64_t(gridDim.x) * (kNarrowThreads / 32);
    uint32_t task, rsub;
    if (WR == 1) {
        rsub = lane / LG;
        task = lane - rsub * LG;
    } else {
        rsub = 0;
        task = uint32_t(gw % WR) * 32 + lane;
    }
    const bool lane_on = WR == 1 ? rsub < RPC : task < LG;
    const uint32_t s = lane_on ? task / G : 0, g = task % G;
    const bool sub_on = lane_on && !(a.active && !a.active[s]);
    // this lane's codewords, pairwise: cb[p][t] = (c_{2p,t}, c_{2p+1,t})
    float2 cb[KP][DS];
    float2 cn[KP];
#pragma unroll
    for (int p = 0; p < KP; ++p) {
        float c0[DS], c1[DS];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const uint32_t j = g * KL + 2 * p + u;
            const bool ok = sub_on && j < a.k;
            float* c = u ? c1 : c0;
#pragma unroll
            for (int t = 0; t < DS; t += 4) {
                const float4 v = ok ? __ldg(reinterpret_cast<const float4*>(a.table + (uint64_t(s) * a.k + j) * DS) + t / 4)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
                c[t] = v.x; c[t + 1] = v.y; c[t + 2] = v.z; c[t + 3] = v.w;
            }
            const float nv = ok ? __ldg(a.cnorm + uint64_t(s) * a.k + j) : 0.f;
            if (u) cn[p].y = nv; else cn[p].x = nv;
        }
#pragma unroll
        for (int t = 0; t < DS; ++t) cb[p][t] = make_float2(c0[t], c1[t]);
    }
    const uint32_t jvalid = a.k > uint64_t(g) * KL ? uint32_t(min(uint64_t(KL), a.k - uint64_t(g) * KL)) : 0u;
    const float cm = sub_on ? a.cmax[s] : 0.f;
    const float cm2 = cm * cm;
    const uint32_t step0 = uint32_t(WR == 1 ? gw : gw / WR);
    const uint32_t steps = uint32_t(WR == 1 ? nwarps : nwarps / WR);
    const uint32_t n = uint32_t(a.n);  // < 2^31 (narrow_variant)
    const uint32_t rstep = steps * RPC;  // rows between a lane's consecutive steps
    const uint64_t ld4 = a.src.ldx / 4;
    const uint64_t dptr = uint64_t(rstep) * ld4;
    // P steps of sub-vectors in flight per lane (a register ring)
    constexpr int PF = DS <= 4 ? 4 : 2;
    float4 xr[PF][DS / 4];
    uint32_t rr = step0 * RPC + rsub;  // the row of ring slot 0
    const float4* xp = reinterpret_cast<const float4*>(a.src.x + uint64_t(s) * a.src.col_stride) + uint64_t(rr) * ld4;
#pragma unroll
    for (int p = 0; p < PF; ++p) {
        if (sub_on && rr + uint32_t(p) * rstep < n) {
#pragma unroll
            for (int t = 0; t < DS / 4; ++t) xr[p][t] = __ldg(xp + uint64_t(p) * dptr + t);
        }
    }
    // the G lanes of a (row, subspace) task are consecutive: their group's bits
    const uint32_t gbase = lane & ~uint32_t(G - 1);
    const uint32_t gmask = G >= 32 ? 0xFFFFFFFFu : (((1u << G) - 1u) << gbase);
    for (; rr - rsub < n; rr += uint32_t(PF) * rstep, xp += uint64_t(PF) * dptr) {
#pragma unroll
        for (int p = 0; p < PF; ++p) {
            const uint32_t crow = rr + uint32_t(p) * rstep;
            if (crow - rsub >= n) break;  // warp-uniform
            const bool cur = sub_on && crow < n;
            float2 xx[DS];
            float nx4 = 0.f;  // ||-2x||^2 = 4 ||x||^2
#pragma unroll
            for (int t = 0; t < DS / 4; ++t) {
                const float v[4] = {-2.f * xr[p][t].x, -2.f * xr[p][t].y, -2.f * xr[p][t].z, -2.f * xr[p][t].w};
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    xx[4 * t + w] = make_float2(v[w], v[w]);
                    nx4 = fmaf(v[w], v[w], nx4);
                }
            }
            if (sub_on && crow + uint32_t(PF) * rstep < n) {  // refill the slot PF steps ahead
#pragma unroll
                for (int t = 0; t < DS / 4; ++t) xr[p][t] = __ldg(xp + uint64_t(p + PF) * dptr + t);
            }
            const float nx = 0.25f * nx4;
            // S >= (||x|| + max||c||)^2 >= every partial sum's magnitude before
            // the offset; the offset window starts at 2^p, p = 1 (mod 16)
            const float S = 2.f * (nx * (1.f + 1e-6f) + cm2) + 1e-6f;
            int e = int((__float_as_uint(S) >> 23) & 0xFF) - 127;
            e = max(-60, min(e, 100));
            const int pw = (e & ~15) + 1;  // smallest p >= e - 14 with p = 1 (mod 16)
            const float O = __uint_as_float(uint32_t(pw + 127) << 23);
            const uint32_t hi4 = uint32_t(pw + 127) >> 4;
            const float E = kE * (S + O) * 1.001f + 1e-30f;
            const float C = nx * (1.f + 2.f * float(DS + 2) * kU) + 2.f * E + O;
            uint32_t m1[NS], m2[NS];
#pragma unroll
            for (int u = 0; u < NS; ++u) m1[u] = m2[u] = 0xFFFFFFFFu;
            narrow_pairs<0, KP, NS, PADK, DS>(cb, cn, xx, make_float2(C, C), m1, m2, m32, jvalid);
            uint32_t k1 = m1[0], k2 = m2[0];
#pragma unroll
            for (int u = 1; u < NS; ++u) {
                k2 = min(min(k2, m2[u]), max(k1, m1[u]));
                k1 = min(k1, m1[u]);
            }
            const uint32_t own = k1;
#pragma unroll
            for (int o = 1; o < G; o <<= 1) {  // merge the G parts of this (row, subspace)
                const uint32_t o1 = __shfl_xor_sync(0xffffffffu, k1, o);
                const uint32_t o2 = __shfl_xor_sync(0xffffffffu, k2, o);
                k2 = min(min(k2, o2), max(k1, o1));
                k1 = min(k1, o1);
            }
            // the part holding the winner (an exact key tie between parts means
            // equal values: the runner-up test below flags the row)
            uint32_t gwin = 0;
            if constexpr (G > 1) {
                const uint32_t bal = __ballot_sync(0xffffffffu, own == k1) & gmask;
                gwin = bal ? uint32_t(__ffs(bal) - 1) - gbase : 0u;
            }
            if (!cur || g != 0) continue;
            const uint32_t i1 = gwin * KL + (k1 & 31u);
            bool unique = false;
            if (isfinite(E) && k1 != 0xFFFFFFFFu) {
                if (k2 == 0xFFFFFFFFu) {
                    unique = true;
                } else {
                    const float f1 = __uint_as_float((k1 >> 5) | (hi4 << 27));
                    const float f2 = __uint_as_float((k2 >> 5) | (hi4 << 27));
                    unique = f2 - f1 > 2.05f * E;
                }
            }
            if (unique && i1 < a.k) {
                if (a.idx_bytes == 1 && a.idx_ps == 1)
                    static_cast<uint8_t*>(a.out_idx)[uint64_t(crow) * a.idx_rs + s] = uint8_t(i1);
                else
                    store_index(a, crow, s, i1);
                if (a.out_dist) {  // -0.5 * (-2x) == x exactly
                    const float* c = a.table + (uint64_t(s) * a.k + i1) * DS;
                    double accd = 0.0;
#pragma unroll
                    for (int t = 0; t < DS; ++t) {
                        const double diff = __dsub_rn((double)(-0.5f * xx[t].x), (double)__ldg(c + t));
                        accd = __dadd_rn(accd, __dmul_rn(diff, diff));
                    }
                    a.out_dist[uint64_t(s) * a.n + crow] = accd;
                }
            } else {
                const unsigned long long slot = atomicAdd(a.flag_count, 1ull);
                a.flags[slot] = (uint64_t(s) << 40) | crow;
            }
        }
    }
}

template <int DS, int KS>
void launch_narrow(pqg_ctx* ctx, const NearestArgs& a) {
    constexpr int G = (KS * DS / 128) > 1 ? KS * DS / 128 : 1;
    const uint32_t LG = a.B * G;
    uint32_t RPC = 1, WR = 1;
    if (LG <= 32) RPC = 32 / LG;
    else WR = (LG + 31) / 32;
    const uint64_t units = (a.n + RPC - 1) / RPC * WR;  // warp steps
    const uint64_t blocks = std::min<uint64_t>((units + 7) / 8, uint64_t(ctx->num_sms) * 16);
    const dim3 grid(unsigned(std::max<uint64_t>(1, blocks)));
    if (a.k == uint64_t(KS))
        launch(ctx, "nearest_narrow", narrow_kernel<DS, KS, G, false>, grid, dim3(kNarrowThreads), 0, a, LG, RPC,
               WR, 32u);
    else
        launch(ctx, "nearest_narrow", narrow_kernel<DS, KS, G, true>, grid, dim3(kNarrowThreads), 0, a, LG, RPC,
               WR, 32u);
}

// Which narrow instance applies (0: none).  LG > 32 needs WR | 8 (warps per CTA).
int narrow_variant(const NearestArgs& a) {
    const char* e = std::getenv("PQG_NARROW");
    if (e && e[0] == '0') return 0;
    if (a.src.codes || a.sse_part || a.out_mat) return 0;
    if (((a.src.ldx | a.src.col_stride) & 3u) != 0 || (reinterpret_cast<uintptr_t>(a.src.x) & 15u) != 0 ||
        (reinterpret_cast<uintptr_t>(a.table) & 15u) != 0)
        return 0;
    if (!(a.d == 4 || a.d == 8 || a.d == 16)) return 0;
    if (a.n >= (uint64_t(1) << 31)) return 0;
    const int KS = a.k <= 16 ? 16 : (a.k <= 32 ? 32 : (a.k <= 64 ? 64 : (a.k <= 128 ? 128 : (a.k <= 256 ? 256 : 0))));
    if (!KS) return 0;
    const int G = std::max(1, KS * int(a.d) / 128);
    if (KS / G > 32 || KS / G < 2) return 0;
    const uint64_t LG = uint64_t(a.B) * G;
    if (LG > 32 && (LG > 256 || 8 % ((LG + 31) / 32) != 0)) return 0;
    if (e && e[0] == '1') return KS;  // forced
    // measured r2 (tools/encode_bench.py, 1M x 128): the tcgen05 screen wins
    // from Ks = 64 up (M=16 Ks=64: 0.42 vs 0.98 ms, M=32 Ks=64: 0.73 vs 1.21)
    if (a.d != 4 || KS > 16) return 0;
    return KS;
}

void narrow(pqg_ctx* ctx, const NearestArgs& a, int KS) {
    auto go = [&](auto ds_tag) {
        constexpr int DS = decltype(ds_tag)::value;
        if constexpr (DS * 16 / 128 <= 32) {
            if (KS == 16) launch_narrow<DS, 16>(ctx, a);
            else if (KS == 32) launch_narrow<DS, 32>(ctx, a);
            else if (KS == 64) launch_narrow<DS, 64>(ctx, a);
            else if (KS == 128) launch_narrow<DS, 128>(ctx, a);
            else launch_narrow<DS, 256>(ctx, a);
        }
    };
    if (a.d == 4) go(std::integral_constant<int, 4>());
    else if (a.d == 8) go(std::integral_constant<int, 8>());
    else go(std::integral_constant<int, 16>());
}

__global__ void __launch_bounds__(256, 1) norms_kernel(const float* table, uint32_t B, uint64_t k, uint32_t d,
                             float* cnorm, unsigned* cmax_bits) {
    const uint64_t total = uint64_t(B) * k;
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += uint64_t(gridDim.x) * blockDim.x) {
        const float* c = table + e * d;
        double s = 0.0;
        for (uint32_t t0 = 0; t0 < d; t0 += 8) {
            float v[8];  // the row's loads issued together (clamped, unpredicated)
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldg(c + min(t0 + u, d - 1));
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (t0 + u < d) s = __dadd_rn(s, __dmul_rn((double)v[u], (double)v[u]));
        }
        cnorm[e] = __double2float_rn(s);
        atomicMax(cmax_bits + e / k, __float_as_uint(__double2float_ru(sqrt(s))));
    }
}

template <int TN, int DP, bool MAT>
size_t smem_bytes() {
    constexpr int BN = 16 * TN;
    constexpr int KCH = DP > 0 ? DP : BK;
    const size_t main = sizeof(float) * (KCH * LDX + KCH * (BN + 4) + BN + 2 * BM);
    const size_t red = size_t(BM) * 16 * (sizeof(uint64_t) + sizeof(uint32_t));
    return main > red + sizeof(float) * 2 * BM ? main : red + sizeof(float) * 2 * BM;
}

template <int TN, int DP, bool MAT>
void launch_nearest(pqg_ctx* ctx, const NearestArgs& a) {
    auto kern = nearest_kernel<TN, DP, MAT>;
    const size_t smem = smem_bytes<TN, DP, MAT>();
    static bool configured = false;
    if (!configured) {
        set_smem(kern, smem);
        configured = true;
    }
    const uint64_t gx = (a.n + BM - 1) / BM;
    launch(ctx, MAT ? "distance_matrix" : "nearest", kern, dim3(unsigned(gx * a.B)), dim3(NT), smem, a);
}

template <int TN, bool MAT>
void dispatch_dp(pqg_ctx* ctx, const NearestArgs& a) {
    const uint32_t dp = (a.d + 3) & ~3u;
    if (dp == 4) launch_nearest<TN, 4, MAT>(ctx, a);
    else if (dp == 8) launch_nearest<TN, 8, MAT>(ctx, a);
    else if (dp == 16) launch_nearest<TN, 16, MAT>(ctx, a);
    else if (dp == 32) launch_nearest<TN, 32, MAT>(ctx, a);
    else launch_nearest<TN, 0, MAT>(ctx, a);
}

template <bool MAT>
void dispatch(pqg_ctx* ctx, const NearestArgs& a) {
    if (a.k >= 128) dispatch_dp<8, MAT>(ctx, a);
    else if (a.k >= 64) dispatch_dp<4, MAT>(ctx, a);
    else if (a.k >= 32) dispatch_dp<2, MAT>(ctx, a);
    else dispatch_dp<1, MAT>(ctx, a);
}

}  // namespace

void table_norms(pqg_ctx* ctx, const float* table, uint32_t B, uint64_t k, uint32_t d,
                 float* cnorm, float* cmax) {
    if (k * d <= 8192 && k <= 4096) {  // PQ codebooks: one block per subspace
        table_norms_small(ctx, table, B, k, d, cnorm, cmax);
        return;
    }
    PQG_CUDA(cudaMemsetAsync(cmax, 0, sizeof(float) * B, ctx->stream));
    launch(ctx, "norms", norms_kernel, dim3(grid1d(uint64_t(B) * k, 256, 4096)), dim3(256), 0,
           table, B, k, d, cnorm, reinterpret_cast<unsigned*>(cmax));
}

void nearest(pqg_ctx* ctx, NearestArgs a) {
    if (a.n == 0 || a.B == 0) return;
    if (a.k >= (uint64_t(1) << 31)) fail(PQG_EUNSUPPORTED, "nearest: k too large");
    if (a.n >= (uint64_t(1) << 40)) fail(PQG_EUNSUPPORTED, "nearest: too many rows");
    // flag list capacity n*B (worst case: every row tied)
    a.flag_count = scratch<unsigned long long>(ctx, 1);
    a.flags = scratch<uint64_t>(ctx, a.n * a.B);
    PQG_CUDA(cudaMemsetAsync(a.flag_count, 0, sizeof(unsigned long long), ctx->stream));
    a.out_mat = nullptr;
    // screen selection: tcgen05 for PQ subspaces unless PQG_SCREEN=fp32
    const char* mode = std::getenv("PQG_SCREEN");
    const bool force_fp32 = mode && std::strcmp(mode, "fp32") == 0;
    // narrow codebooks: the row-wise small-table kernel (PQG_SCREEN=tc keeps
    // the tensor-core screen)
    const bool small_tab = !force_fp32 && !(mode && std::strcmp(mode, "tc") == 0) && a.k <= 16 &&
                           (a.d == 4 || a.d == 8 || a.d == 32) && !a.src.codes && !a.sse_part &&
                           ((a.src.ldx | a.src.col_stride) & 3u) == 0 &&
                           (reinterpret_cast<uintptr_t>(a.src.x) & 15u) == 0 &&
                           (reinterpret_cast<uintptr_t>(a.table) & 15u) == 0 &&
                           uint64_t(a.B) * a.k * (a.d + 1) * sizeof(float) <= 96 * 1024;
    const bool tc_forced = mode && std::strcmp(mode, "tc") == 0;
    const int narrow_ks = force_fp32 || tc_forced ? 0 : narrow_variant(a);
    if (!force_fp32 && !tc_forced && row_screen_supported(a)) {
        row_screen(ctx, a);
    } else if (narrow_ks) {
        narrow(ctx, a, narrow_ks);
    } else if (small_tab) {
        const size_t smem = size_t(a.B) * a.k * (a.d + 1) * sizeof(float);
        const unsigned grid = unsigned(std::min<uint64_t>((a.n + kSmallThreads - 1) / kSmallThreads,
                                                          uint64_t(ctx->num_sms) * 8));
        auto go = [&](auto kern) {
            set_smem(kern, smem);
            launch(ctx, "nearest_small", kern, dim3(grid), dim3(kSmallThreads), smem, a);
        };
        if (a.d == 4) go(small_table_kernel<4>);
        else if (a.d == 8) go(small_table_kernel<8>);
        else go(small_table_kernel<32>);
    } else if (!force_fp32 && umma_screen_supported(a)) umma_screen(ctx, a);
    else if (!force_fp32 && umma_big_supported(a)) umma_big(ctx, a);
    else dispatch<false>(ctx, a);
    // stage the table in shared memory when it fits (PQ tables: <= 33 KB)
    const size_t tbytes = size_t(a.k) * (a.d + 1) * sizeof(float);
    const int tstaged = a.d <= uint32_t(kFixMaxD) && tbytes <= 48 * 1024 ? 1 : 0;
    const bool wvec = !a.src.codes && ((a.src.ldx | a.src.col_stride) & 3u) == 0 &&
                      (reinterpret_cast<uintptr_t>(a.src.x) & 15u) == 0 &&
                      (reinterpret_cast<uintptr_t>(a.table) & 15u) == 0;
    const dim3 wgrid(ctx->num_sms * 16);
    if (wvec && a.d == 16) launch(ctx, "fixup", fixup_warp_kernel<16>, wgrid, dim3(256), 0, a);
    else if (wvec && a.d == 8) launch(ctx, "fixup", fixup_warp_kernel<8>, wgrid, dim3(256), 0, a);
    else if (wvec && a.d == 4) launch(ctx, "fixup", fixup_warp_kernel<4>, wgrid, dim3(256), 0, a);
    else if (wvec && a.d == 32) launch(ctx, "fixup", fixup_warp_kernel<32>, wgrid, dim3(256), 0, a);
    else
        launch(ctx, "fixup", fixup_kernel, dim3(ctx->num_sms * 8), dim3(kFixThreads), tstaged ? tbytes : 0, a,
               tstaged);
    if (std::getenv("PQG_FLAG_STATS")) {  // diagnostics: rows sent to the exact fixup
        unsigned long long h = 0;
        PQG_CUDA(cudaMemcpyAsync(&h, a.flag_count, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
        PQG_CUDA(cudaStreamSynchronize(ctx->stream));
        std::fprintf(stderr, "nearest: n=%llu B=%u k=%llu d=%u flagged=%llu\n", (unsigned long long)a.n,
                     a.B, (unsigned long long)a.k, a.d, h);
    }
}

void distance_matrix(pqg_ctx* ctx, NearestArgs a) {
    if (a.n == 0) return;
    const char* mode = std::getenv("PQG_SCREEN");
    const bool force_fp32 = mode && std::strcmp(mode, "fp32") == 0;
    if (!force_fp32 && umma_big_supported(a)) {
        umma_big(ctx, a);
        return;
    }
    dispatch<true>(ctx, a);
}

}  // namespace pqg
