// kmshard.cu -- the exchange side of a row-sharded k-means iteration
// (pqg_kmshard_*): one NCCL all-reduce of the centroid sums
// and counts per iteration instead of replicating the update.
//
// Each rank owns a contiguous block of the (global, row-ordered) sample.  Per
// iteration it assigns its rows, buckets them stably by cluster and computes
// for every (problem b, cluster c, dim t) the fp64 sum of its members'
// values together with their exponent range (kmeans_local_partials, the
// single-GPU piece machinery).  The packed partials
//     f64 = [ sums B*k*d | counts B*k | inertia B ]       (all-reduce SUM)
//     u8  = [ emax+1 B*k*d | 256-emin B*k*d ]             (all-reduce MAX)
// are reduced across ranks; then every rank finalizes identically:
//   * the stop rule on the global inertia (kmeans.cpp:93-100);
//   * a (b, c, t) whose GLOBAL exponent range and count pass the exactness
//     test (e_max - e_min + ceil(log2 count) <= 28: every partial sum of any
//     subset in any order is exact in fp64) takes float(sum * (1/count)) --
//     each rank's partial is exact, and so is the all-reduce of them, so this
//     IS the reference's row-order sum (kmeans.cpp:103-118);
//   * the other (b, c, t) are replayed exactly as the reference chains them:
//     each rank packs its members' values in local row order, the packs are
//     all-gathered, and the chain runs over rank 0's members, then rank 1's,
//     ... -- the global row order, since ranks own ascending row blocks;
//   * an empty cluster (global count 0) takes, in ascending c, the row of the
//     largest pre-update distance (strict '>', lowest global index on ties;
//     kmeans.cpp:122-130): every rank offers its local top-E positive
//     (dist, index, row) candidates, the merge takes the E best in (dist desc,
//     index asc) order, and once the positive distances are exhausted every
//     distance is 0 and the reference's argmax is global row 0.
// The exponent encodings clamp e_max = 254 to the non-finite code 255; that
// only sends such a column to the exact replay.
#include "kernels.cuh"

namespace pqg {
namespace {

constexpr int kThreads = 256;

__global__ void pack_partials_kernel(uint32_t B, uint64_t k, uint32_t d, const uint64_t* offsets,
                                     const double* csum, const int* cmax, const int* cmin, double* f64,
                                     uint8_t* u8) {
    const uint64_t nkd = uint64_t(B) * k * d;
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < nkd;
         e += uint64_t(gridDim.x) * blockDim.x) {
        f64[e] = csum[e];
        const int ea = cmax[e], ei = cmin[e];
        u8[e] = uint8_t(ea < 0 ? 0 : min(ea + 1, 255));
        u8[nkd + e] = uint8_t(ei > 255 ? 0 : 256 - max(ei, 1));
        if (e % d == 0) {
            const uint64_t bc = e / d, b = bc / k, c = bc - b * k;
            const uint64_t* off = offsets + b * (k + 1);
            f64[nkd + bc] = double(off[c + 1] - off[c]);
        }
    }
}

// warp per (problem, cluster) of an active problem
__global__ void finalize_kernel(uint32_t B, uint64_t k, uint32_t d, const double* f64, const uint8_t* u8,
                                const int* active, float* table, uint32_t* flags, uint32_t* empties) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t bc = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (bc >= uint64_t(B) * k) return;
    const uint64_t b = bc / k;
    const uint64_t nkd = uint64_t(B) * k * d;
    for (uint32_t t = lane; t < d; t += 32) flags[bc * d + t] = 0u;
    if (!active[b]) return;
    const double cntd = f64[nkd + bc];
    if (cntd == 0.0) {
        if (lane == 0) atomicAdd(empties + b, 1u);
        return;
    }
    const uint64_t cnt = uint64_t(cntd);
    int lg = 0;
    while ((uint64_t(1) << lg) < cnt) ++lg;
    const double inv = __ddiv_rn(1.0, cntd);
    for (uint32_t t = lane; t < d; t += 32) {
        const uint64_t e = bc * d + t;
        const int ea = int(u8[e]) - 1;                          // -1: no nonzero member
        const int ei = u8[nkd + e] ? 256 - int(u8[nkd + e]) : (1 << 30);
        if (ea < 0 || (ea < 254 && ea - ei + lg <= 28))
            table[e] = __double2float_rn(__dmul_rn(f64[e], inv));  // kmeans.cpp:112-118
        else
            flags[e] = 1u;
    }
}

__global__ void compact_kernel(const uint32_t* flags, const uint64_t* pos, uint64_t count, uint32_t* work,
                               unsigned long long* res) {
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < count;
         e += uint64_t(gridDim.x) * blockDim.x) {
        if (flags[e]) work[pos[e]] = uint32_t(e);
        if (e == count - 1) res[0] = pos[e] + flags[e];
    }
}

// replay column p < n_fail: its local member count (cnt) and, summed into
// res[2], its global count (the per-rank pack is at most that long)
__global__ void pack_counts_kernel(const uint32_t* work, uint64_t cap, const unsigned long long* res_in,
                                   uint64_t k, uint32_t d, uint32_t B, const uint64_t* offsets, const double* f64,
                                   uint32_t* cnt, unsigned long long* res) {
    const uint64_t n_fail = res_in[0];
    const uint64_t nkd = uint64_t(B) * k * d;
    for (uint64_t p = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < cap;
         p += uint64_t(gridDim.x) * blockDim.x) {
        if (p >= n_fail) {
            cnt[p] = 0u;
            continue;
        }
        const uint64_t bc = work[p] / d, b = bc / k, c = bc - b * k;
        const uint64_t* off = offsets + b * (k + 1);
        cnt[p] = uint32_t(off[c + 1] - off[c]);
        atomicAdd(res + 2, (unsigned long long)f64[nkd + bc]);
    }
}

__global__ void pack_total_kernel(const uint32_t* cnt, const uint64_t* pre, unsigned long long* res) {
    const uint64_t n_fail = res[0];
    res[1] = n_fail ? pre[n_fail - 1] + cnt[n_fail - 1] : 0ull;
}

__global__ void pack_offcnt_kernel(const uint32_t* cnt, const uint64_t* pre, uint64_t n_fail, uint64_t* offcnt) {
    for (uint64_t p = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < n_fail;
         p += uint64_t(gridDim.x) * blockDim.x) {
        offcnt[2 * p] = pre[p];
        offcnt[2 * p + 1] = cnt[p];
    }
}

// warp per failing (b, c, t): the rank's members' values in local row order
__global__ void pack_kernel(RowSrc src, const uint32_t* work, uint64_t n_fail, uint64_t k, uint32_t d,
                            const uint64_t* offsets, const uint32_t* perm, uint64_t n, const uint64_t* offcnt,
                            float* vals) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t p = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (p >= n_fail) return;
    const uint64_t e = work[p], bc = e / d, t = e - bc * d, b = bc / k, c = bc - b * k;
    const uint64_t* off = offsets + b * (k + 1);
    const uint32_t* pb = perm + b * n;
    const float* xb = src.x + b * src.col_stride + t;
    float* out = vals + offcnt[2 * p];
    for (uint64_t m = off[c] + lane; m < off[c + 1]; m += 32)
        out[m - off[c]] = __ldg(xb + uint64_t(__ldg(pb + m)) * src.ldx);
}

// thread per failing (b, c, t): the reference's chain over all ranks' members
__global__ void replay_kernel(const uint32_t* work, uint64_t n_fail, uint64_t k, uint32_t d, uint32_t B,
                              const double* f64, const float* vals, uint64_t stride, const uint64_t* offcnt,
                              uint32_t world, float* table) {
    for (uint64_t p = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < n_fail;
         p += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t e = work[p], bc = e / d;
        double s = 0.0;
        for (uint32_t r = 0; r < world; ++r) {
            const uint64_t o = offcnt[(uint64_t(r) * n_fail + p) * 2], c = offcnt[(uint64_t(r) * n_fail + p) * 2 + 1];
            const float* v = vals + uint64_t(r) * stride + o;
            for (uint64_t j = 0; j < c; ++j) s = __dadd_rn(s, (double)v[j]);
        }
        const double cnt = f64[uint64_t(B) * k * d + bc];
        table[e] = __double2float_rn(__dmul_rn(s, __ddiv_rn(1.0, cnt)));
    }
}

// Chained replay (r2e): the reference's chain of a replay column runs over
// rank 0's members, then rank 1's, ...; rank r continues it from the running
// sums rank r-1 hands over (run[p], one fp64 per column) with its own
// members in local row order -- no member values cross ranks.  Warp per
// column, 32 members per step: a step whose additions provably cannot round
// (every partial sum a multiple of 2^lq and below 2^(lq+53), lq from the
// running sum's lowest set bit and the step's smallest ulp -- any order gives
// the same exact sum) is added as one warp sum, otherwise lane 0 walks the
// 32 members as the reference chains them (kmeans.cpp:103-111).
__device__ __forceinline__ int lowbit_exp64(double r) {  // log2 of r's lowest set bit (r normal, != 0)
    const unsigned long long sb = __double_as_longlong(r);
    const int E = int((sb >> 52) & 0x7FF);
    const unsigned long long mant = (sb & ((1ull << 52) - 1)) | (1ull << 52);
    return E - 1075 + (__ffsll((long long)mant) - 1);
}

__global__ void replay_step_kernel(RowSrc src, const uint32_t* work, uint64_t n_fail, uint64_t k, uint32_t d,
                                   const uint64_t* offsets, const uint32_t* perm, uint64_t n, double* run) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t p = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (p >= n_fail) return;
    const uint64_t e = work[p], bc = e / d, t = e - bc * d, b = bc / k, c = bc - b * k;
    const uint64_t* off = offsets + b * (k + 1);
    const uint32_t* pb = perm + b * n;
    const float* xb = src.x + b * src.col_stride + t;
    double s = run[p];
    for (uint64_t m0 = off[c]; m0 < off[c + 1]; m0 += 32) {
        const uint64_t m = m0 + lane;
        const uint32_t nm = uint32_t(min64(uint64_t(32), off[c + 1] - m0));
        const float v = m < off[c + 1] ? __ldg(xb + uint64_t(__ldg(pb + m)) * src.ldx) : 0.f;
        const int eb = int((__float_as_uint(v) >> 23) & 0xFFu);
        int ehi = v != 0.f ? eb : -1;
        int elo = v != 0.f ? max(eb, 1) : (1 << 30);
        double ws = (double)v;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            ws = __dadd_rn(ws, __shfl_xor_sync(0xffffffffu, ws, o));
            ehi = max(ehi, __shfl_xor_sync(0xffffffffu, ehi, o));
            elo = min(elo, __shfl_xor_sync(0xffffffffu, elo, o));
        }
        bool exact;
        if (ehi < 0) {
            exact = true;  // all zeros
        } else if (ehi == 255 || !isfinite(s)) {
            exact = false;
        } else {
            int lq = elo - 150;  // log2 ulp of the smallest nonzero value
            if (s != 0.0) lq = min(lq, lowbit_exp64(s));
            // every partial sum is at most |s| + 32 values below 2^(ehi-126)
            const double bound = __dadd_ru(fabs(s), ldexp(1.0, ehi - 121));
            const int lb = int((__double_as_longlong(bound) >> 52) & 0x7FF) - 1022;
            exact = lb - lq <= 53;
        }
        if (exact) {
            s = __dadd_rn(s, ws);  // ws is exact too (a subset sum)
        } else {
            for (uint32_t j = 0; j < nm; ++j) s = __dadd_rn(s, (double)__shfl_sync(0xffffffffu, v, j));
        }
    }
    if (lane == 0) run[p] = s;
}

__global__ void replay_finish_kernel(const uint32_t* work, uint64_t n_fail, uint64_t k, uint32_t d, uint32_t B,
                                     const double* f64, const double* run, float* table) {
    for (uint64_t p = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < n_fail;
         p += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t e = work[p], bc = e / d;
        const double cnt = f64[uint64_t(B) * k * d + bc];
        table[e] = __double2float_rn(__dmul_rn(run[p], __ddiv_rn(1.0, cnt)));
    }
}

// block per problem: the rank's E best positive (dist desc, global index asc)
// candidates, plus its local row 0 in slot E (the merge uses rank 0's = global
// row 0 once the positive distances run out)
__global__ void reseed_cand_kernel(RowSrc src, uint64_t n, uint32_t d, const double* dist, const int* active,
                                   const uint32_t* empties, uint32_t E, uint64_t row0, double* cand_d,
                                   uint64_t* cand_i, float* cand_rows) {
    const uint32_t b = blockIdx.x;
    __shared__ double sv[32];
    __shared__ uint64_t si[32];
    __shared__ double lastv;
    __shared__ uint64_t lasti;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const double* db = dist + uint64_t(b) * n;
    double* cd = cand_d + uint64_t(b) * (E + 1);
    uint64_t* ci = cand_i + uint64_t(b) * (E + 1);
    float* cr = cand_rows + uint64_t(b) * (E + 1) * d;
    const uint32_t need = active[b] ? min(empties[b], E) : 0u;
    if (threadIdx.x == 0) { lastv = 0.0; lasti = 0; }
    __syncthreads();
    for (uint32_t s = 0; s < E; ++s) {
        // best (dist, i) strictly after (lastv, lasti) in (dist desc, i asc) order
        double bv = -1.0;
        uint64_t bi = ~uint64_t(0);
        if (s < need) {
            for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) {
                const double v = db[i];
                if (!(v > 0.0)) continue;
                if (s > 0 && !(v < lastv || (v == lastv && i > lasti))) continue;
                if (bi == ~uint64_t(0) || v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
            }
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const uint64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (oi != ~uint64_t(0) && (bi == ~uint64_t(0) || ov > bv || (ov == bv && oi < bi))) { bv = ov; bi = oi; }
        }
        if (lane == 0) { sv[w] = bv; si[w] = bi; }
        __syncthreads();
        if (w == 0) {
            const int nw = blockDim.x >> 5;
            bv = lane < nw ? sv[lane] : -1.0;
            bi = lane < nw ? si[lane] : ~uint64_t(0);
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const uint64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (oi != ~uint64_t(0) && (bi == ~uint64_t(0) || ov > bv || (ov == bv && oi < bi))) { bv = ov; bi = oi; }
            }
            if (lane == 0) {
                cd[s] = bi == ~uint64_t(0) ? -1.0 : bv;
                ci[s] = bi == ~uint64_t(0) ? ~uint64_t(0) : row0 + bi;
                if (bi != ~uint64_t(0)) { lastv = bv; lasti = bi; }
                si[0] = bi;
            }
        }
        __syncthreads();
        const uint64_t pick = si[0];
        for (uint32_t t = threadIdx.x; t < d; t += blockDim.x)
            cr[uint64_t(s) * d + t] = pick == ~uint64_t(0) ? 0.f : src.x[pick * src.ldx + uint64_t(b) * src.col_stride + t];
        __syncthreads();
    }
    if (threadIdx.x == 0) { cd[E] = -2.0; ci[E] = row0; }
    for (uint32_t t = threadIdx.x; t < d; t += blockDim.x)
        cr[uint64_t(E) * d + t] = src.x[uint64_t(b) * src.col_stride + t];
}

// block per problem: merge every rank's candidates and fill the empty
// clusters in ascending order
__global__ void reseed_apply_kernel(uint64_t k, uint32_t d, uint32_t B, const double* f64, const int* active,
                                    uint32_t E, uint32_t world, const double* cand_d, const uint64_t* cand_i,
                                    const float* cand_rows, float* table) {
    const uint32_t b = blockIdx.x;
    if (!active[b]) return;
    __shared__ int pick_r, pick_s;
    __shared__ double lastv;
    __shared__ uint64_t lasti;
    const double* cnt = f64 + uint64_t(B) * k * d + uint64_t(b) * k;
    const uint64_t per = uint64_t(B) * (E + 1);  // one rank's slots
    if (threadIdx.x == 0) { lastv = 0.0; lasti = 0; }
    __syncthreads();
    uint32_t s = 0;
    for (uint64_t c = 0; c < k; ++c) {
        if (cnt[c] != 0.0) continue;
        if (threadIdx.x == 0) {
            // next best positive candidate after (lastv, lasti)
            int br = -1, bs = -1;
            double bv = 0.0;
            uint64_t bi = 0;
            for (uint32_t r = 0; r < world; ++r)
                for (uint32_t j = 0; j < E; ++j) {
                    const uint64_t slot = uint64_t(r) * per + uint64_t(b) * (E + 1) + j;
                    const double v = cand_d[slot];
                    const uint64_t i = cand_i[slot];
                    if (!(v > 0.0)) continue;
                    if (s > 0 && !(v < lastv || (v == lastv && i > lasti))) continue;
                    if (br < 0 || v > bv || (v == bv && i < bi)) { br = int(r); bs = int(j); bv = v; bi = i; }
                }
            if (br >= 0) {
                lastv = bv;
                lasti = bi;
            } else {  // all distances are 0 now: global row 0 (rank 0's slot E)
                br = 0;
                bs = int(E);
            }
            pick_r = br;
            pick_s = bs;
        }
        __syncthreads();
        const float* row = cand_rows + ((uint64_t(pick_r) * per + uint64_t(b) * (E + 1) + pick_s) * d);
        for (uint32_t t = threadIdx.x; t < d; t += blockDim.x) table[(uint64_t(b) * k + c) * d + t] = row[t];
        ++s;
        __syncthreads();
    }
}

// owner rank writes the init rows it holds (bit patterns; zero elsewhere, so
// an integer all-reduce SUM assembles the table exactly)
__global__ void init_gather_kernel(RowSrc src, uint64_t n, uint32_t B, uint32_t d, uint64_t k,
                                   const uint64_t* rows, uint64_t row0, uint32_t* bits) {
    const uint64_t total = uint64_t(B) * k * d;
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t bc = e / d, t = e - bc * d, b = bc / k;
        const uint64_t gi = rows[bc];
        uint32_t v = 0u;
        if (gi >= row0 && gi < row0 + n)
            v = __float_as_uint(src.x[(gi - row0) * src.ldx + b * src.col_stride + t]);
        bits[e] = v;
    }
}

}  // namespace

void shard_init_gather(pqg_ctx* ctx, const RowSrc& src, uint64_t n, uint32_t B, uint32_t d, uint64_t k,
                       const uint64_t* rows, uint64_t row0, uint32_t* bits) {
    launch(ctx, "gather", init_gather_kernel, dim3(grid1d(uint64_t(B) * k * d, kThreads, 4096)), dim3(kThreads),
           0, src, n, B, d, k, rows, row0, bits);
}

void shard_pack_partials(pqg_ctx* ctx, uint32_t B, uint64_t k, uint32_t d, const uint64_t* offsets,
                         const double* csum, const int* cmax, const int* cmin, double* f64, uint8_t* u8) {
    launch(ctx, "kmshard", pack_partials_kernel, dim3(grid1d(uint64_t(B) * k * d, kThreads, 4096)),
           dim3(kThreads), 0, B, k, d, offsets, csum, cmax, cmin, f64, u8);
}

void shard_finalize(pqg_ctx* ctx, uint32_t B, uint64_t k, uint32_t d, const double* f64, const uint8_t* u8,
                    const int* active, float* table, uint32_t* flags, uint32_t* empties) {
    PQG_CUDA(cudaMemsetAsync(empties, 0, sizeof(uint32_t) * B, ctx->stream));
    launch(ctx, "kmshard", finalize_kernel, dim3(grid1d(uint64_t(B) * k * 32, kThreads)), dim3(kThreads), 0, B,
           k, d, f64, u8, active, table, flags, empties);
}

void shard_replay_layout(pqg_ctx* ctx, uint32_t B, uint64_t k, uint32_t d, const uint32_t* flags,
                         const uint64_t* offsets, const double* f64, uint32_t* work, uint32_t* cnt, uint64_t* pre,
                         unsigned long long* res) {
    const uint64_t nkd = uint64_t(B) * k * d;
    PQG_CUDA(cudaMemsetAsync(res, 0, sizeof(unsigned long long) * 3, ctx->stream));
    exclusive_scan_u32(ctx, flags, pre, nkd);
    launch(ctx, "kmshard", compact_kernel, dim3(grid1d(nkd, kThreads, 4096)), dim3(kThreads), 0, flags,
           (const uint64_t*)pre, nkd, work, res);
    launch(ctx, "kmshard", pack_counts_kernel, dim3(grid1d(nkd, kThreads, 4096)), dim3(kThreads), 0,
           (const uint32_t*)work, nkd, (const unsigned long long*)res, k, d, B, offsets, f64, cnt, res);
    exclusive_scan_u32(ctx, cnt, pre, nkd);
    launch(ctx, "kmshard", pack_total_kernel, dim3(1), dim3(1), 0, (const uint32_t*)cnt, (const uint64_t*)pre,
           res);
}

void shard_pack(pqg_ctx* ctx, const RowSrc& src, const uint32_t* work, uint64_t n_fail, uint64_t k,
                uint32_t d, const uint64_t* offsets, const uint32_t* perm, uint64_t n, const uint32_t* cnt,
                const uint64_t* pre, uint64_t* offcnt, float* vals) {
    if (n_fail == 0) return;
    launch(ctx, "kmshard", pack_offcnt_kernel, dim3(grid1d(n_fail, kThreads, 1024)), dim3(kThreads), 0, cnt, pre,
           n_fail, offcnt);
    launch(ctx, "kmshard", pack_kernel, dim3(grid1d(n_fail * 32, kThreads)), dim3(kThreads), 0, src, work,
           n_fail, k, d, offsets, perm, n, (const uint64_t*)offcnt, vals);
}

void shard_replay(pqg_ctx* ctx, const uint32_t* work, uint64_t n_fail, uint64_t k, uint32_t d, uint32_t B,
                  const double* f64, const float* vals, uint64_t stride, const uint64_t* offcnt,
                  uint32_t world, float* table) {
    if (n_fail == 0) return;
    launch(ctx, "kmshard", replay_kernel, dim3(grid1d(n_fail, 64, 4096)), dim3(64), 0, work, n_fail, k, d, B,
           f64, vals, stride, offcnt, world, table);
}

void shard_replay_step(pqg_ctx* ctx, const RowSrc& src, const uint32_t* work, uint64_t n_fail, uint64_t k,
                       uint32_t d, const uint64_t* offsets, const uint32_t* perm, uint64_t n, double* run) {
    if (n_fail == 0) return;
    launch(ctx, "kmshard", replay_step_kernel, dim3(grid1d(n_fail * 32, kThreads)), dim3(kThreads), 0, src, work,
           n_fail, k, d, offsets, perm, n, run);
}

void shard_replay_finish(pqg_ctx* ctx, const uint32_t* work, uint64_t n_fail, uint64_t k, uint32_t d, uint32_t B,
                         const double* f64, const double* run, float* table) {
    if (n_fail == 0) return;
    launch(ctx, "kmshard", replay_finish_kernel, dim3(grid1d(n_fail, 128, 4096)), dim3(128), 0, work, n_fail, k, d,
           B, f64, run, table);
}

void shard_reseed_candidates(pqg_ctx* ctx, const RowSrc& src, uint64_t n, uint32_t B, uint32_t d,
                             const double* dist, const int* active, const uint32_t* empties, uint32_t E,
                             uint64_t row0, double* cand_d, uint64_t* cand_i, float* cand_rows) {
    launch(ctx, "reseed", reseed_cand_kernel, dim3(B), dim3(1024), 0, src, n, d, dist, active, empties, E, row0,
           cand_d, cand_i, cand_rows);
}

void shard_reseed_apply(pqg_ctx* ctx, uint32_t B, uint64_t k, uint32_t d, const double* f64,
                        const int* active, uint32_t E, uint32_t world, const double* cand_d,
                        const uint64_t* cand_i, const float* cand_rows, float* table) {
    launch(ctx, "reseed", reseed_apply_kernel, dim3(B), dim3(128), 0, k, d, B, f64, active, E, world, cand_d,
           cand_i, cand_rows, table);
}

}  // namespace pqg
