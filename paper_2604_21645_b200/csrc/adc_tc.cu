// adc_tc.cu -- batched IVF-PQ search with a tensor-core screen (ivf_query:
// proj/src/ivf.cpp:218-228; adc_table / adc_lookup: proj/src/pq.cpp:132-167;
// scan_list / finalize_hits: proj/src/ivf.cpp:51-77).
//
// The LUT scan (ivf.cu adc_scan_kernel) is bound by its shared-memory gathers
// (ncu: LSU data pipe ~89% busy, 16 random LDS per candidate).  This path
// instead scores (query, candidate) pairs on the 5th-gen tensor cores and
// keeps the LUT arithmetic only for the few candidates that can still enter a
// query's top-k:
//
//   * per index, once (cached with the index): every posting list's
//     candidates are decoded (x^_j = concat_m codeword(m, code_jm)) and stored
//     as the B operand of the 3xTF32 screen, B_j = [-2x^_j, ||x^_j||^2, 1],
//     split hi/lo in the K-major UMMA layout, lists padded to 256-row blocks;
//   * per search: the (query, probe) pairs are bucketed by list (stable
//     counting sort), each list's queries form tasks of <= 128 (the A operand
//     A_q = [q, 1, ||q||^2]), and a persistent warp-specialized kernel
//     (bulk-copy producer, single-thread MMA issuer, 4 epilogue warps; the
//     umma_big.cu pipeline) accumulates the screened ||q - x^||^2 of 128
//     queries x 256 candidates in TMEM;
//   * epilogue thread = query: a candidate whose screened value minus the
//     error bound E (3xTF32 model, umma.cu) exceeds the query's current k-th
//     exact distance cannot be in the top-k (the ADC value is within one fp32
//     rounding of ||q - x^||^2); the others are re-scored exactly as
//     adc_lookup does -- fp64 sum in m order of float(fp64 squared_l2) -- and
//     inserted into the query's list by (dist, id);
//   * each (query, probe) pair yields a top-k; the probes' lists are merged
//     by (dist, id) (topk_merge), exactly finalize_hits' order.
// Thresholds: each query's nearest list is scanned exactly first by the LUT
// kernel (slot 0 of the merge); its k-th distance seeds the query's bound,
// which finished pairs tighten through global memory (atomicMin).  Survivors
// of the screen are re-scored warp-collectively (one survivor per lane), so
// the gathers' latency is paid once per 32 survivors.
#include <cstdlib>
#include <cstring>
#include <limits>

#include "tc_common.cuh"

namespace pqg {

using namespace tc;

namespace {

constexpr uint32_t kQB = 16384;  // queries per batch (bounds the task scratch)

__device__ __forceinline__ uint32_t code_of(const uint8_t* row, uint32_t m, uint32_t w) {
    const uint8_t* p = row + m * w;
    return w == 1 ? uint32_t(p[0]) : (uint32_t(p[0]) | (uint32_t(p[1]) << 8));
}

// ---- per-index operand (cached) ----------------------------------------------
__global__ void tc_list_blocks_kernel(const uint64_t* offsets, uint64_t nlist, uint32_t* nb) {
    for (uint64_t l = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; l < nlist;
         l += uint64_t(gridDim.x) * blockDim.x)
        nb[l] = uint32_t((offsets[l + 1] - offsets[l] + kN - 1) / kN);
}

// One thread per padded candidate slot: decode, ||x^||^2, split into the block.
__global__ void tc_decode_kernel(IndexView ix, const uint64_t* blk_off, uint64_t nblocks,
                                 uint32_t kchunks, uint8_t* Bm, float* maxnorm, int* bad) {
    const uint32_t d = ix.M * ix.ds, rb = ix.M * ix.w;
    for (uint64_t s = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; s < nblocks * kN;
         s += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t b = s / kN;
        const uint32_t jl = uint32_t(s % kN);
        // list of block b: last l with blk_off[l] <= b
        uint64_t lo = 0, hi = ix.nlist;
        while (hi - lo > 1) {
            const uint64_t mid = (lo + hi) >> 1;
            if (blk_off[mid] <= b) lo = mid; else hi = mid;
        }
        const uint64_t l = lo;
        const uint64_t j = (b - blk_off[l]) * kN + jl;
        const uint64_t n_l = ix.offsets[l + 1] - ix.offsets[l];
        const bool valid = j < n_l;
        const uint8_t* row = valid ? ix.codes + (ix.offsets[l] + j) * rb : nullptr;
        float nx = 0.f;
        if (valid)
            for (uint32_t m = 0; m < ix.M; ++m) {
                uint32_t c = code_of(row, m, ix.w);
                if (c >= ix.ks) { atomicExch(bad, 1); c = 0; }
                const float* cw = ix.tables + (uint64_t(m) * ix.ks + c) * ix.ds;
                for (uint32_t t = 0; t < ix.ds; ++t) nx = fmaf(__ldg(cw + t), __ldg(cw + t), nx);
            }
        if (valid) atomicMax(reinterpret_cast<int*>(maxnorm), __float_as_int(sqrtf(nx)));
        for (uint32_t kc = 0; kc < kchunks; ++kc) {
            uint8_t* blk = Bm + (b * kchunks + kc) * (2 * kBChunk);
            for (uint32_t k4 = 0; k4 < kKC; k4 += 4) {
                float h[4], lw[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t t = kc * kKC + k4 + u;
                    float v = 0.f;
                    if (valid) {
                        if (t < d) {
                            const uint32_t m = t / ix.ds, tt = t - m * ix.ds;
                            uint32_t c = code_of(row, m, ix.w);
                            if (c >= ix.ks) c = 0;
                            v = -2.f * __ldg(ix.tables + (uint64_t(m) * ix.ks + c) * ix.ds + tt);
                        } else if (t == d) {
                            v = nx;
                        } else if (t == d + 1) {
                            v = 1.f;
                        }
                    } else if (t == d) {
                        v = 3.0e38f;  // padding slot: never passes the screen
                    }
                    h[u] = tf32_hi(v);
                    lw[u] = tf32_hi(v - h[u]);
                }
                *reinterpret_cast<float4*>(blk + il_off(jl, k4)) = make_float4(h[0], h[1], h[2], h[3]);
                *reinterpret_cast<float4*>(blk + kBChunk + il_off(jl, k4)) =
                    make_float4(lw[0], lw[1], lw[2], lw[3]);
            }
        }
    }
}

// ---- per-search tasks ----------------------------------------------------------
__global__ void tc_task_count_kernel(const uint64_t* pair_off, uint64_t nlist, uint32_t* cnt) {
    for (uint64_t l = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; l < nlist;
         l += uint64_t(gridDim.x) * blockDim.x)
        cnt[l] = uint32_t((pair_off[l + 1] - pair_off[l] + kR - 1) / kR);
}

__global__ void tc_task_fill_kernel(const uint64_t* task_off, uint64_t nlist, uint64_t* tasks) {
    for (uint64_t l = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; l < nlist;
         l += uint64_t(gridDim.x) * blockDim.x)
        for (uint64_t t = task_off[l]; t < task_off[l + 1]; ++t) tasks[t] = (l << 32) | (t - task_off[l]);
}

// One thread per (task, row): A_q = [q, 1, ||q||^2, 0..] split hi/lo, the
// row's pair (q * nprobe + p) and its screen error bound.
__global__ void tc_query_rows_kernel(const float* queries, uint32_t d, uint64_t nprobe,
                                     const uint64_t* tasks, const uint64_t* ntasks_p,
                                     uint64_t max_tasks, const uint64_t* pair_off,
                                     const uint32_t* pair_perm, const float* maxnorm_p,
                                     uint32_t kchunks, uint8_t* At, uint32_t* rowpair,
                                     float* rowE) {
    const uint64_t ntasks = *ntasks_p;
    const float maxnorm = *maxnorm_p;
    for (uint64_t s = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; s < max_tasks * kR;
         s += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t task = s / kR;
        if (task >= ntasks) break;
        const uint32_t r = uint32_t(s % kR);
        const uint64_t l = tasks[task] >> 32, t = tasks[task] & 0xFFFFFFFFu;
        const uint64_t pos = pair_off[l] + t * kR + r;
        const bool valid = pos < pair_off[l + 1];
        const uint32_t pair = valid ? pair_perm[pos] : 0xFFFFFFFFu;
        rowpair[s] = pair;
        const float* qv = valid ? queries + uint64_t(pair / nprobe) * d : nullptr;
        float nq2 = 0.f;
        if (valid)
            for (uint32_t t2 = 0; t2 < d; ++t2) nq2 = fmaf(__ldg(qv + t2), __ldg(qv + t2), nq2);
        const float qn = sqrtf(nq2) * (1.f + 1e-6f) + maxnorm;
        rowE[s] = big_error_bound(qn * qn * 1.01f + 1e-6f, kchunks);
        for (uint32_t kc = 0; kc < kchunks; ++kc) {
            uint8_t* blk = At + (task * kchunks + kc) * (2 * kAChunk);
            for (uint32_t k4 = 0; k4 < kKC; k4 += 4) {
                float h[4], lw[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t t2 = kc * kKC + k4 + u;
                    float v = 0.f;
                    if (valid) v = t2 < d ? __ldg(qv + t2) : (t2 == d ? 1.f : (t2 == d + 1 ? nq2 : 0.f));
                    h[u] = tf32_hi(v);
                    lw[u] = tf32_hi(v - h[u]);
                }
                *reinterpret_cast<float4*>(blk + il_off(r, k4)) = make_float4(h[0], h[1], h[2], h[3]);
                *reinterpret_cast<float4*>(blk + kAChunk + il_off(r, k4)) =
                    make_float4(lw[0], lw[1], lw[2], lw[3]);
            }
        }
    }
}

// Pairs keyed by list for the tensor-core pass; each query's first probe (its
// nearest list, already scanned exactly by the LUT pass) gets key nlist,
// which the bucketing skips.
__global__ void tc_pair_keys_kernel(const uint32_t* probes, uint64_t npairs, uint64_t nprobe,
                                    uint32_t nlist, uint32_t* keys, uint32_t* first) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < npairs;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const bool p0 = i % nprobe == 0;
        keys[i] = p0 ? nlist : probes[i];
        if (p0) first[i / nprobe] = probes[i];
    }
}

// Seeds each query's threshold from the exact top-k of its nearest list (a
// set of real candidates, so its k-th distance bounds the final k-th) and
// moves that top-k into probe slot 0 of the merge.
__global__ void tc_seed_kernel(const uint64_t* ids0, const double* d0, const uint32_t* c0,
                               uint64_t nq, int k, float* thr, uint64_t* slot_ids,
                               double* slot_d, uint32_t* slot_cnt) {
    for (uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nq;
         q += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t c = c0[q];
        for (uint32_t i = 0; i < c; ++i) {
            slot_ids[q * k + i] = ids0[q * k + i];
            slot_d[q * k + i] = d0[q * k + i];
        }
        slot_cnt[q] = c;
        thr[q] = c == uint32_t(k) ? __double2float_ru(d0[q * k + k - 1]) : __int_as_float(0x7f800000);
    }
}

struct TcScanArgs {
    IndexView ix;
    const float* queries;  // batch rows (nq_b x D)
    uint64_t nq_b, nprobe;
    int k;
    int has_max;
    double max_sq;
    const uint64_t* subset;
    uint64_t nsub;
    const uint64_t* tasks;
    const uint64_t* ntasks;
    const uint64_t* blk_off;
    const uint8_t* At;
    const uint8_t* Bm;
    const uint32_t* rowpair;
    const float* rowE;
    float* thr;  // per query of the batch: bound on its k-th distance (float bits, atomicMin)
    const float* luts;  // [nq_b][M][ks] adc_table entries of the batch's queries
    uint64_t* slot_ids;     // [nprobe][nq_b][k]
    double* slot_d;
    uint32_t* slot_cnt;     // [nprobe][nq_b]
    uint32_t kchunks;
};

__device__ __forceinline__ bool hit_less(double a, uint64_t ia, double b, uint64_t ib) {
    return a < b || (a == b && ia < ib);
}

// adc_lookup of one code row (pq.cpp:153-167): the query's table entries
// (float(fp64 squared_l2), built by adc_tables exactly as the LUT scan does)
// summed in fp64 in m order.  The M gathers are independent: one L2 round trip.
__device__ double exact_adc(const float* lutq, uint32_t M, uint32_t ks, uint32_t w,
                            const uint8_t* row) {
    double s = 0.0;
#pragma unroll 8
    for (uint32_t m = 0; m < M; ++m)
        s = __dadd_rn(s, (double)__ldg(lutq + uint64_t(m) * ks + code_of(row, m, w)));
    return s;
}

__global__ void __launch_bounds__(192, 1) tc_scan_kernel(TcScanArgs a) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t full[2], empty[2], tfull[2], tempty[2];
    __shared__ uint32_t tmem_base;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t ntasks = *a.ntasks;
    const uint32_t kchunks = a.kchunks;
    // per-row top-k lists of the epilogue, after the operand ring
    double* ld = reinterpret_cast<double*>(smem + 2 * size_t(kStage));
    uint64_t* li = reinterpret_cast<uint64_t*>(ld + kR * a.k);

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(smem_u32(&tmem_base)), "r"(512u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 32) {
        for (int s = 0; s < 2; ++s) {
            bar_init(&full[s], 1);
            bar_init(&empty[s], 1);
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
            for (uint64_t task = blockIdx.x; task < ntasks; task += gridDim.x) {
                const uint64_t l = a.tasks[task] >> 32;
                const uint64_t b0 = a.blk_off[l], nb = a.blk_off[l + 1] - b0;
                for (uint64_t b = 0; b < nb; ++b) {
                    for (uint32_t kc = 0; kc < kchunks; ++kc, ++q) {
                        const uint32_t s = q & 1, ph = (q >> 1) & 1;
                        bar_wait(&empty[s], ph ^ 1);
                        uint8_t* st = smem + s * kStage;
                        bar_expect_tx(&full[s], kStage);
                        bulk_g2s(st, a.At + (task * kchunks + kc) * (2 * kAChunk), 2 * kAChunk, &full[s]);
                        bulk_g2s(st + 2 * kAChunk, a.Bm + ((b0 + b) * kchunks + kc) * (2 * kBChunk),
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
            for (uint64_t task = blockIdx.x; task < ntasks; task += gridDim.x) {
                const uint64_t l = a.tasks[task] >> 32;
                const uint64_t nb = a.blk_off[l + 1] - a.blk_off[l];
                for (uint64_t b = 0; b < nb; ++b, ++u) {
                    const uint32_t buf = u & 1, tph = (u >> 1) & 1;
                    bar_wait(&tempty[buf], tph ^ 1);
                    fence_after();
                    const uint32_t d_tmem = tmem + buf * 256u;
                    for (uint32_t kc = 0; kc < kchunks; ++kc, ++q) {
                        const uint32_t s = q & 1, ph = (q >> 1) & 1;
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
                        commit(&empty[s]);
                    }
                    commit(&tfull[buf]);
                }
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const uint32_t quarter = warp & 3u;
        const uint32_t r = quarter * 32 + lane;  // query row of the task = TMEM lane
        const uint32_t lane_base = (quarter * 32u) << 16;
        const int k = a.k;
        double* my_d = ld + r * k;
        uint64_t* my_i = li + r * k;
        const uint32_t rb = a.ix.M * a.ix.w;
        const float inf32 = __int_as_float(0x7f800000);
        const float max32 = a.has_max ? __double2float_ru(a.max_sq) : inf32;
        uint32_t u = 0;
        for (uint64_t task = blockIdx.x; task < ntasks; task += gridDim.x) {
            const uint64_t l = a.tasks[task] >> 32;
            const uint64_t nb = a.blk_off[l + 1] - a.blk_off[l];
            const uint64_t lbeg = a.ix.offsets[l], n_l = a.ix.offsets[l + 1] - lbeg;
            const uint32_t pair = a.rowpair[task * kR + r];
            const bool valid = pair != 0xFFFFFFFFu;
            const uint64_t qi = valid ? pair / a.nprobe : 0, pi = valid ? pair % a.nprobe : 0;
            const float E = a.rowE[task * kR + r];
            int cnt = 0;
            float thr = valid ? *reinterpret_cast<volatile float*>(a.thr + qi) : inf32;
            for (uint64_t b = 0; b < nb; ++b, ++u) {
                const uint32_t buf = u & 1, tph = (u >> 1) & 1;
                bar_wait(&tfull[buf], tph);
                fence_after();
                const uint32_t tb = tmem + buf * 256u + lane_base;
                // screen the block's 256 candidates of this row: bit j of mk[c] set when
                // candidate 32c + j may still enter the row's top-k
                const float lim = valid ? fminf(thr, max32) : -inf32;
                uint32_t mk[kN / 32];
#pragma unroll
                for (int c = 0; c < kN / 32; ++c) {
                    uint32_t rr[32];
                    tmem_ld32(tb + c * 32, rr);
                    tmem_wait_ld();
                    uint32_t mask = 0;
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        // lower bound of the ADC value: screen - E, less the fp32
                        // rounding of the float entries and of this product
                        const float lower = (__uint_as_float(rr[j]) - E) * (1.f - 4.f * kU);
                        mask |= (lower <= lim ? 1u : 0u) << j;
                    }
                    // padding slots past the list's end
                    const int64_t left = int64_t(n_l) - int64_t(b * kN + c * 32);
                    if (left < 32) mask &= left <= 0 ? 0u : ((1u << left) - 1u);
                    mk[c] = mask;
                }
                fence_before();
                __syncwarp();
                if (lane == 0) bar_arrive(&tempty[buf]);  // TMEM free: the MMA runs ahead
                // re-score the warp's survivors together, one per lane (the latency of
                // the LUT gathers is paid once per 32 survivors, not per survivor)
                uint32_t mine = 0;
#pragma unroll
                for (int c = 0; c < kN / 32; ++c) mine += __popc(mk[c]);
                uint32_t pre = mine;  // inclusive warp prefix of survivor counts
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t v = __shfl_up_sync(0xffffffffu, pre, o);
                    if (lane >= o) pre += v;
                }
                const uint32_t total = __shfl_sync(0xffffffffu, pre, 31);
                pre -= mine;  // exclusive
                for (uint32_t base = 0; base < total; base += 32) {
                    const uint32_t t = base + lane;
                    // owner lane of survivor t: last lane whose exclusive prefix <= t
                    int owner = 0;
#pragma unroll
                    for (int step = 16; step >= 1; step >>= 1) {
                        const uint32_t pv = __shfl_sync(0xffffffffu, pre, owner + step);
                        if (owner + step < 32 && pv <= t) owner += step;
                    }
                    const uint32_t opre = __shfl_sync(0xffffffffu, pre, owner);
                    uint32_t idx = t - opre;
                    int col = 0;
#pragma unroll
                    for (int c = 0; c < kN / 32; ++c) {
                        const uint32_t om = __shfl_sync(0xffffffffu, mk[c], owner);
                        const uint32_t pc = __popc(om);
                        if (col == 0 && idx < pc) col = c * 32 + int(__fns(om, 0, int(idx) + 1)) + 1;
                        else if (col == 0) idx -= pc;
                    }
                    const uint64_t oq = __shfl_sync(0xffffffffu, qi, owner);
                    double s64 = 0.0;
                    uint64_t id = 0;
                    bool ok = t < total;
                    if (ok) {
                        const uint64_t e = lbeg + b * kN + uint64_t(col - 1);
                        s64 = exact_adc(a.luts + oq * uint64_t(a.ix.M) * a.ix.ks, a.ix.M, a.ix.ks,
                                        a.ix.w, a.ix.codes + e * rb);
                        ok = !(a.has_max && s64 > a.max_sq);
                        if (ok) id = __ldg(a.ix.ids + e);
                        if (ok && a.subset) {
                            uint64_t lo = 0, hi = a.nsub;
                            bool found = false;
                            while (lo < hi) {
                                const uint64_t mid = (lo + hi) >> 1;
                                const uint64_t v = __ldg(a.subset + mid);
                                if (v == id) { found = true; break; }
                                if (v < id) lo = mid + 1; else hi = mid;
                            }
                            ok = found;
                        }
                    }
                    // owners insert their rows' results (in survivor order)
                    uint32_t todo = __ballot_sync(0xffffffffu, ok);
                    while (todo) {
                        const int src = __ffs(todo) - 1;
                        todo &= todo - 1;
                        const int ow = __shfl_sync(0xffffffffu, owner, src);
                        const double cd = __shfl_sync(0xffffffffu, s64, src);
                        const uint64_t cid = __shfl_sync(0xffffffffu, id, src);
                        if (lane == ow && (cnt < k || hit_less(cd, cid, my_d[k - 1], my_i[k - 1]))) {
                            int pos = cnt < k ? cnt : k - 1;
                            while (pos > 0 && hit_less(cd, cid, my_d[pos - 1], my_i[pos - 1])) {
                                my_d[pos] = my_d[pos - 1];
                                my_i[pos] = my_i[pos - 1];
                                --pos;
                            }
                            my_d[pos] = cd;
                            my_i[pos] = cid;
                            if (cnt < k) ++cnt;
                            if (cnt == k) thr = fminf(thr, __double2float_ru(my_d[k - 1]));
                        }
                    }
                }
            }
            if (valid) {
                const uint64_t slot = pi * a.nq_b + qi;
                for (int i = 0; i < cnt; ++i) {
                    a.slot_ids[slot * k + i] = my_i[i];
                    a.slot_d[slot * k + i] = my_d[i];
                }
                a.slot_cnt[slot] = uint32_t(cnt);
                if (cnt == k)
                    atomicMin(reinterpret_cast<int*>(a.thr + qi), __float_as_int(__double2float_ru(my_d[k - 1])));
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

}  // namespace

// Opt-in (PQG_ADC=tc).  Measured on configs[2] (tools/adc_bench.py, r1): the
// decoded operand streams 1.25 KB per candidate from HBM where the LUT scan
// reads 16 B of codes, and list-sized tasks load-balance poorly, so this path
// is slower than the LUT scan there (3.5 ms vs 2.6 ms at M=32, far slower at
// M=8/16 where many candidates sit within the seeded thresholds); it stays as
// an exact, tested alternative, not the default.
bool adc_tc_supported(const IndexView& ix, uint64_t nq, uint64_t k, uint64_t nprobe) {
    const char* env = std::getenv("PQG_ADC");
    if (!(env && std::strcmp(env, "tc") == 0)) return false;
    if (k == 0 || k > 16 || nprobe > 64 || ix.nlist > 16384) return false;
    const uint32_t d = ix.M * ix.ds;
    (void)nq;
    return d >= 16 && d <= 1024 && ix.n > 0;
}

void adc_tc_free(TcCache& c) {
    if (c.Bm) cudaFree(c.Bm);
    if (c.blk_off) cudaFree(c.blk_off);
    if (c.maxnorm) cudaFree(c.maxnorm);
    c = TcCache{};
}

// Builds the decoded, split candidate operand of an index (once; kept with it).
// Returns false (and leaves the cache empty) if a code is out of range, so the
// LUT scan reports the error like adc_lookup does.
bool adc_tc_prepare(pqg_ctx* ctx, const IndexView& ix, TcCache& c) {
    if (c.Bm) return true;
    const uint32_t d = ix.M * ix.ds;
    const uint32_t kchunks = (d + 2 + kKC - 1) / kKC;
    uint32_t* nb = scratch<uint32_t>(ctx, ix.nlist);
    uint64_t* boff = nullptr;
    PQG_CUDA(cudaMalloc(&boff, sizeof(uint64_t) * (ix.nlist + 1)));
    launch(ctx, "tc_prepare", tc_list_blocks_kernel, dim3(grid1d(ix.nlist, 256, 1024)), dim3(256), 0,
           ix.offsets, ix.nlist, nb);
    exclusive_scan_u32(ctx, nb, boff, ix.nlist);
    uint64_t nblocks = 0;
    uint32_t last = 0;
    PQG_CUDA(cudaMemcpyAsync(&nblocks, boff + ix.nlist - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
    PQG_CUDA(cudaMemcpyAsync(&last, nb + ix.nlist - 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
    PQG_CUDA(cudaStreamSynchronize(ctx->stream));
    nblocks += last;
    PQG_CUDA(cudaMemcpyAsync(boff + ix.nlist, &nblocks, sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream));
    const uint64_t bytes = nblocks * kchunks * 2 * kBChunk;
    size_t free_b = 0, total_b = 0;
    PQG_CUDA(cudaMemGetInfo(&free_b, &total_b));
    if (bytes > free_b / 2) {  // keep the cache well inside free memory
        cudaStreamSynchronize(ctx->stream);
        cudaFree(boff);
        return false;
    }
    uint8_t* Bm = nullptr;
    float* mx = nullptr;
    PQG_CUDA(cudaMalloc(&Bm, std::max<uint64_t>(bytes, 1)));
    PQG_CUDA(cudaMalloc(&mx, sizeof(float)));
    PQG_CUDA(cudaMemsetAsync(mx, 0, sizeof(float), ctx->stream));
    int* bad = scratch<int>(ctx, 1);
    PQG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), ctx->stream));
    if (nblocks)
        launch(ctx, "tc_prepare", tc_decode_kernel, dim3(grid1d(nblocks * kN, 128, 1u << 20)), dim3(128), 0,
               ix, (const uint64_t*)boff, nblocks, kchunks, Bm, mx, bad);
    int hbad = 0;
    PQG_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    PQG_CUDA(cudaStreamSynchronize(ctx->stream));
    if (hbad) {
        cudaFree(Bm);
        cudaFree(mx);
        cudaFree(boff);
        return false;
    }
    c.Bm = Bm;
    c.blk_off = boff;
    c.maxnorm = mx;
    c.nblocks = nblocks;
    c.kchunks = kchunks;
    return true;
}

void adc_tc_search(pqg_ctx* ctx, const IndexView& ix, const TcCache& c, const float* queries,
                   uint64_t nq, const uint32_t* probes, uint64_t nprobe, uint64_t k, int has_max,
                   double max_sq, const uint64_t* subset, uint64_t nsub, uint64_t* out_ids,
                   double* out_dists, uint32_t* out_counts) {
    const uint32_t d = ix.M * ix.ds;
    const size_t smem = 2 * size_t(kStage) + size_t(kR) * k * (sizeof(double) + sizeof(uint64_t));
    PQG_CUDA(cudaFuncSetAttribute(tc_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const uint64_t qb_max = std::max<uint64_t>(
        1, std::min<uint64_t>(kQB, (uint64_t(256) << 20) / (uint64_t(ix.M) * ix.ks * 4)));
    const auto mark = ctx->arena.mark();
    for (uint64_t q0 = 0; q0 < nq; q0 += qb_max) {
        ctx->arena.reset_to(mark);
        const uint64_t nqb = std::min<uint64_t>(qb_max, nq - q0);
        const uint64_t npairs = nqb * nprobe;
        // (query, probe) pairs bucketed by list, in pair order within a list
        Bucketing bk{scratch<uint64_t>(ctx, ix.nlist + 1), scratch<uint32_t>(ctx, npairs)};
        uint32_t* keys = scratch<uint32_t>(ctx, npairs);
        uint32_t* first = scratch<uint32_t>(ctx, nqb);
        launch(ctx, "tc_tasks", tc_pair_keys_kernel, dim3(grid1d(npairs, 256, 4096)), dim3(256), 0,
               probes + q0 * nprobe, npairs, nprobe, uint32_t(ix.nlist), keys, first);
        uint64_t* nkept = scratch<uint64_t>(ctx, 1);  // pairs the bucketing keeps (p >= 1)
        const uint64_t hk = npairs - nqb;
        PQG_CUDA(cudaMemcpyAsync(nkept, &hk, sizeof(hk), cudaMemcpyHostToDevice, ctx->stream));
        stable_bucket(ctx, keys, npairs, 1, ix.nlist, nullptr, bk, nkept);
        uint32_t* tcount = scratch<uint32_t>(ctx, ix.nlist);
        uint64_t* toff = scratch<uint64_t>(ctx, ix.nlist + 1);
        launch(ctx, "tc_tasks", tc_task_count_kernel, dim3(grid1d(ix.nlist, 256, 1024)), dim3(256), 0,
               (const uint64_t*)bk.offsets, ix.nlist, tcount);
        // inclusive total lands in toff[nlist]: scan nlist+1 counts with a trailing zero
        uint32_t* tc1 = scratch<uint32_t>(ctx, ix.nlist + 1);
        PQG_CUDA(cudaMemcpyAsync(tc1, tcount, sizeof(uint32_t) * ix.nlist, cudaMemcpyDeviceToDevice, ctx->stream));
        PQG_CUDA(cudaMemsetAsync(tc1 + ix.nlist, 0, sizeof(uint32_t), ctx->stream));
        exclusive_scan_u32(ctx, tc1, toff, ix.nlist + 1);
        const uint64_t max_tasks = ix.nlist + (npairs + kR - 1) / kR;
        uint64_t* tasks = scratch<uint64_t>(ctx, max_tasks);
        launch(ctx, "tc_tasks", tc_task_fill_kernel, dim3(grid1d(ix.nlist, 128, 1024)), dim3(128), 0,
               (const uint64_t*)toff, ix.nlist, tasks);
        uint8_t* At = scratch<uint8_t>(ctx, max_tasks * c.kchunks * 2 * kAChunk);
        uint32_t* rowpair = scratch<uint32_t>(ctx, max_tasks * kR);
        float* rowE = scratch<float>(ctx, max_tasks * kR);
        const float* qb = queries + q0 * d;
        launch(ctx, "tc_tasks", tc_query_rows_kernel, dim3(grid1d(max_tasks * kR, 128, 1u << 16)), dim3(128), 0,
               qb, d, nprobe, (const uint64_t*)tasks, (const uint64_t*)(toff + ix.nlist), max_tasks,
               (const uint64_t*)bk.offsets, (const uint32_t*)bk.perm, (const float*)c.maxnorm,
               c.kchunks, At, rowpair, rowE);
        float* luts = scratch<float>(ctx, nqb * uint64_t(ix.M) * ix.ks);
        adc_tables_dev(ctx, ix.tables, ix.M, ix.ks, ix.ds, qb, nqb, luts);
        uint64_t* sid = scratch<uint64_t>(ctx, npairs * k);
        double* sd = scratch<double>(ctx, npairs * k);
        uint32_t* scnt = scratch<uint32_t>(ctx, npairs);
        // exact top-k of every query's nearest list by the LUT scan (tables from
        // global): slot 0 of the merge and the seed of the screen thresholds
        uint64_t* i0 = scratch<uint64_t>(ctx, nqb * k);
        double* d0 = scratch<double>(ctx, nqb * k);
        uint32_t* c0 = scratch<uint32_t>(ctx, nqb);
        ivf_scan(ctx, ix, qb, nqb, first, 1, k, has_max, max_sq, i0, d0, c0, ctx->d_err, subset, nsub,
                 luts);
        float* thr = scratch<float>(ctx, nqb);
        launch(ctx, "tc_tasks", tc_seed_kernel, dim3(grid1d(nqb, 256, 1024)), dim3(256), 0,
               (const uint64_t*)i0, (const double*)d0, (const uint32_t*)c0, nqb, int(k), thr, sid, sd,
               scnt);
        TcScanArgs a;
        a.ix = ix;
        a.queries = qb;
        a.nq_b = nqb;
        a.nprobe = nprobe;
        a.k = int(k);
        a.has_max = has_max;
        a.max_sq = max_sq;
        a.subset = subset;
        a.nsub = nsub;
        a.tasks = tasks;
        a.ntasks = toff + ix.nlist;
        a.blk_off = c.blk_off;
        a.At = At;
        a.Bm = c.Bm;
        a.rowpair = rowpair;
        a.rowE = rowE;
        a.thr = thr;
        a.luts = luts;
        a.slot_ids = sid;
        a.slot_d = sd;
        a.slot_cnt = scnt;
        a.kchunks = c.kchunks;
        const unsigned grid = unsigned(std::min<uint64_t>(max_tasks, uint64_t(ctx->num_sms)));
        launch(ctx, "adc_scan_tc", tc_scan_kernel, dim3(grid), dim3(192), smem, a);
        topk_merge_dev(ctx, sid, sd, scnt, uint32_t(nprobe), nqb, k, out_ids + q0 * k,
                       out_dists + q0 * k, out_counts + q0);
    }
}

}  // namespace pqg
