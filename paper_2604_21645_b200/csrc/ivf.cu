// ivf.cu -- K6 posting-list scatter, K8 coarse probe selection, K9 ADC scan
// with per-warp exact top-k, K10 shard top-k merge, id-uniqueness checks.
//
//  probe_order   proj/src/ivf.cpp:91-101  nprobe smallest (fp64 dist, list)
//  scan_list     proj/src/ivf.cpp:70-77   adc_lookup + max_sq_dist filter
//  finalize_hits proj/src/ivf.cpp:51-68   k smallest by (dist, id), sorted
//  check_ids_unique proj/src/ivf.cpp:19-26
//
// Exactness.  Probe: the fp32 screen matrix (nearest.cu, error <= E per
// query) gives tau = nprobe-th smallest screened value; every list whose
// screened value exceeds tau + 2E is provably outside the fp64 top-nprobe, so
// only lists within that band are re-scored in the reference's fp64 and
// selected by (dist, index).  Scan: each candidate's fp32 LUT sum s32 bounds
// the reference's fp64 sum (all terms >= 0, relative error <= (M+1) u); a
// candidate is re-scored in fp64 -- the same float entries added in m order,
// exactly adc_lookup -- only if s32 could beat the warp's current k-th hit.
#include <cfloat>
#include <cstdlib>
#include <cstring>

#include "kernels.cuh"

namespace pqg {

namespace {

__device__ __forceinline__ uint32_t code_at(const uint8_t* p, uint32_t m, uint32_t w) {
    p += m * w;
    return w == 1 ? uint32_t(p[0]) : (uint32_t(p[0]) | (uint32_t(p[1]) << 8));
}

// ---------------------------------------------------------------------------
// probe selection
// ---------------------------------------------------------------------------
constexpr int kSelThreads = 64;  // one query per CTA; small CTAs keep ~32 queries in flight per SM
constexpr int kCandCap = 256;
constexpr int kProbeQD = 512;  // query dims staged in fp64 by the probe select

__device__ __forceinline__ bool pair_less(double a, uint64_t ia, double b, uint64_t ib) {
    return a < b || (a == b && ia < ib);
}

// Bitonic sort of (dist, idx) pairs in shared memory, n a power of two.
__device__ void bitonic_sort(double* d, uint32_t* ix, int n) {
    for (int size = 2; size <= n; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            __syncthreads();
            for (int t = threadIdx.x; t < n / 2; t += blockDim.x) {
                const int lo = 2 * t - (t & (stride - 1));
                const int hi = lo + stride;
                const bool up = ((lo & size) == 0);
                const bool sw = up ? pair_less(d[hi], ix[hi], d[lo], ix[lo])
                                   : pair_less(d[lo], ix[lo], d[hi], ix[hi]);
                if (sw) {
                    const double td = d[lo]; d[lo] = d[hi]; d[hi] = td;
                    const uint32_t ti = ix[lo]; ix[lo] = ix[hi]; ix[hi] = ti;
                }
            }
        }
    }
    __syncthreads();
}

// PER > 0: the query's screened row is read once into registers (PER values
// per thread, blockDim * PER >= nlist) and the four digit passes and the band
// test run on them; PER == 0 re-reads the row from global memory per pass.
template <int PER>
__global__ void __launch_bounds__(1024) probe_select_kernel(
    const float* mat, uint64_t ld, const float* row_err, const float* queries, uint64_t D,
    const float* coarse, uint64_t nlist, uint64_t nprobe, uint64_t q0, uint32_t* probes,
    uint32_t* overflow, unsigned* n_overflow) {
    __shared__ uint32_t hist[256];
    __shared__ uint32_t s_prefix, s_rank;
    __shared__ uint32_t cand[kCandCap];
    __shared__ double cd[kCandCap];
    __shared__ unsigned cnt;
    const uint64_t ql = blockIdx.x;  // query within this chunk
    const uint64_t q = q0 + ql;
    const float* v = mat + ql * ld;
    const float E = row_err[ql];
    if (threadIdx.x == 0) { s_prefix = 0; s_rank = uint32_t(nprobe); cnt = 0; }
    float vals[PER > 0 ? PER : 1];
    if constexpr (PER > 0) {
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const uint64_t j = threadIdx.x + uint64_t(i) * blockDim.x;
            vals[i] = j < nlist ? __ldg(v + j) : __int_as_float(0x7f800000);
        }
    }
    uint32_t mask = 0;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        const uint32_t prefix = s_prefix;
        if constexpr (PER > 0) {
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                const uint64_t j = threadIdx.x + uint64_t(i) * blockDim.x;
                const uint32_t bits = __float_as_uint(vals[i]);
                if (j < nlist && (bits & mask) == prefix) atomicAdd(&hist[(bits >> shift) & 255u], 1u);
            }
        } else for (uint64_t j = threadIdx.x; j < nlist; j += blockDim.x) {
            const uint32_t bits = __float_as_uint(v[j]);
            if ((bits & mask) == prefix) atomicAdd(&hist[(bits >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (threadIdx.x < 32) {  // digit holding rank r: warp scan over 8 bins per lane
            const uint32_t lane = threadIdx.x;
            uint32_t h[8], sum = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) { h[i] = hist[lane * 8 + i]; sum += h[i]; }
            uint32_t incl = sum;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, incl, off);
                if (int(lane) >= off) incl += v;
            }
            const uint32_t r = s_rank;
            uint32_t c = incl - sum;
            if (c < r && r <= incl) {
                int dg = int(lane) * 8;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    if (c + h[i] >= r) { dg = int(lane) * 8 + i; break; }
                    c += h[i];
                }
                s_rank = r - c;
                s_prefix = prefix | (uint32_t(dg) << shift);
            }
        }
        mask |= 255u << shift;
        __syncthreads();
    }
    const float tau = __uint_as_float(s_prefix);
    const float band = tau + 2.05f * E;
    // a non-finite band (the query's distances overflow fp32, or a NaN): the
    // exact fallback orders every list in fp64 as probe_order does
    if (!(band < __int_as_float(0x7f800000))) {
        if (threadIdx.x == 0) overflow[atomicAdd(n_overflow, 1u)] = uint32_t(q);
        return;
    }
    if constexpr (PER > 0) {
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const uint64_t j = threadIdx.x + uint64_t(i) * blockDim.x;
            if (j < nlist && vals[i] <= band) {
                const unsigned p = atomicAdd(&cnt, 1u);
                if (p < kCandCap) cand[p] = uint32_t(j);
            }
        }
    } else for (uint64_t j = threadIdx.x; j < nlist; j += blockDim.x) {
        if (v[j] <= band) {
            const unsigned p = atomicAdd(&cnt, 1u);
            if (p < kCandCap) cand[p] = uint32_t(j);
        }
    }
    __syncthreads();
    const unsigned c = cnt;
    if (c > kCandCap) {
        if (threadIdx.x == 0) overflow[atomicAdd(n_overflow, 1u)] = uint32_t(q);
        return;
    }
    int n2 = 1;
    while (n2 < int(c)) n2 <<= 1;
    const float* qv = queries + q * D;
    // squared_l2 (proj/src/kmeans.cpp:11-18) per band candidate: the query in
    // fp64 staged once (shared), each coarse row read 32 coordinates per batch
    // of independent loads (the load latency, not the dadd chain, bounds it)
    __shared__ double qd[kProbeQD];
    const bool staged = D <= uint64_t(kProbeQD) && (D & 3u) == 0 &&
                        (reinterpret_cast<uintptr_t>(coarse) & 15u) == 0;
    if (staged)
        for (uint64_t t = threadIdx.x; t < D; t += blockDim.x) qd[t] = (double)qv[t];
    __syncthreads();
    for (int t = threadIdx.x; t < n2; t += blockDim.x) {
        if (t < int(c)) {
            const float* row = coarse + uint64_t(cand[t]) * D;
            if (staged) {
                double acc = 0.0;
                for (uint32_t t0 = 0; t0 < uint32_t(D); t0 += 32) {
                    float cv[32];
#pragma unroll
                    for (int u = 0; u < 32; u += 4) {
                        const float4 f = t0 + u < D ? __ldg(reinterpret_cast<const float4*>(row + t0 + u))
                                                    : make_float4(0.f, 0.f, 0.f, 0.f);
                        cv[u] = f.x; cv[u + 1] = f.y; cv[u + 2] = f.z; cv[u + 3] = f.w;
                    }
#pragma unroll
                    for (int u = 0; u < 32; ++u) {
                        if (t0 + u < D) {
                            const double diff = __dsub_rn(qd[t0 + u], (double)cv[u]);
                            acc = __dadd_rn(acc, __dmul_rn(diff, diff));
                        }
                    }
                }
                cd[t] = acc;
            } else {
                cd[t] = exact_sq_l2(qv, row, int(D));
            }
        } else { cd[t] = __longlong_as_double(0x7ff0000000000000LL); cand[t] = 0xFFFFFFFFu; }
    }
    bitonic_sort(cd, cand, n2);
    for (uint64_t p = threadIdx.x; p < nprobe; p += blockDim.x) probes[q * nprobe + p] = cand[p];
}

// ---------------------------------------------------------------------------
// r2h: warp per query (nlist <= 1024, nprobe <= 32), no block barriers.  The
// CTA-wide radix select above spends ~6k warp instructions per query (four
// digit passes with shared-atomic histograms, barrier-stalled: ncu
// r2f_probe_select).  Here:
//   1. each lane keeps its <= 32 screened keys in registers (column lane+32i);
//      the nprobe-th smallest LANE MINIMUM (warp bitonic sort of 32 minima)
//      is an upper bound U of tau, the nprobe-th smallest key (>= nprobe keys
//      are <= U: those minima);
//   2. the keys <= U (typically ~nprobe + a few) are compacted into shared
//      memory and tau is the candidate whose rank bracket holds nprobe -- the
//      same key the radix select finds; if more than kWCand keys are <= U
//      (heavy duplicates) tau comes from a bitwise bisection over the
//      registers instead;
//   3. band, overflow rule, fp64 re-score (squared_l2, kmeans.cpp:11-18) and
//      the (dist, index) order are those of probe_select_kernel.
// ---------------------------------------------------------------------------
constexpr int kWarpSelWarps = 8;
constexpr int kWCand = 128;

// ascending warp bitonic sort of one u32 per lane
__device__ __forceinline__ uint32_t warp_sort_u32(uint32_t v, uint32_t lane) {
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const uint32_t o = __shfl_xor_sync(0xffffffffu, v, stride);
            const bool up = (lane & size) == 0 || size == 32;
            const bool low = (lane & stride) == 0;
            v = (low == up) ? min(v, o) : max(v, o);
        }
    }
    return v;
}

// ascending warp bitonic sort of one (dist, index) pair per lane
__device__ __forceinline__ void warp_sort_pair(double& d, uint32_t& ix, uint32_t lane) {
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const double od = __shfl_xor_sync(0xffffffffu, d, stride);
            const uint32_t oi = __shfl_xor_sync(0xffffffffu, ix, stride);
            const bool up = (lane & size) == 0 || size == 32;
            const bool low = (lane & stride) == 0;
            // the lower lane of a pair keeps the smaller (ascending block) or larger
            const bool o_less = pair_less(od, oi, d, ix);
            const bool take = (low == up) ? o_less : pair_less(d, ix, od, oi);
            if (take) { d = od; ix = oi; }
        }
    }
}

// warp-local bitonic sort in shared memory (n a power of two <= 2 * kCandCap)
__device__ void warp_bitonic_sort(double* d, uint32_t* ix, int n, uint32_t lane) {
    for (int size = 2; size <= n; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            __syncwarp();
            for (int t = int(lane); t < n / 2; t += 32) {
                const int lo = 2 * t - (t & (stride - 1));
                const int hi = lo + stride;
                const bool up = ((lo & size) == 0);
                const bool sw = up ? pair_less(d[hi], ix[hi], d[lo], ix[lo])
                                   : pair_less(d[lo], ix[lo], d[hi], ix[hi]);
                if (sw) {
                    const double td = d[lo]; d[lo] = d[hi]; d[hi] = td;
                    const uint32_t ti = ix[lo]; ix[lo] = ix[hi]; ix[hi] = ti;
                }
            }
        }
    }
    __syncwarp();
}

__global__ void __launch_bounds__(kWarpSelWarps * 32) probe_select_warp_kernel(
    const float* mat, uint64_t ld, const float* row_err, const float* queries, uint64_t D,
    const float* coarse, uint64_t nlist, uint64_t nprobe, uint64_t nq, uint64_t q0, uint32_t* probes,
    uint32_t* overflow, unsigned* n_overflow) {
    __shared__ uint32_t s_cand[kWarpSelWarps][kCandCap];
    __shared__ double s_cd[kWarpSelWarps][kCandCap];
    const uint32_t lane = threadIdx.x & 31u, wq = threadIdx.x >> 5;
    const uint64_t ql = uint64_t(blockIdx.x) * kWarpSelWarps + wq;
    if (ql >= nq) return;
    const uint64_t q = q0 + ql;
    uint32_t* cand = s_cand[wq];
    double* cd = s_cd[wq];
    const float* v = mat + ql * ld;
    const float E = row_err[ql];
    const uint32_t r = uint32_t(nprobe);
    constexpr uint32_t kPad = 0xFFFFFFFFu;  // above every real key (NaN keys included)
    uint32_t key[32];
    uint32_t lmin = kPad;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        const uint64_t j = lane + 32u * uint32_t(i);
        key[i] = j < nlist ? __float_as_uint(__ldg(v + j)) : kPad;
        lmin = min(lmin, key[i]);
    }
    // 1. U = the r-th smallest lane minimum (r <= 32 <= lanes holding a real key, or r <= nlist)
    const uint32_t U = __shfl_sync(0xffffffffu, warp_sort_u32(lmin, lane), int(r - 1));
    // 2. tau = the r-th smallest key, among the keys <= U
    uint32_t nle = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) nle += (key[i] != kPad && key[i] <= U) ? 1u : 0u;
    uint32_t incl = nle;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= uint32_t(off)) incl += o;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    uint32_t tau;
    if (total <= uint32_t(kWCand)) {
        uint32_t p = incl - nle;
#pragma unroll
        for (int i = 0; i < 32; ++i)
            if (key[i] != kPad && key[i] <= U) cand[p++] = key[i];
        __syncwarp();
        uint32_t found = 0, mine = 0;
        for (uint32_t c = lane; c < total; c += 32) {
            const uint32_t x = cand[c];
            uint32_t lt = 0, le = 0;
            for (uint32_t t = 0; t < total; ++t) {
                const uint32_t y = cand[t];
                lt += y < x ? 1u : 0u;
                le += y <= x ? 1u : 0u;
            }
            if (lt < r && r <= le) { found = 1; mine = x; }
        }
        const uint32_t who = __ballot_sync(0xffffffffu, found);
        // no bracket holds r (fewer than r real keys): the exact fallback decides
        tau = who ? __shfl_sync(0xffffffffu, mine, __ffs(who) - 1) : 0xFFFFFFFFu;
        __syncwarp();
    } else {
        // bisection: the smallest t with #{keys <= t} >= r
        uint32_t ans = 0;
        for (int b = 31; b >= 0; --b) {
            const uint32_t t = ans | ((1u << b) - 1u);
            uint32_t c = 0;
#pragma unroll
            for (int i = 0; i < 32; ++i) c += (key[i] != kPad && key[i] <= t) ? 1u : 0u;
            c = __reduce_add_sync(0xffffffffu, c);
            if (c < r) ans |= 1u << b;
        }
        tau = ans;
    }
    // 3. the band of probe_select_kernel
    const float band = __uint_as_float(tau) + 2.05f * E;
    if (!(band < __int_as_float(0x7f800000))) {
        if (lane == 0) overflow[atomicAdd(n_overflow, 1u)] = uint32_t(q);
        return;
    }
    uint32_t nb = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) nb += (key[i] != kPad && __uint_as_float(key[i]) <= band) ? 1u : 0u;
    incl = nb;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= uint32_t(off)) incl += o;
    }
    const uint32_t c = __shfl_sync(0xffffffffu, incl, 31);
    if (c > uint32_t(kCandCap)) {
        if (lane == 0) overflow[atomicAdd(n_overflow, 1u)] = uint32_t(q);
        return;
    }
    const float* qv = queries + q * D;
    const bool vec = (D & 3u) == 0 && (reinterpret_cast<uintptr_t>(coarse) & 15u) == 0 &&
                     (reinterpret_cast<uintptr_t>(qv) & 15u) == 0;
    auto rescore = [&](uint32_t j) -> double {
        const float* row = coarse + uint64_t(j) * D;
        if (!vec) return exact_sq_l2(qv, row, int(D));
        double acc = 0.0;
        for (uint64_t t = 0; t < D; t += 4) {
            const float4 f = __ldg(reinterpret_cast<const float4*>(row + t));
            const float4 g = __ldg(reinterpret_cast<const float4*>(qv + t));
            const float cv[4] = {f.x, f.y, f.z, f.w}, xv[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const double diff = __dsub_rn((double)xv[u], (double)cv[u]);
                acc = __dadd_rn(acc, __dmul_rn(diff, diff));
            }
        }
        return acc;
    };
    if (c <= 32u) {
        // one band member per lane (columns compacted through shared memory:
        // a lane may hold several), then a register sort of (dist, index)
        uint32_t p = incl - nb, myj = 0xFFFFFFFFu;
#pragma unroll
        for (int i = 0; i < 32; ++i)
            if (key[i] != kPad && __uint_as_float(key[i]) <= band) cand[p++] = lane + 32u * uint32_t(i);
        __syncwarp();
        double d = __longlong_as_double(0x7ff0000000000000LL);
        if (lane < c) {
            myj = cand[lane];
            d = rescore(myj);
        }
        warp_sort_pair(d, myj, lane);
        if (lane < r) probes[q * nprobe + lane] = myj;
        return;
    }
    uint32_t p = incl - nb;
#pragma unroll
    for (int i = 0; i < 32; ++i)
        if (key[i] != kPad && __uint_as_float(key[i]) <= band) cand[p++] = lane + 32u * uint32_t(i);
    int n2 = 1;
    while (n2 < int(c)) n2 <<= 1;
    __syncwarp();
    for (int t = int(lane); t < n2; t += 32) {
        if (t < int(c)) cd[t] = rescore(cand[t]);
        else { cd[t] = __longlong_as_double(0x7ff0000000000000LL); cand[t] = 0xFFFFFFFFu; }
    }
    warp_bitonic_sort(cd, cand, n2, lane);
    for (uint64_t pp = lane; pp < nprobe; pp += 32) probes[q * nprobe + pp] = cand[pp];
}

// Rare fallback (more than kCandCap lists inside the screen band, e.g. many
// duplicate coarse centroids): exact fp64 for every list, then nprobe rounds
// of a block-wide (dist, index) argmin.
__global__ void probe_exact_kernel(const uint32_t* overflow, const unsigned* n_overflow,
                                   const float* queries, uint64_t D, const float* coarse,
                                   uint64_t nlist, uint64_t nprobe, double* scratch_d,
                                   uint32_t* probes) {
    __shared__ double sv[32];
    __shared__ uint64_t si[32];
    const unsigned total = *n_overflow;
    for (unsigned o = blockIdx.x; o < total; o += gridDim.x) {
        const uint64_t q = overflow[o];
        double* dd = scratch_d + uint64_t(blockIdx.x) * nlist;
        for (uint64_t j = threadIdx.x; j < nlist; j += blockDim.x)
            dd[j] = exact_sq_l2(queries + q * D, coarse + j * D, int(D));
        __syncthreads();
        for (uint64_t p = 0; p < nprobe; ++p) {
            double bv = __longlong_as_double(0x7ff0000000000000LL);
            uint64_t bi = ~uint64_t(0);
            for (uint64_t j = threadIdx.x; j < nlist; j += blockDim.x) {
                const double x = dd[j];
                if (x == -1.0) continue;  // taken
                if (bi == ~uint64_t(0) || pair_less(x, j, bv, bi)) { bv = x; bi = j; }
            }
            for (int off = 16; off >= 1; off >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
                const uint64_t oi = __shfl_xor_sync(0xffffffffu, bi, off);
                if (oi != ~uint64_t(0) && (bi == ~uint64_t(0) || pair_less(ov, oi, bv, bi))) { bv = ov; bi = oi; }
            }
            const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
            if (lane == 0) { sv[w] = bv; si[w] = bi; }
            __syncthreads();
            if (threadIdx.x == 0) {
                for (int i = 1; i < int(blockDim.x >> 5); ++i)
                    if (si[i] != ~uint64_t(0) && (bi == ~uint64_t(0) || pair_less(sv[i], si[i], bv, bi))) { bv = sv[i]; bi = si[i]; }
                probes[q * nprobe + p] = uint32_t(bi);
                dd[bi] = -1.0;
            }
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------------------
// ADC scan with an exact per-warp top-k (k <= 32)
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 256;

struct TopK {
    double d;
    uint64_t id;
};

// Merge the warp's survivor buffer (n <= 32 entries in shared memory) into
// its sorted list (lane l holds entry l; 32 entries kept, the first k are the
// top-k): bitonic sort of the buffer across the lanes, then the first stage
// of a bitonic merge against the list (min of list[l] and buffer[31 - l]
// keeps the 32 smallest of the union) and five half-cleaner steps.  Order is
// (dist, id) as in finalize_hits (proj/src/ivf.cpp:51-56).
__device__ __forceinline__ void warp_merge_buffer(const TopK* buf, uint32_t n, double& my_d, uint64_t& my_id,
                                               int lane) {
    double bd = __longlong_as_double(0x7ff0000000000000LL);
    uint64_t bi = ~uint64_t(0);
    if (uint32_t(lane) < n) { bd = buf[lane].d; bi = buf[lane].id; }
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const double od = __shfl_xor_sync(0xffffffffu, bd, stride);
            const uint64_t oi = __shfl_xor_sync(0xffffffffu, bi, stride);
            const bool take_min = ((lane & stride) == 0) == ((lane & size) == 0 || size == 32);
            const bool o_less = pair_less(od, oi, bd, bi);
            if (take_min == o_less && !(od == bd && oi == bi)) { bd = od; bi = oi; }
        }
    }
    const double rd = __shfl_sync(0xffffffffu, bd, 31 - lane);
    const uint64_t ri = __shfl_sync(0xffffffffu, bi, 31 - lane);
    if (pair_less(rd, ri, my_d, my_id)) { my_d = rd; my_id = ri; }
#pragma unroll
    for (int stride = 16; stride > 0; stride >>= 1) {
        const double od = __shfl_xor_sync(0xffffffffu, my_d, stride);
        const uint64_t oi = __shfl_xor_sync(0xffffffffu, my_id, stride);
        const bool take_min = (lane & stride) == 0;
        const bool o_less = pair_less(od, oi, my_d, my_id);
        if (take_min == o_less && !(od == my_d && oi == my_id)) { my_d = od; my_id = oi; }
    }
}

// Insert (d, id) into the warp's sorted list (lane l < k holds entry l).
__device__ __forceinline__ void warp_insert(double& my_d, uint64_t& my_id, double d, uint64_t id,
                                           int k, int lane) {
    const bool before = lane < k && pair_less(my_d, my_id, d, id);
    const uint32_t m = __ballot_sync(0xffffffffu, before);
    const int pos = __popc(m);
    const double up_d = __shfl_up_sync(0xffffffffu, my_d, 1);
    const uint64_t up_id = __shfl_up_sync(0xffffffffu, my_id, 1);
    if (pos < k) {
        if (lane == pos) { my_d = d; my_id = id; }
        else if (lane > pos && lane < k) { my_d = up_d; my_id = up_id; }
    }
}

__device__ __forceinline__ float lds_f32(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}

// (a0, a1) += (b0, b1) as one packed FADD2 (sm_100): the even and odd
// subspace chains of the screen sum advance together.
__device__ __forceinline__ void add_f32x2(float& a0, float& a1, float b0, float b1) {
    unsigned long long x, y, r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a0), "f"(a1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(y) : "f"(b0), "f"(b1));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(x), "l"(y));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(r));
}

// A code row of RB bytes (RB in {4, 8, 16, 32}) read with vector loads; the
// codes are extracted from registers (RB == 0: generic byte path).
template <int RB>
struct CodeRow {
    uint32_t w[RB > 0 ? RB / 4 : 1];
    __device__ __forceinline__ void load(const uint8_t* p) {
        if constexpr (RB == 4) {
            w[0] = __ldg(reinterpret_cast<const uint32_t*>(p));
        } else if constexpr (RB == 8) {
            const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
            w[0] = v.x; w[1] = v.y;
        } else if constexpr (RB == 16 || RB == 32) {
#pragma unroll
            for (int q = 0; q < RB / 16; ++q) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(p) + q);
                w[4 * q] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
            }
        }
    }
    // code of subspace m for code width W
    template <int W>
    __device__ __forceinline__ uint32_t get(int m) const {
        if constexpr (W == 1) return (w[m >> 2] >> ((m & 3) * 8)) & 0xFFu;
        else return (w[m >> 1] >> ((m & 1) * 16)) & 0xFFFFu;
    }
};

template <int RB, int W, int KS>
__global__ void __launch_bounds__(kScanThreads, (RB >= 32 ? 5 : 6)) adc_scan_kernel(
    const float* tables, uint32_t M, uint32_t ks, uint32_t ds, const float* queries,
    const uint64_t* offsets, const uint64_t* ids, const uint8_t* codes, const uint32_t* probes,
    uint64_t nprobe, int k, int has_max, double max_sq, const uint64_t* subset, uint64_t nsub,
    uint64_t* out_ids, double* out_dists, uint32_t* out_counts, int* err, const float* luts) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* lut = reinterpret_cast<float*>(smem_raw);  // [M][ks]
    TopK* wl = reinterpret_cast<TopK*>(smem_raw + ((sizeof(float) * M * ks + 15) & ~size_t(15)));
    const uint64_t q = blockIdx.x;
    const uint32_t w = ks <= 256 ? 1 : 2;
    // ivf_query_subset (proj/src/ivf.cpp:79-88): candidates outside the sorted
    // subset are skipped before they can enter the top-k
    auto member = [&](uint64_t id) {
        if (!subset) return true;
        uint64_t lo = 0, hi = nsub;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            const uint64_t v = __ldg(subset + mid);
            if (v == id) return true;
            if (v < id) lo = mid + 1; else hi = mid;
        }
        return false;
    };
    const uint32_t rb = M * w;
    const uint64_t D = uint64_t(M) * ds;
    const float* qv = queries + q * D;
    if (luts) {  // tables already built (adc_tables, identical entries)
        const float* lq = luts + q * uint64_t(M) * ks;
        if (((M * ks) & 3u) == 0 && (reinterpret_cast<uintptr_t>(lq) & 15u) == 0) {
            const float4* l4 = reinterpret_cast<const float4*>(lq);
            for (uint32_t e = threadIdx.x; e < M * ks / 4; e += blockDim.x)
                reinterpret_cast<float4*>(lut)[e] = __ldg(l4 + e);
        } else {
            for (uint32_t e = threadIdx.x; e < M * ks; e += blockDim.x) lut[e] = __ldg(lq + e);
        }
    } else {
        // adc_table (proj/src/pq.cpp:132-151): the query converted to fp64 once
        // (shared), then per entry the codeword's conversions and the
        // reference's dsub / dmul / dadd chain in t order
        double* qd = reinterpret_cast<double*>(wl + (kScanThreads / 32) * k);
        for (uint32_t t = threadIdx.x; t < D; t += blockDim.x) qd[t] = (double)qv[t];
        __syncthreads();
        const bool pf = (ds == 8 || ds == 4) && ks <= blockDim.x &&
                        (reinterpret_cast<uintptr_t>(tables) & 15u) == 0;
        if (pf) {
            // Ds <= 8 (one codeword = 1-2 float4): each thread owns codeword j
            // of every subspace and loads subspace m+1's codeword while it
            // computes subspace m's entry (the load latency stays hidden)
            const uint32_t j = threadIdx.x;
            if (j < ks) {
                const uint32_t nv = ds / 4;
                const float4* cp = reinterpret_cast<const float4*>(tables) + uint64_t(j) * nv;
                const uint64_t mstride = uint64_t(ks) * nv;
                float4 n0 = __ldg(cp), n1 = nv > 1 ? __ldg(cp + 1) : n0;
                for (uint32_t m = 0; m < M; ++m) {
                    const float4 u0 = n0, u1 = n1;
                    if (m + 1 < M) {
                        n0 = __ldg(cp + (m + 1) * mstride);
                        if (nv > 1) n1 = __ldg(cp + (m + 1) * mstride + 1);
                    }
                    const float cc[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
                    const double* qm = qd + m * ds;
                    double acc = 0.0;
#pragma unroll
                    for (int v = 0; v < 8; ++v) {
                        if (uint32_t(v) < ds) {
                            const double diff = __dsub_rn(qm[v], (double)cc[v]);
                            acc = __dadd_rn(acc, __dmul_rn(diff, diff));
                        }
                    }
                    lut[m * ks + j] = __double2float_rn(acc);
                }
            }
        } else for (uint32_t m = 0; m < M; ++m) {
            const double* qm = qd + m * ds;
            for (uint32_t j = threadIdx.x; j < ks; j += blockDim.x) {
                const float* c = tables + (uint64_t(m) * ks + j) * ds;
                double acc = 0.0;
                if ((ds & 3u) == 0 && (reinterpret_cast<uintptr_t>(c) & 15u) == 0) {
                    for (uint32_t t = 0; t < ds; t += 4) {
                        const float4 u = __ldg(reinterpret_cast<const float4*>(c + t));
                        const float cc[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                        for (int v = 0; v < 4; ++v) {
                            const double diff = __dsub_rn(qm[t + v], (double)cc[v]);
                            acc = __dadd_rn(acc, __dmul_rn(diff, diff));
                        }
                    }
                } else {
                    for (uint32_t t = 0; t < ds; ++t) {
                        const double diff = __dsub_rn(qm[t], (double)__ldg(c + t));
                        acc = __dadd_rn(acc, __dmul_rn(diff, diff));
                    }
                }
                lut[m * ks + j] = __double2float_rn(acc);
            }
        }
    }
    __syncthreads();
    const uint32_t lut_s = static_cast<uint32_t>(__cvta_generic_to_shared(lut));
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    double my_d = inf;
    uint64_t my_id = ~uint64_t(0);
    // the list's current k-th entry, held by every lane (refreshed after inserts
    // only): the screen and the insertion test need no shuffles
    double kd = inf;
    uint64_t ki = ~uint64_t(0);
    const float shrink = 1.0f - float(M + 2) * kU * 1.05f;
    // Early exit on partial sums (Ks = 256 byte codes: every code is valid, so
    // skipping the rest of a row cannot hide a range error).  LUT entries are
    // >= 0, so a partial sum bounds the full one from below; after each group
    // of subspaces a lane whose bound already exceeds the list's k-th (or
    // max_sq) drops out, and the warp stops when no lane is left.  The fp32
    // test is conservative: partial * shrink_p (rounded) <= the exact partial
    // sum of the fp32 entries for any h <= M terms, and the k-th is rounded up.
    constexpr bool kPrune = RB > 0 && W == 1 && KS == 256;
    const float shrink_p = 1.0f - float(M + 4) * kU * 1.05f;
    const float max32 = has_max ? __double2float_ru(max_sq) : __int_as_float(0x7f800000);
    float lim = max32;  // kPrune: min(k-th rounded up, max_sq), refreshed on insertion
    // the exit test compares the raw fp32 partial sum with lim / shrink_p
    // rounded up: sum > lim_p implies sum * shrink_p > lim in exact arithmetic
    float lim_p = __fdiv_ru(lim, shrink_p);
    // kPrune: per-warp survivor buffer (32 entries) after the fp64 query
    TopK* buf = reinterpret_cast<TopK*>(reinterpret_cast<double*>(wl + (kScanThreads / 32) * k) + D) + wid * 32;
    uint32_t bcnt = 0;
    for (uint64_t p = 0; p < nprobe; ++p) {
        const uint32_t l = probes[q * nprobe + p];
        const uint64_t beg = offsets[l], end = offsets[l + 1];
        // 32-bit offsets within the list (a shard's list is < 2^32 rows)
        const uint32_t len = uint32_t(end - beg);
        const uint8_t* lcodes = codes + beg * RB;
        const uint64_t* lids = ids + beg;
        for (uint32_t o = uint32_t(wid) * 32; o < len; o += kScanThreads) {
            const double th = kd;
            const uint64_t e = beg + o + lane;
            bool want = false;
            double s64 = 0.0;
            uint64_t id = 0;
            if constexpr (kPrune) {
                constexpr int MM = RB;
                constexpr int GS = MM >= 32 ? 8 : 4;
                const uint32_t oe = o + lane;
                const bool valid = oe < len;
                CodeRow<RB> row;
                if (valid) row.load(lcodes + oe * RB);
                else {
#pragma unroll
                    for (int i = 0; i < RB / 4; ++i) row.w[i] = 0;
                }
                bool live = valid;
                float s_even = 0.f, s_odd = 0.f;
#pragma unroll
                for (int g = 0; g < MM; g += GS) {
                    if (g > 0) {
                        live = live && !(s_even + s_odd > lim_p);
                        if (!__any_sync(0xffffffffu, live)) break;
                    }
                    if (live) {
#pragma unroll
                        for (int i = g / 4; i < (g + GS) / 4; ++i) {
                            // the word passes through an opaque move here, so its
                            // byte extraction is not hoisted above the exit test
                            uint32_t cw = row.w[i];
                            asm volatile("" : "+r"(cw));
                            const uint32_t a0 = lut_s + uint32_t(4 * i) * 1024u;
                            const float v0 = lds_f32(a0 + ((cw << 2) & 0x3fcu));
                            const float v1 = lds_f32(a0 + 1024u + ((cw >> 6) & 0x3fcu));
                            const float v2 = lds_f32(a0 + 2048u + ((cw >> 14) & 0x3fcu));
                            const float v3 = lds_f32(a0 + 3072u + ((cw >> 22) & 0x3fcu));
                            add_f32x2(s_even, s_odd, v0, v1);
                            add_f32x2(s_even, s_odd, v2, v3);
                        }
                    }
                }
                if (live) {
                    const double lower = double(s_even + s_odd) * double(shrink);
                    if (lower <= th && !(has_max && lower > max_sq)) {
#pragma unroll
                        for (int m = 0; m < MM; ++m)
                            s64 = __dadd_rn(s64, (double)lut[m * 256 + row.template get<1>(m)]);
                        id = lids[oe];
                        want = !(has_max && s64 > max_sq) && member(id);
                    }
                }
            } else if (e < end) {
                const uint8_t* cr = codes + e * rb;
                float s32 = 0.f;
                bool bad = false;
                if constexpr (RB > 0) {
                    const uint32_t ksc = KS > 0 ? uint32_t(KS) : ks;
                    const bool check = KS == 0 && (W == 2 || ks < 256);
                    CodeRow<RB> row;
                    row.load(cr);
                    constexpr int MM = RB / W;
                    float s_even = 0.f, s_odd = 0.f;  // two chains, one FADD2 per pair
#pragma unroll
                    for (int m = 0; m < MM; m += 2) {
                        uint32_t c0 = row.template get<W>(m), c1 = row.template get<W>(m + 1);
                        if (check) {
                            if (c0 >= ks || c1 >= ks) bad = true;
                            c0 = min(c0, ks - 1);
                            c1 = min(c1, ks - 1);
                        }
                        add_f32x2(s_even, s_odd, lut[m * ksc + c0], lut[(m + 1) * ksc + c1]);
                    }
                    s32 = s_even + s_odd;
                    if (!bad) {
                        const double lower = double(s32) * double(shrink);
                        if (lower <= th && !(has_max && lower > max_sq)) {
#pragma unroll
                            for (int m = 0; m < MM; ++m)
                                s64 = __dadd_rn(s64, (double)lut[m * ksc + row.template get<W>(m)]);
                            id = ids[e];
                            want = !(has_max && s64 > max_sq) && member(id);
                        }
                    }
                } else {
                    for (uint32_t m = 0; m < M; ++m) {
                        const uint32_t c = code_at(cr, m, w);
                        if (c >= ks) { bad = true; break; }
                        s32 += lut[m * ks + c];
                    }
                    if (!bad) {
                        const double lower = double(s32) * double(shrink);
                        if (lower <= th && !(has_max && lower > max_sq)) {
                            for (uint32_t m = 0; m < M; ++m)
                                s64 = __dadd_rn(s64, (double)lut[m * ks + code_at(cr, m, w)]);
                            id = ids[e];
                            want = !(has_max && s64 > max_sq) && member(id);
                        }
                    }
                }
                if (bad) atomicExch(err, 1);
            }
            want = want && pair_less(s64, id, kd, ki);
            if constexpr (kPrune) {
                // survivors are appended to the warp's buffer; a full buffer is
                // sorted and merged into the list (warp_merge_buffer)
                uint32_t ball = __ballot_sync(0xffffffffu, want);
                if (ball) {
                    if (bcnt + uint32_t(__popc(ball)) > 32u) {
                        warp_merge_buffer(buf, bcnt, my_d, my_id, lane);
                        bcnt = 0;
                        kd = __shfl_sync(0xffffffffu, my_d, k - 1);
                        ki = __shfl_sync(0xffffffffu, my_id, k - 1);
                        lim = fminf(__double2float_ru(kd), max32);
                        lim_p = __fdiv_ru(lim, shrink_p);
                        want = want && pair_less(s64, id, kd, ki);
                        ball = __ballot_sync(0xffffffffu, want);
                    }
                    if (want) buf[bcnt + __popc(ball & ((1u << lane) - 1u))] = TopK{s64, id};
                    bcnt += uint32_t(__popc(ball));
                    __syncwarp();
                }
                continue;
            }
            uint32_t ball = __ballot_sync(0xffffffffu, want);
            while (ball) {
                const int src = __ffs(ball) - 1;
                const double cd = __shfl_sync(0xffffffffu, s64, src);
                const uint64_t cid = __shfl_sync(0xffffffffu, id, src);
                warp_insert(my_d, my_id, cd, cid, k, lane);
                kd = __shfl_sync(0xffffffffu, my_d, k - 1);
                ki = __shfl_sync(0xffffffffu, my_id, k - 1);
                want = want && lane != src && pair_less(s64, id, kd, ki);
                ball = __ballot_sync(0xffffffffu, want);
                if constexpr (kPrune) {
                    lim = fminf(__double2float_ru(kd), max32);
                    lim_p = __fdiv_ru(lim, shrink_p);
                }
            }
        }
    }
    if constexpr (kPrune) {
        if (bcnt) warp_merge_buffer(buf, bcnt, my_d, my_id, lane);
    }
    // merge the warps' lists through shared memory into warp 0
    if (lane < k) wl[wid * k + lane] = TopK{my_d, my_id};
    __syncthreads();
    if (wid != 0) return;
    for (int ow = 1; ow < int(kScanThreads / 32); ++ow) {
        for (int j = 0; j < k; ++j) {
            const TopK c = wl[ow * k + j];
            const double thd = __shfl_sync(0xffffffffu, my_d, k - 1);
            const uint64_t thi = __shfl_sync(0xffffffffu, my_id, k - 1);
            if (!pair_less(c.d, c.id, thd, thi)) break;  // lists are sorted
            warp_insert(my_d, my_id, c.d, c.id, k, lane);
        }
    }
    const bool valid = lane < k && my_id != ~uint64_t(0);
    const uint32_t vm = __ballot_sync(0xffffffffu, valid);
    if (lane < k) {
        out_ids[q * k + lane] = valid ? my_id : 0;
        out_dists[q * k + lane] = valid ? my_d : 0.0;
    }
    if (lane == 0) out_counts[q] = __popc(vm);
}

// ---------------------------------------------------------------------------
// CSR scatter, duplicate detection, shard merge
// ---------------------------------------------------------------------------
__global__ void csr_scatter_kernel(const uint32_t* perm, uint64_t n, const uint64_t* ids,
                                   const uint8_t* codes, uint64_t rb, uint64_t* out_ids,
                                   uint8_t* out_codes) {
    for (uint64_t p = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < n;
         p += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t src = perm[p];
        out_ids[p] = ids[src];
        const uint8_t* s = codes + src * rb;
        uint8_t* d = out_codes + p * rb;
        if (rb == 16) {
            *reinterpret_cast<uint4*>(d) = *reinterpret_cast<const uint4*>(s);
        } else if (rb == 8) {
            *reinterpret_cast<uint2*>(d) = *reinterpret_cast<const uint2*>(s);
        } else {
            for (uint64_t j = 0; j < rb; ++j) d[j] = s[j];
        }
    }
}

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return x;
}

// Open-addressing set: state 0 empty / 1 being written / 2 ready; minpos
// keeps the first input position of each id.
__global__ void dup_insert_kernel(const uint64_t* ids, uint64_t n, uint64_t cap_mask,
                                  int* state, uint64_t* keys, unsigned long long* minpos) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t id = ids[i];
        uint64_t s = mix64(id) & cap_mask;
        for (;;) {
            int st = atomicCAS(state + s, 0, 1);
            if (st == 0) {
                keys[s] = id;
                __threadfence();
                atomicExch(state + s, 2);
                atomicMin(minpos + s, (unsigned long long)i);
                break;
            }
            while ((st = atomicAdd(state + s, 0)) != 2) {}
            __threadfence();
            if (keys[s] == id) {
                atomicMin(minpos + s, (unsigned long long)i);
                break;
            }
            s = (s + 1) & cap_mask;
        }
    }
}

__global__ void dup_find_kernel(const uint64_t* ids, uint64_t n, uint64_t cap_mask,
                                const uint64_t* keys, const unsigned long long* minpos,
                                unsigned long long* first_dup) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t id = ids[i];
        uint64_t s = mix64(id) & cap_mask;
        while (keys[s] != id) s = (s + 1) & cap_mask;
        if (minpos[s] != i) atomicMin(first_dup, (unsigned long long)i);
    }
}

__global__ void topk_merge_kernel(const uint64_t* ids, const double* dists, const uint32_t* counts,
                                  uint32_t shards, uint64_t nq, uint64_t k, uint64_t* out_ids,
                                  double* out_dists, uint32_t* out_counts) {
    for (uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nq;
         q += uint64_t(gridDim.x) * blockDim.x) {
        uint32_t pos[64];
        for (uint32_t s = 0; s < shards; ++s) pos[s] = 0;
        uint32_t outc = 0;
        while (outc < k) {
            int best = -1;
            double bd = 0;
            uint64_t bi = 0;
            for (uint32_t s = 0; s < shards; ++s) {
                const uint64_t base = (uint64_t(s) * nq + q) * k;
                if (pos[s] >= counts[uint64_t(s) * nq + q]) continue;
                const double d = dists[base + pos[s]];
                const uint64_t id = ids[base + pos[s]];
                if (best < 0 || pair_less(d, id, bd, bi)) { best = int(s); bd = d; bi = id; }
            }
            if (best < 0) break;
            ++pos[best];
            out_ids[q * k + outc] = bi;
            out_dists[q * k + outc] = bd;
            ++outc;
        }
        for (uint32_t j = outc; j < k; ++j) { out_ids[q * k + j] = 0; out_dists[q * k + j] = 0.0; }
        out_counts[q] = outc;
    }
}

}  // namespace

// r2e: the probe matrix of a few queries (a single ivf_query): thread per
// (query, list), the reference's fp64 squared_l2 (proj/src/kmeans.cpp:11-18)
// rounded to fp32, and row_err = 2^-23 * the row's largest value (rounded
// up) bounds |fp32 - fp64| for the select's band test; a non-finite distance
// makes the band infinite, so the query takes the exact fallback.
__global__ void small_probe_matrix_kernel(const float* queries, uint64_t D, const float* coarse, uint64_t nlist,
                                          uint64_t nq, float* mat, unsigned* row_err_bits) {
    const uint64_t q = blockIdx.y;
    const uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= nq || j >= nlist) return;
    const float* qv = queries + q * D;
    const float* cv = coarse + j * D;
    double acc = 0.0;
    uint64_t t0 = 0;
    if ((D & 3u) == 0 && ((reinterpret_cast<uintptr_t>(qv) | reinterpret_cast<uintptr_t>(cv)) & 15u) == 0) {
        for (; t0 + 16 <= D; t0 += 16) {  // sixteen coordinates' loads in flight
            float4 a[4], c[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                a[u] = __ldg(reinterpret_cast<const float4*>(qv + t0) + u);
                c[u] = __ldg(reinterpret_cast<const float4*>(cv + t0) + u);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float av[4] = {a[u].x, a[u].y, a[u].z, a[u].w}, cc[4] = {c[u].x, c[u].y, c[u].z, c[u].w};
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const double diff = __dsub_rn((double)av[v], (double)cc[v]);
                    acc = __dadd_rn(acc, __dmul_rn(diff, diff));
                }
            }
        }
    }
    for (; t0 < D; ++t0) {
        const double diff = __dsub_rn((double)qv[t0], (double)cv[t0]);
        acc = __dadd_rn(acc, __dmul_rn(diff, diff));
    }
    const float f = __double2float_rn(acc);
    mat[q * nlist + j] = f;
    const unsigned eb = isfinite(f) ? __float_as_uint(__fmul_ru(f, 1.1920929e-07f)) : 0x7f800000u;
    atomicMax(row_err_bits + q, eb);
}

void ivf_probe(pqg_ctx* ctx, const IndexView& ix, const float* queries, uint64_t nq,
               uint64_t nprobe, uint32_t* probes) {
    const uint64_t D = uint64_t(ix.M) * ix.ds;
    // chunk the queries so the screen matrix stays <= 512 MB
    uint64_t chunk = std::max<uint64_t>(1, (uint64_t(128) << 20) / std::max<uint64_t>(1, ix.nlist));
    chunk = std::min<uint64_t>(chunk, nq);
    float* mat = scratch<float>(ctx, chunk * ix.nlist);
    float* rerr = scratch<float>(ctx, chunk);
    uint32_t* overflow = scratch<uint32_t>(ctx, nq);
    unsigned* n_over = scratch<unsigned>(ctx, 1);
    PQG_CUDA(cudaMemsetAsync(n_over, 0, sizeof(unsigned), ctx->stream));
    for (uint64_t q0 = 0; q0 < nq; q0 += chunk) {
        const uint64_t nc = std::min(chunk, nq - q0);
        NearestArgs a;
        a.src.x = queries + q0 * D;
        a.src.ldx = D;
        a.n = nc;
        a.d = uint32_t(D);
        a.B = 1;
        a.table = ix.coarse;
        a.k = ix.nlist;
        a.cnorm = ix.coarse_norm;
        a.cmax = ix.coarse_max;
        a.out_mat = mat;
        a.ld_mat = ix.nlist;
        a.row_err = rerr;
        if (nc <= 16) {  // a few queries: one exact kernel (the tensor-core path pays off for batches)
            PQG_CUDA(cudaMemsetAsync(rerr, 0, sizeof(float) * nc, ctx->stream));
            launch(ctx, "probe_select", small_probe_matrix_kernel,
                   dim3(unsigned((ix.nlist + 127) / 128), unsigned(nc)), dim3(128), 0, queries + q0 * D, D,
                   ix.coarse, ix.nlist, nc, mat, reinterpret_cast<unsigned*>(rerr));
        } else {
            distance_matrix(ctx, a);
        }
        // 16 screened values per thread in registers (nlist <= 16384), else
        // the row is re-read per pass
        constexpr int kPer = 16;
        const char* sel_env = std::getenv("PQG_PROBE_SEL");
        const bool warp_sel = !(sel_env && std::strcmp(sel_env, "cta") == 0);
        if (warp_sel && ix.nlist <= 1024 && nprobe <= 32) {
            launch(ctx, "probe_select", probe_select_warp_kernel,
                   dim3(unsigned((nc + kWarpSelWarps - 1) / kWarpSelWarps)), dim3(kWarpSelWarps * 32), 0,
                   (const float*)mat, ix.nlist, (const float*)rerr, queries, D, ix.coarse, ix.nlist, nprobe,
                   nc, q0, probes, overflow, n_over);
        } else if (ix.nlist <= uint64_t(kPer) * 1024) {
            const unsigned th = unsigned(std::max<uint64_t>(kSelThreads, (ix.nlist + kPer * 32 - 1) / (kPer * 32) * 32));
            launch(ctx, "probe_select", probe_select_kernel<kPer>, dim3(unsigned(nc)), dim3(th), 0,
                   (const float*)mat, ix.nlist, (const float*)rerr, queries, D, ix.coarse, ix.nlist,
                   nprobe, q0, probes, overflow, n_over);
        } else {
            launch(ctx, "probe_select", probe_select_kernel<0>, dim3(unsigned(nc)), dim3(kSelThreads), 0,
                   (const float*)mat, ix.nlist, (const float*)rerr, queries, D, ix.coarse, ix.nlist,
                   nprobe, q0, probes, overflow, n_over);
        }
    }
    const unsigned fb_blocks = 64;
    double* sd = scratch<double>(ctx, uint64_t(fb_blocks) * ix.nlist);
    launch(ctx, "probe_exact", probe_exact_kernel, dim3(fb_blocks), dim3(256), 0,
           (const uint32_t*)overflow, (const unsigned*)n_over, queries, D, ix.coarse, ix.nlist,
           nprobe, sd, probes);
}

__global__ void pairs_prep_kernel(const float* queries, uint64_t D, const uint32_t* probes, uint64_t nq,
                                  uint64_t nprobe, float* qrep, uint32_t* prep) {
    // pair = p * nq + q: query q's p-th probed list as a one-list query
    const uint64_t total = nq * nprobe;
    for (uint64_t pr = blockIdx.x; pr < total; pr += gridDim.x) {
        const uint64_t p = pr / nq, q = pr - p * nq;
        for (uint64_t t = threadIdx.x; t < D; t += blockDim.x) qrep[pr * D + t] = queries[q * D + t];
        if (threadIdx.x == 0) prep[pr] = probes[q * nprobe + p];
    }
}

void ivf_scan(pqg_ctx* ctx, const IndexView& ix, const float* queries, uint64_t nq,
              const uint32_t* probes, uint64_t nprobe, uint64_t k, int has_max, double max_sq,
              uint64_t* out_ids, double* out_dists, uint32_t* out_counts, int* err,
              const uint64_t* subset, uint64_t nsub, const float* luts) {
    // r2e: a few queries would leave all but nq SMs idle -- scan every
    // (query, probed list) pair in its own CTA (a one-list query) and merge
    // the per-list top-k by (dist, id) (finalize_hits' order: the k best of
    // the union are the k best of the per-list k best)
    const char* se = std::getenv("PQG_ADC_SPLIT");
    if (k <= 32 && !luts && nprobe > 1 && nprobe <= 64 && nq * nprobe <= uint64_t(4) * ctx->num_sms && nq < 64 &&
        !(se && se[0] == '0')) {
        const uint64_t D = uint64_t(ix.M) * ix.ds, np = nq * nprobe;
        float* qrep = scratch<float>(ctx, np * D);
        uint32_t* prep = scratch<uint32_t>(ctx, np);
        uint64_t* ti = scratch<uint64_t>(ctx, np * k);
        double* td = scratch<double>(ctx, np * k);
        uint32_t* tc = scratch<uint32_t>(ctx, np);
        launch(ctx, "adc_scan", pairs_prep_kernel, dim3(unsigned(np)), dim3(128), 0, queries, D, probes, nq, nprobe,
               qrep, prep);
        ivf_scan(ctx, ix, qrep, np, prep, 1, k, has_max, max_sq, ti, td, tc, err, subset, nsub, nullptr);
        topk_merge_dev(ctx, ti, td, tc, uint32_t(nprobe), nq, k, out_ids, out_dists, out_counts);
        return;
    }
    if (k > 32) {  // beyond the warp top-k: exact scores + segmented sort (topk_large.cu)
        ivf_scan_large_k(ctx, ix, queries, nq, probes, nprobe, k, has_max, max_sq, out_ids, out_dists,
                         out_counts, err, subset, nsub, luts);
        return;
    }
    const size_t lut_bytes = (sizeof(float) * ix.M * ix.ks + 15) & ~size_t(15);
    const size_t smem = lut_bytes + sizeof(TopK) * k * (kScanThreads / 32) +
                        sizeof(double) * uint64_t(ix.M) * ix.ds +  // fp64 query
                        sizeof(TopK) * 32 * (kScanThreads / 32);   // survivor buffers
    if (smem > 220 * 1024) fail(PQG_EUNSUPPORTED, "search: M*ks lookup table exceeds shared memory");
    const uint32_t rb = ix.M * ix.w;
    // r2: the query LUTs of a batch are built by one batched kernel
    // (adc_luts_kernel) and loaded by the scan; PQG_ADC_LUT=0 builds them
    // inside the scan (r1)
    const char* le = std::getenv("PQG_ADC_LUT");
    const uint64_t qchunk = 16384;  // bounds the LUT scratch (16384 x 16 KB = 256 MB at M=16)
    float* lut_buf = nullptr;
    if (!luts && nq >= 64 && ix.ks <= 256 && !(le && le[0] == '0'))
        lut_buf = scratch<float>(ctx, std::min<uint64_t>(nq, qchunk) * ix.M * ix.ks);
    auto run = [&](auto kern) {
        set_smem(kern, smem);
        for (uint64_t q0 = 0; q0 < nq; q0 += (lut_buf ? qchunk : 65535)) {
            const uint64_t nc = std::min<uint64_t>(lut_buf ? qchunk : 65535, nq - q0);
            const float* lq = luts ? luts + q0 * uint64_t(ix.M) * ix.ks : nullptr;
            if (lut_buf && adc_luts_dev(ctx, ix.tables, ix.M, ix.ks, ix.ds, queries + q0 * ix.M * ix.ds, nc, lut_buf))
                lq = lut_buf;
            launch(ctx, "adc_scan", kern, dim3(unsigned(nc)), dim3(kScanThreads), smem, ix.tables,
                   ix.M, ix.ks, ix.ds, queries + q0 * ix.M * ix.ds, ix.offsets, ix.ids, ix.codes,
                   probes + q0 * nprobe, nprobe, int(k), has_max, max_sq, subset, nsub,
                   out_ids + q0 * k, out_dists + q0 * k, out_counts + q0, err, lq);
        }
    };
    // vector code loads need rb-aligned rows (CSR rows are rb apart from an aligned base)
    const bool aligned = (reinterpret_cast<uintptr_t>(ix.codes) % (rb >= 16 ? 16 : rb)) == 0;
    // PQG_ADC_PRUNE=0: the Ks = 256 scans without the partial-sum early exit
    const char* pe = std::getenv("PQG_ADC_PRUNE");
    const bool k256 = ix.ks == 256 && !(pe && pe[0] == '0');
    if (aligned && ix.w == 1 && rb == 16) k256 ? run(adc_scan_kernel<16, 1, 256>) : run(adc_scan_kernel<16, 1, 0>);
    else if (aligned && ix.w == 1 && rb == 8) k256 ? run(adc_scan_kernel<8, 1, 256>) : run(adc_scan_kernel<8, 1, 0>);
    else if (aligned && ix.w == 1 && rb == 32) k256 ? run(adc_scan_kernel<32, 1, 256>) : run(adc_scan_kernel<32, 1, 0>);
    else if (aligned && ix.w == 1 && rb == 4) run(adc_scan_kernel<4, 1, 0>);
    else if (aligned && ix.w == 2 && rb == 16) run(adc_scan_kernel<16, 2, 0>);
    else if (aligned && ix.w == 2 && rb == 8) run(adc_scan_kernel<8, 2, 0>);
    else run(adc_scan_kernel<0, 1, 0>);
}

void csr_scatter(pqg_ctx* ctx, const uint32_t* perm, uint64_t n, const uint64_t* ids,
                 const uint8_t* codes, uint64_t row_bytes, uint64_t* out_ids, uint8_t* out_codes) {
    launch(ctx, "csr_scatter", csr_scatter_kernel, dim3(grid1d(n, 256, ctx->num_sms * 16)), dim3(256),
           0, perm, n, ids, codes, row_bytes, out_ids, out_codes);
}

void find_duplicate(pqg_ctx* ctx, const uint64_t* ids, uint64_t n, uint64_t* first_dup_pos) {
    uint64_t cap = 1;
    while (cap < 2 * n) cap <<= 1;
    int* state = scratch<int>(ctx, cap);
    uint64_t* keys = scratch<uint64_t>(ctx, cap);
    unsigned long long* minpos = scratch<unsigned long long>(ctx, cap);
    PQG_CUDA(cudaMemsetAsync(state, 0, sizeof(int) * cap, ctx->stream));
    PQG_CUDA(cudaMemsetAsync(minpos, 0xff, sizeof(unsigned long long) * cap, ctx->stream));
    PQG_CUDA(cudaMemsetAsync(first_dup_pos, 0xff, sizeof(uint64_t), ctx->stream));
    const unsigned g = grid1d(n, 256, ctx->num_sms * 16);
    launch(ctx, "dup_check", dup_insert_kernel, dim3(g), dim3(256), 0, ids, n, cap - 1, state, keys,
           minpos);
    launch(ctx, "dup_check", dup_find_kernel, dim3(g), dim3(256), 0, ids, n, cap - 1,
           (const uint64_t*)keys, (const unsigned long long*)minpos,
           reinterpret_cast<unsigned long long*>(first_dup_pos));
}

void topk_merge_dev(pqg_ctx* ctx, const uint64_t* ids, const double* dists,
                    const uint32_t* counts, uint32_t shards, uint64_t nq, uint64_t k,
                    uint64_t* out_ids, double* out_dists, uint32_t* out_counts) {
    if (shards > 64) fail(PQG_EUNSUPPORTED, "topk_merge: at most 64 shards");
    launch(ctx, "topk_merge", topk_merge_kernel, dim3(grid1d(nq, 128, 65535)), dim3(128), 0, ids,
           dists, counts, shards, nq, k, out_ids, out_dists, out_counts);
}

}  // namespace pqg
