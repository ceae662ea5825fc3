// topk_large.cu -- ivf_query / ivf_query_subset / flat_scan for k > 32.
//
// The warp top-k of adc_scan_kernel (ivf.cu) keeps 32 entries per warp.  The
// reference takes any k >= 1 (finalize_hits, proj/src/ivf.cpp:58-68: the k
// smallest hits by (sq_dist, id), sorted; fewer when the probed lists hold
// fewer candidates -- "k beyond n_items saturates", proj/tests/test_ivf.cpp
// :255-259).  For k > 32 every candidate is scored exactly as adc_lookup
// (proj/src/pq.cpp:153-167: fp64 sum of the float entries in m order, from
// 0.0), filtered as scan_list / scan_list_subset (proj/src/ivf.cpp:70-88:
// subset membership first, then the max_sq_dist test), compacted per query,
// and each query's hits are ordered by (sq_dist, id) with two stable
// segmented radix sorts (by id, then by distance -- CUB, the CUDA toolkit's
// sort).  Hit ids are unique (the index rejects duplicates), so the order is
// total and the result is finalize_hits' exactly.  Queries are processed in
// chunks of at most kMaxPairs candidates.
#include <cub/device/device_segmented_sort.cuh>

#include "kernels.cuh"

namespace pqg {
namespace {

constexpr uint64_t kMaxPairs = uint64_t(1) << 25;  // candidates per chunk (32 B each, x2 buffers)
constexpr int kThreads = 256;

__global__ void cand_count_kernel(const uint64_t* offsets, const uint32_t* probes, uint64_t nq,
                                  uint64_t nprobe, uint64_t* cnt) {
    for (uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nq;
         q += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t s = 0;
        for (uint64_t p = 0; p < nprobe; ++p) {
            const uint32_t l = probes[q * nprobe + p];
            s += offsets[l + 1] - offsets[l];
        }
        cnt[q] = s;
    }
}

// grid (nprobe, queries of the chunk); LUT of the query in shared memory
// (SMEM) or read from global memory (tables too wide for shared memory).
template <bool SMEM>
__global__ void __launch_bounds__(kThreads) score_all_kernel(
    const float* luts, uint32_t M, uint32_t ks, uint32_t w, const uint64_t* offsets,
    const uint64_t* ids, const uint8_t* codes, const uint32_t* probes, uint64_t nprobe,
    int has_max, double max_sq, const uint64_t* subset, uint64_t nsub, const int* base,
    unsigned* fill, uint64_t* out_id, double* out_d, int* err) {
    extern __shared__ __align__(16) float slut[];
    const uint64_t qc = blockIdx.y;  // query within the chunk
    const float* glut = luts + qc * uint64_t(M) * ks;
    const float* lut = glut;
    if constexpr (SMEM) {
        for (uint32_t e = threadIdx.x; e < M * ks; e += blockDim.x) slut[e] = __ldg(glut + e);
        __syncthreads();
        lut = slut;
    }
    const uint32_t l = probes[qc * nprobe + blockIdx.x];
    const uint64_t a = offsets[l], b = offsets[l + 1];
    const uint64_t rb = uint64_t(M) * w;
    const int lane = threadIdx.x & 31;
    for (uint64_t i0 = a; i0 < b; i0 += blockDim.x) {
        const uint64_t i = i0 + threadIdx.x;
        bool keep = false;
        double acc = 0.0;
        uint64_t id = 0;
        if (i < b) {
            id = ids[i];
            keep = true;
            if (subset) {  // std::binary_search over the sorted subset
                uint64_t lo = 0, hi = nsub;
                keep = false;
                while (lo < hi) {
                    const uint64_t mid = (lo + hi) >> 1;
                    const uint64_t v = __ldg(subset + mid);
                    if (v == id) { keep = true; break; }
                    if (v < id) lo = mid + 1; else hi = mid;
                }
            }
            if (keep) {
                const uint8_t* row = codes + i * rb;
                for (uint32_t m = 0; m < M; ++m) {
                    const uint32_t code = w == 1 ? uint32_t(row[m])
                                                 : (uint32_t(row[2 * m]) | (uint32_t(row[2 * m + 1]) << 8));
                    if (code >= ks) {  // adc_lookup's out_of_range
                        atomicExch(err, 1);
                        keep = false;
                        break;
                    }
                    acc = __dadd_rn(acc, (double)lut[uint64_t(m) * ks + code]);
                }
                if (keep && has_max && acc > max_sq) keep = false;
            }
        }
        const unsigned mask = __ballot_sync(0xffffffffu, keep);
        if (!mask) continue;
        unsigned pos = 0;
        if (lane == 0) pos = atomicAdd(fill + qc, unsigned(__popc(mask)));
        pos = __shfl_sync(0xffffffffu, pos, 0);
        if (keep) {
            const uint64_t o = uint64_t(base[qc]) + pos + __popc(mask & ((1u << lane) - 1u));
            out_id[o] = id;
            out_d[o] = acc;
        }
    }
}

__global__ void seg_end_kernel(const int* base, const unsigned* fill, uint64_t nqc, int* end) {
    for (uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < nqc;
         q += uint64_t(gridDim.x) * blockDim.x)
        end[q] = base[q] + int(fill[q]);
}

// row q of the outputs: the first min(k, hits) sorted hits, the rest zeroed
__global__ void take_k_kernel(const int* base, const unsigned* fill, const uint64_t* sid,
                              const double* sd, uint64_t k, uint64_t* out_ids, double* out_dists,
                              uint32_t* out_counts) {
    const uint64_t q = blockIdx.x;
    const uint64_t c = min(uint64_t(fill[q]), k);
    for (uint64_t j = threadIdx.x; j < k; j += blockDim.x) {
        const bool v = j < c;
        out_ids[q * k + j] = v ? sid[base[q] + j] : 0;
        out_dists[q * k + j] = v ? sd[base[q] + j] : 0.0;
    }
    if (threadIdx.x == 0) out_counts[q] = uint32_t(c);
}

}  // namespace

void ivf_scan_large_k(pqg_ctx* ctx, const IndexView& ix, const float* queries, uint64_t nq,
                      const uint32_t* probes, uint64_t nprobe, uint64_t k, int has_max,
                      double max_sq, uint64_t* out_ids, double* out_dists, uint32_t* out_counts,
                      int* err, const uint64_t* subset, uint64_t nsub, const float* luts) {
    if (nq == 0) return;
    uint64_t* cnt = scratch<uint64_t>(ctx, nq);
    launch(ctx, "topk_large", cand_count_kernel, dim3(grid1d(nq, 256, 4096)), dim3(256), 0,
           ix.offsets, probes, nq, nprobe, cnt);
    std::vector<uint64_t> h(nq);
    PQG_CUDA(cudaMemcpyAsync(h.data(), cnt, sizeof(uint64_t) * nq, cudaMemcpyDeviceToHost, ctx->stream));
    PQG_CUDA(cudaStreamSynchronize(ctx->stream));
    const uint64_t lut_n = uint64_t(ix.M) * ix.ks;
    const size_t lut_smem = sizeof(float) * lut_n;
    const bool smem = lut_smem <= 200 * 1024;
    if (smem) set_smem(score_all_kernel<true>, lut_smem);
    const auto mark = ctx->arena.mark();
    for (uint64_t q0 = 0; q0 < nq;) {
        // the chunk: as many queries as fit kMaxPairs candidates (at least one)
        uint64_t q1 = q0, tot = 0;
        std::vector<int> hb;
        while (q1 < nq && (q1 == q0 || tot + h[q1] <= kMaxPairs) && q1 - q0 < 65535) {
            hb.push_back(int(tot));
            tot += h[q1];
            ++q1;
        }
        if (tot > uint64_t(INT32_MAX)) fail(PQG_EUNSUPPORTED, "search: too many candidates for one query");
        const uint64_t nqc = q1 - q0;
        ctx->arena.reset_to(mark);
        const float* lq;
        if (luts) {
            lq = luts + q0 * lut_n;
        } else {
            float* e = scratch<float>(ctx, nqc * lut_n);
            adc_tables_dev(ctx, ix.tables, ix.M, ix.ks, ix.ds, queries + q0 * uint64_t(ix.M) * ix.ds,
                           nqc, e);
            lq = e;
        }
        int* base = scratch<int>(ctx, nqc);
        int* end = scratch<int>(ctx, nqc);
        unsigned* fill = scratch<unsigned>(ctx, nqc);
        PQG_CUDA(cudaMemcpyAsync(base, hb.data(), sizeof(int) * nqc, cudaMemcpyHostToDevice, ctx->stream));
        PQG_CUDA(cudaMemsetAsync(fill, 0, sizeof(unsigned) * nqc, ctx->stream));
        const uint64_t T = std::max<uint64_t>(tot, 1);
        uint64_t* id0 = scratch<uint64_t>(ctx, T);
        uint64_t* id1 = scratch<uint64_t>(ctx, T);
        double* d0 = scratch<double>(ctx, T);
        double* d1 = scratch<double>(ctx, T);
        if (nprobe > 65535) fail(PQG_EUNSUPPORTED, "search: nprobe > 65535 with k > 32");
        const dim3 grid{unsigned(nprobe), unsigned(nqc), 1u};
        if (smem)
            launch(ctx, "topk_large", score_all_kernel<true>, grid, dim3(kThreads), lut_smem, lq, ix.M,
                   ix.ks, ix.w, ix.offsets, ix.ids, ix.codes, probes + q0 * nprobe, nprobe, has_max,
                   max_sq, subset, nsub, (const int*)base, fill, id0, d0, err);
        else
            launch(ctx, "topk_large", score_all_kernel<false>, grid, dim3(kThreads), 0, lq, ix.M,
                   ix.ks, ix.w, ix.offsets, ix.ids, ix.codes, probes + q0 * nprobe, nprobe, has_max,
                   max_sq, subset, nsub, (const int*)base, fill, id0, d0, err);
        launch(ctx, "topk_large", seg_end_kernel, dim3(grid1d(nqc, 256, 1024)), dim3(256), 0,
               (const int*)base, (const unsigned*)fill, nqc, end);
        // (dist, id) order: stable sort by id, then stable sort by distance
        size_t b1 = 0, b2 = 0;
        PQG_CUDA(cub::DeviceSegmentedSort::StableSortPairs(nullptr, b1, id0, id1, d0, d1, int(T),
                                                           int(nqc), base, end, ctx->stream));
        PQG_CUDA(cub::DeviceSegmentedSort::StableSortPairs(nullptr, b2, d1, d0, id1, id0, int(T),
                                                           int(nqc), base, end, ctx->stream));
        void* tmp = scratch<uint8_t>(ctx, std::max<size_t>(std::max(b1, b2), 16));
        PQG_CUDA(cub::DeviceSegmentedSort::StableSortPairs(tmp, b1, id0, id1, d0, d1, int(T), int(nqc),
                                                           base, end, ctx->stream));
        PQG_CUDA(cub::DeviceSegmentedSort::StableSortPairs(tmp, b2, d1, d0, id1, id0, int(T), int(nqc),
                                                           base, end, ctx->stream));
        ctx->launches += 2;
        launch(ctx, "topk_large", take_k_kernel, dim3(unsigned(nqc)), dim3(256), 0, (const int*)base,
               (const unsigned*)fill, (const uint64_t*)id0, (const double*)d0, k, out_ids + q0 * k,
               out_dists + q0 * k, out_counts + q0);
        q0 = q1;
    }
    ctx->arena.reset_to(mark);
}

}  // namespace pqg
