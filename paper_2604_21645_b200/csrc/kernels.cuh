// kernels.cuh -- host-side launchers of the libpqg kernels.
#pragma once

#include "common.cuh"

namespace pqg {

// Where the rows of a nearest-centroid problem come from.
//  dense  : x[i * ldx + b * col_stride + t]               (b = problem index)
//  decoded: x[i][t] = tables[m][code(i, m)][t - m*ds]     (pq_decode_row)
struct RowSrc {
    const float* x = nullptr;
    uint64_t ldx = 0;
    uint32_t col_stride = 0;
    const uint8_t* codes = nullptr;  // decoded mode when non-null
    const float* dtab = nullptr;
    uint32_t dM = 0, dks = 0, dds = 0, dw = 1;
};

// B independent argmin problems over the same n rows; problem b has a k x d
// centroid table at table + b*k*d.  Output index of (row i, problem b) goes
// to out_idx[(i*idx_rs + b*idx_ps)] with idx_bytes in {1,2,4}; optional
// fp64 distance to dist[b*n + i].  Rows whose fp32 screen cannot prove the
// fp64 winner are appended to flags and resolved by the fixup kernel.
struct NearestArgs {
    RowSrc src;
    uint64_t n = 0;
    uint32_t d = 0;
    uint32_t B = 1;
    const float* table = nullptr;
    uint64_t k = 0;
    const float* cnorm = nullptr;  // [B][k]
    const float* cmax = nullptr;   // [B]
    void* out_idx = nullptr;
    int idx_bytes = 4;
    uint64_t idx_rs = 1, idx_ps = 0;
    double* out_dist = nullptr;
    // sse mode: accumulate exact (x - c_win)^2 per row into sse_row[i] (fp64)
    double* sse_part = nullptr;
    unsigned long long* flag_count = nullptr;
    uint64_t* flags = nullptr;
    const int* active = nullptr;
    // distance-matrix mode: write screened fp32 distances (plus row margin)
    float* out_mat = nullptr;
    uint64_t ld_mat = 0;
    float* row_err = nullptr;  // [n] screen error bound per row (matrix mode)
    // umma_big: row operand already split (k-means reuses it every iteration)
    const uint8_t* big_rows = nullptr;
    const float* big_nx = nullptr;
};

// nearest.cu
void table_norms(pqg_ctx* ctx, const float* table, uint32_t B, uint64_t k, uint32_t d,
                 float* cnorm, float* cmax);
void nearest(pqg_ctx* ctx, NearestArgs a);           // screen + exact fixup
void distance_matrix(pqg_ctx* ctx, NearestArgs a);   // fp32 screen values only

// umma.cu (tcgen05 3xTF32 screen for PQ subspaces)
bool umma_screen_supported(const NearestArgs& a);
void umma_screen(pqg_ctx* ctx, const NearestArgs& a);
// umma_big.cu (tcgen05 GEMM-argmin / screen matrix for the coarse quantizer)
bool umma_big_supported(const NearestArgs& a);
void umma_big(pqg_ctx* ctx, const NearestArgs& a);
// Split the row operand once (C_r = ||x_r||^2, no margin) for repeated argmin
// calls over the same rows; returns false if the big kernel does not apply.
bool umma_big_prepare_rows(pqg_ctx* ctx, NearestArgs& a);

// kmeans.cu
struct Bucketing {
    uint64_t* offsets;  // [B][k+1]
    uint32_t* perm;     // [B][n] rows in key order, stable
};
void stable_bucket(pqg_ctx* ctx, const uint32_t* keys, uint64_t n, uint32_t B, uint64_t k,
                   const int* active, Bucketing out, const uint64_t* nb = nullptr);
void exclusive_scan_u32(pqg_ctx* ctx, const uint32_t* in, uint64_t* out, uint64_t count);
void transpose_blocks(pqg_ctx* ctx, const float* x, uint64_t n, uint64_t ldx, uint32_t B, uint32_t d,
                      uint32_t col_stride, float* out);
void gather_rows(pqg_ctx* ctx, const float* x, uint64_t ldx, uint32_t B, uint32_t d,
                 uint32_t col_stride, const uint64_t* rows, uint64_t k, float* table);
struct KMeansState {
    int* active;          // [B]
    double* prev;         // [B]
    double* inertia;      // [B]
    double* per_iter;     // [B][max_iters]
    uint32_t* iters;      // [B]
    // [B] zeroed once per fit (r2e): with it the inertia's last partial block
    // runs the stop rule (one launch per pass instead of two); null: stop_kernel
    unsigned* tickets = nullptr;
};
void rows_sum_f64(pqg_ctx* ctx, const double* v, uint64_t n, uint32_t B, double* out);
void kmeans_inertia_and_stop(pqg_ctx* ctx, const double* dist, uint64_t n, uint32_t B,
                             uint32_t it, uint32_t max_iters, double tol, KMeansState st,
                             const uint64_t* nb = nullptr);
// table_norms for small (PQ) tables: a block per problem (kmeans.cu)
void table_norms_small(pqg_ctx* ctx, const float* table, uint32_t B, uint64_t k, uint32_t d, float* cnorm,
                       float* cmax);
void kmeans_update(pqg_ctx* ctx, const RowSrc& src, uint64_t n, uint32_t B, uint32_t d,
                   float* table, uint64_t k, const uint32_t* assign, double* dist,
                   const int* active, const uint64_t* nb = nullptr, float* cnorm = nullptr,
                   float* cmax = nullptr);
// Row-sharded fits (kmshard.cu): one rank's bucketing + exact piece sums with
// exponent ranges, and the stop rule on an already reduced inertia.
bool kmeans_partials_supported(const RowSrc& src, uint32_t d);
void kmeans_local_partials(pqg_ctx* ctx, const RowSrc& src, uint64_t n, uint32_t B, uint32_t d,
                           uint64_t k, const uint32_t* assign, const int* active, uint64_t* offsets,
                           uint32_t* perm, double* csum, int* cmax, int* cmin);
void kmeans_stop_global(pqg_ctx* ctx, const double* inertia, uint32_t B, uint32_t max_iters, double tol,
                        KMeansState st);
// kmshard.cu: the exchange-side kernels of pqg_kmshard_*
void shard_init_gather(pqg_ctx* ctx, const RowSrc& src, uint64_t n, uint32_t B, uint32_t d, uint64_t k,
                       const uint64_t* rows, uint64_t row0, uint32_t* bits);
void shard_pack_partials(pqg_ctx* ctx, uint32_t B, uint64_t k, uint32_t d, const uint64_t* offsets,
                         const double* csum, const int* cmax, const int* cmin, double* f64, uint8_t* u8);
void shard_finalize(pqg_ctx* ctx, uint32_t B, uint64_t k, uint32_t d, const double* f64, const uint8_t* u8,
                    const int* active, float* table, uint32_t* flags, uint32_t* empties);
// ordered replay list (work), per-column local counts (cnt) and their
// exclusive scan (pre); res[0] = n_fail, res[1] = local pack length,
// res[2] = sum of the columns' global counts (a bound on every rank's pack)
void shard_replay_layout(pqg_ctx* ctx, uint32_t B, uint64_t k, uint32_t d, const uint32_t* flags,
                         const uint64_t* offsets, const double* f64, uint32_t* work, uint32_t* cnt, uint64_t* pre,
                         unsigned long long* res);
void shard_pack(pqg_ctx* ctx, const RowSrc& src, const uint32_t* work, uint64_t n_fail, uint64_t k,
                uint32_t d, const uint64_t* offsets, const uint32_t* perm, uint64_t n, const uint32_t* cnt,
                const uint64_t* pre, uint64_t* offcnt, float* vals);
void shard_replay_step(pqg_ctx* ctx, const RowSrc& src, const uint32_t* work, uint64_t n_fail, uint64_t k,
                       uint32_t d, const uint64_t* offsets, const uint32_t* perm, uint64_t n, double* run);
void shard_replay_finish(pqg_ctx* ctx, const uint32_t* work, uint64_t n_fail, uint64_t k, uint32_t d, uint32_t B,
                         const double* f64, const double* run, float* table);
void shard_replay(pqg_ctx* ctx, const uint32_t* work, uint64_t n_fail, uint64_t k, uint32_t d, uint32_t B,
                  const double* f64, const float* vals, uint64_t stride, const uint64_t* offcnt,
                  uint32_t world, float* table);
void shard_reseed_candidates(pqg_ctx* ctx, const RowSrc& src, uint64_t n, uint32_t B, uint32_t d,
                             const double* dist, const int* active, const uint32_t* empties, uint32_t E,
                             uint64_t row0, double* cand_d, uint64_t* cand_i, float* cand_rows);
void shard_reseed_apply(pqg_ctx* ctx, uint32_t B, uint64_t k, uint32_t d, const double* f64,
                        const int* active, uint32_t E, uint32_t world, const double* cand_d,
                        const uint64_t* cand_i, const float* cand_rows, float* table);
// Batched problems of unequal length (nb[b] <= n rows, the rest padding):
// padding rows get key k so the update ignores them.
void kmeans_pad_keys(pqg_ctx* ctx, uint32_t* keys, uint64_t n, uint32_t B, uint64_t k,
                     const uint64_t* nb, uint64_t max_pad);

// pq.cu
void pq_decode_dev(pqg_ctx* ctx, const uint8_t* codes, uint64_t n, uint32_t M, uint32_t ks,
                   uint32_t ds, const float* tables, float* out, int* err);
void sq_error_dev(pqg_ctx* ctx, const float* a, const float* b, uint64_t count, double* sse);
void recon_sse_dev(pqg_ctx* ctx, const float* x, const uint8_t* codes, uint64_t n, uint32_t M,
                   uint32_t ks, uint32_t ds, const float* tables, double* sse, int* err);
// batched search LUTs (one per query, [nq][M][ks]); false if the shape is not covered
bool adc_luts_dev(pqg_ctx* ctx, const float* tables, uint32_t M, uint32_t ks, uint32_t ds,
                  const float* queries, uint64_t nq, float* entries);
void adc_tables_dev(pqg_ctx* ctx, const float* tables, uint32_t M, uint32_t ks, uint32_t ds,
                    const float* queries, uint64_t nq, float* entries);
void adc_lookup_dev(pqg_ctx* ctx, const float* entries, uint32_t M, uint32_t ks,
                    const uint8_t* codes, uint64_t n, double* out, int* err);
void reduce_sum_f64(pqg_ctx* ctx, const double* parts, uint64_t count, double* out);
// the chunked pipeline (proj/src/pipeline.cpp): chunks side by side, decoded
// local codewords, per-chunk reconstruction SSE from the fits' assignments
void interleave_chunks(pqg_ctx* ctx, const float* x, uint64_t D, uint64_t C, uint64_t base,
                       uint64_t extra, uint64_t n_max, float* y);
void chunk_representatives(pqg_ctx* ctx, const float* tables, uint64_t C, uint32_t M, uint32_t ks,
                           uint32_t ds, float* reps);
void chunk_sse(pqg_ctx* ctx, const float* x, uint64_t C, uint32_t M, uint32_t ks, uint32_t ds,
               uint64_t base, uint64_t extra, const uint32_t* assign, uint64_t n_max,
               const float* tables, double* sse);

// ivf.cu
struct IndexView {
    const float* tables;
    uint32_t M, ks, ds, w;
    const float* coarse;
    const float* coarse_norm;
    const float* coarse_max;
    uint64_t nlist;
    const uint64_t* offsets;
    const uint64_t* ids;
    const uint8_t* codes;
    uint64_t n;
};
void ivf_probe(pqg_ctx* ctx, const IndexView& ix, const float* queries, uint64_t nq,
               uint64_t nprobe, uint32_t* probes);
void ivf_scan(pqg_ctx* ctx, const IndexView& ix, const float* queries, uint64_t nq,
              const uint32_t* probes, uint64_t nprobe, uint64_t k, int has_max, double max_sq,
              uint64_t* out_ids, double* out_dists, uint32_t* out_counts, int* err,
              const uint64_t* subset = nullptr, uint64_t nsub = 0, const float* luts = nullptr);
// topk_large.cu: the same search for k > 32 (exact scores of every candidate,
// compacted per query, ordered by (dist, id) with segmented sorts)
void ivf_scan_large_k(pqg_ctx* ctx, const IndexView& ix, const float* queries, uint64_t nq,
                      const uint32_t* probes, uint64_t nprobe, uint64_t k, int has_max,
                      double max_sq, uint64_t* out_ids, double* out_dists, uint32_t* out_counts,
                      int* err, const uint64_t* subset, uint64_t nsub, const float* luts);
void csr_scatter(pqg_ctx* ctx, const uint32_t* perm, uint64_t n, const uint64_t* ids,
                 const uint8_t* codes, uint64_t row_bytes, uint64_t* out_ids, uint8_t* out_codes);
void find_duplicate(pqg_ctx* ctx, const uint64_t* ids, uint64_t n, uint64_t* first_dup_pos);
void topk_merge_dev(pqg_ctx* ctx, const uint64_t* ids, const double* dists,
                    const uint32_t* counts, uint32_t shards, uint64_t nq, uint64_t k,
                    uint64_t* out_ids, double* out_dists, uint32_t* out_counts);
// formats.cu: PQII list section <-> device CSR, load-time validation scans
void pqii_pack(pqg_ctx* ctx, const uint64_t* off, const uint64_t* ids, const uint8_t* codes, uint64_t nlist,
               uint64_t n, uint64_t rb, uint8_t* out);
void pqii_unpack(pqg_ctx* ctx, const uint8_t* sec, const uint64_t* src_off, const uint64_t* off, uint64_t nl,
                 uint64_t n, uint64_t rb, uint64_t* ids, uint8_t* codes);
void first_bad_code(pqg_ctx* ctx, const uint8_t* codes, uint64_t n, uint32_t M, uint32_t ks, uint32_t w,
                    unsigned long long* first);
void first_nonfinite(pqg_ctx* ctx, const float* v, uint64_t count, unsigned long long* first);

}  // namespace pqg
