/*
 * pqg.h -- C ABI of the B200-native PQ / IVF hot path (libpqg.so).
 *
 * Plain pointers and sizes only.  Every data pointer may be HOST memory or
 * DEVICE memory of the context's GPU; the library detects which
 * (cudaPointerGetAttributes) and stages host buffers through its own device
 * scratch, so the same entry points serve the reference-facing host API and
 * device-resident pipelines.  All entry points return PQG_OK (0) or a
 * negative status; pqg_last_error() returns the thread's last message.
 * Status mapping to the reference's exceptions:
 *   PQG_EINVAL -> std::invalid_argument   PQG_ERANGE -> std::out_of_range
 *   PQG_ECUDA / PQG_ENOMEM / PQG_EUNSUPPORTED / PQG_ECHUNK / PQG_EIO -> std::runtime_error
 * Message substrings follow the reference ("not divisible", "exceeds",
 * "no items", "duplicate id", "nprobe", ...).
 *
 * Each function cites the reference function it replaces
 * (/root/reference/proj/<path>:<line>).  Code matrices are the reference's
 * packed layout (proj/include/pqii/pq.hpp:33-55): n rows of M codes, one byte
 * each when ks <= 256, else two bytes little-endian.  Codebooks are
 * [M][ks][ds] fp32 (pq.hpp:15-31).  Posting lists are CSR: offsets[nlist+1]
 * (u64), ids[n] (u64), codes[n][row_bytes] -- list l holds entries
 * offsets[l]..offsets[l+1]-1 in insertion order (ivf.cpp:44-46).
 */
#ifndef PQG_H
#define PQG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PQG_OK 0
#define PQG_EINVAL (-1)
#define PQG_ERANGE (-2)
#define PQG_ECUDA (-3)
#define PQG_ENOMEM (-4)
#define PQG_EUNSUPPORTED (-5)
#define PQG_ECHUNK (-6) /* a pipeline chunk task failed: std::runtime_error("chunk <id>: ...") */
#define PQG_EIO (-7)    /* file / format error: std::runtime_error with the reference's message */

typedef struct pqg_ctx pqg_ctx;     /* one GPU + stream + scratch arena */
typedef struct pqg_index pqg_index; /* device-resident inverted index */

/* ---- context ----------------------------------------------------------- */
int pqg_ctx_create(int device, pqg_ctx** out);
void pqg_ctx_destroy(pqg_ctx* ctx);
/* Run on a caller-owned cudaStream_t (NULL restores the context's own;
 * (void*)1 is cudaStreamLegacy, the default stream of other libraries). */
int pqg_ctx_set_stream(pqg_ctx* ctx, void* cuda_stream);
/* (Switching streams makes the new stream wait for the work already queued
 * on the old one, whose scratch the context reuses.) */
/* The cudaStream_t the context currently launches on. */
void* pqg_ctx_stream(pqg_ctx* ctx);
/* Synchronise the context stream; also reports (PQG_ERANGE) an out-of-range
 * code found by a search whose outputs all stayed on the device. */
int pqg_ctx_sync(pqg_ctx* ctx);
/* Report (PQG_ERANGE, then clear) a pending out-of-range code flagged by a
 * device-output search (adc_lookup's std::out_of_range, pq.cpp:160-163). */
int pqg_ctx_check_errors(pqg_ctx* ctx);
const char* pqg_last_error(void);
/* Number of kernels this context has launched (bench.py's gpu_launches). */
uint64_t pqg_ctx_launches(pqg_ctx* ctx);
/* Per-kernel-class CUDA-event timing on the context stream.  enable=1 starts
 * recording every launch; pqg_profile_read returns (launch count, summed ms)
 * for a class name such as "nearest", "fixup", "kmeans_sum", "adc_scan". */
int pqg_profile_enable(pqg_ctx* ctx, int enable);
int pqg_profile_read(pqg_ctx* ctx, const char* kernel_class, uint64_t* launches,
                     double* total_ms);
const char* pqg_version(void);
/* Measured FP32 FFMA throughput of this GPU (TFLOP/s): the denominator of the
 * fp32-bound kernels' roofline fraction. */
int pqg_fp32_probe(pqg_ctx* ctx, double* tflops);

/* ---- L1: nearest centroid / k-means (proj/src/kmeans.cpp) ---------------- */
/* nearest_in_table (kmeans.cpp:20-31) for n points: index[i], sq_dist[i] are
 * exactly the reference's (fp64 squared_l2, ties to the lowest index). */
int pqg_nearest_batch(pqg_ctx* ctx, const float* points, uint64_t n, uint64_t d,
                      const float* table, uint64_t k, uint32_t* index, double* sq_dist);

/* kmeans_fit (kmeans.cpp:61-133).  centroids k*d, assignments n (nullable),
 * inertia_per_iter max_iters entries (nullable, first *iterations_run valid). */
int pqg_kmeans_fit(pqg_ctx* ctx, const float* points, uint64_t n, uint64_t d, uint64_t k,
                   uint32_t max_iters, uint64_t seed, double tol, float* centroids,
                   uint32_t* assignments, double* inertia, uint32_t* iterations_run,
                   double* inertia_per_iter);

/* ---- L1: product quantization (proj/src/pq.cpp) -------------------------- */
/* pq_fit (pq.cpp:63-93): all M subspace fits batched in one device loop; each
 * keeps the reference's seed+m init and its own tol stop.  tables M*ks*(D/M);
 * iterations_run / inertia per subspace (nullable). */
int pqg_pq_fit(pqg_ctx* ctx, const float* data, uint64_t n, uint64_t D, uint32_t M,
               uint32_t ks, uint32_t max_iters, uint64_t seed, float* tables,
               uint32_t* iterations_run, double* inertia);
/* pq_fit plus each subspace's inertia_per_iter (kmeans.hpp:19): M*max_iters
 * fp64, row m valid for its first iterations_run[m] entries (the rest 0). */
int pqg_pq_fit_ex(pqg_ctx* ctx, const float* data, uint64_t n, uint64_t D, uint32_t M,
                  uint32_t ks, uint32_t max_iters, uint64_t seed, float* tables,
                  uint32_t* iterations_run, double* inertia, double* inertia_per_iter);
/* pq_encode (pq.cpp:95-111): codes n*M*width. */
int pqg_pq_encode(pqg_ctx* ctx, const float* data, uint64_t n, uint32_t M, uint32_t ks,
                  uint32_t ds, const float* tables, uint8_t* codes);
/* pq_decode (pq.cpp:113-130); PQG_ERANGE if a code >= ks. */
int pqg_pq_decode(pqg_ctx* ctx, const uint8_t* codes, uint64_t n, uint32_t M, uint32_t ks,
                  uint32_t ds, const float* tables, float* out);
/* rmse (pq.cpp:169-177) numerator: sum over count elements of (a-b)^2 in fp64. */
int pqg_sq_error(pqg_ctx* ctx, const float* a, const float* b, uint64_t count, double* sse);
/* reconstruction_rmse (pq.cpp:179-181) without materialising the decode:
 * sse = sum (x - decode(codes))^2; rmse = sqrt(sse / (n*M*ds)). */
int pqg_pq_recon_sse(pqg_ctx* ctx, const float* data, const uint8_t* codes, uint64_t n,
                     uint32_t M, uint32_t ks, uint32_t ds, const float* tables, double* sse);
/* Fused encode + reconstruction error: codes as pqg_pq_encode, sse as
 * pqg_pq_recon_sse (sse nullable). */
int pqg_pq_encode_sse(pqg_ctx* ctx, const float* data, uint64_t n, uint32_t M, uint32_t ks,
                      uint32_t ds, const float* tables, uint8_t* codes, double* sse);
/* adc_table (pq.cpp:132-151) for nq queries: entries nq*M*ks, each
 * float(fp64 squared_l2). */
int pqg_adc_tables(pqg_ctx* ctx, const float* tables, uint32_t M, uint32_t ks, uint32_t ds,
                   const float* queries, uint64_t nq, float* entries);
/* adc_lookup (pq.cpp:153-167) for n code rows against one table. */
int pqg_adc_lookup(pqg_ctx* ctx, const float* entries, uint32_t M, uint32_t ks,
                   const uint8_t* codes, uint64_t n, double* out);

/* ---- L2: inverted index (proj/src/ivf.cpp) ------------------------------- */
/* assign_items' list choice (ivf.cpp:36-49): list_of[i] = nearest coarse
 * centroid to the DECODED code row i. */
int pqg_ivf_assign(pqg_ctx* ctx, const uint8_t* codes, uint64_t n, uint32_t M, uint32_t ks,
                   uint32_t ds, const float* tables, const float* coarse, uint64_t nlist,
                   uint32_t* list_of);
/* ivf_build_with_centroids (ivf.cpp:151-166) into a device-resident index.
 * Validates as the reference (no items, coarse shape, duplicate ids). */
int pqg_ivf_build_with_centroids(pqg_ctx* ctx, const float* tables, uint32_t M, uint32_t ks,
                                 uint32_t ds, const uint8_t* codes, const uint64_t* ids,
                                 uint64_t n, const float* coarse, uint64_t nlist,
                                 pqg_index** out);
/* ivf_build (ivf.cpp:123-149): coarse kmeans_fit(decoded, nlist, iters, seed)
 * then lists from its final assignments. */
int pqg_ivf_build(pqg_ctx* ctx, const float* tables, uint32_t M, uint32_t ks, uint32_t ds,
                  const uint8_t* codes, const uint64_t* ids, uint64_t n, uint64_t nlist,
                  uint64_t seed, uint32_t kmeans_iters, pqg_index** out);
/* Wrap an existing CSR index (copied to the device). */
int pqg_index_create(pqg_ctx* ctx, const float* tables, uint32_t M, uint32_t ks, uint32_t ds,
                     const float* coarse, uint64_t nlist, const uint64_t* offsets,
                     const uint64_t* ids, const uint8_t* codes, pqg_index** out);
void pqg_index_destroy(pqg_index* index);
int pqg_index_info(const pqg_index* index, uint64_t* nlist, uint64_t* n_items, uint32_t* M,
                   uint32_t* ks, uint32_t* ds);
/* Copy the CSR out (any of the pointers may be NULL to skip). */
int pqg_index_export(pqg_ctx* ctx, const pqg_index* index, uint64_t* offsets, uint64_t* ids,
                     uint8_t* codes, float* coarse, float* tables);
/* ivf_add (ivf.cpp:168-184): assign and append in order; id collisions and
 * duplicates are rejected before the index changes. */
int pqg_index_add(pqg_ctx* ctx, pqg_index* index, const uint8_t* codes, const uint64_t* ids,
                  uint64_t n);
/* ivf_merge (ivf.cpp:186-216): list l = a's list l then b's. */
int pqg_index_merge(pqg_ctx* ctx, const pqg_index* a, const pqg_index* b, pqg_index** out);
/* Batched ivf_query (ivf.cpp:218-228) -- one call for nq queries.  Row q of
 * out_ids / out_dists (nq*k) holds out_counts[q] <= k hits sorted by
 * (sq_dist, id); has_max enables the max_sq_dist filter (ivf.cpp:70-77). */
int pqg_index_search(pqg_ctx* ctx, const pqg_index* index, const float* queries, uint64_t nq,
                     uint64_t k, uint64_t nprobe, int has_max, double max_sq_dist,
                     uint64_t* out_ids, double* out_dists, uint32_t* out_counts);
/* pqg_index_search that also returns each query's probe lists (out_probes:
 * nq*nprobe u32, host or device; nullable) -- the drop-in uses them to check
 * only the lists a query read against the caller's host index (r2e). */
int pqg_index_search_ex(pqg_ctx* ctx, const pqg_index* index, const float* queries, uint64_t nq,
                        uint64_t k, uint64_t nprobe, int has_max, double max_sq_dist,
                        uint64_t* out_ids, double* out_dists, uint32_t* out_counts, uint32_t* out_probes);
/* ivf_query_subset (ivf.cpp:230-245) for nq queries sharing one subset of
 * ids (sorted ascending, unique; PQG_EINVAL "not sorted" otherwise): hits are
 * restricted to the subset before the top-k. */
int pqg_index_search_subset(pqg_ctx* ctx, const pqg_index* index, const float* queries,
                            uint64_t nq, uint64_t k, const uint64_t* subset, uint64_t nsub,
                            uint64_t nprobe, int has_max, double max_sq_dist, uint64_t* out_ids,
                            double* out_dists, uint32_t* out_counts);
/* probe_order (ivf.cpp:91-101) for nq queries: probes nq*nprobe (u32). */
int pqg_index_probe(pqg_ctx* ctx, const pqg_index* index, const float* queries, uint64_t nq,
                    uint64_t nprobe, uint32_t* probes);
/* flat_scan (ivf.cpp:247-262) for nq queries over n codes. */
int pqg_flat_scan(pqg_ctx* ctx, const float* tables, uint32_t M, uint32_t ks, uint32_t ds,
                  const uint8_t* codes, const uint64_t* ids, uint64_t n, const float* queries,
                  uint64_t nq, uint64_t k, int has_max, double max_sq_dist, uint64_t* out_ids,
                  double* out_dists, uint32_t* out_counts);
/* Merge per-shard top-k lists (S shards x nq x k, counts S x nq) into the
 * global top-k by (dist, id) -- the multi-GPU search combine. */
int pqg_topk_merge(pqg_ctx* ctx, const uint64_t* ids, const double* dists,
                   const uint32_t* counts, uint32_t shards, uint64_t nq, uint64_t k,
                   uint64_t* out_ids, double* out_dists, uint32_t* out_counts);

/* ---- L3: the paper's chunked pipeline (proj/src/pipeline.cpp) ----------- */
#define PQG_MODE_SINGLE 0            /* PipelineMode::kSingle */
#define PQG_MODE_PARALLEL_PQ 1       /* PipelineMode::kParallelPq */
#define PQG_MODE_PARALLEL_PQ_INDEX 2 /* PipelineMode::kParallelPqIndex */
/* phase_seconds[] slots (the reference's phase_seconds keys); -1 = not run */
#define PQG_PHASE_FIT 0
#define PQG_PHASE_CHUNKING 1
#define PQG_PHASE_LOCAL_FIT 2
#define PQG_PHASE_GLOBAL_FIT 3
#define PQG_PHASE_COARSE_FIT 4
#define PQG_PHASE_ENCODE 5
#define PQG_PHASE_INDEX_BUILD 6
#define PQG_PHASE_MERGE 7
#define PQG_PHASE_COUNT 8
/* train_chunk (pipeline.cpp:84-106) for all chunk_rows(n, n_chunks) chunks
 * in one batched k-means (n_chunks*M problems; chunk c seeds seed+c).
 * representatives (n_chunks*ks) x D (the decoded local codewords, in chunk
 * order = aggregate_representatives, :108-135), local_rmse n_chunks,
 * iterations_run n_chunks*M -- all nullable.  Errors as run_chunk_tasks
 * (pipeline.cpp:30-62): PQG_ECHUNK "chunk <id>: ..." for the lowest failing
 * chunk. */
int pqg_train_chunks(pqg_ctx* ctx, const float* data, uint64_t n, uint64_t D, uint64_t n_chunks,
                     uint32_t M, uint32_t ks, uint32_t max_iters, uint64_t seed,
                     float* representatives, double* local_rmse, uint32_t* iterations_run);
/* run_pipeline (pipeline.cpp:142-266) with the data resident on the device
 * between phases.  nlist 0 = default_nlist(n) (capped at n_chunks*ks in
 * PARALLEL_PQ_INDEX mode); nlist_used receives the resolved value.
 * global_tables M*ks*(D/M); representatives (n_chunks*ks) x D and
 * local_rmse[n_chunks] (parallel modes, nullable); merged_index (index mode,
 * nullable; the caller destroys it); phase_seconds[PQG_PHASE_COUNT]
 * (nullable).  The thread count of the reference is not a parameter: the
 * result never depended on it (pipeline.hpp:74-78). */
int pqg_pipeline_run(pqg_ctx* ctx, const float* data, uint64_t n, uint64_t D, uint64_t n_chunks,
                     uint32_t M, uint32_t ks, uint64_t nlist, uint32_t max_iters, uint64_t seed,
                     int mode, float* global_tables, double* global_rmse, float* representatives,
                     double* local_rmse, uint64_t* nlist_used, pqg_index** merged_index,
                     double* phase_seconds);

/* ---- sharded k-means steps (multi-GPU driver) ------------ */
/* One assignment pass of a batch of B k-means problems over a row shard:
 * problem b reads columns [b*col_stride, b*col_stride+d) of rows (n x ld).
 * assign[b*n+i] (u32) and dist[b*n+i] (fp64) are the reference's
 * nearest_in_table results. */
int pqg_assign_pass(pqg_ctx* ctx, const float* rows, uint64_t n, uint64_t ld, uint32_t B,
                    uint32_t d, uint32_t col_stride, const float* tables, uint64_t k,
                    uint32_t* assign, double* dist);
/* The reference's update step (kmeans.cpp:102-130) for B problems given the
 * full (all-shard, row-ordered) assignments and dists: fp64 sums in row
 * order, mean = float(sum * (1/count)), empty clusters reseeded from the
 * pre-update dists.  tables updated in place; dist modified (reseed zeroes). */
int pqg_update_pass(pqg_ctx* ctx, const float* rows, uint64_t n, uint64_t ld, uint32_t B,
                    uint32_t d, uint32_t col_stride, float* tables, uint64_t k,
                    const uint32_t* assign, double* dist, const int* active);
/* Per-problem inertia of B x n fp64 distances with the same fixed-shape tree
 * the single-process fit uses (so sharded and single fits stop identically). */
int pqg_rows_sum_f64(pqg_ctx* ctx, const double* v, uint64_t n, uint32_t B, double* out);
/* The k init rows kmeans_fit draws (proj/src/kmeans.cpp:73-85), host-side. */
int pqg_kmeans_init_rows(uint64_t n, uint64_t k, uint64_t seed, uint64_t* rows);

/* ---- row-sharded k-means, one rank's side -------------
 * The north-star exchange: per iteration ONE all-reduce (SUM) of the packed
 * fp64 partials [centroid sums B*k*d | counts B*k | inertia B] and one
 * all-reduce (MAX) of the u8 exponent ranges [B*k*d | B*k*d]; the caller
 * (paper_2604_21645_b200/dist.py, torch.distributed / NCCL) owns the
 * collectives, these calls own the device work.  Ranks hold ascending
 * contiguous blocks of the global row-ordered sample; the result equals
 * kmeans_fit (kmeans.cpp:61-133) / pq_fit's per-subspace fits bit for bit:
 * sums whose global exponent range proves them exact are reduced in any
 * order, the rest are replayed in global row order from the members the
 * ranks exchange (pqg_kmshard_pack / _replay), empty clusters are reseeded
 * from every rank's best candidates (pqg_kmshard_reseed_*).  rows: device,
 * n x ld; problem b reads columns [b*col_stride, b*col_stride + d); d % 4 ==
 * 0 and d <= 128 (else PQG_EUNSUPPORTED).  Every call runs on ctx's stream. */
typedef struct pqg_kmshard pqg_kmshard;
int pqg_kmshard_create(pqg_ctx* ctx, const float* rows, uint64_t n, uint64_t ld, uint32_t B, uint32_t d,
                       uint32_t col_stride, uint64_t k, uint32_t max_iters, double tol, pqg_kmshard** out);
void pqg_kmshard_destroy(pqg_kmshard* h);
/* element counts of the two packed partial buffers */
int pqg_kmshard_sizes(const pqg_kmshard* h, uint64_t* n_f64, uint64_t* n_u8);
/* table_bits (device, B*k*d u32): the bit patterns of the init rows this rank
 * owns (global row ids init_rows[B*k], host; this rank holds rows
 * [row0, row0 + n)), zero elsewhere -- an integer all-reduce SUM assembles
 * the initial centroids (kmeans.cpp:73-88). */
int pqg_kmshard_init_table(pqg_ctx* ctx, pqg_kmshard* h, const uint64_t* init_rows, uint64_t row0,
                           uint32_t* table_bits);
/* assignment pass (kmeans.cpp:46-57) of the local rows against tables
 * (device B*k*d) and the local partials into f64 / u8 (device) */
int pqg_kmshard_partials(pqg_ctx* ctx, pqg_kmshard* h, const float* tables, double* f64, uint8_t* u8);
/* after the all-reduces: stop rule, exact means, the ordered list of the
 * n_fail (b, c, t) columns that need the row-order replay and *stride (an
 * upper bound on every rank's pack length: the columns' global member
 * counts), the largest number of empty clusters of a continuing problem
 * (*max_empty), *any_active.  The iteration's one host synchronisation. */
int pqg_kmshard_apply(pqg_ctx* ctx, pqg_kmshard* h, float* tables, const double* f64, const uint8_t* u8,
                      uint64_t* n_fail, uint64_t* stride, uint32_t* max_empty, int* any_active);
/* this rank's members of the replay columns in local row order: vals (device,
 * cap >= stride floats) and offcnt (device, 2*n_fail u64: offset, count) */
int pqg_kmshard_pack(pqg_ctx* ctx, pqg_kmshard* h, float* vals, uint64_t cap, uint64_t* offcnt);
/* the reference's chain over every rank's packed members, rank order:
 * all_vals world x stride floats, all_offcnt world x 2*n_fail */
int pqg_kmshard_replay(pqg_ctx* ctx, pqg_kmshard* h, float* tables, const double* f64, const float* all_vals,
                       uint64_t stride, const uint64_t* all_offcnt, uint32_t world);
/* The chained replay (r2e; no member values cross ranks): run (device,
 * n_fail fp64) holds each replay column's running row-order sum over the
 * members of the ranks before this one (zeros on rank 0); _step continues
 * every chain over this rank's members in local row order (the caller then
 * hands run to the next rank), _finish writes the means from the last
 * rank's run (broadcast to every rank). */
int pqg_kmshard_replay_step(pqg_ctx* ctx, pqg_kmshard* h, double* run);
int pqg_kmshard_replay_finish(pqg_ctx* ctx, pqg_kmshard* h, float* tables, const double* f64, const double* run);
/* per problem the E+1 candidate slots (dist, global index, row) of this rank */
int pqg_kmshard_reseed_candidates(pqg_ctx* ctx, pqg_kmshard* h, uint64_t row0, uint32_t E, double* cand_d,
                                  uint64_t* cand_i, float* cand_rows);
int pqg_kmshard_reseed_apply(pqg_ctx* ctx, pqg_kmshard* h, float* tables, const double* f64, uint32_t E,
                             uint32_t world, const double* all_d, const uint64_t* all_i, const float* all_rows);
/* iterations_run[B], inertia[B], inertia_per_iter[B*max_iters], the last
 * pass's local assignments [B*n] (any nullable; host or device) */
int pqg_kmshard_result(pqg_ctx* ctx, pqg_kmshard* h, uint32_t* iterations_run, double* inertia,
                       double* inertia_per_iter, uint32_t* assignments);

/* ---- the native host of the row-sharded fit (kmnccl.cu; r2e) --------------
 * One rank per GPU with its own NCCL communicator (libnccl.so.2, opened at
 * run time): pqg_kmeans_fit_sharded runs the whole pqg_kmshard_* protocol
 * above in C++ -- grouped ncclAllReduce of the partials, the row-order chain
 * by ncclSend / ncclRecv / ncclBroadcast, ncclAllGather of the reseed
 * candidates -- on ctx's stream, one host synchronisation per iteration.
 * rows: this rank's n_local x ld device rows (ranks hold ascending contiguous
 * blocks of the global row-ordered sample); seeds[B]; tables_out B*k*d (host
 * or device); iterations_run[B], inertia[B], inertia_per_iter[B*max_iters],
 * assignments_local[B*n_local] as pqg_kmshard_result (nullable); stats[4]
 * (nullable): iterations, replay columns, reseeds, all-reduced bytes per
 * iteration.  Equals kmeans_fit / pq_fit's subspace fits bit for bit. */
int pqg_nccl_get_unique_id(void* id128);
int pqg_nccl_comm_init(int device, int world, int rank, const void* id128, void** comm);
int pqg_nccl_comm_init_all(int ndev, const int* devices, void** comms);
void pqg_nccl_comm_destroy(void* comm);
int pqg_kmeans_fit_sharded(pqg_ctx* ctx, void* comm, const float* rows, uint64_t n_local, uint64_t ld,
                           uint32_t B, uint32_t d, uint32_t col_stride, uint64_t k, uint32_t max_iters,
                           const uint64_t* seeds, double tol, float* tables_out, uint32_t* iterations_run,
                           double* inertia, double* inertia_per_iter, uint32_t* assignments_local,
                           uint64_t* stats);

/* ---- on-disk formats ----------------------------------
 * Byte-identical to the reference's files; load errors carry the reference's
 * messages ("<format>: bad magic", "truncated read of <what>",
 * "<path>: unsupported version N", "<path>: duplicate id N",
 * "<path>: code out of range", "<path>: trailing data after payload", ...) as
 * PQG_EIO (std::runtime_error), except the codebook-parameter checks
 * (PQG_EINVAL, std::invalid_argument) the reference raises on the way. */

/* PQII index image (save_index / load_index, ivf.cpp:264-355).  The posting
 * lists are packed / unpacked by device kernels (formats.cu) straight from /
 * into the device CSR; ids are checked for duplicates and codes for range on
 * the device.  serialize: buf (host or device) NULL -> only *size. */
int pqg_index_serialize(pqg_ctx* ctx, const pqg_index* index, void* buf, uint64_t cap, uint64_t* size);
int pqg_index_deserialize(pqg_ctx* ctx, const void* buf, uint64_t size, const char* name, pqg_index** out);
int pqg_index_save(pqg_ctx* ctx, const pqg_index* index, const char* path);
int pqg_index_load(pqg_ctx* ctx, const char* path, pqg_index** out);

/* PQCM code file (save_codes / load_codes, pq.cpp:221-259): codes host or
 * device; load validates every code on the device ("code out of range at
 * row N").  file_info reads only the header (n, M, ks). */
int pqg_codes_save(pqg_ctx* ctx, const uint8_t* codes, uint64_t n, uint32_t M, uint32_t ks, const char* path);
int pqg_codes_file_info(const char* path, uint64_t* n, uint32_t* M, uint32_t* ks);
int pqg_codes_load(pqg_ctx* ctx, const char* path, uint8_t* codes, uint64_t cap_bytes);

/* PQCB codebook file (save_codebook / load_codebook, pq.cpp:183-219). */
int pqg_codebook_save(pqg_ctx* ctx, const float* tables, uint32_t M, uint32_t ks, uint32_t ds, const char* path);
int pqg_codebook_file_info(const char* path, uint32_t* M, uint32_t* ks, uint32_t* ds);
int pqg_codebook_load(pqg_ctx* ctx, const char* path, float* tables, uint64_t cap_floats);

#ifdef __cplusplus
}
#endif
#endif /* PQG_H */
