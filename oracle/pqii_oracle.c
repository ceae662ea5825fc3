/*
 * pqii_oracle.c -- CPU restatement of the reference's PQ / IVF hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path in paper_2604_21645_b200/.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * library never links or calls it.
 *
 * Every function restates one reference function; the citation in front of
 * each names /root/reference/proj/<file>:<lines>.  Arithmetic order matters:
 * distances are fp64, accumulated left to right with separate multiply and
 * add (the reference is built for baseline x86-64, which has no FMA), so
 * this file must be compiled with -ffp-contract=off.
 *
 * Pinning: tests/test_oracle.py checks every function here against
 *   (a) the reference compiled from its own sources (oracle/_ref, built by
 *       oracle/Makefile) and
 *   (b) the committed golden fixtures tests/golden/*.npz written by
 *       tests/golden/make_golden.py from that compiled reference, and
 *   (c) the reference's own known-answer tests (test_kmeans.cpp, test_pq.cpp).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EINVAL (-1)
#define ORC_ERANGE (-2)
#define ORC_ENOMEM (-3)

/* ------------------------------------------------------------------------ */
/* std::mt19937_64 (fully specified by the C++ standard, [rand.eng.mers]).   */
/* Used by kmeans_fit's init (proj/src/kmeans.cpp:74) and the test helpers. */
/* ------------------------------------------------------------------------ */
#define MT_N 312
#define MT_M 156
typedef struct {
    uint64_t s[MT_N];
    int i;
} orc_mt64;

void orc_mt_seed(orc_mt64* g, uint64_t seed) {
    g->s[0] = seed;
    for (int k = 1; k < MT_N; ++k) {
        uint64_t prev = g->s[k - 1];
        g->s[k] = 6364136223846793005ULL * (prev ^ (prev >> 62)) + (uint64_t)k;
    }
    g->i = MT_N;
}

static void mt_twist(orc_mt64* g) {
    const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
    for (int k = 0; k < MT_N; ++k) {
        uint64_t y = (g->s[k] & upper) | (g->s[(k + 1) % MT_N] & lower);
        uint64_t v = g->s[(k + MT_M) % MT_N] ^ (y >> 1);
        if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
        g->s[k] = v;
    }
    g->i = 0;
}

uint64_t orc_mt_next(orc_mt64* g) {
    if (g->i >= MT_N) mt_twist(g);
    uint64_t z = g->s[g->i++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= z >> 43;
    return z;
}

/* libstdc++ (GCC 13) std::uniform_int_distribution<size_t>(lo, hi) driven by
 * a 64-bit engine: Lemire's multiply-shift with rejection ("_S_nd" in
 * bits/uniform_int_dist.h).  The reference relies on this implementation-
 * defined algorithm for its k-means init (proj/src/kmeans.cpp:77-80). */
uint64_t orc_uniform_index(orc_mt64* g, uint64_t lo, uint64_t hi) {
    const uint64_t urange = hi - lo;
    if (urange == UINT64_MAX) return orc_mt_next(g) + lo;
    const uint64_t range = urange + 1;
    unsigned __int128 prod = (unsigned __int128)orc_mt_next(g) * range;
    uint64_t low = (uint64_t)prod;
    if (low < range) {
        const uint64_t threshold = (0 - range) % range;
        while (low < threshold) {
            prod = (unsigned __int128)orc_mt_next(g) * range;
            low = (uint64_t)prod;
        }
    }
    return (uint64_t)(prod >> 64) + lo;
}

/* libstdc++ std::uniform_real_distribution<float>(lo, hi) over mt19937_64:
 * generate_canonical<float, 24> takes one 64-bit draw, converts it to float,
 * divides by 2^64 and clamps to nextafter(1, 0); the result is scaled as
 * u * (hi - lo) + lo in float.  Restates proj/tests/test_helpers.cpp:26-33
 * (random_matrix), the fixture behind most of the reference's unit tests. */
static float uniform_float(orc_mt64* g, float lo, float hi) {
    float sum = (float)orc_mt_next(g);
    float r = sum / 18446744073709551616.0f;
    if (r >= 1.0f) r = nextafterf(1.0f, 0.0f);
    return r * (hi - lo) + lo;
}

void orc_random_matrix(uint64_t rows, uint64_t dims, uint64_t seed, float lo, float hi,
                       float* out) {
    orc_mt64 g;
    orc_mt_seed(&g, seed);
    for (uint64_t i = 0; i < rows * dims; ++i) out[i] = uniform_float(&g, lo, hi);
}

/* ------------------------------------------------------------------------ */
/* Distances and argmin: proj/src/kmeans.cpp:11-40                            */
/* ------------------------------------------------------------------------ */

/* proj/src/kmeans.cpp:11-18 -- sequential fp64 sum of squared differences. */
double orc_squared_l2(const float* a, const float* b, uint64_t d) {
    double acc = 0.0;
    for (uint64_t i = 0; i < d; ++i) {
        const double diff = (double)a[i] - (double)b[i];
        acc += diff * diff;
    }
    return acc;
}

/* proj/src/kmeans.cpp:20-31 -- strict '<' keeps the lowest index on ties. */
void orc_nearest_in_table(const float* point, const float* table, uint64_t k, uint64_t d,
                          uint64_t* index, double* sq_dist) {
    uint64_t best = 0;
    double best_d = orc_squared_l2(point, table, d);
    for (uint64_t c = 1; c < k; ++c) {
        const double dist = orc_squared_l2(point, table + c * d, d);
        if (dist < best_d) {
            best = c;
            best_d = dist;
        }
    }
    *index = best;
    *sq_dist = best_d;
}

/* Batched form of nearest_in_table over n points (used by the tests). */
void orc_nearest_batch(const float* points, uint64_t n, uint64_t d, const float* table,
                       uint64_t k, uint32_t* index, double* sq_dist) {
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t idx;
        double dist;
        orc_nearest_in_table(points + i * d, table, k, d, &idx, &dist);
        index[i] = (uint32_t)idx;
        sq_dist[i] = dist;
    }
}

/* ------------------------------------------------------------------------ */
/* Threaded helpers (parity at BASELINE sizes).  Each row's nearest centroid */
/* is computed exactly as above, independently of the others; the threads   */
/* only split the row range, and every order-dependent reduction (inertia,   */
/* sums) stays sequential on the calling thread, so results are bit-identical */
/* to the single-threaded restatement for any thread count.                  */
/* ------------------------------------------------------------------------ */
typedef struct {
    const float* points;
    const float* table;
    uint64_t b, e, d, k;
    uint32_t* index;
    double* sq_dist;
} orc_nb_task;

static void* nb_worker(void* p) {
    const orc_nb_task* t = (const orc_nb_task*)p;
    orc_nearest_batch(t->points + t->b * t->d, t->e - t->b, t->d, t->table, t->k,
                      t->index + t->b, t->sq_dist + t->b);
    return NULL;
}

void orc_nearest_batch_mt(const float* points, uint64_t n, uint64_t d, const float* table,
                          uint64_t k, uint32_t* index, double* sq_dist, int threads) {
    if (threads > 256) threads = 256;
    if (threads < 2 || n < 2 * (uint64_t)threads) {
        orc_nearest_batch(points, n, d, table, k, index, sq_dist);
        return;
    }
    pthread_t tid[256];
    orc_nb_task task[256];
    for (int t = 0; t < threads; ++t) {
        task[t] = (orc_nb_task){points, table, n * t / threads, n * (t + 1) / threads, d, k, index,
                                sq_dist};
        pthread_create(&tid[t], NULL, nb_worker, &task[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
}

/* The update step of proj/src/kmeans.cpp:102-130 given one pass's
 * assignments and fp64 distances: fp64 sums in row order, mean =
 * float(sum * (1/count)) for non-empty clusters, then each empty cluster in
 * ascending order takes the row of the (strict '>') largest pre-update
 * distance and zeroes it.  centroids and dists are updated in place; also the
 * parity checker for one Lloyd step from the GPU's centroids. */
int orc_lloyd_update(const float* points, uint64_t n, uint64_t d, uint64_t k,
                     const uint32_t* assignments, double* dists, float* centroids) {
    double* sums = (double*)calloc(k * d, sizeof(double));
    uint64_t* counts = (uint64_t*)calloc(k, sizeof(uint64_t));
    if (!sums || !counts) {
        free(sums); free(counts);
        return ORC_ENOMEM;
    }
    for (uint64_t i = 0; i < n; ++i) {
        const uint32_t c = assignments[i];
        if (c >= k) {
            free(sums); free(counts);
            return ORC_ERANGE;
        }
        const float* row = points + i * d;
        double* s = sums + (uint64_t)c * d;
        for (uint64_t j = 0; j < d; ++j) s[j] += row[j];
        ++counts[c];
    }
    for (uint64_t c = 0; c < k; ++c) {
        if (counts[c] == 0) continue;
        const double inv = 1.0 / (double)counts[c];
        for (uint64_t j = 0; j < d; ++j) centroids[c * d + j] = (float)(sums[c * d + j] * inv);
    }
    for (uint64_t c = 0; c < k; ++c) {
        if (counts[c] != 0) continue;
        uint64_t far = 0;
        for (uint64_t i = 1; i < n; ++i)
            if (dists[i] > dists[far]) far = i;
        memcpy(centroids + c * d, points + far * d, d * sizeof(float));
        dists[far] = 0.0;
    }
    free(sums);
    free(counts);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Lloyd k-means: proj/src/kmeans.cpp:61-133                                 */
/* ------------------------------------------------------------------------ */
/* threads > 1 splits only the assignment pass's rows (see above). */
int orc_kmeans_fit_mt(const float* points, uint64_t n, uint64_t d, uint64_t k, uint32_t max_iters,
                      uint64_t seed, double tol, float* centroids, uint32_t* assignments,
                      double* inertia_out, uint32_t* iterations_run, double* inertia_per_iter,
                      int threads) {
    /* validation, :65-71 */
    if (k == 0 || k > n || max_iters < 1 || tol < 0.0) return ORC_EINVAL;

    /* init: k distinct rows by partial Fisher-Yates, :73-88 */
    uint64_t* idx = (uint64_t*)malloc(n * sizeof(uint64_t));
    double* dists = (double*)malloc(n * sizeof(double));
    if (!idx || !dists) {
        free(idx); free(dists);
        return ORC_ENOMEM;
    }
    orc_mt64 g;
    orc_mt_seed(&g, seed);
    for (uint64_t i = 0; i < n; ++i) idx[i] = i;
    for (uint64_t i = 0; i < k; ++i) {
        const uint64_t j = orc_uniform_index(&g, i, n - 1);
        const uint64_t t = idx[i];
        idx[i] = idx[j];
        idx[j] = t;
    }
    for (uint64_t c = 0; c < k; ++c) memcpy(centroids + c * d, points + idx[c] * d, d * sizeof(float));
    free(idx);

    double inertia = 0.0, prev = 0.0;
    uint32_t it_run = 0;
    int rc = ORC_OK;
    for (uint32_t it = 1; it <= max_iters; ++it) {
        /* assign pass, :46-57; inertia summed sequentially in row order */
        orc_nearest_batch_mt(points, n, d, centroids, k, assignments, dists, threads);
        inertia = 0.0;
        for (uint64_t i = 0; i < n; ++i) inertia += dists[i];
        if (inertia_per_iter) inertia_per_iter[it - 1] = inertia;
        it_run = it;
        /* stop rules, :98-100 */
        const double floor1 = prev > 1.0 ? prev : 1.0;
        if (it > 1 && prev - inertia < tol * floor1) break;
        if (it == max_iters) break;
        prev = inertia;
        /* update + empty-cluster reseed, :102-130 */
        rc = orc_lloyd_update(points, n, d, k, assignments, dists, centroids);
        if (rc) break;
    }
    *inertia_out = inertia;
    *iterations_run = it_run;
    free(dists);
    return rc;
}

int orc_kmeans_fit(const float* points, uint64_t n, uint64_t d, uint64_t k, uint32_t max_iters,
                   uint64_t seed, double tol, float* centroids, uint32_t* assignments,
                   double* inertia_out, uint32_t* iterations_run, double* inertia_per_iter) {
    return orc_kmeans_fit_mt(points, n, d, k, max_iters, seed, tol, centroids, assignments,
                             inertia_out, iterations_run, inertia_per_iter, 1);
}

/* ------------------------------------------------------------------------ */
/* Product quantization: proj/src/pq.cpp                                     */
/* ------------------------------------------------------------------------ */
static uint32_t code_width(uint32_t ks) { return ks <= 256 ? 1u : 2u; } /* pq.hpp:45 */

static uint32_t code_at(const uint8_t* codes, uint64_t i, uint32_t m, uint32_t M, uint32_t w) {
    const uint64_t off = (i * M + m) * w; /* pq.cpp:41-45 */
    if (w == 1) return codes[off];
    return (uint32_t)codes[off] | ((uint32_t)codes[off + 1] << 8);
}

static void code_set(uint8_t* codes, uint64_t i, uint32_t m, uint32_t M, uint32_t w, uint32_t v) {
    const uint64_t off = (i * M + m) * w; /* pq.cpp:47-51 */
    codes[off] = (uint8_t)(v & 0xff);
    if (w == 2) codes[off + 1] = (uint8_t)(v >> 8);
}

/* proj/src/pq.cpp:63-93: one kmeans_fit per column block, seed + sub,
 * default tol (kmeans.hpp:12).  iters_out[m] (optional) gets iterations_run. */
int orc_pq_fit(const float* data, uint64_t n, uint64_t D, uint32_t M, uint32_t ks,
               uint32_t max_iters, uint64_t seed, float* tables, uint32_t* iters_out,
               double* inertia_out) {
    if (M == 0 || D % M != 0 || ks > n || ks == 0 || ks > 65536) return ORC_EINVAL;
    const uint64_t ds = D / M;
    float* slice = (float*)malloc(n * ds * sizeof(float));
    uint32_t* assign = (uint32_t*)malloc(n * sizeof(uint32_t));
    if (!slice || !assign) {
        free(slice); free(assign);
        return ORC_ENOMEM;
    }
    int rc = ORC_OK;
    for (uint32_t sub = 0; sub < M && rc == ORC_OK; ++sub) {
        for (uint64_t i = 0; i < n; ++i)
            memcpy(slice + i * ds, data + i * D + sub * ds, ds * sizeof(float));
        double inertia;
        uint32_t iters;
        rc = orc_kmeans_fit(slice, n, ds, ks, max_iters, seed + sub, 1e-4,
                            tables + (uint64_t)sub * ks * ds, assign, &inertia, &iters, NULL);
        if (iters_out) iters_out[sub] = iters;
        if (inertia_out) inertia_out[sub] = inertia;
    }
    free(slice);
    free(assign);
    return rc;
}

/* proj/src/pq.cpp:95-111 */
void orc_pq_encode(const float* data, uint64_t n, uint32_t M, uint32_t ks, uint32_t ds,
                   const float* tables, uint8_t* codes) {
    const uint32_t w = code_width(ks);
    const uint64_t D = (uint64_t)M * ds;
    for (uint64_t i = 0; i < n; ++i) {
        for (uint32_t m = 0; m < M; ++m) {
            uint64_t best;
            double bd;
            orc_nearest_in_table(data + i * D + m * ds, tables + (uint64_t)m * ks * ds, ks, ds,
                                 &best, &bd);
            code_set(codes, i, m, M, w, (uint32_t)best);
        }
    }
}

/* proj/src/pq.cpp:113-130; returns ORC_ERANGE for a code >= ks (:117-120). */
int orc_pq_decode(const uint8_t* codes, uint64_t n, uint32_t M, uint32_t ks, uint32_t ds,
                  const float* tables, float* out) {
    const uint32_t w = code_width(ks);
    const uint64_t D = (uint64_t)M * ds;
    for (uint64_t i = 0; i < n; ++i) {
        for (uint32_t m = 0; m < M; ++m) {
            const uint32_t code = code_at(codes, i, m, M, w);
            if (code >= ks) return ORC_ERANGE;
            memcpy(out + i * D + m * ds, tables + ((uint64_t)m * ks + code) * ds,
                   ds * sizeof(float));
        }
    }
    return ORC_OK;
}

/* proj/src/pq.cpp:169-177: fp64 sequential sum over all elements. */
double orc_rmse(const float* a, const float* b, uint64_t rows, uint64_t dims) {
    double total = 0.0;
    for (uint64_t i = 0; i < rows * dims; ++i) {
        const double diff = (double)a[i] - (double)b[i];
        total += diff * diff;
    }
    return sqrt(total / (double)(rows * dims));
}

/* proj/src/pipeline.cpp:84-106 (train_chunk): a local pq_fit with the chunk's
 * seed, representative j = codeword j of every subspace concatenated
 * (reps ks x D), and the chunk's reconstruction rmse under its own codebook
 * (reconstruction_rmse = rmse(chunk, decode(encode(chunk))), pq.cpp:179-181). */
int orc_train_chunk(const float* chunk, uint64_t n, uint64_t D, uint32_t M, uint32_t ks,
                    uint32_t max_iters, uint64_t chunk_seed, float* reps, double* local_rmse) {
    if (n < ks) return ORC_EINVAL; /* pipeline.cpp:86-89 */
    if (M == 0 || D % M != 0) return ORC_EINVAL;
    const uint64_t ds = D / M;
    float* tables = (float*)malloc((uint64_t)M * ks * ds * sizeof(float));
    uint8_t* codes = (uint8_t*)malloc(n * M * code_width(ks));
    float* dec = (float*)malloc(n * D * sizeof(float));
    int rc = (tables && codes && dec) ? ORC_OK : ORC_ENOMEM;
    if (rc == ORC_OK) rc = orc_pq_fit(chunk, n, D, M, ks, max_iters, chunk_seed, tables, NULL, NULL);
    if (rc == ORC_OK) {
        for (uint32_t j = 0; j < ks; ++j)
            for (uint32_t m = 0; m < M; ++m)
                memcpy(reps + (uint64_t)j * D + m * ds, tables + ((uint64_t)m * ks + j) * ds,
                       ds * sizeof(float));
        orc_pq_encode(chunk, n, M, ks, (uint32_t)ds, tables, codes);
        rc = orc_pq_decode(codes, n, M, ks, (uint32_t)ds, tables, dec);
        if (rc == ORC_OK) *local_rmse = orc_rmse(chunk, dec, n, D);
    }
    free(tables);
    free(codes);
    free(dec);
    return rc;
}

/* proj/src/pq.cpp:132-151: entries are float(fp64 squared_l2). */
void orc_adc_table(const float* tables, uint32_t M, uint32_t ks, uint32_t ds, const float* query,
                   float* entries) {
    for (uint32_t m = 0; m < M; ++m)
        for (uint32_t j = 0; j < ks; ++j)
            entries[(uint64_t)m * ks + j] =
                (float)orc_squared_l2(query + m * ds, tables + ((uint64_t)m * ks + j) * ds, ds);
}

/* proj/src/pq.cpp:153-167: fp64 sum of float entries in m order. */
int orc_adc_lookup(const float* entries, uint32_t M, uint32_t ks, const uint8_t* codes,
                   uint64_t row, double* out) {
    const uint32_t w = code_width(ks);
    double acc = 0.0;
    for (uint32_t m = 0; m < M; ++m) {
        const uint32_t code = code_at(codes, row, m, M, w);
        if (code >= ks) return ORC_ERANGE;
        acc += entries[(uint64_t)m * ks + code];
    }
    *out = acc;
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Inverted index: proj/src/ivf.cpp                                          */
/* ------------------------------------------------------------------------ */

/* proj/src/ivf.cpp:36-49 (assign_items): list of the coarse centroid nearest
 * the DECODED code row. */
int orc_ivf_assign(const uint8_t* codes, uint64_t n, uint32_t M, uint32_t ks, uint32_t ds,
                   const float* tables, const float* coarse, uint64_t nlist, uint32_t* list_of) {
    const uint64_t D = (uint64_t)M * ds;
    float* dec = (float*)malloc(D * sizeof(float));
    if (!dec) return ORC_ENOMEM;
    for (uint64_t i = 0; i < n; ++i) {
        int rc = orc_pq_decode(codes + i * M * code_width(ks), 1, M, ks, ds, tables, dec);
        if (rc) {
            free(dec);
            return rc;
        }
        uint64_t best;
        double bd;
        orc_nearest_in_table(dec, coarse, nlist, D, &best, &bd);
        list_of[i] = (uint32_t)best;
    }
    free(dec);
    return ORC_OK;
}

/* Posting lists as CSR.  The reference appends in input order
 * (proj/src/ivf.cpp:44-46), i.e. a stable counting sort on list id. */
void orc_ivf_csr(const uint32_t* list_of, const uint64_t* ids, const uint8_t* codes, uint64_t n,
                 uint64_t row_bytes, uint64_t nlist, uint64_t* offsets, uint64_t* out_ids,
                 uint8_t* out_codes) {
    memset(offsets, 0, (nlist + 1) * sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) offsets[list_of[i] + 1]++;
    for (uint64_t l = 0; l < nlist; ++l) offsets[l + 1] += offsets[l];
    uint64_t* cursor = (uint64_t*)malloc(nlist * sizeof(uint64_t));
    memcpy(cursor, offsets, nlist * sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t p = cursor[list_of[i]]++;
        out_ids[p] = ids[i];
        memcpy(out_codes + p * row_bytes, codes + i * row_bytes, row_bytes);
    }
    free(cursor);
}

typedef struct {
    uint64_t id;
    double d;
} orc_hit;

static int hit_less(const void* pa, const void* pb) { /* HitLess, proj/src/ivf.cpp:51-56 */
    const orc_hit* a = (const orc_hit*)pa;
    const orc_hit* b = (const orc_hit*)pb;
    if (a->d != b->d) return a->d < b->d ? -1 : 1;
    return a->id < b->id ? -1 : (a->id > b->id ? 1 : 0);
}

typedef struct {
    double d;
    uint64_t c;
} orc_probe;

static int probe_less(const void* pa, const void* pb) { /* std::pair order, ivf.cpp:97 */
    const orc_probe* a = (const orc_probe*)pa;
    const orc_probe* b = (const orc_probe*)pb;
    if (a->d != b->d) return a->d < b->d ? -1 : 1;
    return a->c < b->c ? -1 : (a->c > b->c ? 1 : 0);
}

/* proj/src/ivf.cpp:91-101 (probe_order): the nprobe smallest (dist, c). */
void orc_probe_order(const float* coarse, uint64_t nlist, uint64_t D, const float* query,
                     uint64_t nprobe, uint32_t* probes) {
    orc_probe* order = (orc_probe*)malloc(nlist * sizeof(orc_probe));
    for (uint64_t c = 0; c < nlist; ++c) {
        order[c].d = orc_squared_l2(query, coarse + c * D, D);
        order[c].c = c;
    }
    qsort(order, nlist, sizeof(orc_probe), probe_less);
    for (uint64_t p = 0; p < nprobe; ++p) probes[p] = (uint32_t)order[p].c;
    free(order);
}

/* proj/src/ivf.cpp:58-68 (finalize_hits): k smallest by (dist, id), sorted. */
static uint64_t finalize(orc_hit* hits, uint64_t nh, uint64_t k, uint64_t* out_ids,
                         double* out_d) {
    qsort(hits, nh, sizeof(orc_hit), hit_less);
    const uint64_t cnt = nh < k ? nh : k;
    for (uint64_t i = 0; i < cnt; ++i) {
        out_ids[i] = hits[i].id;
        out_d[i] = hits[i].d;
    }
    return cnt;
}

/* proj/src/ivf.cpp:218-228 (ivf_query) over a CSR index; has_max selects the
 * optional max_sq_dist filter (:70-77).  Returns the hit count (<= k) or a
 * negative status. */
int64_t orc_ivf_query(const float* tables, uint32_t M, uint32_t ks, uint32_t ds,
                      const float* coarse, uint64_t nlist, const uint64_t* offsets,
                      const uint64_t* list_ids, const uint8_t* list_codes, const float* query,
                      uint64_t k, uint64_t nprobe, int has_max, double max_sq_dist,
                      uint64_t* out_ids, double* out_d) {
    if (k == 0 || nprobe == 0 || nprobe > nlist) return ORC_EINVAL; /* check_query :103-114 */
    const uint64_t D = (uint64_t)M * ds;
    float* table = (float*)malloc((uint64_t)M * ks * sizeof(float));
    uint32_t* probes = (uint32_t*)malloc(nprobe * sizeof(uint32_t));
    orc_adc_table(tables, M, ks, ds, query, table);
    orc_probe_order(coarse, nlist, D, query, nprobe, probes);
    uint64_t cap = 0;
    for (uint64_t p = 0; p < nprobe; ++p) cap += offsets[probes[p] + 1] - offsets[probes[p]];
    orc_hit* hits = (orc_hit*)malloc((cap ? cap : 1) * sizeof(orc_hit));
    uint64_t nh = 0;
    const uint64_t rb = (uint64_t)M * code_width(ks);
    int rc = 0;
    for (uint64_t p = 0; p < nprobe && !rc; ++p) {
        const uint64_t l = probes[p];
        for (uint64_t e = offsets[l]; e < offsets[l + 1]; ++e) {
            double dist;
            rc = orc_adc_lookup(table, M, ks, list_codes + e * rb, 0, &dist);
            if (rc) break;
            if (has_max && dist > max_sq_dist) continue;
            hits[nh].id = list_ids[e];
            hits[nh].d = dist;
            ++nh;
        }
    }
    int64_t cnt = rc ? rc : (int64_t)finalize(hits, nh, k, out_ids, out_d);
    free(hits);
    free(table);
    free(probes);
    return cnt;
}

/* proj/src/ivf.cpp:247-262 (flat_scan). */
int64_t orc_flat_scan(const float* tables, uint32_t M, uint32_t ks, uint32_t ds,
                      const uint8_t* codes, const uint64_t* ids, uint64_t n, const float* query,
                      uint64_t k, int has_max, double max_sq_dist, uint64_t* out_ids,
                      double* out_d) {
    if (k == 0) return ORC_EINVAL;
    float* table = (float*)malloc((uint64_t)M * ks * sizeof(float));
    orc_adc_table(tables, M, ks, ds, query, table);
    orc_hit* hits = (orc_hit*)malloc((n ? n : 1) * sizeof(orc_hit));
    uint64_t nh = 0;
    int rc = 0;
    for (uint64_t i = 0; i < n; ++i) {
        double dist;
        rc = orc_adc_lookup(table, M, ks, codes, i, &dist);
        if (rc) break;
        if (has_max && dist > max_sq_dist) continue;
        hits[nh].id = ids[i];
        hits[nh].d = dist;
        ++nh;
    }
    int64_t cnt = rc ? rc : (int64_t)finalize(hits, nh, k, out_ids, out_d);
    free(hits);
    free(table);
    return cnt;
}

/* proj/src/dataset_io.cpp:322-339 (chunk_rows): the first n % c ranges carry
 * one extra row.  Writes c+1 boundaries. */
int orc_chunk_rows(uint64_t n, uint64_t c, uint64_t* bounds) {
    if (c == 0 || c > n) return ORC_EINVAL;
    const uint64_t base = n / c, extra = n % c;
    bounds[0] = 0;
    for (uint64_t i = 0; i < c; ++i) bounds[i + 1] = bounds[i] + base + (i < extra ? 1 : 0);
    return ORC_OK;
}

/* The sequence of uniform_int_distribution(i, n-1) draws kmeans_fit makes
 * during init (proj/src/kmeans.cpp:74-80); used to pin orc_uniform_index. */
void orc_init_draws(uint64_t seed, uint64_t n, uint64_t k, uint64_t* out) {
    orc_mt64 g;
    orc_mt_seed(&g, seed);
    for (uint64_t i = 0; i < k; ++i) out[i] = orc_uniform_index(&g, i, n - 1);
}

static int in_sorted(const uint64_t* s, uint64_t n, uint64_t v) { /* std::binary_search */
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) / 2;
        if (s[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo < n && s[lo] == v;
}

/* proj/src/ivf.cpp:230-245 (ivf_query_subset) with scan_list_subset (:79-88):
 * candidates whose id is not in the sorted subset are skipped before the
 * distance test.  Returns the hit count or a negative status. */
int64_t orc_ivf_query_subset(const float* tables, uint32_t M, uint32_t ks, uint32_t ds,
                             const float* coarse, uint64_t nlist, const uint64_t* offsets,
                             const uint64_t* list_ids, const uint8_t* list_codes, const float* query,
                             uint64_t k, const uint64_t* subset, uint64_t nsub, uint64_t nprobe,
                             int has_max, double max_sq_dist, uint64_t* out_ids, double* out_d) {
    if (k == 0 || nprobe == 0 || nprobe > nlist) return ORC_EINVAL;
    for (uint64_t i = 1; i < nsub; ++i)
        if (subset[i - 1] >= subset[i]) return ORC_EINVAL;
    const uint64_t D = (uint64_t)M * ds;
    float* table = (float*)malloc((uint64_t)M * ks * sizeof(float));
    uint32_t* probes = (uint32_t*)malloc(nprobe * sizeof(uint32_t));
    orc_adc_table(tables, M, ks, ds, query, table);
    orc_probe_order(coarse, nlist, D, query, nprobe, probes);
    uint64_t cap = 0;
    for (uint64_t p = 0; p < nprobe; ++p) cap += offsets[probes[p] + 1] - offsets[probes[p]];
    orc_hit* hits = (orc_hit*)malloc((cap ? cap : 1) * sizeof(orc_hit));
    uint64_t nh = 0;
    const uint64_t rb = (uint64_t)M * code_width(ks);
    int rc = 0;
    for (uint64_t p = 0; p < nprobe && !rc; ++p) {
        const uint64_t l = probes[p];
        for (uint64_t e = offsets[l]; e < offsets[l + 1]; ++e) {
            if (!in_sorted(subset, nsub, list_ids[e])) continue;
            double dist;
            rc = orc_adc_lookup(table, M, ks, list_codes + e * rb, 0, &dist);
            if (rc) break;
            if (has_max && dist > max_sq_dist) continue;
            hits[nh].id = list_ids[e];
            hits[nh].d = dist;
            ++nh;
        }
    }
    int64_t cnt = rc ? rc : (int64_t)finalize(hits, nh, k, out_ids, out_d);
    free(hits);
    free(table);
    free(probes);
    return cnt;
}
