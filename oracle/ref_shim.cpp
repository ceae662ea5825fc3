// ref_shim.cpp -- extern "C" entry points over the REFERENCE's own C++ code.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together with
// the reference sources where they lie (/root/reference/proj/src/*.cpp) into
// oracle/_ref/libpqii_ref.so.  Nothing here restates an algorithm: every
// function forwards to the reference implementation so the tests, the golden
// generator (tests/golden/make_golden.py) and bench.py's reference arm can
// run the reference on plain arrays.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <mutex>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "pqii/dataset_io.hpp"
#include "pqii/ivf.hpp"
#include "pqii/kmeans.hpp"
#include "pqii/pipeline.hpp"
#include "pqii/pq.hpp"

using namespace pqii;

namespace {

VectorMatrix as_matrix(const float* p, std::uint64_t n, std::uint64_t d) {
    VectorMatrix m(n, d);
    if (n * d) std::memcpy(m.values.data(), p, n * d * sizeof(float));
    return m;
}

Codebook as_codebook(const float* tables, std::uint32_t M, std::uint32_t ks, std::uint32_t ds) {
    Codebook cb;
    cb.m_subspaces = M;
    cb.ks = ks;
    cb.sub_dim = ds;
    cb.tables.assign(tables, tables + std::size_t(M) * ks * ds);
    return cb;
}

CodeMatrix as_codes(const std::uint8_t* bytes, std::uint64_t n, std::uint32_t M, std::uint32_t ks) {
    CodeMatrix c(n, M, ks);
    if (!c.bytes.empty()) std::memcpy(c.bytes.data(), bytes, c.bytes.size());
    return c;
}

// 0 ok, -1 invalid_argument, -2 out_of_range, -4 other
template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    } catch (const std::out_of_range&) {
        return -2;
    } catch (...) {
        return -4;
    }
}

struct RefIndex {
    InvertedIndex index;
};

}  // namespace

extern "C" {

int ref_random_matrix(std::uint64_t rows, std::uint64_t dims, std::uint64_t seed, float lo,
                      float hi, float* out) {
    // proj/tests/test_helpers.cpp:26-33 restated through the same libstdc++.
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<float> dist(lo, hi);
    for (std::uint64_t i = 0; i < rows * dims; ++i) out[i] = dist(rng);
    return 0;
}

int ref_uniform_indices(std::uint64_t seed, std::uint64_t n, std::uint64_t k, std::uint64_t* out) {
    // The exact draw sequence of kmeans_fit's init (proj/src/kmeans.cpp:74-80).
    std::mt19937_64 rng(seed);
    for (std::uint64_t i = 0; i < k; ++i) {
        std::uniform_int_distribution<std::size_t> pick(i, n - 1);
        out[i] = pick(rng);
    }
    return 0;
}

int ref_nearest_batch(const float* points, std::uint64_t n, std::uint64_t d, const float* table,
                      std::uint64_t k, std::uint32_t* index, double* sq_dist) {
    return guarded([&] {
        for (std::uint64_t i = 0; i < n; ++i) {
            const auto nc = nearest_in_table(points + i * d, table, k, d);
            index[i] = static_cast<std::uint32_t>(nc.index);
            sq_dist[i] = nc.sq_dist;
        }
    });
}

int ref_kmeans_fit(const float* points, std::uint64_t n, std::uint64_t d, std::uint64_t k,
                   std::uint32_t max_iters, std::uint64_t seed, double tol, float* centroids,
                   std::uint32_t* assignments, double* inertia, std::uint32_t* iterations_run,
                   double* inertia_per_iter) {
    return guarded([&] {
        const KMeansResult r = kmeans_fit(as_matrix(points, n, d), k, max_iters, seed, tol);
        std::memcpy(centroids, r.centroids.values.data(), k * d * sizeof(float));
        std::memcpy(assignments, r.assignments.data(), n * sizeof(std::uint32_t));
        *inertia = r.inertia;
        *iterations_run = r.iterations_run;
        if (inertia_per_iter)
            std::copy(r.inertia_per_iter.begin(), r.inertia_per_iter.end(), inertia_per_iter);
    });
}

int ref_pq_fit(const float* data, std::uint64_t n, std::uint64_t D, std::uint32_t M,
               std::uint32_t ks, std::uint32_t max_iters, std::uint64_t seed, float* tables) {
    return guarded([&] {
        const Codebook cb = pq_fit(as_matrix(data, n, D), M, ks, max_iters, seed);
        std::memcpy(tables, cb.tables.data(), cb.tables.size() * sizeof(float));
    });
}

// pq_fit with the subspaces fitted on `threads` threads (kmeans_fit is safe for
// concurrent disjoint fits, proj/include/pqii/kmeans.hpp:40); bit-identical to
// pq_fit because each subspace is an independent fit with seed + m.
int ref_pq_fit_threads(const float* data, std::uint64_t n, std::uint64_t D, std::uint32_t M,
                       std::uint32_t ks, std::uint32_t max_iters, std::uint64_t seed,
                       float* tables, int threads) {
    return guarded([&] {
        const std::uint64_t ds = D / M;
        std::vector<std::thread> pool;
        std::vector<int> err(M, 0);
        std::uint32_t next = 0;
        std::mutex mu;
        auto work = [&] {
            for (;;) {
                std::uint32_t m;
                {
                    std::lock_guard<std::mutex> g(mu);
                    if (next >= M) return;
                    m = next++;
                }
                VectorMatrix slice(n, ds);
                for (std::uint64_t i = 0; i < n; ++i)
                    std::memcpy(slice.row(i), data + i * D + m * ds, ds * sizeof(float));
                try {
                    const KMeansResult km = kmeans_fit(slice, ks, max_iters, seed + m);
                    std::memcpy(tables + std::size_t(m) * ks * ds, km.centroids.values.data(),
                                std::size_t(ks) * ds * sizeof(float));
                } catch (...) {
                    err[m] = 1;
                }
            }
        };
        for (int t = 0; t < std::max(1, threads); ++t) pool.emplace_back(work);
        for (auto& t : pool) t.join();
        for (int e : err)
            if (e) throw std::invalid_argument("pq_fit failed");
    });
}

int ref_pq_encode(const float* data, std::uint64_t n, std::uint32_t M, std::uint32_t ks,
                  std::uint32_t ds, const float* tables, std::uint8_t* codes) {
    return guarded([&] {
        const CodeMatrix c =
            pq_encode(as_codebook(tables, M, ks, ds), as_matrix(data, n, std::uint64_t(M) * ds));
        std::memcpy(codes, c.bytes.data(), c.bytes.size());
    });
}

// pq_encode over chunk_rows(n, threads) ranges on `threads` threads -- the
// reference's own chunk-parallel encode (proj/src/pipeline.cpp:226-231).
int ref_pq_encode_threads(const float* data, std::uint64_t n, std::uint32_t M, std::uint32_t ks,
                          std::uint32_t ds, const float* tables, std::uint8_t* codes,
                          int threads) {
    return guarded([&] {
        const Codebook cb = as_codebook(tables, M, ks, ds);
        const std::uint64_t D = std::uint64_t(M) * ds;
        const auto ranges = chunk_rows(n, std::min<std::uint64_t>(n, std::max(1, threads)));
        const std::size_t rb = std::size_t(M) * (ks <= 256 ? 1 : 2);
        std::vector<std::thread> pool;
        for (const RowRange r : ranges) {
            pool.emplace_back([&, r] {
                VectorMatrix part(r.size(), D);
                std::memcpy(part.values.data(), data + r.begin * D, r.size() * D * sizeof(float));
                const CodeMatrix c = pq_encode(cb, part);
                std::memcpy(codes + r.begin * rb, c.bytes.data(), c.bytes.size());
            });
        }
        for (auto& t : pool) t.join();
    });
}

int ref_pq_decode(const std::uint8_t* codes, std::uint64_t n, std::uint32_t M, std::uint32_t ks,
                  std::uint32_t ds, const float* tables, float* out) {
    return guarded([&] {
        const VectorMatrix v = pq_decode(as_codebook(tables, M, ks, ds), as_codes(codes, n, M, ks));
        std::memcpy(out, v.values.data(), v.values.size() * sizeof(float));
    });
}

int ref_rmse(const float* a, const float* b, std::uint64_t rows, std::uint64_t dims, double* out) {
    return guarded([&] { *out = rmse(as_matrix(a, rows, dims), as_matrix(b, rows, dims)); });
}

int ref_reconstruction_rmse(const float* data, std::uint64_t n, std::uint32_t M, std::uint32_t ks,
                            std::uint32_t ds, const float* tables, double* out) {
    return guarded([&] {
        *out = reconstruction_rmse(as_codebook(tables, M, ks, ds),
                                   as_matrix(data, n, std::uint64_t(M) * ds));
    });
}

int ref_adc_table(const float* tables, std::uint32_t M, std::uint32_t ks, std::uint32_t ds,
                  const float* query, float* entries) {
    return guarded([&] {
        const DistanceTable t = adc_table(as_codebook(tables, M, ks, ds),
                                          std::span<const float>(query, std::size_t(M) * ds));
        std::memcpy(entries, t.entries.data(), t.entries.size() * sizeof(float));
    });
}

int ref_adc_lookup_all(const float* entries, std::uint32_t M, std::uint32_t ks,
                       const std::uint8_t* codes, std::uint64_t n, double* out) {
    return guarded([&] {
        DistanceTable t;
        t.m_subspaces = M;
        t.ks = ks;
        t.entries.assign(entries, entries + std::size_t(M) * ks);
        const CodeMatrix c = as_codes(codes, n, M, ks);
        for (std::uint64_t i = 0; i < n; ++i) out[i] = adc_lookup(t, c, i);
    });
}

// ivf_build_with_centroids (proj/src/ivf.cpp:151-166) returned as a handle.
void* ref_ivf_build_with_centroids(const float* tables, std::uint32_t M, std::uint32_t ks,
                                   std::uint32_t ds, const std::uint8_t* codes,
                                   const std::uint64_t* ids, std::uint64_t n,
                                   const float* coarse, std::uint64_t nlist, int* status) {
    RefIndex* h = nullptr;
    *status = guarded([&] {
        auto idx = ivf_build_with_centroids(as_codebook(tables, M, ks, ds),
                                            as_codes(codes, n, M, ks),
                                            std::span<const std::uint64_t>(ids, n),
                                            as_matrix(coarse, nlist, std::uint64_t(M) * ds));
        h = new RefIndex{std::move(idx)};
    });
    return h;
}

// ivf_build (proj/src/ivf.cpp:123-149): coarse k-means over decoded codes.
void* ref_ivf_build(const float* tables, std::uint32_t M, std::uint32_t ks, std::uint32_t ds,
                    const std::uint8_t* codes, const std::uint64_t* ids, std::uint64_t n,
                    std::uint64_t nlist, std::uint64_t seed, std::uint32_t iters, int* status) {
    RefIndex* h = nullptr;
    *status = guarded([&] {
        auto idx = ivf_build(as_codebook(tables, M, ks, ds), as_codes(codes, n, M, ks),
                             std::span<const std::uint64_t>(ids, n), nlist, seed, iters);
        h = new RefIndex{std::move(idx)};
    });
    return h;
}

void ref_ivf_free(void* h) { delete static_cast<RefIndex*>(h); }

std::uint64_t ref_ivf_nlist(void* h) { return static_cast<RefIndex*>(h)->index.nlist(); }

std::uint64_t ref_ivf_n_items(void* h) { return static_cast<RefIndex*>(h)->index.n_items; }

// Copies the index out as CSR: offsets[nlist+1], ids[n], codes[n*row_bytes];
// coarse (nlist*D) optional.
int ref_ivf_export(void* h, std::uint64_t* offsets, std::uint64_t* ids, std::uint8_t* codes,
                   float* coarse) {
    const InvertedIndex& idx = static_cast<RefIndex*>(h)->index;
    std::uint64_t off = 0;
    offsets[0] = 0;
    for (std::size_t l = 0; l < idx.lists.size(); ++l) {
        const PostingList& pl = idx.lists[l];
        const std::size_t rb = pl.codes.row_bytes();
        for (std::size_t i = 0; i < pl.ids.size(); ++i) {
            ids[off + i] = pl.ids[i];
            std::memcpy(codes + (off + i) * rb, pl.codes.bytes.data() + i * rb, rb);
        }
        off += pl.ids.size();
        offsets[l + 1] = off;
    }
    if (coarse)
        std::memcpy(coarse, idx.coarse_centroids.values.data(),
                    idx.coarse_centroids.values.size() * sizeof(float));
    return 0;
}

// ivf_add (proj/src/ivf.cpp:168-184)
int ref_ivf_add(void* h, const std::uint8_t* codes, const std::uint64_t* ids, std::uint64_t n) {
    InvertedIndex& idx = static_cast<RefIndex*>(h)->index;
    return guarded([&] {
        ivf_add(idx, as_codes(codes, n, idx.codebook.m_subspaces, idx.codebook.ks),
                std::span<const std::uint64_t>(ids, n));
    });
}

// ivf_merge (proj/src/ivf.cpp:186-216)
void* ref_ivf_merge(void* a, void* b, int* status) {
    RefIndex* h = nullptr;
    *status = guarded([&] {
        auto idx = ivf_merge(static_cast<RefIndex*>(a)->index, static_cast<RefIndex*>(b)->index);
        h = new RefIndex{std::move(idx)};
    });
    return h;
}

// ivf_query (proj/src/ivf.cpp:218-228) over nq queries on `threads` threads
// (a frozen index is reader-safe, proj/include/pqii/ivf.hpp:20-22).
// Row q of out_ids/out_dists holds counts[q] <= k hits.
int ref_ivf_query_batch(void* h, const float* queries, std::uint64_t nq, std::uint64_t k,
                        std::uint64_t nprobe, int has_max, double max_sq_dist,
                        std::uint64_t* out_ids, double* out_dists, std::uint32_t* counts,
                        int threads) {
    const InvertedIndex& idx = static_cast<RefIndex*>(h)->index;
    const std::size_t D = idx.codebook.dims();
    std::vector<int> rc(std::max(1, threads), 0);
    auto run = [&](int t, std::uint64_t b, std::uint64_t e) {
        rc[t] = guarded([&] {
            for (std::uint64_t q = b; q < e; ++q) {
                const auto r = ivf_query(idx, std::span<const float>(queries + q * D, D), k,
                                         nprobe,
                                         has_max ? std::optional<double>(max_sq_dist)
                                                 : std::nullopt);
                counts[q] = static_cast<std::uint32_t>(r.hits.size());
                for (std::size_t j = 0; j < r.hits.size(); ++j) {
                    out_ids[q * k + j] = r.hits[j].id;
                    out_dists[q * k + j] = r.hits[j].sq_dist;
                }
            }
        });
    };
    const int T = std::max(1, std::min<int>(threads, int(std::max<std::uint64_t>(1, nq))));
    std::vector<std::thread> pool;
    for (int t = 0; t < T; ++t) {
        const std::uint64_t b = nq * t / T, e = nq * (t + 1) / T;
        pool.emplace_back(run, t, b, e);
    }
    for (auto& t : pool) t.join();
    for (int r : rc)
        if (r) return r;
    return 0;
}

int ref_ivf_query_subset(void* h, const float* query, std::uint64_t k, const std::uint64_t* subset,
                         std::uint64_t nsub, std::uint64_t nprobe, int has_max,
                         double max_sq_dist, std::uint64_t* out_ids, double* out_dists,
                         std::uint32_t* count) {
    const InvertedIndex& idx = static_cast<RefIndex*>(h)->index;
    const std::size_t D = idx.codebook.dims();
    return guarded([&] {
        const auto r = ivf_query_subset(
            idx, std::span<const float>(query, D), k, std::span<const std::uint64_t>(subset, nsub),
            nprobe, has_max ? std::optional<double>(max_sq_dist) : std::nullopt);
        *count = static_cast<std::uint32_t>(r.hits.size());
        for (std::size_t j = 0; j < r.hits.size(); ++j) {
            out_ids[j] = r.hits[j].id;
            out_dists[j] = r.hits[j].sq_dist;
        }
    });
}

int ref_flat_scan(const float* tables, std::uint32_t M, std::uint32_t ks, std::uint32_t ds,
                  const std::uint8_t* codes, const std::uint64_t* ids, std::uint64_t n,
                  const float* query, std::uint64_t k, int has_max, double max_sq_dist,
                  std::uint64_t* out_ids, double* out_dists, std::uint32_t* count) {
    return guarded([&] {
        const auto r = flat_scan(as_codebook(tables, M, ks, ds), as_codes(codes, n, M, ks),
                                 std::span<const std::uint64_t>(ids, n),
                                 std::span<const float>(query, std::size_t(M) * ds), k,
                                 has_max ? std::optional<double>(max_sq_dist) : std::nullopt);
        *count = static_cast<std::uint32_t>(r.hits.size());
        for (std::size_t j = 0; j < r.hits.size(); ++j) {
            out_ids[j] = r.hits[j].id;
            out_dists[j] = r.hits[j].sq_dist;
        }
    });
}

std::uint64_t ref_default_nlist(std::uint64_t n) { return default_nlist(n); }

int ref_chunk_rows(std::uint64_t n, std::uint64_t c, std::uint64_t* bounds) {
    return guarded([&] {
        const auto r = chunk_rows(n, c);
        bounds[0] = 0;
        for (std::size_t i = 0; i < r.size(); ++i) bounds[i + 1] = r[i].end;
    });
}

unsigned ref_hardware_concurrency() { return std::thread::hardware_concurrency(); }

// train_chunk (proj/src/pipeline.cpp:84-106) on one chunk of rows.
int ref_train_chunk(const float* chunk, std::uint64_t n, std::uint64_t D, std::uint32_t M,
                    std::uint32_t ks, std::uint32_t iters, std::uint64_t chunk_seed, float* reps,
                    double* local_rmse) {
    return guarded([&] {
        const ChunkOutput out = train_chunk(as_matrix(chunk, n, D), M, ks, iters, chunk_seed);
        std::memcpy(reps, out.representatives.values.data(),
                    out.representatives.values.size() * sizeof(float));
        *local_rmse = out.local_rmse;
    });
}

// run_pipeline (proj/src/pipeline.cpp:142-266).  reps: n_chunks*ks*D (parallel
// modes, nullable); index: the merged index as a RefIndex handle (index mode,
// nullable); phases: fit, chunking, local_fit, global_fit, coarse_fit, encode,
// index_build, merge seconds (-1 when absent), total last (9 entries).
int ref_run_pipeline(const float* data, std::uint64_t n, std::uint64_t D, std::uint64_t n_chunks,
                     std::uint32_t M, std::uint32_t ks, std::uint64_t nlist, std::uint32_t iters,
                     std::uint64_t seed, std::uint64_t threads, int mode, float* tables,
                     double* global_rmse, float* reps, std::uint64_t* nlist_used, void** index,
                     double* phases, char* err, std::uint64_t err_len) {
    int rc = -4;
    std::string msg;
    try {
        PipelineConfig cfg;
        cfg.n_chunks = n_chunks;
        cfg.m_subspaces = M;
        cfg.ks = ks;
        cfg.nlist = nlist;
        cfg.kmeans_iters = iters;
        cfg.seed = seed;
        cfg.n_threads = threads;
        cfg.mode = mode == 0 ? PipelineMode::kSingle
                             : (mode == 1 ? PipelineMode::kParallelPq : PipelineMode::kParallelPqIndex);
        PipelineReport r = run_pipeline(as_matrix(data, n, D), cfg);
        std::memcpy(tables, r.global_codebook.tables.data(),
                    r.global_codebook.tables.size() * sizeof(float));
        *global_rmse = r.global_rmse;
        if (nlist_used) *nlist_used = r.config.nlist;
        if (reps && r.representatives)
            std::memcpy(reps, r.representatives->values.data(),
                        r.representatives->values.size() * sizeof(float));
        if (index) *index = r.merged_index ? new RefIndex{std::move(*r.merged_index)} : nullptr;
        if (phases) {
            const char* names[8] = {"fit", "chunking", "local_fit", "global_fit",
                                    "coarse_fit", "encode", "index_build", "merge"};
            for (int i = 0; i < 8; ++i) {
                auto it = r.phase_seconds.find(names[i]);
                phases[i] = it == r.phase_seconds.end() ? -1.0 : it->second;
            }
            phases[8] = r.total_seconds;
        }
        rc = 0;
    } catch (const std::invalid_argument& e) {
        rc = -1;
        msg = e.what();
    } catch (const std::out_of_range& e) {
        rc = -2;
        msg = e.what();
    } catch (const std::exception& e) {
        rc = -4;
        msg = e.what();
    }
    if (err && err_len) {
        std::strncpy(err, msg.c_str(), err_len - 1);
        err[err_len - 1] = 0;
    }
    return rc;
}


}  // extern "C"

// ---- on-disk formats: the reference's own writers / readers
// (proj/src/pq.cpp:183-259, ivf.cpp:264-355).  The exception message of a
// failed call is kept for ref_last_message().
namespace {
thread_local std::string g_msg;
thread_local CodeMatrix g_codes;
thread_local Codebook g_cb;
template <class F>
int guarded_msg(F&& f) {
    try {
        f();
        g_msg.clear();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_msg = e.what();
        return -1;
    } catch (const std::out_of_range& e) {
        g_msg = e.what();
        return -2;
    } catch (const std::exception& e) {
        g_msg = e.what();
        return -4;
    }
}
}  // namespace

extern "C" {

const char* ref_last_message() { return g_msg.c_str(); }

int ref_save_index(void* h, const char* path) {
    return guarded_msg([&] { save_index(static_cast<RefIndex*>(h)->index, path); });
}

void* ref_load_index(const char* path, int* status) {
    RefIndex* h = nullptr;
    *status = guarded_msg([&] { h = new RefIndex{load_index(path)}; });
    return h;
}

int ref_save_codes(const std::uint8_t* codes, std::uint64_t n, std::uint32_t M, std::uint32_t ks, const char* path) {
    return guarded_msg([&] { save_codes(as_codes(codes, n, M, ks), path); });
}

// loads into a thread-local CodeMatrix; out (cap bytes) may be null to query the shape
int ref_load_codes(const char* path, std::uint64_t* n, std::uint32_t* M, std::uint32_t* ks, std::uint8_t* out,
                   std::uint64_t cap) {
    return guarded_msg([&] {
        g_codes = load_codes(path);
        *n = g_codes.rows;
        *M = g_codes.m_subspaces;
        *ks = g_codes.ks;
        if (out && cap >= g_codes.bytes.size()) std::memcpy(out, g_codes.bytes.data(), g_codes.bytes.size());
    });
}

int ref_save_codebook(const float* tables, std::uint32_t M, std::uint32_t ks, std::uint32_t ds, const char* path) {
    return guarded_msg([&] { save_codebook(as_codebook(tables, M, ks, ds), path); });
}

int ref_load_codebook(const char* path, std::uint32_t* M, std::uint32_t* ks, std::uint32_t* ds, float* out,
                      std::uint64_t cap) {
    return guarded_msg([&] {
        g_cb = load_codebook(path);
        *M = g_cb.m_subspaces;
        *ks = g_cb.ks;
        *ds = g_cb.sub_dim;
        if (out && cap >= g_cb.tables.size()) std::memcpy(out, g_cb.tables.data(), g_cb.tables.size() * 4);
    });
}

}  // extern "C"
