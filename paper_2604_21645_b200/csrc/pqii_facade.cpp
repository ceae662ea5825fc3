// pqii_facade.cpp -- the reference's C++ API (namespace pqii) implemented
// over the C ABI of libpqg.so, so unchanged reference callers (pipeline,
// bench, CLI, tests: /root/reference/proj/src/pipeline.cpp:84-266,
// proj/tests/*) link against libpqg_pqii.so instead of libpqii.a.
//
// Every numeric result comes from the device (include/pqg.h); this file only
// validates with the reference's messages, marshals the reference's structs
// and maintains the host-side data structures the API returns by value
// (posting-list vectors, id_set).  One pqg context per calling thread keeps
// the API re-entrant as run_pipeline requires (SURVEY.md 8(b) Threading).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iomanip>
#include <sstream>
#include <list>
#include <memory>
#include <optional>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>

#include "pqg.h"
#include "pqii/ivf.hpp"
#include "pqii/kmeans.hpp"
#include "pqii/matrix.hpp"
#include "pqii/pipeline.hpp"
#include "pqii/pq.hpp"

namespace pqii {

namespace {

// ---------------------------------------------------------------------------
// context and error mapping
// ---------------------------------------------------------------------------
int device_index() {
    const char* e = std::getenv("PQG_DEVICE");
    return e ? std::atoi(e) : 0;
}

void raise(int rc) {
    if (rc == PQG_OK) return;
    const std::string msg = pqg_last_error();
    if (rc == PQG_EINVAL) throw std::invalid_argument(msg);
    if (rc == PQG_ERANGE) throw std::out_of_range(msg);
    throw std::runtime_error(msg);
}

struct CtxHolder {
    pqg_ctx* c = nullptr;
    ~CtxHolder() {
        if (c) pqg_ctx_destroy(c);
    }
};

pqg_ctx* ctx() {
    thread_local CtxHolder h;
    if (!h.c) raise(pqg_ctx_create(device_index(), &h.c));
    return h.c;
}

// ---------------------------------------------------------------------------
// device-index cache for repeated queries on the same (unmodified) index.
// Pointer identity is never trusted: a freed index's blocks are reused by
// malloc for the next one of the same shape, and the reference's structs have
// public fields that callers may edit in place.
// ---------------------------------------------------------------------------
// r2e: each cache entry keeps a host copy of what it uploaded (the CSR the
// upload packs anyway) and reuse is decided by EXACT comparison -- no hash,
// no collision.  The head (header, codebook, coarse centroids, list sizes)
// is compared on every call; the lists only where the call reads them: a
// query batch that probes fewer than half the lists runs on the cached copy,
// gets its probe lists back (pqg_index_search_ex) and compares just those
// lists -- a list the batch does not probe cannot change its result -- and
// re-uploads and re-runs if one differs.  A single ivf_query therefore reads
// ~the head plus nprobe lists of host memory, not the whole index (r2 hashed
// every list: 4.2 ms per call at 1M items; tools/facade_latency.cpp).
struct IndexDeleter {
    void operator()(pqg_index* p) const { pqg_index_destroy(p); }
};
using IndexPtr = std::shared_ptr<pqg_index>;

struct HostCopy {  // what the device copy was built from
    std::uint64_t hdr[4];
    std::vector<float> tables, coarse;
    std::vector<std::uint64_t> offsets, ids;
    std::vector<std::uint8_t> codes;
    std::size_t rb = 0;
};

struct CacheEntry {
    std::shared_ptr<const HostCopy> host;
    IndexPtr dev;
};
std::mutex g_cache_mu;
std::list<CacheEntry> g_cache;  // most recent first

bool head_equal(const HostCopy& h, const InvertedIndex& ix) {
    const std::uint64_t hdr[4] = {ix.lists.size(), ix.n_items, ix.codebook.m_subspaces, ix.codebook.ks};
    if (std::memcmp(hdr, h.hdr, sizeof(hdr)) != 0) return false;
    if (ix.codebook.tables.size() != h.tables.size() || ix.coarse_centroids.values.size() != h.coarse.size())
        return false;
    for (std::size_t l = 0; l < ix.lists.size(); ++l)
        if (ix.lists[l].ids.size() != h.offsets[l + 1] - h.offsets[l] ||
            ix.lists[l].codes.bytes.size() != ix.lists[l].ids.size() * h.rb)
            return false;
    return std::memcmp(ix.codebook.tables.data(), h.tables.data(), h.tables.size() * sizeof(float)) == 0 &&
           std::memcmp(ix.coarse_centroids.values.data(), h.coarse.data(), h.coarse.size() * sizeof(float)) == 0;
}

bool list_equal(const HostCopy& h, const InvertedIndex& ix, std::size_t l) {
    const PostingList& pl = ix.lists[l];
    const std::size_t a = h.offsets[l], n = h.offsets[l + 1] - a;
    return std::memcmp(pl.ids.data(), h.ids.data() + a, n * sizeof(std::uint64_t)) == 0 &&
           std::memcmp(pl.codes.bytes.data(), h.codes.data() + a * h.rb, n * h.rb) == 0;
}

CacheEntry upload(const InvertedIndex& ix) {
    auto h = std::make_shared<HostCopy>();
    const std::size_t nlist = ix.lists.size();
    h->rb = ix.codebook.m_subspaces * (ix.codebook.ks <= 256 ? 1 : 2);
    h->hdr[0] = nlist;
    h->hdr[1] = ix.n_items;
    h->hdr[2] = ix.codebook.m_subspaces;
    h->hdr[3] = ix.codebook.ks;
    h->tables = ix.codebook.tables;
    h->coarse = ix.coarse_centroids.values;
    h->offsets.assign(nlist + 1, 0);
    for (std::size_t l = 0; l < nlist; ++l) {
        if (ix.lists[l].codes.bytes.size() != ix.lists[l].ids.size() * h->rb)
            throw std::invalid_argument("index: posting list ids and codes differ in length");
        h->offsets[l + 1] = h->offsets[l] + ix.lists[l].ids.size();
    }
    h->ids.reserve(h->offsets[nlist]);
    h->codes.reserve(h->offsets[nlist] * h->rb);
    for (const auto& pl : ix.lists) {
        h->ids.insert(h->ids.end(), pl.ids.begin(), pl.ids.end());
        h->codes.insert(h->codes.end(), pl.codes.bytes.begin(), pl.codes.bytes.end());
    }
    pqg_index* d = nullptr;
    raise(pqg_index_create(ctx(), ix.codebook.tables.data(), ix.codebook.m_subspaces,
                           ix.codebook.ks, ix.codebook.sub_dim, ix.coarse_centroids.values.data(),
                           nlist, h->offsets.data(), h->ids.data(), h->codes.data(), &d));
    return CacheEntry{h, IndexPtr(d, IndexDeleter())};
}

CacheEntry cache_insert(const InvertedIndex& ix) {
    CacheEntry e = upload(ix);
    std::lock_guard<std::mutex> g(g_cache_mu);
    g_cache.push_front(e);
    while (g_cache.size() > 8) g_cache.pop_back();
    return e;
}

// A cached entry whose head equals ix's (lists not yet compared), or none.
std::optional<CacheEntry> cache_find(const InvertedIndex& ix) {
    std::lock_guard<std::mutex> g(g_cache_mu);
    for (auto it = g_cache.begin(); it != g_cache.end(); ++it) {
        if (head_equal(*it->host, ix)) {
            g_cache.splice(g_cache.begin(), g_cache, it);
            return g_cache.front();
        }
    }
    return std::nullopt;
}

void cache_drop(const CacheEntry& e) {
    std::lock_guard<std::mutex> g(g_cache_mu);
    g_cache.remove_if([&](const CacheEntry& x) { return x.dev == e.dev; });
}

// The device copy of ix, every list compared (merge, save, batches that
// probe most lists).
IndexPtr device_index_for(const InvertedIndex& ix) {
    if (auto e = cache_find(ix)) {
        bool ok = true;
        for (std::size_t l = 0; l < ix.lists.size() && ok; ++l) ok = list_equal(*e->host, ix, l);
        if (ok) return e->dev;
        cache_drop(*e);
    }
    return cache_insert(ix).dev;
}

// Build the reference's host structure from a device index (CSR export).
InvertedIndex to_host(pqg_index* h, const Codebook& cb) {
    std::uint64_t nlist = 0, n = 0;
    std::uint32_t M = 0, ks = 0, ds = 0;
    raise(pqg_index_info(h, &nlist, &n, &M, &ks, &ds));
    const std::size_t rb = std::size_t(M) * (ks <= 256 ? 1 : 2);
    std::vector<std::uint64_t> offsets(nlist + 1), ids(std::max<std::uint64_t>(n, 1));
    std::vector<std::uint8_t> codes(std::max<std::uint64_t>(n, 1) * rb);
    InvertedIndex ix;
    ix.codebook = cb;
    ix.coarse_centroids = VectorMatrix(nlist, std::size_t(M) * ds);
    raise(pqg_index_export(ctx(), h, offsets.data(), ids.data(), codes.data(),
                           ix.coarse_centroids.values.data(), nullptr));
    ix.lists.resize(nlist);
    for (std::size_t l = 0; l < nlist; ++l) {
        PostingList& pl = ix.lists[l];
        const std::size_t a = offsets[l], b = offsets[l + 1];
        pl.ids.assign(ids.begin() + a, ids.begin() + b);
        pl.codes = CodeMatrix(0, M, ks);
        pl.codes.bytes.assign(codes.begin() + a * rb, codes.begin() + b * rb);
        pl.codes.rows = b - a;
    }
    ix.n_items = n;
    ix.id_set.reserve(n);
    ix.id_set.insert(ids.begin(), ids.begin() + n);
    return ix;
}

void check_codebook_params(std::uint32_t m, std::uint32_t ks, std::uint32_t sub_dim) {
    if (m == 0) throw std::invalid_argument("codebook: M must be >= 1");
    if (ks == 0 || ks > 65536) throw std::invalid_argument("codebook: Ks must be in [1, 65536]");
    if (sub_dim == 0) throw std::invalid_argument("codebook: sub_dim must be >= 1");
}

void check_codes_match(const Codebook& cb, const CodeMatrix& codes, const char* who) {
    if (codes.m_subspaces != cb.m_subspaces || codes.ks != cb.ks)
        throw std::invalid_argument(std::string(who) + ": codes do not match the codebook");
}

void check_query(const InvertedIndex& index, std::span<const float> query, std::size_t k,
                 std::size_t nprobe) {
    if (k == 0) throw std::invalid_argument("query: k must be >= 1");
    if (query.size() != index.codebook.dims()) throw std::invalid_argument("query: dimension mismatch");
    if (nprobe == 0 || nprobe > index.nlist())
        throw std::invalid_argument("query: nprobe (" + std::to_string(nprobe) +
                                    ") must be in [1, nlist=" + std::to_string(index.nlist()) + "]");
}

QueryResult result_of(const std::uint64_t* ids, const double* d, std::uint32_t cnt, std::size_t k) {
    QueryResult r;
    r.k_requested = k;
    r.hits.reserve(cnt);
    for (std::uint32_t j = 0; j < cnt; ++j) r.hits.push_back({ids[j], d[j]});
    return r;
}

}  // namespace

// ===========================================================================
// matrix.hpp
// ===========================================================================
VectorMatrix slice_rows(const VectorMatrix& m, RowRange r) {
    if (r.begin >= r.end || r.end > m.rows) throw std::invalid_argument("slice_rows: range out of bounds");
    VectorMatrix out(r.size(), m.dims);
    std::memcpy(out.values.data(), m.row(r.begin), r.size() * m.dims * sizeof(float));
    return out;
}

// ===========================================================================
// kmeans.hpp
// ===========================================================================
NearestCentroid nearest_in_table(const float* point, const float* table, std::size_t k,
                                 std::size_t d) {
    if (d == 0) return {0, 0.0};
    std::uint32_t idx = 0;
    double dist = 0.0;
    raise(pqg_nearest_batch(ctx(), point, 1, d, table, k, &idx, &dist));
    return {idx, dist};
}

double squared_l2(const float* a, const float* b, std::size_t d) {
    return nearest_in_table(a, b, 1, d).sq_dist;
}

NearestCentroid nearest_centroid(std::span<const float> point, const VectorMatrix& centroids) {
    if (centroids.rows == 0) throw std::invalid_argument("nearest_centroid: empty centroid set");
    if (point.size() != centroids.dims) throw std::invalid_argument("nearest_centroid: dimension mismatch");
    return nearest_in_table(point.data(), centroids.values.data(), centroids.rows, centroids.dims);
}

KMeansResult kmeans_fit(const VectorMatrix& points, std::size_t k, std::uint32_t max_iters,
                        std::uint64_t seed, double tol) {
    KMeansResult r;
    r.centroids = VectorMatrix(k <= points.rows ? k : 0, points.dims);
    r.assignments.resize(points.rows);
    r.inertia_per_iter.resize(std::max<std::uint32_t>(max_iters, 1));
    raise(pqg_kmeans_fit(ctx(), points.values.data(), points.rows, points.dims, k, max_iters, seed,
                         tol, r.centroids.values.data(), r.assignments.data(), &r.inertia,
                         &r.iterations_run, r.inertia_per_iter.data()));
    r.inertia_per_iter.resize(r.iterations_run);
    return r;
}

// ===========================================================================
// pq.hpp
// ===========================================================================
CodeMatrix::CodeMatrix(std::size_t n, std::uint32_t m, std::uint32_t ks_)
    : rows(n), m_subspaces(m), ks(ks_) {
    check_codebook_params(m, ks_, 1);
    bytes.assign(n * row_bytes(), 0);
}

std::uint32_t CodeMatrix::at(std::size_t i, std::size_t m) const {
    const std::size_t off = i * row_bytes() + m * code_width();
    return code_width() == 1 ? bytes[off] : (std::uint32_t(bytes[off]) | std::uint32_t(bytes[off + 1]) << 8);
}

void CodeMatrix::set(std::size_t i, std::size_t m, std::uint32_t value) {
    const std::size_t off = i * row_bytes() + m * code_width();
    bytes[off] = std::uint8_t(value & 0xff);
    if (code_width() == 2) bytes[off + 1] = std::uint8_t(value >> 8);
}

void CodeMatrix::append_row_from(const CodeMatrix& src, std::size_t src_row) {
    if (src.m_subspaces != m_subspaces || src.ks != ks)
        throw std::invalid_argument("CodeMatrix: shape mismatch on append");
    const std::size_t rb = row_bytes();
    const std::uint8_t* p = src.bytes.data() + src_row * rb;
    bytes.insert(bytes.end(), p, p + rb);
    ++rows;
}

Codebook pq_fit(const VectorMatrix& data, std::uint32_t m, std::uint32_t ks,
                std::uint32_t max_iters, std::uint64_t seed) {
    Codebook cb;
    cb.m_subspaces = m;
    cb.ks = ks;
    cb.sub_dim = m ? std::uint32_t(data.dims / m) : 0;
    cb.tables.resize(std::size_t(m) * ks * cb.sub_dim);
    raise(pqg_pq_fit(ctx(), data.values.data(), data.rows, data.dims, m, ks, max_iters, seed,
                     cb.tables.data(), nullptr, nullptr));
    return cb;
}

CodeMatrix pq_encode(const Codebook& cb, const VectorMatrix& data) {
    if (data.dims != cb.dims())
        throw std::invalid_argument("pq_encode: data dimension " + std::to_string(data.dims) +
                                    " does not match codebook dimension " + std::to_string(cb.dims()));
    CodeMatrix codes(data.rows, cb.m_subspaces, cb.ks);
    raise(pqg_pq_encode(ctx(), data.values.data(), data.rows, cb.m_subspaces, cb.ks, cb.sub_dim,
                        cb.tables.data(), codes.bytes.data()));
    return codes;
}

void pq_decode_row(const Codebook& cb, const CodeMatrix& codes, std::size_t i, float* out) {
    raise(pqg_pq_decode(ctx(), codes.bytes.data() + i * codes.row_bytes(), 1, cb.m_subspaces, cb.ks,
                        cb.sub_dim, cb.tables.data(), out));
}

VectorMatrix pq_decode(const Codebook& cb, const CodeMatrix& codes) {
    check_codes_match(cb, codes, "pq_decode");
    VectorMatrix out(codes.rows, cb.dims());
    raise(pqg_pq_decode(ctx(), codes.bytes.data(), codes.rows, cb.m_subspaces, cb.ks, cb.sub_dim,
                        cb.tables.data(), out.values.data()));
    return out;
}

DistanceTable adc_table(const Codebook& cb, std::span<const float> query) {
    if (query.size() != cb.dims())
        throw std::invalid_argument("adc_table: query dimension " + std::to_string(query.size()) +
                                    " does not match codebook dimension " + std::to_string(cb.dims()));
    DistanceTable t;
    t.m_subspaces = cb.m_subspaces;
    t.ks = cb.ks;
    t.entries.resize(std::size_t(cb.m_subspaces) * cb.ks);
    raise(pqg_adc_tables(ctx(), cb.tables.data(), cb.m_subspaces, cb.ks, cb.sub_dim, query.data(), 1,
                         t.entries.data()));
    return t;
}

double adc_lookup(const DistanceTable& table, const CodeMatrix& codes, std::size_t row) {
    if (codes.m_subspaces != table.m_subspaces || codes.ks != table.ks)
        throw std::invalid_argument("adc_lookup: codes do not match the table");
    double out = 0.0;
    raise(pqg_adc_lookup(ctx(), table.entries.data(), table.m_subspaces, table.ks,
                         codes.bytes.data() + row * codes.row_bytes(), 1, &out));
    return out;
}

double rmse(const VectorMatrix& a, const VectorMatrix& b) {
    if (!a.same_shape(b)) throw std::invalid_argument("rmse: shape mismatch");
    double sse = 0.0;
    raise(pqg_sq_error(ctx(), a.values.data(), b.values.data(), a.values.size(), &sse));
    return std::sqrt(sse / double(a.rows * a.dims));
}

double reconstruction_rmse(const Codebook& cb, const VectorMatrix& data) {
    if (data.dims != cb.dims())
        throw std::invalid_argument("pq_encode: data dimension " + std::to_string(data.dims) +
                                    " does not match codebook dimension " + std::to_string(cb.dims()));
    double sse = 0.0;
    raise(pqg_pq_encode_sse(ctx(), data.values.data(), data.rows, cb.m_subspaces, cb.ks, cb.sub_dim,
                            cb.tables.data(), nullptr, &sse));
    return std::sqrt(sse / double(data.rows * data.dims));
}

// On-disk formats (pq.cpp:183-259) through the C ABI: byte-identical files,
// the reference's messages; payload validation runs on the device.
void save_codebook(const Codebook& cb, const std::string& path) {
    raise(pqg_codebook_save(ctx(), cb.tables.data(), cb.m_subspaces, cb.ks, cb.sub_dim, path.c_str()));
}

Codebook load_codebook(const std::string& path) {
    Codebook cb;
    raise(pqg_codebook_file_info(path.c_str(), &cb.m_subspaces, &cb.ks, &cb.sub_dim));
    cb.tables.resize(std::size_t(cb.m_subspaces) * cb.ks * cb.sub_dim);
    raise(pqg_codebook_load(ctx(), path.c_str(), cb.tables.data(), cb.tables.size()));
    return cb;
}

void save_codes(const CodeMatrix& codes, const std::string& path) {
    raise(pqg_codes_save(ctx(), codes.bytes.data(), codes.rows, codes.m_subspaces, codes.ks, path.c_str()));
}

CodeMatrix load_codes(const std::string& path) {
    std::uint64_t n = 0;
    std::uint32_t m = 0, ks = 0;
    raise(pqg_codes_file_info(path.c_str(), &n, &m, &ks));
    CodeMatrix codes(std::size_t(n), m, ks);
    raise(pqg_codes_load(ctx(), path.c_str(), codes.bytes.data(), codes.bytes.size()));
    return codes;
}

// ===========================================================================
// ivf.hpp
// ===========================================================================
std::size_t default_nlist(std::size_t n_items) {
    const auto r = static_cast<std::size_t>(std::llround(std::sqrt(double(n_items))));
    return std::clamp<std::size_t>(r, 1, n_items == 0 ? 1 : n_items);
}

InvertedIndex ivf_build(const Codebook& cb, const CodeMatrix& codes,
                        std::span<const std::uint64_t> ids, std::size_t nlist, std::uint64_t seed,
                        std::uint32_t kmeans_iters) {
    if (ids.empty()) throw std::invalid_argument("ivf_build: no items");
    if (ids.size() != codes.rows) throw std::invalid_argument("ivf_build: ids/codes length mismatch");
    check_codes_match(cb, codes, "pq_decode");
    pqg_index* h = nullptr;
    raise(pqg_ivf_build(ctx(), cb.tables.data(), cb.m_subspaces, cb.ks, cb.sub_dim,
                        codes.bytes.data(), ids.data(), codes.rows, nlist, seed, kmeans_iters, &h));
    IndexPtr p(h, IndexDeleter());
    return to_host(h, cb);
}

InvertedIndex ivf_build_with_centroids(const Codebook& cb, const CodeMatrix& codes,
                                       std::span<const std::uint64_t> ids,
                                       const VectorMatrix& coarse_centroids) {
    if (ids.empty()) throw std::invalid_argument("ivf_build: no items");
    if (ids.size() != codes.rows) throw std::invalid_argument("ivf_build: ids/codes length mismatch");
    if (coarse_centroids.rows == 0 || coarse_centroids.dims != cb.dims())
        throw std::invalid_argument("ivf_build: coarse centroids do not match the codebook");
    pqg_index* h = nullptr;
    raise(pqg_ivf_build_with_centroids(ctx(), cb.tables.data(), cb.m_subspaces, cb.ks, cb.sub_dim,
                                       codes.bytes.data(), ids.data(), codes.rows,
                                       coarse_centroids.values.data(), coarse_centroids.rows, &h));
    IndexPtr p(h, IndexDeleter());
    return to_host(h, cb);
}

void ivf_add(InvertedIndex& index, const CodeMatrix& codes, std::span<const std::uint64_t> ids) {
    if (ids.size() != codes.rows) throw std::invalid_argument("ivf_add: ids/codes length mismatch");
    if (codes.m_subspaces != index.codebook.m_subspaces || codes.ks != index.codebook.ks)
        throw std::invalid_argument("ivf_add: codes do not match the index codebook");
    if (ids.empty()) return;
    std::unordered_set<std::uint64_t> fresh;
    fresh.reserve(ids.size());
    for (const std::uint64_t id : ids)
        if (!fresh.insert(id).second) throw std::invalid_argument("duplicate id " + std::to_string(id));
    for (const std::uint64_t id : ids)
        if (index.id_set.contains(id))
            throw std::invalid_argument("ivf_add: id collision on id " + std::to_string(id));
    std::vector<std::uint32_t> list_of(codes.rows);
    const Codebook& cb = index.codebook;
    raise(pqg_ivf_assign(ctx(), codes.bytes.data(), codes.rows, cb.m_subspaces, cb.ks, cb.sub_dim,
                         cb.tables.data(), index.coarse_centroids.values.data(), index.nlist(),
                         list_of.data()));
    for (std::size_t i = 0; i < codes.rows; ++i) {  // append in input order (ivf.cpp:44-46)
        PostingList& pl = index.lists[list_of[i]];
        pl.ids.push_back(ids[i]);
        pl.codes.append_row_from(codes, i);
    }
    index.n_items += codes.rows;
    index.id_set.merge(fresh);
}

InvertedIndex ivf_merge(const InvertedIndex& a, const InvertedIndex& b) {
    // the device merge (pqg_index_merge: codebook / coarse / id-collision
    // checks, then list l = a's then b's with csr_concat) on the cached
    // device copies of both operands
    IndexPtr da = device_index_for(a), db = device_index_for(b);
    pqg_index* h = nullptr;
    raise(pqg_index_merge(ctx(), da.get(), db.get(), &h));
    IndexPtr p(h, IndexDeleter());
    return to_host(h, a.codebook);
}

std::vector<QueryResult> ivf_query_batch(const InvertedIndex& index, const VectorMatrix& queries,
                                         std::size_t k, std::size_t nprobe,
                                         std::optional<double> max_sq_dist) {
    const std::size_t nq = queries.rows;
    if (nq == 0) return {};
    check_query(index, queries.row_span(0), k, nprobe);
    std::vector<std::uint64_t> ids(nq * k);
    std::vector<double> d(nq * k);
    std::vector<std::uint32_t> cnt(nq);
    auto run = [&](pqg_index* h, std::uint32_t* probes) {
        raise(pqg_index_search_ex(ctx(), h, queries.values.data(), nq, k, nprobe, max_sq_dist.has_value(),
                                  max_sq_dist.value_or(0.0), ids.data(), d.data(), cnt.data(), probes));
    };
    bool done = false;
    if (nq * nprobe * 2 < index.lists.size()) {
        // few probed lists: search the cached copy, then compare only the
        // lists the queries read against the caller's index
        if (auto e = cache_find(index)) {
            std::vector<std::uint32_t> probes(nq * nprobe);
            run(e->dev.get(), probes.data());
            std::sort(probes.begin(), probes.end());
            probes.erase(std::unique(probes.begin(), probes.end()), probes.end());
            done = true;
            for (std::uint32_t l : probes)
                if (!list_equal(*e->host, index, l)) { done = false; break; }
            if (!done) cache_drop(*e);
        }
        if (!done) {
            run(cache_insert(index).dev.get(), nullptr);
            done = true;
        }
    }
    if (!done) run(device_index_for(index).get(), nullptr);
    std::vector<QueryResult> out;
    out.reserve(nq);
    for (std::size_t q = 0; q < nq; ++q) out.push_back(result_of(&ids[q * k], &d[q * k], cnt[q], k));
    return out;
}

QueryResult ivf_query(const InvertedIndex& index, std::span<const float> query, std::size_t k,
                      std::size_t nprobe, std::optional<double> max_sq_dist) {
    check_query(index, query, k, nprobe);
    VectorMatrix q(1, query.size());
    std::memcpy(q.values.data(), query.data(), query.size() * sizeof(float));
    return ivf_query_batch(index, q, k, nprobe, max_sq_dist)[0];
}

QueryResult ivf_query_subset(const InvertedIndex& index, std::span<const float> query,
                             std::size_t k, std::span<const std::uint64_t> subset,
                             std::size_t nprobe, std::optional<double> max_sq_dist) {
    check_query(index, query, k, nprobe);
    IndexPtr dev = device_index_for(index);
    std::vector<std::uint64_t> ids(k);
    std::vector<double> d(k);
    std::uint32_t cnt = 0;
    raise(pqg_index_search_subset(ctx(), dev.get(), query.data(), 1, k, subset.data(), subset.size(),
                                  nprobe, max_sq_dist.has_value(), max_sq_dist.value_or(0.0),
                                  ids.data(), d.data(), &cnt));
    return result_of(ids.data(), d.data(), cnt, k);
}

QueryResult flat_scan(const Codebook& cb, const CodeMatrix& codes,
                      std::span<const std::uint64_t> ids, std::span<const float> query,
                      std::size_t k, std::optional<double> max_sq_dist) {
    if (k == 0) throw std::invalid_argument("flat_scan: k must be >= 1");
    if (ids.size() != codes.rows) throw std::invalid_argument("flat_scan: ids/codes length mismatch");
    if (query.size() != cb.dims()) throw std::invalid_argument("flat_scan: dimension mismatch");
    std::vector<std::uint64_t> oi(k);
    std::vector<double> od(k);
    std::uint32_t cnt = 0;
    if (codes.rows == 0) return result_of(oi.data(), od.data(), 0, k);
    raise(pqg_flat_scan(ctx(), cb.tables.data(), cb.m_subspaces, cb.ks, cb.sub_dim,
                        codes.bytes.data(), ids.data(), codes.rows, query.data(), 1, k,
                        max_sq_dist.has_value(), max_sq_dist.value_or(0.0), oi.data(), od.data(), &cnt));
    return result_of(oi.data(), od.data(), cnt, k);
}

// PQII (ivf.cpp:264-355): the device index (cached upload) is packed into the
// file image by the device; loading unpacks the lists into a device CSR,
// checks ids and codes there, and exports the reference's host structure.
void save_index(const InvertedIndex& index, const std::string& path) {
    IndexPtr dev = device_index_for(index);
    raise(pqg_index_save(ctx(), dev.get(), path.c_str()));
}

InvertedIndex load_index(const std::string& path) {
    pqg_index* h = nullptr;
    raise(pqg_index_load(ctx(), path.c_str(), &h));
    IndexPtr dev(h, IndexDeleter());
    std::uint64_t nlist = 0, n = 0;
    std::uint32_t M = 0, ks = 0, ds = 0;
    raise(pqg_index_info(h, &nlist, &n, &M, &ks, &ds));
    Codebook cb;
    cb.m_subspaces = M;
    cb.ks = ks;
    cb.sub_dim = ds;
    cb.tables.resize(std::size_t(M) * ks * ds);
    raise(pqg_index_export(ctx(), h, nullptr, nullptr, nullptr, nullptr, cb.tables.data()));
    return to_host(h, cb);
}

// ===========================================================================
// pipeline.hpp (proj/src/pipeline.cpp) -- one batched device fit for all
// chunks, data resident on the device between phases (pqg_pipeline_run)
// ===========================================================================
const char* to_string(PipelineMode mode) {
    switch (mode) {
        case PipelineMode::kSingle: return "single";
        case PipelineMode::kParallelPq: return "parallel_pq";
        case PipelineMode::kParallelPqIndex: return "parallel_pq_index";
    }
    return "unknown";
}

std::optional<PipelineMode> parse_mode(std::string_view name) {
    for (PipelineMode m : {PipelineMode::kSingle, PipelineMode::kParallelPq,
                           PipelineMode::kParallelPqIndex})
        if (name == to_string(m)) return m;
    return std::nullopt;
}

ChunkOutput train_chunk(const VectorMatrix& chunk, std::uint32_t m, std::uint32_t ks,
                        std::uint32_t iters, std::uint64_t chunk_seed) {
    const auto t0 = std::chrono::steady_clock::now();
    ChunkOutput out;
    out.representatives = VectorMatrix(ks, chunk.dims);
    const int rc = pqg_train_chunks(ctx(), chunk.values.data(), chunk.rows, chunk.dims, 1, m, ks,
                                    iters, chunk_seed, out.representatives.values.data(),
                                    &out.local_rmse, nullptr);
    if (rc == PQG_ECHUNK) {
        // train_chunk itself throws invalid_argument without the task prefix
        // (pipeline.cpp:84-90)
        std::string msg = pqg_last_error();
        if (msg.rfind("chunk 0: ", 0) == 0) msg = msg.substr(9);
        throw std::invalid_argument(msg);
    }
    raise(rc);
    out.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return out;
}

VectorMatrix aggregate_representatives(const std::vector<ChunkOutput>& outputs) {
    if (outputs.empty()) throw std::invalid_argument("aggregate_representatives: no outputs");
    std::vector<const ChunkOutput*> order;
    for (const auto& o : outputs) order.push_back(&o);
    std::stable_sort(order.begin(), order.end(),
                     [](const ChunkOutput* a, const ChunkOutput* b) { return a->chunk_id < b->chunk_id; });
    const std::size_t d = outputs.front().representatives.dims;
    std::size_t rows = 0;
    for (const auto& o : outputs) {
        if (o.representatives.dims != d)
            throw std::invalid_argument("aggregate_representatives: dimension mismatch at chunk " +
                                        std::to_string(o.chunk_id));
        rows += o.representatives.rows;
    }
    VectorMatrix all(rows, d);
    std::size_t at = 0;
    for (const ChunkOutput* o : order) {
        std::copy(o->representatives.values.begin(), o->representatives.values.end(),
                  all.values.begin() + at * d);
        at += o->representatives.rows;
    }
    return all;
}

Codebook fit_global(const VectorMatrix& representatives, std::uint32_t m, std::uint32_t ks,
                    std::uint32_t iters, std::uint64_t seed) {
    return pq_fit(representatives, m, ks, iters, seed);
}

PipelineReport run_pipeline(const VectorMatrix& data, const PipelineConfig& config) {
    if (data.rows == 0 || data.dims == 0) throw std::invalid_argument("run_pipeline: empty dataset");
    if (config.n_threads == 0) throw std::invalid_argument("run_pipeline: n_threads must be >= 1");
    const auto t0 = std::chrono::steady_clock::now();
    PipelineReport r;
    r.config = config;
    const std::uint32_t M = config.m_subspaces, ks = config.ks;
    const bool parallel = config.mode != PipelineMode::kSingle;
    const std::size_t ds = (M && data.dims % M == 0) ? data.dims / M : 1;
    r.global_codebook.m_subspaces = M;
    r.global_codebook.ks = ks;
    r.global_codebook.sub_dim = static_cast<std::uint32_t>(ds);
    r.global_codebook.tables.assign(std::size_t(M) * ks * ds, 0.0f);
    VectorMatrix reps;
    if (parallel) reps = VectorMatrix(config.n_chunks * ks, data.dims);
    std::vector<double> local(parallel ? std::max<std::size_t>(config.n_chunks, 1) : 0);
    std::uint64_t nlist = 0;
    pqg_index* h = nullptr;
    double ph[PQG_PHASE_COUNT];
    const int mode = config.mode == PipelineMode::kSingle
                         ? PQG_MODE_SINGLE
                         : (config.mode == PipelineMode::kParallelPq ? PQG_MODE_PARALLEL_PQ
                                                                     : PQG_MODE_PARALLEL_PQ_INDEX);
    raise(pqg_pipeline_run(ctx(), data.values.data(), data.rows, data.dims, config.n_chunks, M, ks,
                           config.nlist, config.kmeans_iters, config.seed, mode,
                           r.global_codebook.tables.data(), &r.global_rmse,
                           parallel ? reps.values.data() : nullptr,
                           parallel ? local.data() : nullptr, &nlist,
                           mode == PQG_MODE_PARALLEL_PQ_INDEX ? &h : nullptr, ph));
    r.config.nlist = nlist;
    static const char* names[PQG_PHASE_COUNT] = {"fit",        "chunking", "local_fit",
                                                 "global_fit", "coarse_fit", "encode",
                                                 "index_build", "merge"};
    for (int i = 0; i < PQG_PHASE_COUNT; ++i)
        if (ph[i] >= 0.0) r.phase_seconds[names[i]] = ph[i];
    if (!parallel) r.single_rmse = r.global_rmse;
    else r.representatives = std::move(reps);
    if (h) {
        IndexPtr p(h, IndexDeleter());
        r.merged_index = to_host(h, r.global_codebook);
    }
    r.total_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return r;
}

std::string PipelineReport::summary() const {
    std::ostringstream out;
    out << "mode: " << to_string(config.mode) << '\n';
    out << "params: M=" << config.m_subspaces << " Ks=" << config.ks << " C=" << config.n_chunks
        << " T=" << config.n_threads << " nlist=" << config.nlist << " iters=" << config.kmeans_iters
        << " seed=" << config.seed << '\n';
    out << "phases:";
    for (const auto& [phase, secs] : phase_seconds)
        out << ' ' << phase << '=' << std::fixed << std::setprecision(3) << secs << 's'
            << std::defaultfloat;
    out << '\n';
    out << "total: " << std::fixed << std::setprecision(3) << total_seconds << "s\n"
        << std::defaultfloat;
    out << std::setprecision(9) << "rmse: " << global_rmse << '\n';
    if (merged_index)
        out << "index: " << merged_index->n_items << " items across " << merged_index->nlist()
            << " lists\n";
    return out.str();
}

}  // namespace pqii
