// facade_test.cpp -- the reference's unit-test cases (proj/tests/test_kmeans.cpp,
// test_pq.cpp, test_ivf.cpp) restated against the drop-in libpqg_pqii.so
// through the pqii headers of this repo.  A tiny CHECK harness replaces the
// absent doctest.  Run by tests/test_facade_cpp.py on a GPU.
#include <algorithm>
#include <unistd.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "pqii/ivf.hpp"
#include "pqii/kmeans.hpp"
#include "pqii/pipeline.hpp"
#include "pqii/pq.hpp"

using namespace pqii;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                              \
    do {                                                                      \
        ++g_checks;                                                           \
        if (!(c)) {                                                           \
            ++g_fail;                                                         \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);          \
        }                                                                     \
    } while (0)
#define CHECK_THROWS_WITH(expr, type, sub)                                    \
    do {                                                                      \
        ++g_checks;                                                           \
        bool ok = false;                                                      \
        try {                                                                 \
            expr;                                                             \
        } catch (const type& e) {                                             \
            ok = std::string(e.what()).find(sub) != std::string::npos;        \
        } catch (...) {                                                       \
        }                                                                     \
        if (!ok) {                                                            \
            ++g_fail;                                                         \
            std::printf("FAIL %s:%d: %s does not throw %s(%s)\n", __FILE__,   \
                        __LINE__, #expr, #type, sub);                         \
        }                                                                     \
    } while (0)

// proj/tests/test_helpers.cpp:26-33
static VectorMatrix random_matrix(std::size_t rows, std::size_t dims, std::uint64_t seed,
                                  float lo = -1.0f, float hi = 1.0f) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<float> dist(lo, hi);
    VectorMatrix m(rows, dims);
    for (auto& v : m.values) v = dist(rng);
    return m;
}

// a 12-cluster mixture standing in for the reference's gen_synthetic
// (its tests use clustered_data, proj/tests/test_pipeline.cpp:15-18)
static VectorMatrix clustered(std::size_t n, std::size_t d, std::uint64_t seed) {
    const VectorMatrix centers = random_matrix(12, d, seed * 7 + 1, -8.0f, 8.0f);
    std::mt19937_64 rng(seed);
    std::normal_distribution<float> z(0.0f, 0.7f);
    VectorMatrix m(n, d);
    for (std::size_t i = 0; i < n; ++i) {
        const float* c = centers.row(rng() % 12);
        for (std::size_t t = 0; t < d; ++t) m.row(i)[t] = c[t] + z(rng);
    }
    return m;
}

static bool rows_equal_as_sets(const VectorMatrix& a, const VectorMatrix& b, double tol) {
    if (!a.same_shape(b)) return false;
    std::vector<bool> used(b.rows, false);
    for (std::size_t i = 0; i < a.rows; ++i) {
        bool matched = false;
        for (std::size_t j = 0; j < b.rows && !matched; ++j) {
            if (used[j]) continue;
            bool close = true;
            for (std::size_t t = 0; t < a.dims && close; ++t)
                close = std::fabs(double(a.row(i)[t]) - double(b.row(j)[t])) <= tol;
            if (close) used[j] = matched = true;
        }
        if (!matched) return false;
    }
    return true;
}

static double exhaustive(const float* p, const float* t, std::size_t k, std::size_t d, std::size_t* best) {
    double bd = INFINITY;
    for (std::size_t c = 0; c < k; ++c) {
        double acc = 0;
        for (std::size_t j = 0; j < d; ++j) {
            const double diff = double(p[j]) - double(t[c * d + j]);
            acc += diff * diff;
        }
        if (acc < bd) { bd = acc; *best = c; }
    }
    return bd;
}

int main() {
    // ---- test_kmeans.cpp
    {   // :48-64 k=1 centroid is the coordinate-wise mean
        const VectorMatrix pts = random_matrix(50, 4, 21);
        const KMeansResult r = kmeans_fit(pts, 1, 20, 3);
        for (std::size_t d = 0; d < 4; ++d) {
            double mean = 0;
            for (std::size_t i = 0; i < pts.rows; ++i) mean += pts.row(i)[d];
            mean /= double(pts.rows);
            CHECK(std::fabs(r.centroids.row(0)[d] - mean) <= 1e-6 * std::max(1.0, std::fabs(mean)));
        }
    }
    {   // :80-96 {0,1,9,10}
        VectorMatrix pts(4, 1);
        pts.values = {0, 1, 9, 10};
        for (std::uint64_t seed = 0; seed < 6; ++seed) {
            const KMeansResult r = kmeans_fit(pts, 2, 20, seed);
            CHECK(std::fabs(r.inertia - 1.0) < 1e-9);
            CHECK(std::min(r.centroids.values[0], r.centroids.values[1]) == 0.5f);
            CHECK(std::max(r.centroids.values[0], r.centroids.values[1]) == 9.5f);
        }
    }
    {   // :98-144 nearest_centroid
        const VectorMatrix table = random_matrix(16, 8, 31);
        const auto nc = nearest_centroid(table.row_span(3), table);
        CHECK(nc.index == 3 && nc.sq_dist == 0.0);
        VectorMatrix two(2, 1);
        two.values = {1.0f, 3.0f};
        const float probe = 2.0f;
        CHECK(nearest_centroid({&probe, 1}, two).index == 0);
        std::mt19937_64 rng(77);
        std::uniform_real_distribution<float> dist(-1, 1);
        for (int trial = 0; trial < 100; ++trial) {
            std::vector<float> p(8);
            for (auto& v : p) v = dist(rng);
            const auto n2 = nearest_centroid({p.data(), 8}, table);
            std::size_t best = 0;
            const double bd = exhaustive(p.data(), table.values.data(), 16, 8, &best);
            CHECK(n2.index == best);
            CHECK(n2.sq_dist == bd);
        }
        const VectorMatrix empty;
        const float z = 0;
        CHECK_THROWS_WITH(nearest_centroid({&z, 1}, empty), std::invalid_argument, "empty centroid set");
    }
    {   // :146-157 determinism
        const VectorMatrix pts = random_matrix(300, 6, 41);
        const KMeansResult a = kmeans_fit(pts, 12, 15, 9), b = kmeans_fit(pts, 12, 15, 9);
        CHECK(a.centroids == b.centroids && a.assignments == b.assignments && a.inertia == b.inertia);
    }
    {   // :174-187 duplicates, validation
        VectorMatrix pts(6, 2, 1.5f);
        const KMeansResult r = kmeans_fit(pts, 3, 10, 0);
        CHECK(r.inertia == 0.0);
        for (const float v : r.centroids.values) CHECK(std::isfinite(v));
        const VectorMatrix p5 = random_matrix(5, 2, 1);
        CHECK_THROWS_WITH(kmeans_fit(p5, 0, 10, 0), std::invalid_argument, "");
        CHECK_THROWS_WITH(kmeans_fit(p5, 6, 10, 0), std::invalid_argument, "exceeds");
        CHECK_THROWS_WITH(kmeans_fit(p5, 2, 0, 0), std::invalid_argument, "");
        CHECK_THROWS_WITH(kmeans_fit(p5, 2, 10, 0, -1.0), std::invalid_argument, "");
    }
    // ---- test_pq.cpp
    {   // :37-60 shapes, M=1 == kmeans_fit, errors
        const VectorMatrix data = random_matrix(64, 4, 17);
        const Codebook cb = pq_fit(data, 2, 8, 10, 1);
        CHECK(cb.m_subspaces == 2 && cb.sub_dim == 2 && cb.ks == 8 && cb.tables.size() == 32u);
        const Codebook c1 = pq_fit(data, 1, 8, 10, 42);
        CHECK(c1.tables == kmeans_fit(data, 8, 10, 42).centroids.values);
        CHECK_THROWS_WITH(pq_fit(data, 3, 8, 10, 1), std::invalid_argument, "not divisible");
        CHECK_THROWS_WITH(pq_fit(data, 2, 65, 10, 1), std::invalid_argument, "exceeds");
    }
    {   // :102-127 encode == exhaustive fp64 scan
        const VectorMatrix data = random_matrix(120, 8, 57);
        const Codebook cb = pq_fit(data, 4, 16, 15, 5);
        const CodeMatrix codes = pq_encode(cb, data);
        for (std::size_t i = 0; i < data.rows; ++i)
            for (std::uint32_t m = 0; m < 4; ++m) {
                std::size_t best = 0;
                exhaustive(data.row(i) + m * 2, cb.sub_table(m), 16, 2, &best);
                CHECK(codes.at(i, m) == best);
            }
        CodeMatrix bad(1, 4, 16);
        bad.bytes[0] = 200;
        CHECK_THROWS_WITH(pq_decode(cb, bad), std::out_of_range, "");
    }
    {   // :163-214 adc arithmetic; :238-242 rmse
        Codebook cb;
        cb.m_subspaces = 1; cb.ks = 1; cb.sub_dim = 1; cb.tables = {3.0f};
        const float q = 1.0f;
        CHECK(adc_table(cb, {&q, 1}).entry(0, 0) == 4.0f);
        VectorMatrix a(1, 2), b(1, 2);
        b.values = {3, 4};
        CHECK(std::fabs(rmse(a, b) - std::sqrt(25.0 / 2.0)) < 1e-12);
        CHECK_THROWS_WITH(rmse(random_matrix(2, 2, 1), random_matrix(2, 3, 1)), std::invalid_argument, "");
    }
    // ---- test_ivf.cpp
    {
        VectorMatrix data = random_matrix(2000, 16, 3, 0, 10);
        const Codebook cb = pq_fit(data, 4, 16, 10, 2);
        const CodeMatrix codes = pq_encode(cb, data);
        std::vector<std::uint64_t> ids(codes.rows);
        std::iota(ids.begin(), ids.end(), 100);
        const InvertedIndex ix = ivf_build(cb, codes, ids, 12, 5);
        CHECK(ix.nlist() == 12 && ix.n_items == 2000 && ix.id_set.size() == 2000);
        // membership == nearest coarse centroid of the decoded vector (:66-81)
        for (std::size_t l = 0; l < ix.nlist(); ++l)
            for (std::size_t i = 0; i < ix.lists[l].ids.size(); ++i) {
                std::vector<float> dec(16);
                pq_decode_row(cb, ix.lists[l].codes, i, dec.data());
                CHECK(nearest_centroid({dec.data(), 16}, ix.coarse_centroids).index == l);
            }
        // query at nprobe = nlist == flat_scan (:246-253)
        const VectorMatrix qs = random_matrix(20, 16, 9, 0, 10);
        for (std::size_t q = 0; q < qs.rows; ++q) {
            const auto a = ivf_query(ix, qs.row_span(q), 10, ix.nlist());
            const auto f = flat_scan(cb, codes, ids, qs.row_span(q), 10);
            CHECK(a.hits == f.hits);
        }
        // merge of halves == monolithic with the same centroids (:171-186)
        CodeMatrix lo(0, 4, 16), hi(0, 4, 16);
        for (std::size_t i = 0; i < codes.rows; ++i) (i < 700 ? lo : hi).append_row_from(codes, i);
        const std::vector<std::uint64_t> ilo(ids.begin(), ids.begin() + 700), ihi(ids.begin() + 700, ids.end());
        const InvertedIndex m = ivf_merge(ivf_build_with_centroids(cb, lo, ilo, ix.coarse_centroids),
                                          ivf_build_with_centroids(cb, hi, ihi, ix.coarse_centroids));
        const InvertedIndex mono = ivf_build_with_centroids(cb, codes, ids, ix.coarse_centroids);
        for (std::size_t l = 0; l < m.nlist(); ++l) {
            CHECK(m.lists[l].ids == mono.lists[l].ids);
            CHECK(m.lists[l].codes == mono.lists[l].codes);
        }
        InvertedIndex add = ivf_build_with_centroids(cb, lo, ilo, ix.coarse_centroids);
        ivf_add(add, hi, ihi);
        for (std::size_t l = 0; l < add.nlist(); ++l) CHECK(add.lists[l].ids == mono.lists[l].ids);
        CHECK_THROWS_WITH(ivf_add(add, hi, ihi), std::invalid_argument, "id collision");
        CHECK_THROWS_WITH(ivf_query(ix, qs.row_span(0), 10, 0), std::invalid_argument, "nprobe");
        std::vector<std::uint64_t> dup = ids;
        dup[5] = dup[2];
        CHECK_THROWS_WITH(ivf_build_with_centroids(cb, codes, dup, ix.coarse_centroids),
                          std::invalid_argument, "duplicate id");
        CHECK(default_nlist(10000) == 100 && default_nlist(0) == 1 && default_nlist(2) == 1);
        // the device-index cache never serves a stale index: same-shape indexes
        // built and freed in a loop (malloc reuses their blocks), and a list
        // edited in place through the public fields
        for (int rep = 0; rep < 3; ++rep) {
            const VectorMatrix d2 = random_matrix(2000, 16, 100 + rep, 0, 10);
            const CodeMatrix c2 = pq_encode(cb, d2);
            const InvertedIndex i2 = ivf_build_with_centroids(cb, c2, ids, ix.coarse_centroids);
            const auto r2 = ivf_query(i2, qs.row_span(2), 10, i2.nlist());
            const auto f2 = flat_scan(cb, c2, ids, qs.row_span(2), 10);
            CHECK(r2.hits == f2.hits);
        }
        {
            InvertedIndex edit = ivf_build_with_centroids(cb, codes, ids, ix.coarse_centroids);
            const auto before = ivf_query(edit, qs.row_span(3), 5, edit.nlist());
            const std::uint64_t top = before.hits[0].id;
            for (auto& pl : edit.lists)  // move the best hit's code far away
                for (std::size_t i = 0; i < pl.ids.size(); ++i)
                    if (pl.ids[i] == top)
                        for (std::uint32_t m = 0; m < 4; ++m) {
                            const std::uint32_t c = pl.codes.at(i, m);
                            pl.codes.set(i, m, (c + 8) % 16);
                        }
            const auto after = ivf_query(edit, qs.row_span(3), 5, edit.nlist());
            CodeMatrix c3(0, 4, 16);
            std::vector<std::uint64_t> i3;
            for (const auto& pl : edit.lists)
                for (std::size_t i = 0; i < pl.ids.size(); ++i) {
                    c3.append_row_from(pl.codes, i);
                    i3.push_back(pl.ids[i]);
                }
            CHECK(after.hits == flat_scan(cb, c3, i3, qs.row_span(3), 5).hits);
            // r2e: a small-nprobe query verifies only the lists it probes --
            // an in-place edit of a probed list must still be seen: expected =
            // flat_scan over the items of the two nearest lists (fp64 probe order)
            const auto q4 = qs.row_span(4);
            std::vector<std::pair<double, std::size_t>> pd;
            for (std::size_t l = 0; l < edit.nlist(); ++l) {
                double acc = 0.0;
                for (std::size_t t = 0; t < q4.size(); ++t) {
                    const double df = double(q4[t]) - double(edit.coarse_centroids.row(l)[t]);
                    acc += df * df;
                }
                pd.emplace_back(acc, l);
            }
            std::sort(pd.begin(), pd.end());
            auto probed_flat = [&](std::size_t kk) {
                CodeMatrix cp(0, 4, 16);
                std::vector<std::uint64_t> ip;
                for (int j = 0; j < 2; ++j) {
                    const PostingList& pl = edit.lists[pd[j].second];
                    for (std::size_t i = 0; i < pl.ids.size(); ++i) {
                        cp.append_row_from(pl.codes, i);
                        ip.push_back(pl.ids[i]);
                    }
                }
                return flat_scan(cb, cp, ip, q4, kk).hits;
            };
            const auto b4 = ivf_query(edit, q4, 5, 2);
            CHECK(b4.hits == probed_flat(5));
            PostingList& hot = edit.lists[pd[0].second];
            for (std::size_t i = 0; i < hot.ids.size(); ++i)
                for (std::uint32_t m = 0; m < 4; ++m) hot.codes.set(i, m, (hot.codes.at(i, m) + 5) % 16);
            const auto a4 = ivf_query(edit, q4, 5, 2);
            CHECK(a4.hits == probed_flat(5));
        }
        // k > 32 (the CTA-wide path) and k beyond n_items saturating (test_ivf.cpp:255-259)
        const QueryResult sat = ivf_query(ix, qs.row_span(0), 1000, ix.nlist());
        CHECK(sat.hits.size() == 1000 && sat.k_requested == 1000);
        const QueryResult sat2 = ivf_query(mono, qs.row_span(1), 5000, mono.nlist());
        CHECK(sat2.hits.size() == 2000 && sat2.k_requested == 5000);
        const QueryResult flat_big = flat_scan(cb, codes, ids, qs.row_span(1), 5000);
        CHECK(flat_big.hits == sat2.hits);
        for (std::size_t j = 1; j < sat2.hits.size(); ++j)
            CHECK(sat2.hits[j - 1].sq_dist < sat2.hits[j].sq_dist ||
                  (sat2.hits[j - 1].sq_dist == sat2.hits[j].sq_dist && sat2.hits[j - 1].id < sat2.hits[j].id));
    }
    // ---- test_pq.cpp:302-329 "codebook and code files round-trip", and
    // ---- test_ivf.cpp:357-407 "index serialization round-trips bit-exactly"
    {
        const std::string dir = std::string(std::getenv("TMPDIR") ? std::getenv("TMPDIR") : "/tmp") + "/pqg_fmt_" +
                                std::to_string(::getpid());
        if (std::system(("mkdir -p " + dir).c_str()) != 0) std::printf("mkdir failed\n");
        auto read_file = [](const std::string& p) {
            std::FILE* f = std::fopen(p.c_str(), "rb");
            std::string out;
            if (!f) return out;
            char buf[4096];
            std::size_t n;
            while ((n = std::fread(buf, 1, sizeof(buf), f)) > 0) out.append(buf, n);
            std::fclose(f);
            return out;
        };
        auto write_file = [](const std::string& p, const std::string& b) {
            std::FILE* f = std::fopen(p.c_str(), "wb");
            std::fwrite(b.data(), 1, b.size(), f);
            std::fclose(f);
        };
        const VectorMatrix data = random_matrix(64, 8, 3);
        const Codebook cb = pq_fit(data, 4, 8, 10, 5);
        save_codebook(cb, dir + "/cb.pqcb");
        CHECK(load_codebook(dir + "/cb.pqcb") == cb);
        const CodeMatrix codes = pq_encode(cb, data);
        save_codes(codes, dir + "/codes.pqcm");
        CHECK(load_codes(dir + "/codes.pqcm") == codes);
        save_codebook(load_codebook(dir + "/cb.pqcb"), dir + "/cb2.pqcb");
        CHECK(read_file(dir + "/cb2.pqcb") == read_file(dir + "/cb.pqcb"));
        std::string bytes = read_file(dir + "/cb.pqcb");
        bytes[1] = 'x';
        write_file(dir + "/bad.pqcb", bytes);
        CHECK_THROWS_WITH(load_codebook(dir + "/bad.pqcb"), std::runtime_error, "bad magic");

        // byte codes (Ks <= 256): make_fixture(150, 61) shape -- 16-d data, M=4, Ks=16
        const VectorMatrix d16 = random_matrix(150, 16, 61, -10, 10);
        const Codebook cb16 = pq_fit(d16, 4, 16, 15, 3);
        const CodeMatrix c16 = pq_encode(cb16, d16);
        std::vector<std::uint64_t> ids16(150);
        std::iota(ids16.begin(), ids16.end(), std::uint64_t{0});
        const InvertedIndex index = ivf_build(cb16, c16, ids16, 10, 67);
        save_index(index, dir + "/a.pqii");
        const InvertedIndex loaded = load_index(dir + "/a.pqii");
        save_index(loaded, dir + "/b.pqii");
        CHECK(read_file(dir + "/a.pqii") == read_file(dir + "/b.pqii"));
        CHECK(loaded.n_items == index.n_items);
        CHECK(loaded.codebook == index.codebook);
        CHECK(loaded.coarse_centroids == index.coarse_centroids);
        CHECK(loaded.id_set.size() == index.id_set.size());
        const VectorMatrix q = random_matrix(1, 16, 9);
        CHECK(ivf_query(loaded, q.row_span(0), 5, 10).hits == ivf_query(index, q.row_span(0), 5, 10).hits);
        // wide codes (Ks > 256)
        const VectorMatrix dw = random_matrix(600, 8, 71, -10, 10);
        const Codebook cbw = pq_fit(dw, 2, 300, 8, 3);
        const CodeMatrix cw = pq_encode(cbw, dw);
        CHECK(cw.code_width() == 2);
        std::vector<std::uint64_t> idw(600);
        std::iota(idw.begin(), idw.end(), std::uint64_t{0});
        const InvertedIndex iw = ivf_build(cbw, cw, idw, 5, 7);
        save_index(iw, dir + "/wide.pqii");
        const InvertedIndex lw = load_index(dir + "/wide.pqii");
        CHECK(lw.codebook == iw.codebook);
        for (std::size_t l = 0; l < iw.nlist(); ++l) {
            CHECK(lw.lists[l].ids == iw.lists[l].ids);
            CHECK(lw.lists[l].codes == iw.lists[l].codes);
        }
        // bad magic
        std::string ib = read_file(dir + "/a.pqii");
        ib[0] = 'Z';
        write_file(dir + "/bad.pqii", ib);
        CHECK_THROWS_WITH(load_index(dir + "/bad.pqii"), std::runtime_error, "bad magic");
        if (std::system(("rm -rf " + dir).c_str()) != 0) std::printf("rm failed\n");
    }
    // ---- test_pipeline.cpp
    {   // train_chunk :44-92
        const VectorMatrix chunk = clustered(120, 8, 5);
        const ChunkOutput one = train_chunk(chunk, 4, 1, 10, 3);
        CHECK(one.representatives.rows == 1 && one.representatives.dims == 8);
        for (std::size_t d = 0; d < 8; ++d) {
            double mean = 0.0;
            for (std::size_t i = 0; i < chunk.rows; ++i) mean += chunk.row(i)[d];
            mean /= double(chunk.rows);
            CHECK(std::fabs(one.representatives.row(0)[d] - mean) <= 1e-5 * std::max(1.0, std::fabs(mean)));
        }
        for (std::uint32_t ks : {2u, 8u, 32u}) {
            const ChunkOutput o = train_chunk(chunk, 4, ks, 10, 3);
            CHECK(o.representatives.rows == ks && o.representatives.dims == 8);
        }
        const VectorMatrix base = random_matrix(8, 8, 17, -5, 5);
        VectorMatrix data(96, 8);
        for (std::size_t i = 0; i < data.rows; ++i) std::memcpy(data.row(i), base.row(i % 8), 8 * sizeof(float));
        const ChunkOutput out = train_chunk(data, 4, 8, 25, 7);
        CHECK(out.local_rmse <= 1e-6);
        for (std::uint32_t m = 0; m < 4; ++m) {
            VectorMatrix got(8, 2), want(8, 2);
            for (std::size_t j = 0; j < 8; ++j) {
                std::memcpy(got.row(j), out.representatives.row(j) + m * 2, 2 * sizeof(float));
                std::memcpy(want.row(j), base.row(j) + m * 2, 2 * sizeof(float));
            }
            CHECK(rows_equal_as_sets(got, want, 1e-6));
        }
        CHECK(reconstruction_rmse(fit_global(out.representatives, 4, 8, 25, 3), data) <= 1e-6);
        CHECK_THROWS_WITH(train_chunk(clustered(4, 8, 1), 4, 8, 10, 0), std::invalid_argument,
                          "fewer than ks");
    }
    {   // aggregate_representatives :94-129
        std::vector<ChunkOutput> ordered(5);
        for (std::size_t c = 0; c < 5; ++c) {
            ordered[c].chunk_id = c;
            ordered[c].representatives = random_matrix(3, 2, c + 1);
        }
        std::vector<ChunkOutput> shuffled = {ordered[3], ordered[0], ordered[4], ordered[2], ordered[1]};
        CHECK(aggregate_representatives(ordered) == aggregate_representatives(shuffled));
        CHECK(aggregate_representatives({ordered[0]}) == ordered[0].representatives);
        std::vector<ChunkOutput> bad(2);
        bad[0].representatives = random_matrix(2, 3, 1);
        bad[1].chunk_id = 1;
        bad[1].representatives = random_matrix(2, 4, 2);
        CHECK_THROWS_WITH(aggregate_representatives(bad), std::invalid_argument, "dimension mismatch");
    }
    {   // fit_global :131-157
        const VectorMatrix data = clustered(600, 8, 21);
        ChunkOutput out = train_chunk(data, 4, 16, 20, 42);
        const Codebook global = fit_global(aggregate_representatives({out}), 4, 16, 20, 42);
        const Codebook local = pq_fit(data, 4, 16, 20, 42);
        for (std::uint32_t m = 0; m < 4; ++m) {
            VectorMatrix g(16, 2), l(16, 2);
            std::memcpy(g.values.data(), global.sub_table(m), 16 * 2 * sizeof(float));
            std::memcpy(l.values.data(), local.sub_table(m), 16 * 2 * sizeof(float));
            CHECK(rows_equal_as_sets(g, l, 1e-6));
        }
        const Codebook cb = fit_global(VectorMatrix(10, 4, 2.5f), 2, 4, 10, 1);
        CodeMatrix codes(1, 2, 4);
        codes.set(0, 0, 3);
        codes.set(0, 1, 1);
        const VectorMatrix dec = pq_decode(cb, codes);
        for (std::size_t t = 0; t < 4; ++t) CHECK(dec.row(0)[t] == 2.5f);
    }
    {   // run_pipeline :159-255
        const VectorMatrix data = clustered(800, 8, 33);
        PipelineConfig config;
        config.m_subspaces = 4;
        config.ks = 16;
        config.kmeans_iters = 15;
        config.seed = 3;
        const PipelineReport a = run_pipeline(data, config);
        config.mode = PipelineMode::kParallelPq;
        const PipelineReport b = run_pipeline(data, config);
        CHECK(std::fabs(a.global_rmse - b.global_rmse) <= 1e-6);
        CHECK(a.single_rmse.has_value() && !b.single_rmse.has_value() && b.representatives.has_value());

        const VectorMatrix d2 = clustered(700, 8, 61);
        PipelineConfig c2;
        c2.mode = PipelineMode::kParallelPqIndex;
        c2.n_chunks = 5;
        c2.m_subspaces = 4;
        c2.ks = 16;
        c2.nlist = 9;
        c2.kmeans_iters = 10;
        c2.seed = 11;
        c2.n_threads = 2;
        const PipelineReport r = run_pipeline(d2, c2);
        c2.n_threads = 1;
        const PipelineReport r1 = run_pipeline(d2, c2);
        CHECK(r.global_codebook == r1.global_codebook && r.global_rmse == r1.global_rmse);
        CHECK(r.merged_index.has_value() && r.merged_index->n_items == d2.rows);
        const CodeMatrix codes = pq_encode(r.global_codebook, d2);
        std::vector<std::uint64_t> ids(d2.rows);
        std::iota(ids.begin(), ids.end(), std::uint64_t{0});
        const VectorMatrix qs = random_matrix(12, 8, 5, -2, 12);
        for (std::size_t q = 0; q < qs.rows; ++q) {
            const auto x = ivf_query(*r.merged_index, qs.row_span(q), 8, r.merged_index->nlist());
            CHECK(x.hits == flat_scan(r.global_codebook, codes, ids, qs.row_span(q), 8).hits);
        }
        for (const char* ph : {"chunking", "local_fit", "global_fit", "coarse_fit", "encode",
                               "index_build", "merge"})
            CHECK(r.phase_seconds.count(ph) && r.phase_seconds.at(ph) >= 0.0);
        CHECK(r.summary().find("index: 700 items across 9 lists") != std::string::npos);

        PipelineConfig bad;
        bad.mode = PipelineMode::kParallelPq;
        bad.n_chunks = 5;
        bad.m_subspaces = 2;
        bad.ks = 3;
        bad.n_threads = 2;
        CHECK_THROWS_WITH(run_pipeline(clustered(10, 4, 71), bad), std::runtime_error, "chunk ");
        CHECK_THROWS_WITH(run_pipeline(clustered(10, 4, 71), bad), std::runtime_error, "fewer than ks");
        CHECK(parse_mode("parallel_pq_index") == PipelineMode::kParallelPqIndex && !parse_mode("x"));

        const VectorMatrix d3 = clustered(200, 8, 81);
        const ChunkOutput o = train_chunk(d3, 4, 8, 10, 9);
        CHECK(std::fabs(o.local_rmse - reconstruction_rmse(pq_fit(d3, 4, 8, 10, 9), d3)) <=
              1e-12 * o.local_rmse);
    }
    std::printf("facade_test: %d checks, %d failures\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
