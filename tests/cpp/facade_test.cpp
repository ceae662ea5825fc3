// facade_test.cpp -- the reference's unit-test cases (proj/tests/test_kmeans.cpp,
// test_pq.cpp, test_ivf.cpp) restated against the drop-in libpqg_pqii.so
// through the pqii headers of this repo.  A tiny CHECK harness replaces the
// absent doctest.  Run by tests/test_facade_cpp.py on a GPU.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "pqii/ivf.hpp"
#include "pqii/kmeans.hpp"
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
    }
    std::printf("facade_test: %d checks, %d failures\n", g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
