// Per-call latency of the C++ drop-in (libpqg_pqii.so) on a configs[2]-sized
// index built directly through the public structs: 1M items, D = 128, M = 16,
// Ks = 256, nlist = 1024.  Times the first ivf_query (upload), then single
// ivf_query calls (nprobe 16, k 10), then one 10k-query ivf_query_batch.
// One JSON line.
//   g++ -std=c++20 -O2 -Iinclude tools/facade_latency.cpp -Lpaper_2604_21645_b200 \
//       -lpqg_pqii -lpqg -Wl,-rpath,$PWD/paper_2604_21645_b200 -o /tmp/fl && /tmp/fl
#include <chrono>
#include <cstdio>
#include <random>

#include "pqii/ivf.hpp"

using namespace pqii;
using Clock = std::chrono::steady_clock;

static double ms_since(Clock::time_point t) {
    return std::chrono::duration<double, std::milli>(Clock::now() - t).count();
}

int main() {
    const std::size_t N = 1000000, D = 128, nlist = 1024, nq = 10000;
    const std::uint32_t M = 16, ks = 256;
    std::mt19937_64 rng(2604);
    std::normal_distribution<float> g(0.f, 1.f);
    InvertedIndex ix;
    ix.codebook.m_subspaces = M;
    ix.codebook.ks = ks;
    ix.codebook.sub_dim = D / M;
    ix.codebook.tables.resize(std::size_t(M) * ks * (D / M));
    for (auto& v : ix.codebook.tables) v = g(rng);
    ix.coarse_centroids = VectorMatrix(nlist, D);
    for (auto& v : ix.coarse_centroids.values) v = g(rng);
    ix.lists.resize(nlist);
    for (auto& pl : ix.lists) pl.codes = CodeMatrix(0, M, ks);
    std::uniform_int_distribution<std::size_t> pick(0, nlist - 1);
    for (std::size_t i = 0; i < N; ++i) {
        PostingList& pl = ix.lists[pick(rng)];
        pl.ids.push_back(i);
        for (std::uint32_t m = 0; m < M; ++m) pl.codes.bytes.push_back(std::uint8_t(rng() & 255u));
        ++pl.codes.rows;
    }
    ix.n_items = N;
    ix.id_set.reserve(N);
    for (std::size_t i = 0; i < N; ++i) ix.id_set.insert(i);
    VectorMatrix qs(nq, D);
    for (auto& v : qs.values) v = g(rng);

    auto t0 = Clock::now();
    QueryResult r = ivf_query(ix, qs.row_span(0), 10, 16);
    const double first_ms = ms_since(t0);
    const int reps = 500;
    t0 = Clock::now();
    std::size_t hits = 0;
    for (int i = 0; i < reps; ++i) hits += ivf_query(ix, qs.row_span(1 + i), 10, 16).hits.size();
    const double per_call_us = ms_since(t0) * 1e3 / reps;
    t0 = Clock::now();
    const auto batch = ivf_query_batch(ix, qs, 10, 16);
    const double batch_ms = ms_since(t0);
    std::printf("{\"items\": %zu, \"nlist\": %zu, \"M\": %u, \"Ks\": %u, \"nprobe\": 16, \"k\": 10, "
                "\"first_query_ms\": %.3f, \"ivf_query_us_per_call\": %.2f, \"calls\": %d, "
                "\"batch_10k_ms\": %.3f, \"batch_queries_per_s\": %.1f, \"hits_checked\": %zu}\n",
                N, nlist, M, ks, first_ms, per_call_us, reps, batch_ms, nq / (batch_ms / 1e3),
                hits + r.hits.size() + batch.size());
    return 0;
}
