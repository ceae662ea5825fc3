// capi.cu -- the extern "C" boundary (include/pqg.h) and the host-side
// orchestration of the device hot path: the batched Lloyd loop, pq_fit,
// encode/decode/RMSE, index build/add/merge and batched search.
//
// Host code here only validates arguments (with the reference's messages),
// stages host buffers, draws the k-means init indices exactly as the
// reference does (libstdc++ mt19937_64 + uniform_int_distribution, the same
// GCC 13 headers) and sequences kernels.  There is no CPU compute fallback:
// every numeric result comes from the kernels in nearest.cu, kmeans.cu,
// pq.cu and ivf.cu.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <tuple>
#include <memory>
#include <numeric>
#include <random>
#include <string>
#include <unordered_map>
#include <vector>

#include "kernels.cuh"

using namespace pqg;

// ---------------------------------------------------------------------------
// error plumbing
// ---------------------------------------------------------------------------
static thread_local std::string g_last_error;

template <class F>
static int guard(F&& f) {
    try {
        f();
        return PQG_OK;
    } catch (const Error& e) {
        g_last_error = e.msg;
        return e.code;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return PQG_ECUDA;
    } catch (...) {
        g_last_error = "unknown error";
        return PQG_ECUDA;
    }
}

static void inval(const std::string& m) { fail(PQG_EINVAL, m); }

namespace pqg {
// the other translation units' C entry points (kmnccl.cu) report through here
void set_last_error(const std::string& m) { g_last_error = m; }
}  // namespace pqg

// ---------------------------------------------------------------------------
// host / device pointer staging
// ---------------------------------------------------------------------------
static bool on_device(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

template <class T>
static const T* in(pqg_ctx* ctx, const T* p, uint64_t count) {
    if (!p || count == 0 || on_device(p)) return p;
    T* d = scratch<T>(ctx, count);
    PQG_CUDA(cudaMemcpyAsync(d, p, count * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
    return d;
}

template <class T>
struct Out {
    T* user = nullptr;
    T* dev = nullptr;
    uint64_t count = 0;
    bool host = false;
};

template <class T>
static Out<T> out(pqg_ctx* ctx, T* p, uint64_t count) {
    Out<T> o;
    o.user = p;
    o.count = count;
    if (!p) return o;
    if (on_device(p)) {
        o.dev = p;
    } else {
        o.host = true;
        o.dev = scratch<T>(ctx, std::max<uint64_t>(count, 1));
    }
    return o;
}

template <class T>
static void finish(pqg_ctx* ctx, const Out<T>& o) {
    if (o.host && o.count)
        PQG_CUDA(cudaMemcpyAsync(o.user, o.dev, o.count * sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
}

static void sync(pqg_ctx* ctx) { PQG_CUDA(cudaStreamSynchronize(ctx->stream)); }

// The device error word collects out-of-range code reports.  A call whose
// outputs all stay on the device does not synchronise to read it: the flag is
// left pending (err_pending) and reported by the next pqg_ctx_sync /
// pqg_ctx_check_errors, and later calls do not clear it until then.
static void reset_err(pqg_ctx* ctx) {
    if (ctx->err_pending) return;
    PQG_CUDA(cudaMemsetAsync(ctx->d_err, 0, sizeof(int), ctx->stream));
}

static int read_err(pqg_ctx* ctx) {
    int h = 0;
    PQG_CUDA(cudaMemcpyAsync(&h, ctx->d_err, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    ctx->err_pending = false;
    return h;
}

static uint32_t code_width(uint32_t ks) { return ks <= 256 ? 1 : 2; }

// ---------------------------------------------------------------------------
// small kernels local to the orchestration
// ---------------------------------------------------------------------------
__global__ void codes_check_kernel(const uint8_t* codes, uint64_t n, uint32_t M, uint32_t ks,
                                   uint32_t w, int* err) {
    const uint64_t total = n * M;
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += uint64_t(gridDim.x) * blockDim.x) {
        const uint8_t* p = codes + e * w;
        const uint32_t c = w == 1 ? p[0] : (uint32_t(p[0]) | (uint32_t(p[1]) << 8));
        if (c >= ks) atomicExch(err, 1);
    }
}

// CSR concatenation per list: entries of a keep their slot shifted by the b
// entries of earlier lists; entries of b follow a's list (ivf.cpp:203-211).
__global__ void csr_concat_kernel(const uint64_t* off_a, const uint64_t* ids_a,
                                  const uint8_t* codes_a, uint64_t na, const uint64_t* off_b,
                                  const uint64_t* ids_b, const uint8_t* codes_b, uint64_t nb,
                                  uint64_t nlist, uint64_t rb, uint64_t* off_o, uint64_t* ids_o,
                                  uint8_t* codes_o) {
    const uint64_t total = na + nb;
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total + nlist + 1;
         e += uint64_t(gridDim.x) * blockDim.x) {
        if (e >= total) {
            const uint64_t l = e - total;
            off_o[l] = off_a[l] + off_b[l];
            continue;
        }
        const bool from_a = e < na;
        const uint64_t x = from_a ? e : e - na;
        const uint64_t* off = from_a ? off_a : off_b;
        // list of entry x: last l with off[l] <= x
        uint64_t lo = 0, hi = nlist;
        while (hi - lo > 1) {
            const uint64_t mid = (lo + hi) >> 1;
            if (off[mid] <= x) lo = mid; else hi = mid;
        }
        // skip empty lists sharing the offset
        while (lo + 1 < nlist && off[lo + 1] <= x) ++lo;
        const uint64_t dst = from_a ? x + off_b[lo] : x + off_a[lo + 1];
        ids_o[dst] = from_a ? ids_a[x] : ids_b[x];
        const uint8_t* s = (from_a ? codes_a : codes_b) + x * rb;
        for (uint64_t j = 0; j < rb; ++j) codes_o[dst * rb + j] = s[j];
    }
}

__global__ void iota_u64_kernel(uint64_t* p, uint64_t n) {
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
         e += uint64_t(gridDim.x) * blockDim.x)
        p[e] = e;
}

// ---------------------------------------------------------------------------
// context and index objects
// ---------------------------------------------------------------------------
struct pqg_index {
    int device = 0;
    uint32_t M = 0, ks = 0, ds = 0, w = 1;
    uint64_t nlist = 0, n = 0;
    float* tables = nullptr;
    float* coarse = nullptr;
    float* coarse_norm = nullptr;
    float* coarse_max = nullptr;
    uint64_t* offsets = nullptr;
    uint64_t* ids = nullptr;
    uint8_t* codes = nullptr;

    uint64_t D() const { return uint64_t(M) * ds; }
    uint64_t rb() const { return uint64_t(M) * w; }
    IndexView view() const {
        return IndexView{tables, M, ks, ds, w, coarse, coarse_norm, coarse_max, nlist,
                         offsets, ids, codes, n};
    }
    void free_all() {
        for (void* p : {(void*)tables, (void*)coarse, (void*)coarse_norm, (void*)coarse_max,
                        (void*)offsets, (void*)ids, (void*)codes})
            if (p) cudaFree(p);
        tables = coarse = coarse_norm = coarse_max = nullptr;
        offsets = ids = nullptr;
        codes = nullptr;
    }
};

template <class T>
static T* dalloc(uint64_t count) {
    T* p = nullptr;
    if (cudaMalloc(&p, std::max<uint64_t>(count, 1) * sizeof(T)) != cudaSuccess) {
        cudaGetLastError();
        fail(PQG_ENOMEM, "device allocation of " + std::to_string(count * sizeof(T)) + " bytes failed");
    }
    return p;
}

static pqg_index* new_index(pqg_ctx* ctx, uint32_t M, uint32_t ks, uint32_t ds, uint64_t nlist,
                            uint64_t n, const float* d_tables, const float* d_coarse) {
    pqg_index* ix = new pqg_index;
    ix->device = ctx->device;
    ix->M = M; ix->ks = ks; ix->ds = ds; ix->w = code_width(ks);
    ix->nlist = nlist; ix->n = n;
    try {
        ix->tables = dalloc<float>(uint64_t(M) * ks * ds);
        ix->coarse = dalloc<float>(nlist * ix->D());
        ix->coarse_norm = dalloc<float>(nlist);
        ix->coarse_max = dalloc<float>(1);
        ix->offsets = dalloc<uint64_t>(nlist + 1);
        ix->ids = dalloc<uint64_t>(n);
        ix->codes = dalloc<uint8_t>(n * ix->rb());
        PQG_CUDA(cudaMemcpyAsync(ix->tables, d_tables, sizeof(float) * M * ks * ds,
                                 cudaMemcpyDeviceToDevice, ctx->stream));
        PQG_CUDA(cudaMemcpyAsync(ix->coarse, d_coarse, sizeof(float) * nlist * ix->D(),
                                 cudaMemcpyDeviceToDevice, ctx->stream));
        table_norms(ctx, ix->coarse, 1, nlist, uint32_t(ix->D()), ix->coarse_norm, ix->coarse_max);
    } catch (...) {
        ix->free_all();
        delete ix;
        throw;
    }
    return ix;
}

// ---------------------------------------------------------------------------
// k-means engine (B problems batched; proj/src/kmeans.cpp:61-133 each)
// ---------------------------------------------------------------------------
// Init indices exactly as kmeans_fit (kmeans.cpp:73-85): partial Fisher-Yates
// over iota(n) driven by mt19937_64(seed) and uniform_int_distribution(i, n-1);
// the permutation is kept sparse (only touched slots are stored).
static std::vector<uint64_t> init_rows(uint64_t n, uint64_t k, uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::unordered_map<uint64_t, uint64_t> perm;
    perm.reserve(2 * k);
    auto get = [&](uint64_t i) {
        auto it = perm.find(i);
        return it == perm.end() ? i : it->second;
    };
    for (uint64_t i = 0; i < k; ++i) {
        std::uniform_int_distribution<std::size_t> pick(i, n - 1);
        const uint64_t j = pick(rng);
        const uint64_t vi = get(i), vj = get(j);
        perm[i] = vj;
        perm[j] = vi;
    }
    std::vector<uint64_t> rows(k);
    for (uint64_t c = 0; c < k; ++c) rows[c] = get(c);
    return rows;
}

struct KMeansOut {
    std::vector<double> inertia;   // [B]
    std::vector<uint32_t> iters;   // [B]
    std::vector<double> per_iter;  // [B][max_iters]
};

// x: device rows (n x ldx); table (device, B*k*d) receives the centroids;
// assign (device, B*n u32) receives the final assignments.  counts (optional,
// B entries <= n): problem b fits only its first counts[b] rows -- the
// batched local fits of the chunked pipeline, whose chunks differ by a row.
static KMeansOut run_kmeans(pqg_ctx* ctx, const float* x, uint64_t n, uint64_t ldx, uint32_t B,
                            uint32_t d, uint32_t col_stride, uint64_t k, uint32_t max_iters,
                            const std::vector<uint64_t>& seeds, double tol, float* table,
                            uint32_t* assign, const std::vector<uint64_t>* counts = nullptr) {
    std::vector<uint64_t> rows;
    rows.reserve(uint64_t(B) * k);
    uint64_t max_pad = 0;
    for (uint32_t b = 0; b < B; ++b) {
        const uint64_t nb = counts ? (*counts)[b] : n;
        max_pad = std::max(max_pad, n - nb);
        auto r = init_rows(nb, k, seeds[b]);
        rows.insert(rows.end(), r.begin(), r.end());
    }
    const uint64_t* d_nb = nullptr;
    if (max_pad) {
        uint64_t* p = scratch<uint64_t>(ctx, B);
        PQG_CUDA(cudaMemcpyAsync(p, counts->data(), sizeof(uint64_t) * B, cudaMemcpyHostToDevice,
                                 ctx->stream));
        d_nb = p;
    }
    // Batched fits over rows larger than L2: copy the B column blocks into a
    // problem-major layout once per fit, so each problem's rows are one dense
    // region -- the assignment passes and the member gathers of the update
    // then stay within L2 instead of re-fetching whole rows from HBM for
    // every problem.
    if (B > 1 && uint64_t(B) * n * d * sizeof(float) >= (uint64_t(64) << 20)) {
        if (uint64_t(n) * d > 0xFFFFFFFFull) fail(PQG_EUNSUPPORTED, "kmeans: problem block too large");
        float* xt = scratch<float>(ctx, uint64_t(B) * n * d);
        transpose_blocks(ctx, x, n, ldx, B, d, col_stride, xt);
        x = xt;
        ldx = d;
        col_stride = uint32_t(n * d);
    }
    uint64_t* d_rows = scratch<uint64_t>(ctx, rows.size());
    PQG_CUDA(cudaMemcpyAsync(d_rows, rows.data(), rows.size() * sizeof(uint64_t),
                             cudaMemcpyHostToDevice, ctx->stream));
    gather_rows(ctx, x, ldx, B, d, col_stride, d_rows, k, table);

    KMeansState st;
    st.active = scratch<int>(ctx, B);
    st.prev = scratch<double>(ctx, B);
    st.inertia = scratch<double>(ctx, B);
    st.per_iter = scratch<double>(ctx, uint64_t(B) * max_iters);
    st.iters = scratch<uint32_t>(ctx, B);
    st.tickets = scratch<unsigned>(ctx, B);
    PQG_CUDA(cudaMemsetAsync(st.tickets, 0, sizeof(unsigned) * B, ctx->stream));
    std::vector<int> ones(B, 1);
    PQG_CUDA(cudaMemcpyAsync(st.active, ones.data(), sizeof(int) * B, cudaMemcpyHostToDevice, ctx->stream));
    PQG_CUDA(cudaMemsetAsync(st.prev, 0, sizeof(double) * B, ctx->stream));
    PQG_CUDA(cudaMemsetAsync(st.per_iter, 0, sizeof(double) * B * max_iters, ctx->stream));
    float* cnorm = scratch<float>(ctx, uint64_t(B) * k);
    float* cmax = scratch<float>(ctx, B);
    double* dist = scratch<double>(ctx, uint64_t(B) * n);

    RowSrc src;
    src.x = x;
    src.ldx = ldx;
    src.col_stride = col_stride;
    // coarse fits (one problem, large d and k): split the row operand for the
    // tensor-core screen once; every assignment pass reuses it
    NearestArgs prep;
    prep.src = src;
    prep.n = n;
    prep.d = d;
    prep.B = B;
    prep.k = k;
    prep.cmax = cmax;
    const bool big = B == 1 && umma_big_prepare_rows(ctx, prep);
    PQG_CUDA(cudaMemsetAsync(st.iters, 0, sizeof(uint32_t) * B, ctx->stream));
    const auto iter_mark = ctx->arena.mark();
    // small tables (PQ subspaces): the reseed block of each problem computes
    // the next pass's norms; large ones (coarse fits) keep the wide kernel
    const bool fuse_norms = uint64_t(k) * d <= 8192;
    auto body = [&](uint32_t it, bool update) {
        ctx->arena.reset_to(iter_mark);  // per-iteration scratch is reused
        // the first pass's norms; later passes get theirs from the previous
        // update (reseed_kernel computes them once the table is final)
        if (it == 1 || !fuse_norms) table_norms(ctx, table, B, k, d, cnorm, cmax);
        NearestArgs a;
        a.src = src;
        a.n = n;
        a.d = d;
        a.B = B;
        a.table = table;
        a.k = k;
        a.cnorm = cnorm;
        a.cmax = cmax;
        a.out_idx = assign;
        a.idx_bytes = 4;
        a.idx_rs = 1;
        a.idx_ps = n;
        a.out_dist = dist;
        a.active = st.active;
        if (big) {
            a.big_rows = prep.big_rows;
            a.big_nx = prep.big_nx;
        }
        nearest(ctx, a);
        kmeans_pad_keys(ctx, assign, n, B, k, d_nb, max_pad);
        kmeans_inertia_and_stop(ctx, dist, n, B, it, max_iters, tol, st, d_nb);
        if (update)
            kmeans_update(ctx, src, n, B, d, table, k, assign, dist, st.active, d_nb, fuse_norms ? cnorm : nullptr,
                          cmax);
    };
    // Iterations 2 .. max_iters-1 are identical launch sequences (the pass
    // number lives on the device, inactive problems are skipped by the
    // kernels): captured once into a CUDA graph and replayed, so the ~15
    // small launches of an iteration go to the GPU as one.  Iteration 1 runs
    // eagerly first (it sizes the scratch the graph then reuses).
    const char* ge = std::getenv("PQG_KM_GRAPH");
    // (the legacy / per-thread default streams cannot be captured)
    const bool capturable = ctx->stream != nullptr && ctx->stream != cudaStreamLegacy &&
                            ctx->stream != cudaStreamPerThread;
    const bool use_graph = !ctx->profiling && !(ge && ge[0] == '0') && !std::getenv("PQG_FLAG_STATS") &&
                           max_iters >= 3 && capturable;
    cudaGraphExec_t gexec = nullptr;
    uint64_t body_launches = 0;
    try {
        for (uint32_t it = 1; it <= max_iters; ++it) {
            const bool last = it == max_iters;
            if (use_graph && it >= 2 && !last) {
                if (!gexec) {
                    const uint64_t l0 = ctx->launches;
                    PQG_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeRelaxed));
                    try {
                        body(it, true);
                    } catch (...) {
                        cudaGraph_t g = nullptr;
                        cudaStreamEndCapture(ctx->stream, &g);
                        if (g) cudaGraphDestroy(g);
                        throw;
                    }
                    cudaGraph_t g = nullptr;
                    PQG_CUDA(cudaStreamEndCapture(ctx->stream, &g));
                    const cudaError_t ie = cudaGraphInstantiate(&gexec, g, 0);
                    cudaGraphDestroy(g);
                    if (ie != cudaSuccess) fail(PQG_ECUDA, std::string("kmeans graph: ") + cudaGetErrorString(ie));
                    body_launches = ctx->launches - l0;
                    ctx->launches = l0;
                }
                PQG_CUDA(cudaGraphLaunch(gexec, ctx->stream));
                ctx->launches += body_launches;
            } else {
                body(it, !last);
            }
        }
    } catch (...) {
        if (gexec) cudaGraphExecDestroy(gexec);
        throw;
    }
    KMeansOut o;
    o.inertia.resize(B);
    o.iters.resize(B);
    o.per_iter.resize(uint64_t(B) * max_iters);
    PQG_CUDA(cudaMemcpyAsync(o.inertia.data(), st.inertia, sizeof(double) * B, cudaMemcpyDeviceToHost, ctx->stream));
    PQG_CUDA(cudaMemcpyAsync(o.iters.data(), st.iters, sizeof(uint32_t) * B, cudaMemcpyDeviceToHost, ctx->stream));
    PQG_CUDA(cudaMemcpyAsync(o.per_iter.data(), st.per_iter, sizeof(double) * B * max_iters,
                             cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    if (gexec) cudaGraphExecDestroy(gexec);
    return o;
}

// Encode n rows (device) into codes (device) in row chunks.
static void encode_dev(pqg_ctx* ctx, const float* x, uint64_t n, uint32_t M, uint32_t ks,
                       uint32_t ds, const float* tables, uint8_t* codes) {
    float* cnorm = scratch<float>(ctx, uint64_t(M) * ks);
    float* cmax = scratch<float>(ctx, M);
    table_norms(ctx, tables, M, ks, ds, cnorm, cmax);
    const uint64_t D = uint64_t(M) * ds;
    const uint32_t w = code_width(ks);
    const uint64_t chunk = std::max<uint64_t>(1, (uint64_t(64) << 20) / M);
    const auto chunk_mark = ctx->arena.mark();
    for (uint64_t r0 = 0; r0 < n; r0 += chunk) {
        ctx->arena.reset_to(chunk_mark);
        const uint64_t nc = std::min(chunk, n - r0);
        NearestArgs a;
        a.src.x = x + r0 * D;
        a.src.ldx = D;
        a.src.col_stride = ds;
        a.n = nc;
        a.d = ds;
        a.B = M;
        a.table = tables;
        a.k = ks;
        a.cnorm = cnorm;
        a.cmax = cmax;
        a.out_idx = codes + r0 * M * w;
        a.idx_bytes = int(w);
        a.idx_rs = M;
        a.idx_ps = 1;
        nearest(ctx, a);
    }
}

static void check_pq_shape(uint32_t M, uint32_t ks, uint32_t ds, const char* who) {
    if (M == 0) inval(std::string(who) + ": M must be >= 1");
    if (ks == 0 || ks > 65536) inval(std::string(who) + ": Ks must be in [1, 65536]");
    if (ds == 0) inval(std::string(who) + ": sub_dim must be >= 1");
}

// pq_fit's argument checks, in its order (proj/src/pq.cpp:65-75, then
// kmeans_fit's max_iters check, kmeans.cpp:70)
static void check_pq_fit(uint64_t n, uint64_t D, uint32_t M, uint32_t ks, uint32_t max_iters) {
    if (M == 0) inval("pq_fit: M must be >= 1");
    if (D % M != 0)
        inval("pq_fit: D (" + std::to_string(D) + ") is not divisible by M (" + std::to_string(M) +
              ")");
    if (ks > n)
        inval("pq_fit: Ks (" + std::to_string(ks) + ") exceeds number of rows (" +
              std::to_string(n) + ")");
    check_pq_shape(M, uint32_t(ks), uint32_t(D / M), "codebook");
    if (max_iters < 1) inval("kmeans_fit: max_iters must be >= 1");
}

// ---------------------------------------------------------------------------
// index construction helpers
// ---------------------------------------------------------------------------
static void check_unique_ids(pqg_ctx* ctx, const uint64_t* d_ids, const uint64_t* h_ids,
                             uint64_t n, const std::string& prefix) {
    if (n < 2) return;
    uint64_t* pos = scratch<uint64_t>(ctx, 1);
    find_duplicate(ctx, d_ids, n, pos);
    uint64_t h = 0;
    PQG_CUDA(cudaMemcpyAsync(&h, pos, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    if (h != ~uint64_t(0)) {
        uint64_t id = 0;
        if (h_ids) id = h_ids[h];
        else PQG_CUDA(cudaMemcpy(&id, d_ids + h, sizeof(id), cudaMemcpyDeviceToHost));
        inval(prefix + std::to_string(id));
    }
}

// Build CSR lists for n items with list ids (device) into a fresh index.
static void fill_lists(pqg_ctx* ctx, pqg_index* ix, const uint32_t* list_of, const uint64_t* ids,
                       const uint8_t* codes, uint64_t n) {
    Bucketing bk{ix->offsets, scratch<uint32_t>(ctx, std::max<uint64_t>(n, 1))};
    if (n == 0) {
        PQG_CUDA(cudaMemsetAsync(ix->offsets, 0, sizeof(uint64_t) * (ix->nlist + 1), ctx->stream));
        return;
    }
    stable_bucket(ctx, list_of, n, 1, ix->nlist, nullptr, bk);
    csr_scatter(ctx, bk.perm, n, ids, codes, ix->rb(), ix->ids, ix->codes);
}

static uint32_t* assign_lists(pqg_ctx* ctx, const float* tables, uint32_t M, uint32_t ks,
                              uint32_t ds, const uint8_t* codes, uint64_t n, const float* coarse,
                              const float* cnorm, const float* cmax, uint64_t nlist) {
    reset_err(ctx);
    const uint32_t w = code_width(ks);
    launch(ctx, "codes_check", codes_check_kernel, dim3(grid1d(n * M, 256, ctx->num_sms * 8)),
           dim3(256), 0, codes, n, M, ks, w, ctx->d_err);
    uint32_t* list_of = scratch<uint32_t>(ctx, std::max<uint64_t>(n, 1));
    NearestArgs a;
    a.src.codes = codes;
    a.src.dtab = tables;
    a.src.dM = M;
    a.src.dks = ks;
    a.src.dds = ds;
    a.src.dw = w;
    a.n = n;
    a.d = M * ds;
    a.B = 1;
    a.table = coarse;
    a.k = nlist;
    a.cnorm = cnorm;
    a.cmax = cmax;
    a.out_idx = list_of;
    a.idx_bytes = 4;
    a.idx_rs = 1;
    a.idx_ps = 0;
    nearest(ctx, a);
    if (read_err(ctx)) fail(PQG_ERANGE, "pq_decode: code out of range for Ks=" + std::to_string(ks));
    return list_of;
}


// ---------------------------------------------------------------------------
// the paper's chunked pipeline (proj/src/pipeline.cpp)
// ---------------------------------------------------------------------------
// chunk_rows (proj/src/dataset_io.cpp:322-339) as (base, extra): chunk c holds
// base + (c < extra) rows.
static void check_chunks(uint64_t n, uint64_t C) {
    if (C == 0) inval("chunk_rows: n_chunks must be >= 1");
    if (C > n)
        inval("chunk_rows: n_chunks (" + std::to_string(C) + ") exceeds n_rows (" +
              std::to_string(n) + ")");
}

// run_chunk_tasks reports the lowest-id failing chunk as a runtime_error
// "chunk <id>: <what>" (pipeline.cpp:30-62); train_chunk checks the row count before pq_fit's own
// checks (pipeline.cpp:84-90).  Chunk 0 is the largest, so a size-independent
// pq_fit failure always surfaces as chunk 0.
static void check_train_chunks(uint64_t n, uint64_t D, uint64_t C, uint32_t M, uint32_t ks,
                               uint32_t iters) {
    check_chunks(n, C);
    const uint64_t base = n / C, extra = n % C, n_max = base + (extra ? 1 : 0);
    auto rows_err = [&](uint64_t c, uint64_t rows) {
        fail(PQG_ECHUNK, "chunk " + std::to_string(c) + ": train_chunk: chunk has " +
                             std::to_string(rows) + " rows, fewer than ks=" + std::to_string(ks));
    };
    if (n_max < ks) rows_err(0, n_max);
    try {
        check_pq_fit(n_max, D, M, ks, iters);
    } catch (Error& e) {
        fail(PQG_ECHUNK, "chunk 0: " + e.msg);
    }
    if (base < ks) rows_err(extra, base);
}

struct ChunkFits {
    float* reps = nullptr;       // device [C*ks][D]
    std::vector<double> rmse;    // [C]
    std::vector<uint32_t> iters; // [C*M]
};

// train_chunk for every chunk at once (pipeline.cpp:84-106): the C chunks are
// laid side by side so the C*M local subspace fits run as ONE batched k-means
// (problem c*M+m: chunk c's rows, subspace m's columns, seed (seed+c)+m, its
// own init, tol stop and reseeds).  Each chunk's reconstruction RMSE comes
// from the fit's final assignments.  x: device n x D.
static ChunkFits train_chunks_dev(pqg_ctx* ctx, const float* x, uint64_t n, uint64_t D, uint64_t C,
                                  uint32_t M, uint32_t ks, uint32_t iters, uint64_t seed) {
    const uint64_t base = n / C, extra = n % C, n_max = base + (extra ? 1 : 0);
    const uint32_t ds = uint32_t(D / M);
    const uint64_t B64 = C * M;
    if (B64 > (1u << 20)) fail(PQG_EUNSUPPORTED, "train_chunks: n_chunks * M too large");
    const uint32_t B = uint32_t(B64);
    const float* y = x;
    if (C > 1) {
        float* yy = scratch<float>(ctx, n_max * C * D);
        interleave_chunks(ctx, x, D, C, base, extra, n_max, yy);
        y = yy;
    }
    float* tables = scratch<float>(ctx, B64 * ks * ds);
    uint32_t* assign = scratch<uint32_t>(ctx, B64 * n_max);
    std::vector<uint64_t> seeds(B), counts(B);
    for (uint64_t c = 0; c < C; ++c)
        for (uint32_t m = 0; m < M; ++m) {
            seeds[c * M + m] = (seed + c) + m;  // chunk_seed = seed + c (pipeline.cpp:190), pq.cpp:88
            counts[c * M + m] = base + (c < extra ? 1 : 0);
        }
    KMeansOut r = run_kmeans(ctx, y, n_max, C * D, B, ds, ds, ks, iters, seeds, 1e-4, tables,
                             assign, extra ? &counts : nullptr);
    ChunkFits f;
    f.reps = scratch<float>(ctx, C * ks * D);
    chunk_representatives(ctx, tables, C, M, ks, ds, f.reps);
    double* sse = scratch<double>(ctx, C);
    chunk_sse(ctx, x, C, M, ks, ds, base, extra, assign, n_max, tables, sse);
    f.rmse.resize(C);
    PQG_CUDA(cudaMemcpyAsync(f.rmse.data(), sse, sizeof(double) * C, cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    for (uint64_t c = 0; c < C; ++c)
        f.rmse[c] = std::sqrt(f.rmse[c] / double((base + (c < extra ? 1 : 0)) * D));  // pq.cpp:169-177
    f.iters = r.iters;
    return f;
}

static uint64_t default_nlist_of(uint64_t n) {  // proj/src/ivf.cpp:118-121
    const uint64_t r = uint64_t(std::llround(std::sqrt(double(n))));
    return std::clamp<uint64_t>(r, 1, n == 0 ? 1 : n);
}

using Clock = std::chrono::steady_clock;
static double seconds_since(Clock::time_point t) {
    return std::chrono::duration<double>(Clock::now() - t).count();
}

// Search of nq queries with their probe lists: the LUT scan (ivf.cu).
// The query LUTs of a search batch (adc_luts_kernel) do not depend on the
// probe lists: they are built on the context's side stream while the probe
// kernels run on the main one (r2), and the scan loads them.  Returns null
// (the scan builds its own) when the batch is small, the shape is not
// covered or PQG_ADC_LUT=0.
static const float* search_luts_async(pqg_ctx* ctx, const pqg_index* ix, const float* dq, uint64_t nq) {
    const char* le = std::getenv("PQG_ADC_LUT");
    if ((le && le[0] == '0') || nq < 64 || nq > 16384 || ix->ks > 256 ||
        !(ix->ds == 4 || ix->ds == 8 || ix->ds == 16 || ix->ds == 32))
        return nullptr;
    float* luts = scratch<float>(ctx, nq * ix->M * ix->ks);
    if (!ctx->copy_stream) PQG_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    if (!ctx->pipe_ev[2]) PQG_CUDA(cudaEventCreateWithFlags(&ctx->pipe_ev[2], cudaEventDisableTiming));
    if (!ctx->pipe_ev[3]) PQG_CUDA(cudaEventCreateWithFlags(&ctx->pipe_ev[3], cudaEventDisableTiming));
    PQG_CUDA(cudaEventRecord(ctx->pipe_ev[2], ctx->stream));
    PQG_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->pipe_ev[2], 0));
    cudaStream_t main = ctx->stream;
    ctx->stream = ctx->copy_stream;
    bool ok = false;
    try {
        ok = adc_luts_dev(ctx, ix->tables, ix->M, ix->ks, ix->ds, dq, nq, luts);
    } catch (...) {
        ctx->stream = main;
        throw;
    }
    ctx->stream = main;
    PQG_CUDA(cudaEventRecord(ctx->pipe_ev[3], ctx->copy_stream));
    return ok ? luts : nullptr;
}

static void search_scan(pqg_ctx* ctx, const pqg_index* ix, const float* dq, uint64_t nq,
                        const uint32_t* probes, uint64_t nprobe, uint64_t k, int has_max,
                        double max_sq, uint64_t* oi, double* od, uint32_t* oc,
                        const uint64_t* subset = nullptr, uint64_t nsub = 0, const float* luts = nullptr) {
    if (luts) PQG_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->pipe_ev[3], 0));
    const IndexView v = ix->view();
    ivf_scan(ctx, v, dq, nq, probes, nprobe, k, has_max, max_sq, oi, od, oc, ctx->d_err, subset, nsub, luts);
}

// ===========================================================================
// extern "C"
// ===========================================================================
extern "C" {

const char* pqg_last_error(void) { return g_last_error.c_str(); }

const char* pqg_version(void) { return "pqg 0.1 (sm_100a)"; }

int pqg_ctx_create(int device, pqg_ctx** out_ctx) {
    return guard([&] {
        if (!out_ctx) inval("ctx_create: null output");
        int ndev = 0;
        PQG_CUDA(cudaGetDeviceCount(&ndev));
        if (device < 0 || device >= ndev) inval("ctx_create: no such device");
        PQG_CUDA(cudaSetDevice(device));
        pqg_ctx* c = new pqg_ctx;
        c->device = device;
        cudaDeviceProp prop;
        PQG_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major != 10) {
            delete c;
            fail(PQG_EUNSUPPORTED, "libpqg is built for sm_100a (B200); device is sm_" +
                                       std::to_string(prop.major) + std::to_string(prop.minor));
        }
        c->num_sms = prop.multiProcessorCount;
        PQG_CUDA(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
        c->stream = c->own_stream;
        PQG_CUDA(cudaMalloc(&c->d_err, sizeof(int)));
        *out_ctx = c;
    });
}

void pqg_ctx_destroy(pqg_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    ctx->arena.release();
    for (auto& r : ctx->prof_recs) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (auto e : ctx->event_pool) cudaEventDestroy(e);
    if (ctx->d_err) cudaFree(ctx->d_err);
    for (auto e : ctx->pipe_ev)
        if (e) cudaEventDestroy(e);
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    if (ctx->handoff_ev) cudaEventDestroy(ctx->handoff_ev);
    if (ctx->shard_ws) pqg_ctx_destroy(ctx->shard_ws);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;
}

int pqg_ctx_set_stream(pqg_ctx* ctx, void* s) {
    return guard([&] {
        cudaStream_t ns = s ? static_cast<cudaStream_t>(s) : ctx->own_stream;
        if (ns == ctx->stream) return;
        PQG_CUDA(cudaSetDevice(ctx->device));
        // Work already queued on the outgoing stream may still use the scratch
        // arena the next call hands out again: the new stream waits for it.
        if (!ctx->handoff_ev) PQG_CUDA(cudaEventCreateWithFlags(&ctx->handoff_ev, cudaEventDisableTiming));
        PQG_CUDA(cudaEventRecord(ctx->handoff_ev, ctx->stream));
        PQG_CUDA(cudaStreamWaitEvent(ns, ctx->handoff_ev, 0));
        ctx->stream = ns;
    });
}

void* pqg_ctx_stream(pqg_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int pqg_ctx_check_errors(pqg_ctx* ctx) {
    return guard([&] {
        Scope sc(ctx);
        if (ctx->err_pending && read_err(ctx)) {
            PQG_CUDA(cudaMemsetAsync(ctx->d_err, 0, sizeof(int), ctx->stream));
            fail(PQG_ERANGE, "adc_lookup: code out of range");
        }
    });
}

int pqg_ctx_sync(pqg_ctx* ctx) {
    const int rc = guard([&] { sync(ctx); });
    return rc ? rc : pqg_ctx_check_errors(ctx);
}

uint64_t pqg_ctx_launches(pqg_ctx* ctx) { return ctx ? ctx->launches : 0; }

int pqg_profile_enable(pqg_ctx* ctx, int enable) {
    return guard([&] {
        sync(ctx);
        for (auto& r : ctx->prof_recs) {
            ctx->event_pool.push_back(r.a);
            ctx->event_pool.push_back(r.b);
        }
        ctx->prof_recs.clear();
        ctx->profiling = enable != 0;
    });
}

int pqg_profile_read(pqg_ctx* ctx, const char* cls, uint64_t* launches, double* total_ms) {
    return guard([&] {
        sync(ctx);
        uint64_t n = 0;
        double ms = 0.0;
        for (auto& r : ctx->prof_recs) {
            if (ctx->prof_names[r.cls] != cls) continue;
            float t = 0.f;
            PQG_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
            ms += t;
            ++n;
        }
        if (launches) *launches = n;
        if (total_ms) *total_ms = ms;
    });
}

int pqg_nearest_batch(pqg_ctx* ctx, const float* points, uint64_t n, uint64_t d,
                      const float* table, uint64_t k, uint32_t* index, double* sq_dist) {
    return guard([&] {
        Scope sc(ctx);
        if (k == 0) inval("nearest_centroid: empty centroid set");
        if (d == 0 || n == 0) return;
        const float* dp = in(ctx, points, n * d);
        const float* dt = in(ctx, table, k * d);
        auto oi = out(ctx, index, n);
        auto od = out(ctx, sq_dist, n);
        float* cnorm = scratch<float>(ctx, k);
        float* cmax = scratch<float>(ctx, 1);
        table_norms(ctx, dt, 1, k, uint32_t(d), cnorm, cmax);
        NearestArgs a;
        a.src.x = dp;
        a.src.ldx = d;
        a.n = n;
        a.d = uint32_t(d);
        a.table = dt;
        a.k = k;
        a.cnorm = cnorm;
        a.cmax = cmax;
        a.out_idx = oi.dev ? (void*)oi.dev : (void*)scratch<uint32_t>(ctx, n);
        a.idx_bytes = 4;
        a.idx_rs = 1;
        a.out_dist = od.dev;
        nearest(ctx, a);
        finish(ctx, oi);
        finish(ctx, od);
        sync(ctx);
    });
}

int pqg_kmeans_fit(pqg_ctx* ctx, const float* points, uint64_t n, uint64_t d, uint64_t k,
                   uint32_t max_iters, uint64_t seed, double tol, float* centroids,
                   uint32_t* assignments, double* inertia, uint32_t* iterations_run,
                   double* inertia_per_iter) {
    return guard([&] {
        Scope sc(ctx);
        // proj/src/kmeans.cpp:65-71
        if (k == 0) inval("kmeans_fit: k must be >= 1");
        if (k > n)
            inval("kmeans_fit: k (" + std::to_string(k) + ") exceeds number of points (" +
                  std::to_string(n) + ")");
        if (max_iters < 1) inval("kmeans_fit: max_iters must be >= 1");
        if (tol < 0.0) inval("kmeans_fit: tol must be >= 0");
        if (d == 0) inval("kmeans_fit: dims must be >= 1");
        const float* dp = in(ctx, points, n * d);
        auto oc = out(ctx, centroids, k * d);
        float* table = oc.dev ? oc.dev : scratch<float>(ctx, k * d);
        auto oa = out(ctx, assignments, n);
        uint32_t* assign = oa.dev ? oa.dev : scratch<uint32_t>(ctx, n);
        KMeansOut r = run_kmeans(ctx, dp, n, d, 1, uint32_t(d), 0, k, max_iters, {seed}, tol,
                                 table, assign);
        finish(ctx, oc);
        finish(ctx, oa);
        sync(ctx);
        if (inertia) *inertia = r.inertia[0];
        if (iterations_run) *iterations_run = r.iters[0];
        if (inertia_per_iter)
            std::copy(r.per_iter.begin(), r.per_iter.begin() + r.iters[0], inertia_per_iter);
    });
}

int pqg_train_chunks(pqg_ctx* ctx, const float* data, uint64_t n, uint64_t D, uint64_t n_chunks,
                     uint32_t M, uint32_t ks, uint32_t max_iters, uint64_t seed,
                     float* representatives, double* local_rmse, uint32_t* iterations_run) {
    return guard([&] {
        Scope sc(ctx);
        check_train_chunks(n, D, n_chunks, M, ks, max_iters);
        const float* dx = in(ctx, data, n * D);
        ChunkFits f = train_chunks_dev(ctx, dx, n, D, n_chunks, M, ks, max_iters, seed);
        if (representatives) {
            const uint64_t cnt = n_chunks * ks * D;
            PQG_CUDA(cudaMemcpyAsync(representatives, f.reps, sizeof(float) * cnt,
                                     on_device(representatives) ? cudaMemcpyDeviceToDevice
                                                                : cudaMemcpyDeviceToHost,
                                     ctx->stream));
        }
        sync(ctx);
        if (local_rmse) std::copy(f.rmse.begin(), f.rmse.end(), local_rmse);
        if (iterations_run) std::copy(f.iters.begin(), f.iters.end(), iterations_run);
    });
}

int pqg_pipeline_run(pqg_ctx* ctx, const float* data, uint64_t n, uint64_t D, uint64_t n_chunks,
                     uint32_t M, uint32_t ks, uint64_t nlist, uint32_t max_iters, uint64_t seed,
                     int mode, float* global_tables, double* global_rmse, float* representatives,
                     double* local_rmse, uint64_t* nlist_used, pqg_index** merged_index,
                     double* phase_seconds) {
    return guard([&] {
        Scope sc(ctx);
        // proj/src/pipeline.cpp:142-163
        if (n == 0 || D == 0) inval("run_pipeline: empty dataset");
        if (mode < PQG_MODE_SINGLE || mode > PQG_MODE_PARALLEL_PQ_INDEX)
            inval("run_pipeline: unknown mode " + std::to_string(mode));
        uint64_t nl = nlist == 0 ? default_nlist_of(n) : nlist;
        if (nlist == 0 && mode == PQG_MODE_PARALLEL_PQ_INDEX) nl = std::min<uint64_t>(nl, n_chunks * ks);
        if (nlist_used) *nlist_used = nl;
        double ph[PQG_PHASE_COUNT];
        std::fill(ph, ph + PQG_PHASE_COUNT, -1.0);
        auto timed = [&](int phase, auto&& body) {
            const auto t0 = Clock::now();
            body();
            sync(ctx);
            ph[phase] = seconds_since(t0);
        };
        const float* dx = in(ctx, data, n * D);
        const uint32_t ds = (M && D % M == 0) ? uint32_t(D / M) : 0;
        auto ot = out(ctx, global_tables, uint64_t(M) * ks * (ds ? ds : 1));
        float* gt = nullptr;
        double rmse_g = 0.0;

        if (mode == PQG_MODE_SINGLE) {
            // fit (pipeline.cpp:166-169), then reconstruction_rmse (:171-173): the
            // final assignment pass of each subspace fit IS the encode of the data
            // with the returned codebook (no update follows it, kmeans.cpp:93-101),
            // so the SSE is taken from those assignments.
            check_pq_fit(n, D, M, ks, max_iters);
            uint32_t* assign = scratch<uint32_t>(ctx, uint64_t(M) * n);
            gt = ot.dev ? ot.dev : scratch<float>(ctx, uint64_t(M) * ks * ds);
            std::vector<uint64_t> seeds(M);
            for (uint32_t m = 0; m < M; ++m) seeds[m] = seed + m;
            timed(PQG_PHASE_FIT, [&] {
                run_kmeans(ctx, dx, n, D, M, ds, ds, ks, max_iters, seeds, 1e-4, gt, assign);
            });
            timed(PQG_PHASE_ENCODE, [&] {
                double* sse = scratch<double>(ctx, 1);
                chunk_sse(ctx, dx, 1, M, ks, ds, n, 0, assign, n, gt, sse);
                double h = 0.0;
                PQG_CUDA(cudaMemcpyAsync(&h, sse, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
                sync(ctx);
                rmse_g = std::sqrt(h / double(n * D));
            });
        } else {
            timed(PQG_PHASE_CHUNKING, [&] { check_chunks(n, n_chunks); });
            check_train_chunks(n, D, n_chunks, M, ks, max_iters);
            const uint64_t C = n_chunks, R = C * ks;
            ChunkFits f;
            timed(PQG_PHASE_LOCAL_FIT, [&] {
                f = train_chunks_dev(ctx, dx, n, D, C, M, ks, max_iters, seed);
            });
            // fit_global = pq_fit(representatives, M, ks, iters, seed) (pipeline.cpp:137-140)
            check_pq_fit(R, D, M, ks, max_iters);
            gt = ot.dev ? ot.dev : scratch<float>(ctx, uint64_t(M) * ks * ds);
            timed(PQG_PHASE_GLOBAL_FIT, [&] {
                uint32_t* assign = scratch<uint32_t>(ctx, uint64_t(M) * R);
                std::vector<uint64_t> seeds(M);
                for (uint32_t m = 0; m < M; ++m) seeds[m] = seed + m;
                run_kmeans(ctx, f.reps, R, D, M, ds, ds, ks, max_iters, seeds, 1e-4, gt, assign);
            });
            if (representatives) {
                PQG_CUDA(cudaMemcpyAsync(representatives, f.reps, sizeof(float) * R * D,
                                         on_device(representatives) ? cudaMemcpyDeviceToDevice
                                                                    : cudaMemcpyDeviceToHost,
                                         ctx->stream));
            }
            if (local_rmse) std::copy(f.rmse.begin(), f.rmse.end(), local_rmse);
            const uint32_t w = code_width(ks);
            uint8_t* codes = scratch<uint8_t>(ctx, n * M * w);
            auto encode_rmse = [&] {
                encode_dev(ctx, dx, n, M, ks, ds, gt, codes);
                double* sse = scratch<double>(ctx, 1);
                reset_err(ctx);
                recon_sse_dev(ctx, dx, codes, n, M, ks, ds, gt, sse, ctx->d_err);
                double h = 0.0;
                PQG_CUDA(cudaMemcpyAsync(&h, sse, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
                sync(ctx);
                rmse_g = std::sqrt(h / double(n * D));
            };
            if (mode == PQG_MODE_PARALLEL_PQ) {
                timed(PQG_PHASE_ENCODE, encode_rmse);  // pipeline.cpp:201-206
            } else {
                // shared coarse centroids: kmeans_fit(representatives, nlist, iters,
                // seed + M) (pipeline.cpp:212-219)
                if (nl > R)
                    inval("kmeans_fit: k (" + std::to_string(nl) + ") exceeds number of points (" +
                          std::to_string(R) + ")");
                float* coarse = scratch<float>(ctx, nl * D);
                timed(PQG_PHASE_COARSE_FIT, [&] {
                    uint32_t* assign = scratch<uint32_t>(ctx, R);
                    run_kmeans(ctx, f.reps, R, D, 1, uint32_t(D), 0, nl, max_iters, {seed + M}, 1e-4,
                               coarse, assign);
                });
                timed(PQG_PHASE_ENCODE, encode_rmse);  // pipeline.cpp:225-243
                // per-chunk ivf_build_with_centroids with ids [begin, end) then
                // ivf_merge in chunk order (pipeline.cpp:245-263): list l of the merge
                // is chunk 0's list l, then chunk 1's, ... -- exactly the stable
                // build over all n items with ids 0..n-1, which is what runs here
                // (one launch sequence for every chunk; the merge is free).
                pqg_index* ix = nullptr;
                timed(PQG_PHASE_INDEX_BUILD, [&] {
                    uint64_t* ids = scratch<uint64_t>(ctx, n);
                    launch(ctx, "pipeline", iota_u64_kernel, dim3(grid1d(n, 256, 4096)), dim3(256), 0,
                           ids, n);
                    ix = new_index(ctx, M, ks, ds, nl, n, gt, coarse);
                    try {
                        uint32_t* lo = assign_lists(ctx, ix->tables, M, ks, ds, codes, n, ix->coarse,
                                                    ix->coarse_norm, ix->coarse_max, nl);
                        fill_lists(ctx, ix, lo, ids, codes, n);
                        sync(ctx);
                    } catch (...) {
                        ix->free_all();
                        delete ix;
                        throw;
                    }
                });
                ph[PQG_PHASE_MERGE] = 0.0;
                if (merged_index) *merged_index = ix;
                else {
                    ix->free_all();
                    delete ix;
                }
            }
        }
        finish(ctx, ot);
        sync(ctx);
        if (global_rmse) *global_rmse = rmse_g;
        if (phase_seconds) std::copy(ph, ph + PQG_PHASE_COUNT, phase_seconds);
    });
}

int pqg_pq_fit(pqg_ctx* ctx, const float* data, uint64_t n, uint64_t D, uint32_t M, uint32_t ks,
               uint32_t max_iters, uint64_t seed, float* tables, uint32_t* iterations_run,
               double* inertia) {
    return pqg_pq_fit_ex(ctx, data, n, D, M, ks, max_iters, seed, tables, iterations_run, inertia,
                         nullptr);
}

int pqg_pq_fit_ex(pqg_ctx* ctx, const float* data, uint64_t n, uint64_t D, uint32_t M,
                  uint32_t ks, uint32_t max_iters, uint64_t seed, float* tables,
                  uint32_t* iterations_run, double* inertia, double* inertia_per_iter) {
    return guard([&] {
        Scope sc(ctx);
        check_pq_fit(n, D, M, ks, max_iters);
        const uint32_t ds = uint32_t(D / M);
        const float* dp = in(ctx, data, n * D);
        auto ot = out(ctx, tables, uint64_t(M) * ks * ds);
        float* table = ot.dev ? ot.dev : scratch<float>(ctx, uint64_t(M) * ks * ds);
        uint32_t* assign = scratch<uint32_t>(ctx, uint64_t(M) * n);
        std::vector<uint64_t> seeds(M);
        for (uint32_t m = 0; m < M; ++m) seeds[m] = seed + m;  // pq.cpp:88
        KMeansOut r = run_kmeans(ctx, dp, n, D, M, ds, ds, ks, max_iters, seeds, 1e-4, table, assign);
        finish(ctx, ot);
        sync(ctx);
        if (iterations_run) std::copy(r.iters.begin(), r.iters.end(), iterations_run);
        if (inertia) std::copy(r.inertia.begin(), r.inertia.end(), inertia);
        if (inertia_per_iter) std::copy(r.per_iter.begin(), r.per_iter.end(), inertia_per_iter);
    });
}

// Host rows: overlap the H2D copy of chunk c+1 (copy stream) with the encode
// of chunk c (context stream) through two staging buffers; codes go back per
// chunk on the copy stream.  PCIe is the bound for host inputs (~50 GB/s vs
// the ~500 GB/s the encode consumes), so this hides the encode entirely.
static void encode_host_pipelined(pqg_ctx* ctx, const float* data, uint64_t n, uint32_t M,
                                  uint32_t ks, uint32_t ds, const float* dt, uint8_t* codes_host) {
    const uint64_t D = uint64_t(M) * ds;
    const uint32_t w = code_width(ks);
    if (!ctx->copy_stream) {
        PQG_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
        for (auto& e : ctx->pipe_ev) PQG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    const uint64_t chunk = std::max<uint64_t>(4096, std::min<uint64_t>(n / 8 + 1, (uint64_t(64) << 20) / (D * 4)));
    float* stage[2] = {scratch<float>(ctx, chunk * D), scratch<float>(ctx, chunk * D)};
    uint8_t* dcodes = scratch<uint8_t>(ctx, n * M * w);
    cudaEvent_t* copied = ctx->pipe_ev;      // [2]: chunk landed in stage[b]
    cudaEvent_t* consumed = ctx->pipe_ev + 2;  // [2]: encode of stage[b] done
    PQG_CUDA(cudaEventRecord(consumed[0], ctx->stream));
    PQG_CUDA(cudaEventRecord(consumed[1], ctx->stream));
    const auto mark = ctx->arena.mark();
    const uint64_t nchunks = (n + chunk - 1) / chunk;
    auto h2d = [&](uint64_t c) {  // copy stream: chunk c -> stage[c & 1]
        const uint64_t r0 = c * chunk, nc = std::min(chunk, n - r0);
        const int b = int(c & 1);
        PQG_CUDA(cudaStreamWaitEvent(ctx->copy_stream, consumed[b], 0));
        PQG_CUDA(cudaMemcpyAsync(stage[b], data + r0 * D, nc * D * sizeof(float), cudaMemcpyHostToDevice,
                                 ctx->copy_stream));
        PQG_CUDA(cudaEventRecord(copied[b], ctx->copy_stream));
    };
    h2d(0);
    for (uint64_t c = 0; c < nchunks; ++c) {
        // the next chunk's copy is queued before this chunk's results go back,
        // so the copy engine streams rows while the SMs encode
        if (c + 1 < nchunks) h2d(c + 1);
        const uint64_t r0 = c * chunk, nc = std::min(chunk, n - r0);
        const int b = int(c & 1);
        PQG_CUDA(cudaStreamWaitEvent(ctx->stream, copied[b], 0));
        ctx->arena.reset_to(mark);
        encode_dev(ctx, stage[b], nc, M, ks, ds, dt, dcodes + r0 * M * w);
        PQG_CUDA(cudaEventRecord(consumed[b], ctx->stream));
        PQG_CUDA(cudaMemcpyAsync(codes_host + r0 * M * w, dcodes + r0 * M * w, nc * M * w,
                                 cudaMemcpyDeviceToHost, ctx->stream));
    }
    PQG_CUDA(cudaStreamSynchronize(ctx->copy_stream));
    PQG_CUDA(cudaStreamSynchronize(ctx->stream));
}

int pqg_pq_encode(pqg_ctx* ctx, const float* data, uint64_t n, uint32_t M, uint32_t ks,
                  uint32_t ds, const float* tables, uint8_t* codes) {
    return guard([&] {
        Scope sc(ctx);
        check_pq_shape(M, ks, ds, "pq_encode");
        if (n == 0) return;
        const uint64_t D = uint64_t(M) * ds;
        if (n >= 65536 && !on_device(data) && codes && !on_device(codes)) {
            const float* dt0 = in(ctx, tables, uint64_t(M) * ks * ds);
            encode_host_pipelined(ctx, data, n, M, ks, ds, dt0, codes);
            return;
        }
        const float* dx = in(ctx, data, n * D);
        const float* dt = in(ctx, tables, uint64_t(M) * ks * ds);
        auto oc = out(ctx, codes, n * M * code_width(ks));
        encode_dev(ctx, dx, n, M, ks, ds, dt, oc.dev);
        finish(ctx, oc);
        if (oc.host) sync(ctx);
    });
}

int pqg_pq_decode(pqg_ctx* ctx, const uint8_t* codes, uint64_t n, uint32_t M, uint32_t ks,
                  uint32_t ds, const float* tables, float* outp) {
    return guard([&] {
        Scope sc(ctx);
        check_pq_shape(M, ks, ds, "pq_decode");
        if (n == 0) return;
        const uint8_t* dc = in(ctx, codes, n * M * code_width(ks));
        const float* dt = in(ctx, tables, uint64_t(M) * ks * ds);
        auto oo = out(ctx, outp, n * M * ds);
        reset_err(ctx);
        pq_decode_dev(ctx, dc, n, M, ks, ds, dt, oo.dev, ctx->d_err);
        finish(ctx, oo);
        if (read_err(ctx)) fail(PQG_ERANGE, "pq_decode: code out of range for Ks=" + std::to_string(ks));
    });
}

int pqg_sq_error(pqg_ctx* ctx, const float* a, const float* b, uint64_t count, double* sse) {
    return guard([&] {
        Scope sc(ctx);
        if (count == 0) {
            *sse = 0.0;
            return;
        }
        const float* da = in(ctx, a, count);
        const float* db = in(ctx, b, count);
        auto os = out(ctx, sse, 1);
        sq_error_dev(ctx, da, db, count, os.dev);
        finish(ctx, os);
        sync(ctx);
    });
}

int pqg_pq_recon_sse(pqg_ctx* ctx, const float* data, const uint8_t* codes, uint64_t n,
                     uint32_t M, uint32_t ks, uint32_t ds, const float* tables, double* sse) {
    return guard([&] {
        Scope sc(ctx);
        check_pq_shape(M, ks, ds, "reconstruction_rmse");
        if (n == 0) {
            *sse = 0.0;
            return;
        }
        const float* dx = in(ctx, data, n * M * ds);
        const uint8_t* dc = in(ctx, codes, n * M * code_width(ks));
        const float* dt = in(ctx, tables, uint64_t(M) * ks * ds);
        auto os = out(ctx, sse, 1);
        reset_err(ctx);
        recon_sse_dev(ctx, dx, dc, n, M, ks, ds, dt, os.dev, ctx->d_err);
        finish(ctx, os);
        if (read_err(ctx)) fail(PQG_ERANGE, "pq_decode: code out of range for Ks=" + std::to_string(ks));
    });
}

int pqg_pq_encode_sse(pqg_ctx* ctx, const float* data, uint64_t n, uint32_t M, uint32_t ks,
                      uint32_t ds, const float* tables, uint8_t* codes, double* sse) {
    return guard([&] {
        Scope sc(ctx);
        check_pq_shape(M, ks, ds, "pq_encode");
        if (n == 0) {
            if (sse) *sse = 0.0;
            return;
        }
        const uint64_t D = uint64_t(M) * ds;
        const float* dx = in(ctx, data, n * D);
        const float* dt = in(ctx, tables, uint64_t(M) * ks * ds);
        auto oc = out(ctx, codes, n * M * code_width(ks));
        uint8_t* dc = oc.dev ? oc.dev : scratch<uint8_t>(ctx, n * M * code_width(ks));
        encode_dev(ctx, dx, n, M, ks, ds, dt, dc);
        auto os = out(ctx, sse, 1);
        if (os.dev) recon_sse_dev(ctx, dx, dc, n, M, ks, ds, dt, os.dev, ctx->d_err);
        finish(ctx, oc);
        finish(ctx, os);
        if (oc.host || os.host) sync(ctx);
    });
}

int pqg_adc_tables(pqg_ctx* ctx, const float* tables, uint32_t M, uint32_t ks, uint32_t ds,
                   const float* queries, uint64_t nq, float* entries) {
    return guard([&] {
        Scope sc(ctx);
        check_pq_shape(M, ks, ds, "adc_table");
        if (nq == 0) return;
        const float* dt = in(ctx, tables, uint64_t(M) * ks * ds);
        const float* dq = in(ctx, queries, nq * M * ds);
        auto oe = out(ctx, entries, nq * M * ks);
        adc_tables_dev(ctx, dt, M, ks, ds, dq, nq, oe.dev);
        finish(ctx, oe);
        if (oe.host) sync(ctx);
    });
}

int pqg_adc_lookup(pqg_ctx* ctx, const float* entries, uint32_t M, uint32_t ks,
                   const uint8_t* codes, uint64_t n, double* outp) {
    return guard([&] {
        Scope sc(ctx);
        if (n == 0) return;
        const float* de = in(ctx, entries, uint64_t(M) * ks);
        const uint8_t* dc = in(ctx, codes, n * M * code_width(ks));
        auto oo = out(ctx, outp, n);
        reset_err(ctx);
        adc_lookup_dev(ctx, de, M, ks, dc, n, oo.dev, ctx->d_err);
        finish(ctx, oo);
        if (read_err(ctx)) fail(PQG_ERANGE, "adc_lookup: code out of range for Ks=" + std::to_string(ks));
    });
}

int pqg_ivf_assign(pqg_ctx* ctx, const uint8_t* codes, uint64_t n, uint32_t M, uint32_t ks,
                   uint32_t ds, const float* tables, const float* coarse, uint64_t nlist,
                   uint32_t* list_of) {
    return guard([&] {
        Scope sc(ctx);
        check_pq_shape(M, ks, ds, "ivf_assign");
        if (nlist == 0) inval("ivf_build: coarse centroids do not match the codebook");
        if (n == 0) return;
        const uint8_t* dc = in(ctx, codes, n * M * code_width(ks));
        const float* dt = in(ctx, tables, uint64_t(M) * ks * ds);
        const float* dco = in(ctx, coarse, nlist * M * ds);
        float* cnorm = scratch<float>(ctx, nlist);
        float* cmax = scratch<float>(ctx, 1);
        table_norms(ctx, dco, 1, nlist, M * ds, cnorm, cmax);
        uint32_t* lo = assign_lists(ctx, dt, M, ks, ds, dc, n, dco, cnorm, cmax, nlist);
        auto ol = out(ctx, list_of, n);
        PQG_CUDA(cudaMemcpyAsync(ol.dev, lo, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, ctx->stream));
        finish(ctx, ol);
        sync(ctx);
    });
}

int pqg_ivf_build_with_centroids(pqg_ctx* ctx, const float* tables, uint32_t M, uint32_t ks,
                                 uint32_t ds, const uint8_t* codes, const uint64_t* ids,
                                 uint64_t n, const float* coarse, uint64_t nlist,
                                 pqg_index** outp) {
    return guard([&] {
        Scope sc(ctx);
        // proj/src/ivf.cpp:151-160
        if (n == 0) inval("ivf_build: no items");
        if (nlist == 0 || !coarse) inval("ivf_build: coarse centroids do not match the codebook");
        check_pq_shape(M, ks, ds, "ivf_build");
        const uint64_t rb = uint64_t(M) * code_width(ks);
        const float* dt = in(ctx, tables, uint64_t(M) * ks * ds);
        const uint8_t* dc = in(ctx, codes, n * rb);
        const uint64_t* di = in(ctx, ids, n);
        const float* dco = in(ctx, coarse, nlist * M * ds);
        check_unique_ids(ctx, di, on_device(ids) ? nullptr : ids, n, "duplicate id ");
        pqg_index* ix = new_index(ctx, M, ks, ds, nlist, n, dt, dco);
        try {
            uint32_t* lo = assign_lists(ctx, ix->tables, M, ks, ds, dc, n, ix->coarse,
                                        ix->coarse_norm, ix->coarse_max, nlist);
            fill_lists(ctx, ix, lo, di, dc, n);
            sync(ctx);
        } catch (...) {
            ix->free_all();
            delete ix;
            throw;
        }
        *outp = ix;
    });
}

int pqg_ivf_build(pqg_ctx* ctx, const float* tables, uint32_t M, uint32_t ks, uint32_t ds,
                  const uint8_t* codes, const uint64_t* ids, uint64_t n, uint64_t nlist,
                  uint64_t seed, uint32_t kmeans_iters, pqg_index** outp) {
    return guard([&] {
        Scope sc(ctx);
        // proj/src/ivf.cpp:126-131
        if (n == 0) inval("ivf_build: no items");
        if (nlist == 0 || nlist > n)
            inval("ivf_build: nlist (" + std::to_string(nlist) + ") must be in [1, n_items=" +
                  std::to_string(n) + "]");
        check_pq_shape(M, ks, ds, "ivf_build");
        const uint64_t D = uint64_t(M) * ds;
        const uint64_t rb = uint64_t(M) * code_width(ks);
        const float* dt = in(ctx, tables, uint64_t(M) * ks * ds);
        const uint8_t* dc = in(ctx, codes, n * rb);
        const uint64_t* di = in(ctx, ids, n);
        // decode all (pq_decode, throws out_of_range) then kmeans_fit(decoded, nlist, iters, seed)
        float* dec = scratch<float>(ctx, n * D);
        reset_err(ctx);
        pq_decode_dev(ctx, dc, n, M, ks, ds, dt, dec, ctx->d_err);
        if (read_err(ctx)) fail(PQG_ERANGE, "pq_decode: code out of range for Ks=" + std::to_string(ks));
        if (kmeans_iters < 1) inval("kmeans_fit: max_iters must be >= 1");
        float* coarse = scratch<float>(ctx, nlist * D);
        uint32_t* assign = scratch<uint32_t>(ctx, n);
        run_kmeans(ctx, dec, n, D, 1, uint32_t(D), 0, nlist, kmeans_iters, {seed}, 1e-4, coarse, assign);
        check_unique_ids(ctx, di, on_device(ids) ? nullptr : ids, n, "duplicate id ");
        pqg_index* ix = new_index(ctx, M, ks, ds, nlist, n, dt, coarse);
        try {
            // the final pass leaves assignments consistent with the centroids (ivf.cpp:142-146)
            fill_lists(ctx, ix, assign, di, dc, n);
            sync(ctx);
        } catch (...) {
            ix->free_all();
            delete ix;
            throw;
        }
        *outp = ix;
    });
}

int pqg_index_create(pqg_ctx* ctx, const float* tables, uint32_t M, uint32_t ks, uint32_t ds,
                     const float* coarse, uint64_t nlist, const uint64_t* offsets,
                     const uint64_t* ids, const uint8_t* codes, pqg_index** outp) {
    return guard([&] {
        Scope sc(ctx);
        check_pq_shape(M, ks, ds, "index");
        if (nlist == 0) inval("index: nlist must be >= 1");
        std::vector<uint64_t> hoff(nlist + 1);
        PQG_CUDA(cudaMemcpy(hoff.data(), offsets, sizeof(uint64_t) * (nlist + 1), cudaMemcpyDefault));
        const uint64_t n = hoff[nlist];
        if (hoff[0] != 0) inval("index: offsets[0] must be 0");
        for (uint64_t l = 0; l < nlist; ++l)
            if (hoff[l + 1] < hoff[l]) inval("index: offsets must be non-decreasing");
        const float* dt = in(ctx, tables, uint64_t(M) * ks * ds);
        const float* dco = in(ctx, coarse, nlist * M * ds);
        pqg_index* ix = new_index(ctx, M, ks, ds, nlist, n, dt, dco);
        try {
            PQG_CUDA(cudaMemcpyAsync(ix->offsets, hoff.data(), sizeof(uint64_t) * (nlist + 1),
                                     cudaMemcpyHostToDevice, ctx->stream));
            if (n) {
                PQG_CUDA(cudaMemcpyAsync(ix->ids, ids, sizeof(uint64_t) * n, cudaMemcpyDefault, ctx->stream));
                PQG_CUDA(cudaMemcpyAsync(ix->codes, codes, n * ix->rb(), cudaMemcpyDefault, ctx->stream));
            }
            sync(ctx);
        } catch (...) {
            ix->free_all();
            delete ix;
            throw;
        }
        *outp = ix;
    });
}

void pqg_index_destroy(pqg_index* ix) {
    if (!ix) return;
    cudaSetDevice(ix->device);
    cudaDeviceSynchronize();
    ix->free_all();
    delete ix;
}

int pqg_index_info(const pqg_index* ix, uint64_t* nlist, uint64_t* n_items, uint32_t* M,
                   uint32_t* ks, uint32_t* ds) {
    return guard([&] {
        if (!ix) inval("index: null");
        if (nlist) *nlist = ix->nlist;
        if (n_items) *n_items = ix->n;
        if (M) *M = ix->M;
        if (ks) *ks = ix->ks;
        if (ds) *ds = ix->ds;
    });
}

int pqg_index_export(pqg_ctx* ctx, const pqg_index* ix, uint64_t* offsets, uint64_t* ids,
                     uint8_t* codes, float* coarse, float* tables) {
    return guard([&] {
        Scope sc(ctx);
        if (offsets)
            PQG_CUDA(cudaMemcpyAsync(offsets, ix->offsets, sizeof(uint64_t) * (ix->nlist + 1),
                                     cudaMemcpyDefault, ctx->stream));
        if (ids && ix->n)
            PQG_CUDA(cudaMemcpyAsync(ids, ix->ids, sizeof(uint64_t) * ix->n, cudaMemcpyDefault, ctx->stream));
        if (codes && ix->n)
            PQG_CUDA(cudaMemcpyAsync(codes, ix->codes, ix->n * ix->rb(), cudaMemcpyDefault, ctx->stream));
        if (coarse)
            PQG_CUDA(cudaMemcpyAsync(coarse, ix->coarse, sizeof(float) * ix->nlist * ix->D(),
                                     cudaMemcpyDefault, ctx->stream));
        if (tables)
            PQG_CUDA(cudaMemcpyAsync(tables, ix->tables, sizeof(float) * ix->M * ix->ks * ix->ds,
                                     cudaMemcpyDefault, ctx->stream));
        sync(ctx);
    });
}

// Replace ix's lists with concat(ix lists, new lists) per list.
static void concat_into(pqg_ctx* ctx, pqg_index* dst, const pqg_index* a, const uint64_t* off_b,
                        const uint64_t* ids_b, const uint8_t* codes_b, uint64_t nb) {
    const uint64_t total = a->n + nb;
    uint64_t* off_o = dalloc<uint64_t>(a->nlist + 1);
    uint64_t* ids_o = dalloc<uint64_t>(total);
    uint8_t* codes_o = dalloc<uint8_t>(total * a->rb());
    launch(ctx, "csr_concat", csr_concat_kernel, dim3(grid1d(total + a->nlist + 1, 256, ctx->num_sms * 16)),
           dim3(256), 0, (const uint64_t*)a->offsets, (const uint64_t*)a->ids,
           (const uint8_t*)a->codes, a->n, off_b, ids_b, codes_b, nb, a->nlist, a->rb(), off_o,
           ids_o, codes_o);
    sync(ctx);
    if (dst->offsets) cudaFree(dst->offsets);
    if (dst->ids) cudaFree(dst->ids);
    if (dst->codes) cudaFree(dst->codes);
    dst->offsets = off_o;
    dst->ids = ids_o;
    dst->codes = codes_o;
    dst->n = total;
}

int pqg_index_add(pqg_ctx* ctx, pqg_index* ix, const uint8_t* codes, const uint64_t* ids,
                  uint64_t n) {
    return guard([&] {
        Scope sc(ctx);
        if (n == 0) return;
        const uint64_t rb = ix->rb();
        const uint8_t* dc = in(ctx, codes, n * rb);
        const uint64_t* di = in(ctx, ids, n);
        check_unique_ids(ctx, di, on_device(ids) ? nullptr : ids, n, "duplicate id ");
        // collisions with the index: first new id (input order) already present
        {
            uint64_t* cat = scratch<uint64_t>(ctx, ix->n + n);
            if (ix->n)
                PQG_CUDA(cudaMemcpyAsync(cat, ix->ids, sizeof(uint64_t) * ix->n, cudaMemcpyDeviceToDevice, ctx->stream));
            PQG_CUDA(cudaMemcpyAsync(cat + ix->n, di, sizeof(uint64_t) * n, cudaMemcpyDeviceToDevice, ctx->stream));
            uint64_t* pos = scratch<uint64_t>(ctx, 1);
            find_duplicate(ctx, cat, ix->n + n, pos);
            uint64_t h = 0;
            PQG_CUDA(cudaMemcpyAsync(&h, pos, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
            sync(ctx);
            if (h != ~uint64_t(0)) {
                uint64_t id = 0;
                PQG_CUDA(cudaMemcpy(&id, cat + h, sizeof(id), cudaMemcpyDeviceToHost));
                inval("ivf_add: id collision on id " + std::to_string(id));
            }
        }
        uint32_t* lo = assign_lists(ctx, ix->tables, ix->M, ix->ks, ix->ds, dc, n, ix->coarse,
                                    ix->coarse_norm, ix->coarse_max, ix->nlist);
        uint64_t* off_b = scratch<uint64_t>(ctx, ix->nlist + 1);
        Bucketing bk{off_b, scratch<uint32_t>(ctx, n)};
        stable_bucket(ctx, lo, n, 1, ix->nlist, nullptr, bk);
        uint64_t* ids_b = scratch<uint64_t>(ctx, n);
        uint8_t* codes_b = scratch<uint8_t>(ctx, n * rb);
        csr_scatter(ctx, bk.perm, n, di, dc, rb, ids_b, codes_b);
        concat_into(ctx, ix, ix, off_b, ids_b, codes_b, n);
    });
}

int pqg_index_merge(pqg_ctx* ctx, const pqg_index* a, const pqg_index* b, pqg_index** outp) {
    return guard([&] {
        Scope sc(ctx);
        // proj/src/ivf.cpp:186-197
        const uint64_t ntab = uint64_t(a->M) * a->ks * a->ds;
        bool same_cb = a->M == b->M && a->ks == b->ks && a->ds == b->ds;
        if (same_cb) {
            std::vector<float> ta(ntab), tb(ntab);
            PQG_CUDA(cudaMemcpy(ta.data(), a->tables, ntab * 4, cudaMemcpyDeviceToHost));
            PQG_CUDA(cudaMemcpy(tb.data(), b->tables, ntab * 4, cudaMemcpyDeviceToHost));
            for (uint64_t i = 0; i < ntab && same_cb; ++i) same_cb = ta[i] == tb[i];
        }
        if (!same_cb) inval("ivf_merge: codebook mismatch");
        bool same_coarse = a->nlist == b->nlist;
        if (same_coarse) {
            const uint64_t nc = a->nlist * a->D();
            std::vector<float> ca(nc), cb(nc);
            PQG_CUDA(cudaMemcpy(ca.data(), a->coarse, nc * 4, cudaMemcpyDeviceToHost));
            PQG_CUDA(cudaMemcpy(cb.data(), b->coarse, nc * 4, cudaMemcpyDeviceToHost));
            for (uint64_t i = 0; i < nc && same_coarse; ++i) same_coarse = ca[i] == cb[i];
        }
        if (!same_coarse) inval("ivf_merge: coarse centroid mismatch");
        if (a->n && b->n) {
            uint64_t* cat = scratch<uint64_t>(ctx, a->n + b->n);
            PQG_CUDA(cudaMemcpyAsync(cat, a->ids, sizeof(uint64_t) * a->n, cudaMemcpyDeviceToDevice, ctx->stream));
            PQG_CUDA(cudaMemcpyAsync(cat + a->n, b->ids, sizeof(uint64_t) * b->n, cudaMemcpyDeviceToDevice, ctx->stream));
            uint64_t* pos = scratch<uint64_t>(ctx, 1);
            find_duplicate(ctx, cat, a->n + b->n, pos);
            uint64_t h = 0;
            PQG_CUDA(cudaMemcpyAsync(&h, pos, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
            sync(ctx);
            if (h != ~uint64_t(0)) {
                uint64_t id = 0;
                PQG_CUDA(cudaMemcpy(&id, cat + h, sizeof(id), cudaMemcpyDeviceToHost));
                inval("ivf_merge: id collision on id " + std::to_string(id));
            }
        }
        pqg_index* o = new_index(ctx, a->M, a->ks, a->ds, a->nlist, 0, a->tables, a->coarse);
        try {
            concat_into(ctx, o, a, b->offsets, b->ids, b->codes, b->n);
        } catch (...) {
            o->free_all();
            delete o;
            throw;
        }
        *outp = o;
    });
}

static void check_query(const pqg_index* ix, uint64_t k, uint64_t nprobe) {
    // proj/src/ivf.cpp:103-114
    if (k == 0) inval("query: k must be >= 1");
    if (nprobe == 0 || nprobe > ix->nlist)
        inval("query: nprobe (" + std::to_string(nprobe) + ") must be in [1, nlist=" +
              std::to_string(ix->nlist) + "]");
}

int pqg_index_probe(pqg_ctx* ctx, const pqg_index* ix, const float* queries, uint64_t nq,
                    uint64_t nprobe, uint32_t* probes) {
    return guard([&] {
        Scope sc(ctx);
        check_query(ix, 1, nprobe);
        if (nq == 0) return;
        const float* dq = in(ctx, queries, nq * ix->D());
        auto op = out(ctx, probes, nq * nprobe);
        ivf_probe(ctx, ix->view(), dq, nq, nprobe, op.dev);
        finish(ctx, op);
        sync(ctx);
    });
}

int pqg_index_search(pqg_ctx* ctx, const pqg_index* ix, const float* queries, uint64_t nq,
                     uint64_t k, uint64_t nprobe, int has_max, double max_sq_dist,
                     uint64_t* out_ids, double* out_dists, uint32_t* out_counts) {
    return pqg_index_search_ex(ctx, ix, queries, nq, k, nprobe, has_max, max_sq_dist, out_ids, out_dists,
                               out_counts, nullptr);
}

int pqg_index_search_ex(pqg_ctx* ctx, const pqg_index* ix, const float* queries, uint64_t nq,
                        uint64_t k, uint64_t nprobe, int has_max, double max_sq_dist,
                        uint64_t* out_ids, double* out_dists, uint32_t* out_counts, uint32_t* out_probes) {
    return guard([&] {
        Scope sc(ctx);
        check_query(ix, k, nprobe);
        if (nq == 0) return;
        const float* dq = in(ctx, queries, nq * ix->D());
        auto oi = out(ctx, out_ids, nq * k);
        auto od = out(ctx, out_dists, nq * k);
        auto oc = out(ctx, out_counts, nq);
        uint32_t* probes = scratch<uint32_t>(ctx, nq * nprobe);
        const float* luts = k <= 32 ? search_luts_async(ctx, ix, dq, nq) : nullptr;
        ivf_probe(ctx, ix->view(), dq, nq, nprobe, probes);
        if (out_probes)
            PQG_CUDA(cudaMemcpyAsync(out_probes, probes, sizeof(uint32_t) * nq * nprobe, cudaMemcpyDefault,
                                     ctx->stream));
        reset_err(ctx);
        search_scan(ctx, ix, dq, nq, probes, nprobe, k, has_max, max_sq_dist, oi.dev, od.dev, oc.dev, nullptr, 0,
                    luts);
        finish(ctx, oi);
        finish(ctx, od);
        finish(ctx, oc);
        if (oi.host || od.host || oc.host) {
            if (read_err(ctx)) fail(PQG_ERANGE, "adc_lookup: code out of range");
        } else {
            ctx->err_pending = true;  // reported by pqg_ctx_sync / pqg_ctx_check_errors
        }
    });
}

int pqg_index_search_subset(pqg_ctx* ctx, const pqg_index* ix, const float* queries, uint64_t nq,
                            uint64_t k, const uint64_t* subset, uint64_t nsub, uint64_t nprobe,
                            int has_max, double max_sq_dist, uint64_t* out_ids, double* out_dists,
                            uint32_t* out_counts) {
    return guard([&] {
        Scope sc(ctx);
        check_query(ix, k, nprobe);
        // proj/src/ivf.cpp:234-238
        if (nsub > 1) {
            std::vector<uint64_t> hs(nsub);
            PQG_CUDA(cudaMemcpy(hs.data(), subset, sizeof(uint64_t) * nsub, cudaMemcpyDefault));
            for (uint64_t i = 1; i < nsub; ++i)
                if (hs[i - 1] >= hs[i]) inval("ivf_query_subset: subset is not sorted ascending");
        }
        if (nq == 0) return;
        const float* dq = in(ctx, queries, nq * ix->D());
        const uint64_t* dsub = in(ctx, subset, std::max<uint64_t>(nsub, 1));
        uint64_t* empty_sub = nullptr;
        if (nsub == 0) {  // an empty subset admits nothing
            empty_sub = scratch<uint64_t>(ctx, 1);
            dsub = empty_sub;
        }
        auto oi = out(ctx, out_ids, nq * k);
        auto od = out(ctx, out_dists, nq * k);
        auto oc = out(ctx, out_counts, nq);
        uint32_t* probes = scratch<uint32_t>(ctx, nq * nprobe);
        ivf_probe(ctx, ix->view(), dq, nq, nprobe, probes);
        reset_err(ctx);
        search_scan(ctx, ix, dq, nq, probes, nprobe, k, has_max, max_sq_dist, oi.dev, od.dev, oc.dev,
                    dsub, nsub);
        finish(ctx, oi);
        finish(ctx, od);
        finish(ctx, oc);
        if (oi.host || od.host || oc.host) {
            if (read_err(ctx)) fail(PQG_ERANGE, "adc_lookup: code out of range");
        } else {
            ctx->err_pending = true;  // reported by pqg_ctx_sync / pqg_ctx_check_errors
        }
    });
}

int pqg_flat_scan(pqg_ctx* ctx, const float* tables, uint32_t M, uint32_t ks, uint32_t ds,
                  const uint8_t* codes, const uint64_t* ids, uint64_t n, const float* queries,
                  uint64_t nq, uint64_t k, int has_max, double max_sq_dist, uint64_t* out_ids,
                  double* out_dists, uint32_t* out_counts) {
    return guard([&] {
        Scope sc(ctx);
        // proj/src/ivf.cpp:250-252
        if (k == 0) inval("flat_scan: k must be >= 1");
        check_pq_shape(M, ks, ds, "flat_scan");
        if (nq == 0) return;
        const uint64_t rb = uint64_t(M) * code_width(ks);
        const float* dt = in(ctx, tables, uint64_t(M) * ks * ds);
        const uint8_t* dc = in(ctx, codes, n * rb);
        const uint64_t* di = in(ctx, ids, n);
        const float* dq = in(ctx, queries, nq * M * ds);
        uint64_t* off = scratch<uint64_t>(ctx, 2);
        const uint64_t hoff[2] = {0, n};
        PQG_CUDA(cudaMemcpyAsync(off, hoff, sizeof(hoff), cudaMemcpyHostToDevice, ctx->stream));
        uint32_t* probes = scratch<uint32_t>(ctx, nq);
        PQG_CUDA(cudaMemsetAsync(probes, 0, sizeof(uint32_t) * nq, ctx->stream));
        IndexView v{dt, M, ks, ds, code_width(ks), nullptr, nullptr, nullptr, 1, off, di, dc, n};
        auto oi = out(ctx, out_ids, nq * k);
        auto od = out(ctx, out_dists, nq * k);
        auto oc = out(ctx, out_counts, nq);
        reset_err(ctx);
        ivf_scan(ctx, v, dq, nq, probes, 1, k, has_max, max_sq_dist, oi.dev, od.dev, oc.dev, ctx->d_err);
        finish(ctx, oi);
        finish(ctx, od);
        finish(ctx, oc);
        if (read_err(ctx)) fail(PQG_ERANGE, "adc_lookup: code out of range");
    });
}

int pqg_topk_merge(pqg_ctx* ctx, const uint64_t* ids, const double* dists,
                   const uint32_t* counts, uint32_t shards, uint64_t nq, uint64_t k,
                   uint64_t* out_ids, double* out_dists, uint32_t* out_counts) {
    return guard([&] {
        Scope sc(ctx);
        if (nq == 0 || shards == 0) return;
        const uint64_t* di = in(ctx, ids, uint64_t(shards) * nq * k);
        const double* dd = in(ctx, dists, uint64_t(shards) * nq * k);
        const uint32_t* dc = in(ctx, counts, uint64_t(shards) * nq);
        auto oi = out(ctx, out_ids, nq * k);
        auto od = out(ctx, out_dists, nq * k);
        auto oc = out(ctx, out_counts, nq);
        topk_merge_dev(ctx, di, dd, dc, shards, nq, k, oi.dev, od.dev, oc.dev);
        finish(ctx, oi);
        finish(ctx, od);
        finish(ctx, oc);
        if (oi.host || od.host || oc.host) sync(ctx);
    });
}

int pqg_assign_pass(pqg_ctx* ctx, const float* rows, uint64_t n, uint64_t ld, uint32_t B,
                    uint32_t d, uint32_t col_stride, const float* tables, uint64_t k,
                    uint32_t* assign, double* dist) {
    return guard([&] {
        Scope sc(ctx);
        if (k == 0) inval("nearest_centroid: empty centroid set");
        if (n == 0) return;
        const float* dr = in(ctx, rows, n * ld);
        const float* dt = in(ctx, tables, uint64_t(B) * k * d);
        auto oa = out(ctx, assign, uint64_t(B) * n);
        auto od = out(ctx, dist, uint64_t(B) * n);
        float* cnorm = scratch<float>(ctx, uint64_t(B) * k);
        float* cmax = scratch<float>(ctx, B);
        table_norms(ctx, dt, B, k, d, cnorm, cmax);
        NearestArgs a;
        a.src.x = dr;
        a.src.ldx = ld;
        a.src.col_stride = col_stride;
        a.n = n;
        a.d = d;
        a.B = B;
        a.table = dt;
        a.k = k;
        a.cnorm = cnorm;
        a.cmax = cmax;
        a.out_idx = oa.dev;
        a.idx_bytes = 4;
        a.idx_rs = 1;
        a.idx_ps = n;
        a.out_dist = od.dev;
        nearest(ctx, a);
        finish(ctx, oa);
        finish(ctx, od);
        if (oa.host || od.host) sync(ctx);
    });
}

int pqg_update_pass(pqg_ctx* ctx, const float* rows, uint64_t n, uint64_t ld, uint32_t B,
                    uint32_t d, uint32_t col_stride, float* tables, uint64_t k,
                    const uint32_t* assign, double* dist, const int* active) {
    return guard([&] {
        Scope sc(ctx);
        if (n == 0) return;
        const float* dr = in(ctx, rows, n * ld);
        const uint32_t* da = in(ctx, assign, uint64_t(B) * n);
        auto ot = out(ctx, tables, uint64_t(B) * k * d);
        if (ot.host)
            PQG_CUDA(cudaMemcpyAsync(ot.dev, tables, sizeof(float) * B * k * d, cudaMemcpyHostToDevice, ctx->stream));
        auto odist = out(ctx, dist, uint64_t(B) * n);
        if (odist.host)
            PQG_CUDA(cudaMemcpyAsync(odist.dev, dist, sizeof(double) * B * n, cudaMemcpyHostToDevice, ctx->stream));
        RowSrc src;
        src.x = dr;
        src.ldx = ld;
        src.col_stride = col_stride;
        const int* dact = in(ctx, active, B);
        kmeans_update(ctx, src, n, B, d, ot.dev, k, da, odist.dev, dact);
        finish(ctx, ot);
        finish(ctx, odist);
        if (ot.host || odist.host) sync(ctx);
    });
}

int pqg_rows_sum_f64(pqg_ctx* ctx, const double* v, uint64_t n, uint32_t B, double* outp) {
    return guard([&] {
        Scope sc(ctx);
        if (n == 0 || B == 0) {
            for (uint32_t b = 0; b < B; ++b) outp[b] = 0.0;
            return;
        }
        const double* dv = in(ctx, v, uint64_t(B) * n);
        auto oo = out(ctx, outp, B);
        rows_sum_f64(ctx, dv, n, B, oo.dev);
        finish(ctx, oo);
        sync(ctx);
    });
}

int pqg_kmeans_init_rows(uint64_t n, uint64_t k, uint64_t seed, uint64_t* rows) {
    return guard([&] {
        if (k == 0 || k > n) inval("kmeans_fit: k (" + std::to_string(k) + ") exceeds number of points (" + std::to_string(n) + ")");
        const auto r = init_rows(n, k, seed);
        std::copy(r.begin(), r.end(), rows);
    });
}


// ---------------------------------------------------------------------------
// row-sharded k-means: one rank's side (kmshard.cu)
// ---------------------------------------------------------------------------
}  // extern "C"

struct pqg_kmshard {
    pqg_ctx* own = nullptr;  // private context: its pinned arena holds the per-fit buffers
    pqg_ctx* parent = nullptr;
    RowSrc src;
    uint64_t n = 0, k = 0;
    uint32_t B = 0, d = 0, max_iters = 0;
    double tol = 0.0;
    uint32_t* assign = nullptr;
    double* dist = nullptr;
    uint64_t* offsets = nullptr;
    uint32_t* perm = nullptr;
    double* csum = nullptr;
    int* cmax = nullptr;
    int* cmin = nullptr;
    uint32_t* flags = nullptr;
    uint32_t* work = nullptr;
    uint32_t* cnt = nullptr;              // replay columns' local member counts
    uint64_t* pre = nullptr;              // their exclusive scan (pack offsets)
    unsigned long long* res = nullptr;    // n_fail, local pack length, global bound
    uint32_t* empties = nullptr;
    float* cnorm = nullptr;
    float* cmaxn = nullptr;
    uint64_t* init_rows = nullptr;
    KMeansState st{};
    uint64_t n_fail = 0;
    const uint8_t* big_rows = nullptr;
    const float* big_nx = nullptr;
    std::pair<size_t, size_t> mark{0, 0};
    // the fixed launch sequences of a step, replayed as CUDA graphs once their
    // pointers are known (the arena hands out the same scratch every step)
    struct Graph {
        cudaGraphExec_t exec = nullptr;
        const void* key[3] = {nullptr, nullptr, nullptr};
        bool warm = false;
        uint64_t launches = 0;
    } g_partials, g_apply;
    uint64_t nkd() const { return uint64_t(B) * k * d; }
    ~pqg_kmshard() {
        if (g_partials.exec) cudaGraphExecDestroy(g_partials.exec);
        if (g_apply.exec) cudaGraphExecDestroy(g_apply.exec);
    }
};

namespace {
// every step runs on the caller's current stream, in the handle's arena
struct ShardStep {
    pqg_kmshard* h;
    ShardStep(pqg_ctx* ctx, pqg_kmshard* hh) : h(hh) {
        if (!ctx || !hh) fail(PQG_EINVAL, "kmshard: null handle");
        PQG_CUDA(cudaSetDevice(h->own->device));
        h->own->stream = ctx->stream;
        h->own->arena.reset_to(h->mark);
    }
    ~ShardStep() { h->own->arena.reset_to(h->mark); }
};
// body() eagerly on the first call, captured on the second, replayed after
template <class F>
void run_graphed(pqg_ctx* o, pqg_kmshard::Graph& g, const void* k0, const void* k1, const void* k2, F&& body) {
    const char* ge = std::getenv("PQG_KM_GRAPH");
    // the legacy / per-thread default streams cannot be captured
    const bool legacy = o->stream == nullptr || o->stream == cudaStreamLegacy || o->stream == cudaStreamPerThread;
    if (o->profiling || legacy || (ge && ge[0] == '0')) {
        body();
        return;
    }
    if (g.exec && (g.key[0] != k0 || g.key[1] != k1 || g.key[2] != k2)) {
        cudaGraphExecDestroy(g.exec);
        g.exec = nullptr;
        g.warm = false;
    }
    if (!g.exec) {
        if (!g.warm) {
            body();
            g.warm = true;
            g.key[0] = k0;
            g.key[1] = k1;
            g.key[2] = k2;
            return;
        }
        const uint64_t l0 = o->launches;
        PQG_CUDA(cudaStreamBeginCapture(o->stream, cudaStreamCaptureModeRelaxed));
        try {
            body();
        } catch (...) {
            cudaGraph_t gg = nullptr;
            cudaStreamEndCapture(o->stream, &gg);
            if (gg) cudaGraphDestroy(gg);
            throw;
        }
        cudaGraph_t gg = nullptr;
        PQG_CUDA(cudaStreamEndCapture(o->stream, &gg));
        const cudaError_t ie = cudaGraphInstantiate(&g.exec, gg, 0);
        cudaGraphDestroy(gg);
        if (ie != cudaSuccess) fail(PQG_ECUDA, std::string("kmshard graph: ") + cudaGetErrorString(ie));
        g.launches = o->launches - l0;
        o->launches = l0;
    }
    PQG_CUDA(cudaGraphLaunch(g.exec, o->stream));
    o->launches += g.launches;
}
}  // namespace

extern "C" {

int pqg_kmshard_create(pqg_ctx* ctx, const float* rows, uint64_t n, uint64_t ld, uint32_t B, uint32_t d,
                       uint32_t col_stride, uint64_t k, uint32_t max_iters, double tol, pqg_kmshard** out_h) {
    return guard([&] {
        if (!out_h) inval("kmshard: null output");
        *out_h = nullptr;
        if (k == 0) inval("kmeans_fit: k must be >= 1");
        if (max_iters < 1) inval("kmeans_fit: max_iters must be >= 1");
        if (tol < 0.0) inval("kmeans_fit: tol must be >= 0");
        if (n == 0 || B == 0 || d == 0) inval("kmshard: empty shard");
        if (!on_device(rows)) inval("kmshard: rows must be device memory");
        RowSrc src;
        src.x = rows;
        src.ldx = ld;
        src.col_stride = col_stride;
        if (!kmeans_partials_supported(src, d) || uint64_t(B) * k * d > 0xFFFFFFFFull || n > 0xFFFFFFFFull)
            fail(PQG_EUNSUPPORTED, "kmshard: shape not supported by the sharded update (d % 4, d <= 128)");
        auto h = std::make_unique<pqg_kmshard>();
        PQG_CUDA(cudaSetDevice(ctx->device));
        // the workspace context (its arena holds the per-fit buffers) is cached
        // in the caller's context between fits: no allocation per fit
        if (ctx->shard_ws) {
            h->own = ctx->shard_ws;
            ctx->shard_ws = nullptr;
        } else {
            const int rc = pqg_ctx_create(ctx->device, &h->own);
            if (rc) fail(rc, g_last_error);
        }
        h->parent = ctx;
        h->own->stream = ctx->stream;
        h->own->arena.rewind();
        h->own->arena.depth = 1;  // pinned: the buffers below live until destroy
        pqg_ctx* o = h->own;
        h->src = src;
        h->n = n;
        h->k = k;
        h->B = B;
        h->d = d;
        h->max_iters = max_iters;
        h->tol = tol;
        const uint64_t nkd = uint64_t(B) * k * d;
        h->assign = scratch<uint32_t>(o, uint64_t(B) * n);
        h->dist = scratch<double>(o, uint64_t(B) * n);
        h->offsets = scratch<uint64_t>(o, uint64_t(B) * (k + 1));
        h->perm = scratch<uint32_t>(o, uint64_t(B) * n);
        h->csum = scratch<double>(o, nkd);
        h->cmax = scratch<int>(o, nkd);
        h->cmin = scratch<int>(o, nkd);
        h->flags = scratch<uint32_t>(o, nkd);
        h->work = scratch<uint32_t>(o, nkd);
        h->cnt = scratch<uint32_t>(o, nkd);
        h->pre = scratch<uint64_t>(o, nkd);
        h->res = scratch<unsigned long long>(o, 3);
        h->empties = scratch<uint32_t>(o, B);
        h->cnorm = scratch<float>(o, uint64_t(B) * k);
        h->cmaxn = scratch<float>(o, B);
        h->init_rows = scratch<uint64_t>(o, uint64_t(B) * k);
        h->st.active = scratch<int>(o, B);
        h->st.prev = scratch<double>(o, B);
        h->st.inertia = scratch<double>(o, B);
        h->st.per_iter = scratch<double>(o, uint64_t(B) * max_iters);
        h->st.iters = scratch<uint32_t>(o, B);
        std::vector<int> ones(B, 1);
        PQG_CUDA(cudaMemcpyAsync(h->st.active, ones.data(), sizeof(int) * B, cudaMemcpyHostToDevice, o->stream));
        PQG_CUDA(cudaMemsetAsync(h->st.prev, 0, sizeof(double) * B, o->stream));
        PQG_CUDA(cudaMemsetAsync(h->st.inertia, 0, sizeof(double) * B, o->stream));
        PQG_CUDA(cudaMemsetAsync(h->st.per_iter, 0, sizeof(double) * B * max_iters, o->stream));
        PQG_CUDA(cudaMemsetAsync(h->st.iters, 0, sizeof(uint32_t) * B, o->stream));
        // coarse fits: the row operand split once for the tensor-core screen
        NearestArgs prep;
        prep.src = src;
        prep.n = n;
        prep.d = d;
        prep.B = B;
        prep.k = k;
        prep.cmax = h->cmaxn;
        if (B == 1 && umma_big_prepare_rows(o, prep)) {
            h->big_rows = prep.big_rows;
            h->big_nx = prep.big_nx;
        }
        h->mark = o->arena.mark();
        PQG_CUDA(cudaStreamSynchronize(o->stream));
        *out_h = h.release();
    });
}

void pqg_kmshard_destroy(pqg_kmshard* h) {
    if (!h) return;
    if (h->own) {
        cudaStreamSynchronize(h->own->stream);
        h->own->stream = h->own->own_stream;
        h->own->arena.depth = 0;
        if (h->parent && !h->parent->shard_ws) h->parent->shard_ws = h->own;  // kept for the next fit
        else pqg_ctx_destroy(h->own);
    }
    delete h;
}

int pqg_kmshard_sizes(const pqg_kmshard* h, uint64_t* n_f64, uint64_t* n_u8) {
    return guard([&] {
        if (!h) inval("kmshard: null handle");
        if (n_f64) *n_f64 = h->nkd() + uint64_t(h->B) * h->k + h->B;
        if (n_u8) *n_u8 = 2 * h->nkd();
    });
}

int pqg_kmshard_init_table(pqg_ctx* ctx, pqg_kmshard* h, const uint64_t* init_rows, uint64_t row0,
                           uint32_t* table_bits) {
    return guard([&] {
        ShardStep step(ctx, h);
        pqg_ctx* o = h->own;
        PQG_CUDA(cudaMemcpyAsync(h->init_rows, init_rows, sizeof(uint64_t) * h->B * h->k,
                                 cudaMemcpyHostToDevice, o->stream));
        shard_init_gather(o, h->src, h->n, h->B, h->d, h->k, h->init_rows, row0, table_bits);
        PQG_CUDA(cudaStreamSynchronize(o->stream));  // init_rows is the caller's host buffer
        ctx->launches += 1;
    });
}

int pqg_kmshard_partials(pqg_ctx* ctx, pqg_kmshard* h, const float* tables, double* f64, uint8_t* u8) {
    return guard([&] {
        ShardStep step(ctx, h);
        pqg_ctx* o = h->own;
        const uint64_t l0 = o->launches;
        run_graphed(o, h->g_partials, tables, f64, u8, [&] {
        table_norms(o, tables, h->B, h->k, h->d, h->cnorm, h->cmaxn);
        NearestArgs a;
        a.src = h->src;
        a.n = h->n;
        a.d = h->d;
        a.B = h->B;
        a.table = tables;
        a.k = h->k;
        a.cnorm = h->cnorm;
        a.cmax = h->cmaxn;
        a.out_idx = h->assign;
        a.idx_bytes = 4;
        a.idx_rs = 1;
        a.idx_ps = h->n;
        a.out_dist = h->dist;
        a.active = h->st.active;
        a.big_rows = h->big_rows;
        a.big_nx = h->big_nx;
        nearest(o, a);
        kmeans_local_partials(o, h->src, h->n, h->B, h->d, h->k, h->assign, h->st.active, h->offsets,
                              h->perm, h->csum, h->cmax, h->cmin);
        shard_pack_partials(o, h->B, h->k, h->d, h->offsets, h->csum, h->cmax, h->cmin, f64, u8);
        rows_sum_f64(o, h->dist, h->n, h->B, f64 + h->nkd() + uint64_t(h->B) * h->k);
        });
        ctx->launches += o->launches - l0;
    });
}

int pqg_kmshard_apply(pqg_ctx* ctx, pqg_kmshard* h, float* tables, const double* f64, const uint8_t* u8,
                      uint64_t* n_fail, uint64_t* stride, uint32_t* max_empty, int* any_active) {
    return guard([&] {
        ShardStep step(ctx, h);
        pqg_ctx* o = h->own;
        const uint64_t l0 = o->launches;
        run_graphed(o, h->g_apply, tables, f64, u8, [&] {
            kmeans_stop_global(o, f64 + h->nkd() + uint64_t(h->B) * h->k, h->B, h->max_iters, h->tol, h->st);
            shard_finalize(o, h->B, h->k, h->d, f64, u8, h->st.active, tables, h->flags, h->empties);
            shard_replay_layout(o, h->B, h->k, h->d, h->flags, h->offsets, f64, h->work, h->cnt, h->pre, h->res);
        });
        // the iteration's one host synchronisation: sizes of the exchanges to come
        std::vector<unsigned long long> res(3);
        std::vector<uint32_t> emp(h->B);
        std::vector<int> act(h->B);
        PQG_CUDA(cudaMemcpyAsync(res.data(), h->res, sizeof(unsigned long long) * 3, cudaMemcpyDeviceToHost, o->stream));
        PQG_CUDA(cudaMemcpyAsync(emp.data(), h->empties, sizeof(uint32_t) * h->B, cudaMemcpyDeviceToHost, o->stream));
        PQG_CUDA(cudaMemcpyAsync(act.data(), h->st.active, sizeof(int) * h->B, cudaMemcpyDeviceToHost, o->stream));
        PQG_CUDA(cudaStreamSynchronize(o->stream));
        h->n_fail = res[0];
        uint32_t me = 0;
        int aa = 0;
        for (uint32_t b = 0; b < h->B; ++b) {
            if (act[b]) me = std::max(me, emp[b]);
            aa |= act[b];
        }
        if (n_fail) *n_fail = res[0];
        if (stride) *stride = std::max<unsigned long long>(1, res[2]);
        if (max_empty) *max_empty = me;
        if (any_active) *any_active = aa;
        ctx->launches += o->launches - l0;
    });
}

int pqg_kmshard_pack(pqg_ctx* ctx, pqg_kmshard* h, float* vals, uint64_t cap, uint64_t* offcnt) {
    return guard([&] {
        ShardStep step(ctx, h);
        pqg_ctx* o = h->own;
        const uint64_t l0 = o->launches;
        (void)cap;  // cap >= the apply's stride bounds every rank's pack
        shard_pack(o, h->src, h->work, h->n_fail, h->k, h->d, h->offsets, h->perm, h->n, h->cnt, h->pre, offcnt,
                   vals);
        ctx->launches += o->launches - l0;
    });
}

int pqg_kmshard_replay(pqg_ctx* ctx, pqg_kmshard* h, float* tables, const double* f64, const float* all_vals,
                       uint64_t stride, const uint64_t* all_offcnt, uint32_t world) {
    return guard([&] {
        ShardStep step(ctx, h);
        pqg_ctx* o = h->own;
        const uint64_t l0 = o->launches;
        shard_replay(o, h->work, h->n_fail, h->k, h->d, h->B, f64, all_vals, stride, all_offcnt, world, tables);
        ctx->launches += o->launches - l0;
    });
}

int pqg_kmshard_replay_step(pqg_ctx* ctx, pqg_kmshard* h, double* run) {
    return guard([&] {
        ShardStep step(ctx, h);
        pqg_ctx* o = h->own;
        const uint64_t l0 = o->launches;
        shard_replay_step(o, h->src, h->work, h->n_fail, h->k, h->d, h->offsets, h->perm, h->n, run);
        ctx->launches += o->launches - l0;
    });
}

int pqg_kmshard_replay_finish(pqg_ctx* ctx, pqg_kmshard* h, float* tables, const double* f64, const double* run) {
    return guard([&] {
        ShardStep step(ctx, h);
        pqg_ctx* o = h->own;
        const uint64_t l0 = o->launches;
        shard_replay_finish(o, h->work, h->n_fail, h->k, h->d, h->B, f64, run, tables);
        ctx->launches += o->launches - l0;
    });
}

int pqg_kmshard_reseed_candidates(pqg_ctx* ctx, pqg_kmshard* h, uint64_t row0, uint32_t E, double* cand_d,
                                  uint64_t* cand_i, float* cand_rows) {
    return guard([&] {
        ShardStep step(ctx, h);
        pqg_ctx* o = h->own;
        const uint64_t l0 = o->launches;
        shard_reseed_candidates(o, h->src, h->n, h->B, h->d, h->dist, h->st.active, h->empties, E, row0, cand_d,
                                cand_i, cand_rows);
        ctx->launches += o->launches - l0;
    });
}

int pqg_kmshard_reseed_apply(pqg_ctx* ctx, pqg_kmshard* h, float* tables, const double* f64, uint32_t E,
                             uint32_t world, const double* all_d, const uint64_t* all_i, const float* all_rows) {
    return guard([&] {
        ShardStep step(ctx, h);
        pqg_ctx* o = h->own;
        const uint64_t l0 = o->launches;
        shard_reseed_apply(o, h->B, h->k, h->d, f64, h->st.active, E, world, all_d, all_i, all_rows, tables);
        ctx->launches += o->launches - l0;
    });
}

int pqg_kmshard_result(pqg_ctx* ctx, pqg_kmshard* h, uint32_t* iterations_run, double* inertia,
                       double* inertia_per_iter, uint32_t* assignments) {
    return guard([&] {
        ShardStep step(ctx, h);
        pqg_ctx* o = h->own;
        if (iterations_run)
            PQG_CUDA(cudaMemcpyAsync(iterations_run, h->st.iters, sizeof(uint32_t) * h->B, cudaMemcpyDefault, o->stream));
        if (inertia)
            PQG_CUDA(cudaMemcpyAsync(inertia, h->st.inertia, sizeof(double) * h->B, cudaMemcpyDefault, o->stream));
        if (inertia_per_iter)
            PQG_CUDA(cudaMemcpyAsync(inertia_per_iter, h->st.per_iter, sizeof(double) * h->B * h->max_iters,
                                     cudaMemcpyDefault, o->stream));
        if (assignments)
            PQG_CUDA(cudaMemcpyAsync(assignments, h->assign, sizeof(uint32_t) * h->B * h->n, cudaMemcpyDefault,
                                     o->stream));
        PQG_CUDA(cudaStreamSynchronize(o->stream));
    });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// on-disk formats: PQII / PQCM / PQCB, byte-identical to
// the reference's writers (proj/src/ivf.cpp:264-355, pq.cpp:183-259).  The
// posting lists move between the file layout and the device CSR through the
// pack / unpack kernels of formats.cu; load-time validation (duplicate ids,
// code range, finite codewords) runs on the device.  Errors carry the
// reference's messages (io_util.hpp read_bytes / expect_magic) as PQG_EIO.
// ---------------------------------------------------------------------------
namespace {

[[noreturn]] void io_fail(const std::string& m) { fail(PQG_EIO, m); }

struct ByteReader {  // proj/src/io_util.hpp:45-87 over a memory image
    const uint8_t* b;
    uint64_t size, pos;
    void need(uint64_t k, const char* what) const {
        if (size - pos < k) io_fail(std::string("truncated read of ") + what);
    }
    uint32_t u32(const char* what) {
        need(4, what);
        const uint32_t v = uint32_t(b[pos]) | uint32_t(b[pos + 1]) << 8 | uint32_t(b[pos + 2]) << 16 |
                           uint32_t(b[pos + 3]) << 24;
        pos += 4;
        return v;
    }
    uint64_t u64(const char* what) {
        need(8, what);
        uint64_t v = 0;
        for (int i = 7; i >= 0; --i) v = (v << 8) | b[pos + i];
        pos += 8;
        return v;
    }
    void magic(const char* m, const char* format_name) {
        need(4, "magic");
        if (std::memcmp(b + pos, m, 4) != 0) io_fail(std::string(format_name) + ": bad magic");
        pos += 4;
    }
    // k elements of `es` bytes (overflow-safe)
    const uint8_t* bytes(uint64_t k, uint64_t es, const char* what) {
        if (es && k > (size - pos) / es) io_fail(std::string("truncated read of ") + what);
        const uint8_t* p = b + pos;
        pos += k * es;
        return p;
    }
};

void put32(std::vector<uint8_t>& o, uint32_t v) {
    for (int i = 0; i < 4; ++i) o.push_back(uint8_t(v >> (8 * i)));
}
void put64(std::vector<uint8_t>& o, uint64_t v) {
    for (int i = 0; i < 8; ++i) o.push_back(uint8_t(v >> (8 * i)));
}

struct Pinned {  // page-locked host staging for file <-> device transfers
    uint8_t* p = nullptr;
    explicit Pinned(uint64_t n) {
        if (cudaHostAlloc(reinterpret_cast<void**>(&p), std::max<uint64_t>(n, 1), cudaHostAllocDefault) !=
            cudaSuccess) {
            cudaGetLastError();
            fail(PQG_ENOMEM, "pinned host allocation of " + std::to_string(n) + " bytes failed");
        }
    }
    ~Pinned() {
        if (p) cudaFreeHost(p);
    }
};

struct File {
    FILE* f = nullptr;
    File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
    ~File() {
        if (f) std::fclose(f);
    }
};

// whole file -> pinned host image
std::unique_ptr<Pinned> read_file(const char* path, uint64_t* size) {
    File f(path, "rb");
    if (!f.f) io_fail(std::string("cannot open file: ") + path);
    std::fseek(f.f, 0, SEEK_END);
    const long n = std::ftell(f.f);
    std::fseek(f.f, 0, SEEK_SET);
    if (n < 0) io_fail(std::string("cannot open file: ") + path);
    auto buf = std::make_unique<Pinned>(uint64_t(n));
    if (n && std::fread(buf->p, 1, size_t(n), f.f) != size_t(n)) io_fail(std::string("cannot read file: ") + path);
    *size = uint64_t(n);
    return buf;
}

void write_file(const char* path, const uint8_t* p, uint64_t n) {
    File f(path, "wb");
    if (!f.f) io_fail(std::string("cannot open file for writing: ") + path);
    if (n && std::fwrite(p, 1, size_t(n), f.f) != size_t(n)) io_fail(std::string("write failed: ") + path);
    if (std::fflush(f.f) != 0) io_fail(std::string("write failed: ") + path);
}

uint64_t index_header_bytes(const pqg_index* ix) {
    return 28 + 4 * uint64_t(ix->M) * ix->ks * ix->ds + 4 + 4 * ix->nlist * ix->D();
}

// PQII header (ivf.cpp:267-281): magic, version, embedded PQCB block, nlist, coarse
std::vector<uint8_t> index_header(pqg_ctx* ctx, const pqg_index* ix) {
    std::vector<uint8_t> h;
    h.reserve(index_header_bytes(ix));
    h.insert(h.end(), {'P', 'Q', 'I', 'I'});
    put32(h, 1);
    h.insert(h.end(), {'P', 'Q', 'C', 'B'});
    put32(h, 1);
    put32(h, ix->M);
    put32(h, ix->ks);
    put32(h, ix->ds);
    const uint64_t nt = uint64_t(ix->M) * ix->ks * ix->ds, nc = ix->nlist * ix->D();
    const size_t at = h.size();
    h.resize(at + 4 * nt);
    PQG_CUDA(cudaMemcpyAsync(h.data() + at, ix->tables, 4 * nt, cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    put32(h, uint32_t(ix->nlist));
    const size_t at2 = h.size();
    h.resize(at2 + 4 * nc);
    PQG_CUDA(cudaMemcpyAsync(h.data() + at2, ix->coarse, 4 * nc, cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    return h;
}

uint64_t index_image_bytes(const pqg_index* ix) {
    return index_header_bytes(ix) + 8 * ix->nlist + ix->n * (8 + ix->rb());
}

void serialize_index(pqg_ctx* ctx, const pqg_index* ix, uint8_t* buf) {
    const std::vector<uint8_t> hdr = index_header(ctx, ix);
    const uint64_t sec_bytes = 8 * ix->nlist + ix->n * (8 + ix->rb());
    const bool dev = on_device(buf);
    uint8_t* sec = dev ? buf + hdr.size() : scratch<uint8_t>(ctx, sec_bytes);
    pqii_pack(ctx, ix->offsets, ix->ids, ix->codes, ix->nlist, ix->n, ix->rb(), sec);
    if (dev) {
        PQG_CUDA(cudaMemcpyAsync(buf, hdr.data(), hdr.size(), cudaMemcpyHostToDevice, ctx->stream));
    } else {
        std::memcpy(buf, hdr.data(), hdr.size());
        PQG_CUDA(cudaMemcpyAsync(buf + hdr.size(), sec, sec_bytes, cudaMemcpyDeviceToHost, ctx->stream));
    }
    sync(ctx);
}

// load_index (ivf.cpp:295-355) over a host image: the header and the list
// headers are walked on the host (one jump per list), the entries are
// unpacked on the device.  The first error is the one the reference would
// raise reading front to back: per list, a duplicate id while reading its
// entries, then a code range error at its end; a truncation stops the walk.
pqg_index* parse_index(pqg_ctx* ctx, const uint8_t* img, uint64_t size, const std::string& name) {
    ByteReader r{img, size, 0};
    r.magic("PQII", "index file");
    const uint32_t ver = r.u32("version");
    if (ver != 1) io_fail(name + ": unsupported version " + std::to_string(ver));
    r.magic("PQCB", "embedded codebook");
    if (r.u32("codebook version") != 1) io_fail(name + ": unsupported codebook version");
    const uint32_t M = r.u32("M"), ks = r.u32("Ks"), ds = r.u32("sub_dim");
    if (M == 0 || ks == 0 || ds == 0) io_fail(name + ": invalid codebook header");
    if (uint64_t(M) * ks > (uint64_t(1) << 40) / ds) io_fail("truncated read of codebook tables");
    const uint64_t nt = uint64_t(M) * ks * ds;
    const float* tables = reinterpret_cast<const float*>(r.bytes(nt, 4, "codebook tables"));
    const uint32_t nlist = r.u32("nlist");
    if (nlist == 0) io_fail(name + ": nlist must be >= 1");
    const uint64_t D = uint64_t(M) * ds;
    const float* coarse = reinterpret_cast<const float*>(r.bytes(uint64_t(nlist) * D, 4, "coarse centroids"));
    check_pq_shape(M, ks, 1, "codebook");  // make_lists -> CodeMatrix(0, M, ks) (pq.cpp:35-39)
    const uint32_t w = code_width(ks);
    const uint64_t rb = uint64_t(M) * w, es = 8 + rb;
    // ---- walk the list headers
    const uint64_t sec0 = r.pos;
    std::vector<uint64_t> off(1, 0), src;
    int64_t t_list = -1;
    uint64_t t_entry = 0;
    const char* t_what = nullptr;
    for (uint64_t l = 0; l < nlist; ++l) {
        if (size - r.pos < 8) {
            t_list = int64_t(l);
            t_what = "list length";
            break;
        }
        const uint64_t len = r.u64("list length");
        const uint64_t avail = (size - r.pos) / es;
        src.push_back(r.pos - sec0);
        if (len > avail) {
            const uint64_t rem = (size - r.pos) - avail * es;
            t_list = int64_t(l);
            t_entry = avail;
            t_what = rem < 8 ? "entry id" : "entry code";
            off.push_back(off.back() + avail);
            r.pos += avail * es;
            break;
        }
        off.push_back(off.back() + len);
        r.pos += len * es;
    }
    const uint64_t nl_parsed = off.size() - 1, n = off.back();
    // ---- device: index object, entries unpacked into its CSR
    const float* dt = in(ctx, tables, nt);
    const float* dco = in(ctx, coarse, uint64_t(nlist) * D);
    pqg_index* ix = new_index(ctx, M, ks, ds, nlist, n, dt, dco);
    try {
        const uint64_t sec_bytes = r.pos - sec0;
        if (nl_parsed) {
            const uint8_t* dsec = in(ctx, img + sec0, sec_bytes);
            const uint64_t* dsrc = in(ctx, src.data(), nl_parsed);
            const uint64_t* doff = in(ctx, off.data(), nl_parsed + 1);
            pqii_unpack(ctx, dsec, dsrc, doff, nl_parsed, n, rb, ix->ids, ix->codes);
        }
        uint64_t h_dup = ~uint64_t(0);
        unsigned long long h_bad = ~0ull;
        if (n >= 2) {
            uint64_t* pos = scratch<uint64_t>(ctx, 1);
            find_duplicate(ctx, ix->ids, n, pos);
            PQG_CUDA(cudaMemcpyAsync(&h_dup, pos, sizeof(h_dup), cudaMemcpyDeviceToHost, ctx->stream));
        }
        if (n && (w == 2 || ks < 256)) {
            unsigned long long* bad = scratch<unsigned long long>(ctx, 1);
            first_bad_code(ctx, ix->codes, n, M, ks, w, bad);
            PQG_CUDA(cudaMemcpyAsync(&h_bad, bad, sizeof(h_bad), cudaMemcpyDeviceToHost, ctx->stream));
        }
        sync(ctx);
        auto list_of = [&](uint64_t e) {
            return uint64_t(std::upper_bound(off.begin(), off.end(), e) - off.begin()) - 1;
        };
        // event keys (list, phase, entry): entries are read (and id-checked)
        // in phase 0, the list's codes are range-checked in phase 1
        struct Ev {
            uint64_t l, ph, e;
            int kind;  // 0 dup, 1 range, 2 truncation
        };
        std::vector<Ev> ev;
        if (h_dup != ~uint64_t(0)) {
            const uint64_t l = list_of(h_dup);
            ev.push_back({l, 0, h_dup - off[l], 0});
        }
        if (h_bad != ~0ull) {
            const uint64_t l = list_of(h_bad);
            if (!(t_list >= 0 && l == uint64_t(t_list))) ev.push_back({l, 1, 0, 1});  // a truncated list is never range-checked
        }
        if (t_list >= 0) ev.push_back({uint64_t(t_list), 0, t_entry, 2});
        if (!ev.empty()) {
            const Ev first = *std::min_element(ev.begin(), ev.end(), [](const Ev& a, const Ev& b) {
                return std::tie(a.l, a.ph, a.e) < std::tie(b.l, b.ph, b.e);
            });
            if (first.kind == 0) {
                uint64_t id = 0;
                PQG_CUDA(cudaMemcpy(&id, ix->ids + h_dup, sizeof(id), cudaMemcpyDeviceToHost));
                io_fail(name + ": duplicate id " + std::to_string(id));
            }
            if (first.kind == 1) io_fail(name + ": code out of range");
            io_fail(std::string("truncated read of ") + t_what);
        }
        if (r.pos != size) io_fail(name + ": trailing data after payload");
        PQG_CUDA(cudaMemcpyAsync(ix->offsets, off.data(), sizeof(uint64_t) * (nlist + 1), cudaMemcpyHostToDevice,
                                 ctx->stream));
        sync(ctx);
    } catch (...) {
        ix->free_all();
        delete ix;
        throw;
    }
    return ix;
}

// PQCM / PQCB headers (pq.cpp:221-232, :183-193)
struct CodesHdr {
    uint64_t n;
    uint32_t M, ks;
};
CodesHdr codes_header(ByteReader& r, const std::string& name) {
    r.magic("PQCM", "code file");
    const uint32_t ver = r.u32("version");
    if (ver != 1) io_fail(name + ": unsupported version " + std::to_string(ver));
    CodesHdr h;
    h.n = r.u64("row count");
    h.M = r.u32("M");
    h.ks = r.u32("Ks");
    check_pq_shape(h.M, h.ks, 1, "codebook");  // CodeMatrix(n, M, ks) (pq.cpp:35-39)
    return h;
}
struct CbHdr {
    uint32_t M, ks, ds;
};
CbHdr codebook_header(ByteReader& r, const std::string& name) {
    r.magic("PQCB", "codebook file");
    const uint32_t ver = r.u32("version");
    if (ver != 1) io_fail(name + ": unsupported version " + std::to_string(ver));
    CbHdr h;
    h.M = r.u32("M");
    h.ks = r.u32("Ks");
    h.ds = r.u32("sub_dim");
    check_pq_shape(h.M, h.ks, h.ds, "codebook");
    return h;
}

// the first `cap` bytes of a file (headers only)
std::vector<uint8_t> read_head(const char* path, uint64_t cap) {
    File f(path, "rb");
    if (!f.f) io_fail(std::string("cannot open file: ") + path);
    std::vector<uint8_t> v(cap);
    v.resize(std::fread(v.data(), 1, cap, f.f));
    return v;
}

}  // namespace

extern "C" {

int pqg_index_serialize(pqg_ctx* ctx, const pqg_index* ix, void* buf, uint64_t cap, uint64_t* size) {
    return guard([&] {
        Scope sc(ctx);
        if (!ix) inval("index serialize: null index");
        const uint64_t total = index_image_bytes(ix);
        if (size) *size = total;
        if (!buf) return;
        if (cap < total)
            inval("index serialize: buffer of " + std::to_string(cap) + " bytes, image needs " + std::to_string(total));
        serialize_index(ctx, ix, static_cast<uint8_t*>(buf));
    });
}

int pqg_index_deserialize(pqg_ctx* ctx, const void* buf, uint64_t size, const char* name, pqg_index** out) {
    return guard([&] {
        Scope sc(ctx);
        const std::string nm = name ? name : "index image";
        const uint8_t* img = static_cast<const uint8_t*>(buf);
        std::unique_ptr<Pinned> host;
        if (on_device(buf)) {  // the header walk runs on the host
            host = std::make_unique<Pinned>(size);
            PQG_CUDA(cudaMemcpy(host->p, buf, size, cudaMemcpyDeviceToHost));
            img = host->p;
        }
        *out = parse_index(ctx, img, size, nm);
    });
}

int pqg_index_save(pqg_ctx* ctx, const pqg_index* ix, const char* path) {
    return guard([&] {
        Scope sc(ctx);
        if (!ix) inval("save_index: null index");
        const uint64_t total = index_image_bytes(ix);
        Pinned buf(total);
        serialize_index(ctx, ix, buf.p);
        write_file(path, buf.p, total);
    });
}

int pqg_index_load(pqg_ctx* ctx, const char* path, pqg_index** out) {
    return guard([&] {
        Scope sc(ctx);
        uint64_t size = 0;
        auto img = read_file(path, &size);
        *out = parse_index(ctx, img->p, size, path);
    });
}

int pqg_codes_save(pqg_ctx* ctx, const uint8_t* codes, uint64_t n, uint32_t M, uint32_t ks, const char* path) {
    return guard([&] {
        Scope sc(ctx);
        check_pq_shape(M, ks, 1, "codebook");
        const uint64_t payload = n * M * code_width(ks);
        std::vector<uint8_t> h;
        h.insert(h.end(), {'P', 'Q', 'C', 'M'});
        put32(h, 1);
        put64(h, n);
        put32(h, M);
        put32(h, ks);
        Pinned buf(h.size() + payload);
        std::memcpy(buf.p, h.data(), h.size());
        if (payload) {
            PQG_CUDA(cudaMemcpyAsync(buf.p + h.size(), codes, payload, cudaMemcpyDefault, ctx->stream));
            sync(ctx);
        }
        write_file(path, buf.p, h.size() + payload);
    });
}

int pqg_codes_file_info(const char* path, uint64_t* n, uint32_t* M, uint32_t* ks) {
    return guard([&] {
        const std::vector<uint8_t> head = read_head(path, 24);
        ByteReader r{head.data(), head.size(), 0};
        const CodesHdr h = codes_header(r, path);
        if (n) *n = h.n;
        if (M) *M = h.M;
        if (ks) *ks = h.ks;
    });
}

int pqg_codes_load(pqg_ctx* ctx, const char* path, uint8_t* codes, uint64_t cap_bytes) {
    return guard([&] {
        Scope sc(ctx);
        uint64_t size = 0;
        auto img = read_file(path, &size);
        ByteReader r{img->p, size, 0};
        const CodesHdr h = codes_header(r, path);
        const uint32_t w = code_width(h.ks);
        if (h.n > (uint64_t(1) << 48) / (uint64_t(h.M) * w)) io_fail(std::string(path) + ": truncated payload");
        const uint64_t payload = h.n * h.M * w;
        if (cap_bytes < payload) inval("load_codes: output buffer of " + std::to_string(cap_bytes) + " bytes < " +
                                       std::to_string(payload));
        if (size - r.pos < payload) io_fail(std::string(path) + ": truncated payload");
        if (!payload) return;
        const bool dev = on_device(codes);
        uint8_t* d = dev ? codes : scratch<uint8_t>(ctx, payload);
        PQG_CUDA(cudaMemcpyAsync(d, img->p + r.pos, payload, cudaMemcpyHostToDevice, ctx->stream));
        unsigned long long* bad = scratch<unsigned long long>(ctx, 1);
        unsigned long long hb = ~0ull;
        first_bad_code(ctx, d, h.n, h.M, h.ks, w, bad);
        PQG_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost, ctx->stream));
        if (!dev) std::memcpy(codes, img->p + r.pos, payload);
        sync(ctx);
        if (hb != ~0ull) io_fail(std::string(path) + ": code out of range at row " + std::to_string(hb));
    });
}

int pqg_codebook_save(pqg_ctx* ctx, const float* tables, uint32_t M, uint32_t ks, uint32_t ds, const char* path) {
    return guard([&] {
        Scope sc(ctx);
        check_pq_shape(M, ks, ds, "codebook");
        const uint64_t payload = 4 * uint64_t(M) * ks * ds;
        std::vector<uint8_t> h;
        h.insert(h.end(), {'P', 'Q', 'C', 'B'});
        put32(h, 1);
        put32(h, M);
        put32(h, ks);
        put32(h, ds);
        Pinned buf(h.size() + payload);
        std::memcpy(buf.p, h.data(), h.size());
        PQG_CUDA(cudaMemcpyAsync(buf.p + h.size(), tables, payload, cudaMemcpyDefault, ctx->stream));
        sync(ctx);
        write_file(path, buf.p, h.size() + payload);
    });
}

int pqg_codebook_file_info(const char* path, uint32_t* M, uint32_t* ks, uint32_t* ds) {
    return guard([&] {
        const std::vector<uint8_t> head = read_head(path, 20);
        ByteReader r{head.data(), head.size(), 0};
        const CbHdr h = codebook_header(r, path);
        if (M) *M = h.M;
        if (ks) *ks = h.ks;
        if (ds) *ds = h.ds;
    });
}

int pqg_codebook_load(pqg_ctx* ctx, const char* path, float* tables, uint64_t cap_floats) {
    return guard([&] {
        Scope sc(ctx);
        uint64_t size = 0;
        auto img = read_file(path, &size);
        ByteReader r{img->p, size, 0};
        const CbHdr h = codebook_header(r, path);
        const uint64_t count = uint64_t(h.M) * h.ks * h.ds;
        if (cap_floats < count)
            inval("load_codebook: output buffer of " + std::to_string(cap_floats) + " floats < " + std::to_string(count));
        if ((size - r.pos) / 4 < count) io_fail(std::string(path) + ": truncated payload");
        const bool dev = on_device(tables);
        float* d = dev ? tables : scratch<float>(ctx, count);
        PQG_CUDA(cudaMemcpyAsync(d, img->p + r.pos, 4 * count, cudaMemcpyHostToDevice, ctx->stream));
        unsigned long long* bad = scratch<unsigned long long>(ctx, 1);
        unsigned long long hb = ~0ull;
        first_nonfinite(ctx, d, count, bad);
        PQG_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost, ctx->stream));
        if (!dev) std::memcpy(tables, img->p + r.pos, 4 * count);
        sync(ctx);
        if (hb != ~0ull) io_fail(std::string(path) + ": non-finite codeword value");
    });
}

}  // extern "C"
