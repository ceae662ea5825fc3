// kmeans.cu -- K2: the Lloyd update of proj/src/kmeans.cpp:93-130 for a batch
// of B problems, plus the stable bucketing (histogram -> prefix scan ->
// stable scatter) shared with the inverted-index build (K6).
//
// Exactness.  The reference accumulates centroid sums in fp64 in row order
// (kmeans.cpp:103-111).  Floating-point addition is not associative in
// general, so the rows are first bucketed by cluster with a STABLE counting
// sort (members of each cluster in ascending row order).  The sums are then
// taken in parallel where that provably equals the row-order sum (all partial
// sums exact, see mean_exact_kernel) and in row order otherwise.  The mean is
// float(sum * (1.0 / count)) (:112-118) and empty clusters are reseeded from
// the pre-update fp64 distances, ascending cluster order, strict '>' argmax
// (:122-130).  The resulting centroids are bit-identical to the reference's.
#include "kernels.cuh"
#include "tc_common.cuh"

namespace pqg {

namespace {

// Bucketing geometry: a tile of T rows per CTA of W warps (each warp walks
// T/W consecutive rows); W is bounded by the per-warp key counters in shared
// memory, T by the size of the [k][tiles] count matrix that is scanned.
struct BucketGeom {
    uint32_t W, T, ntiles;
};
BucketGeom bucket_geom(uint64_t n, uint64_t k) {
    BucketGeom g;
    // W a power of two (T / W rows per warp must tile T exactly)
    const uint64_t wmax = std::max<uint64_t>(1, std::min<uint64_t>(8, (96 * 1024) / (4 * std::max<uint64_t>(k, 1))));
    g.W = 1;
    while (uint64_t(g.W) * 2 <= wmax) g.W *= 2;
    g.T = k <= 1024 ? 1024u : 4096u;  // multiples of 32 * W for every W <= 8
    g.ntiles = uint32_t((n + g.T - 1) / g.T);
    return g;
}

// Accumulators a later kernel of the same update adds into (csum = 0,
// cmax = -1, cmin = 2^30 per (problem, cluster, dim)): zeroed by the
// histogram launch, which has the grid for it (r2e: pieces_setup's B CTAs
// spent ~40% of its 8 us on this).
struct SumInit {
    double* csum = nullptr;
    int* cmax = nullptr;
    int* cmin = nullptr;
    uint64_t count = 0;
};

__global__ void hist_kernel(const uint32_t* keys, uint64_t n, uint64_t k, uint32_t ntiles, uint32_t T,
                            uint32_t* tile_counts, SumInit zi) {
    extern __shared__ uint32_t hist[];
    const uint32_t tile = blockIdx.x, b = blockIdx.y;
    if (zi.count) {
        const uint64_t nthr = uint64_t(gridDim.x) * gridDim.y * blockDim.x;
        for (uint64_t e = (uint64_t(b) * gridDim.x + tile) * blockDim.x + threadIdx.x; e < zi.count; e += nthr) {
            zi.csum[e] = 0.0;
            zi.cmax[e] = -1;
            zi.cmin[e] = 1 << 30;
        }
    }
    for (uint64_t c = threadIdx.x; c < k; c += blockDim.x) hist[c] = 0;
    __syncthreads();
    const uint64_t r0 = uint64_t(tile) * T;
    const uint64_t r1 = min64(n, r0 + T);
    const uint32_t* kb = keys + uint64_t(b) * n;
    for (uint64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
        const uint32_t c = __ldg(kb + i);
        if (c < k) atomicAdd(&hist[c], 1u);  // key k marks a padding row (no cluster)
    }
    __syncthreads();
    uint32_t* out = tile_counts + uint64_t(b) * k * ntiles;
    for (uint64_t c = threadIdx.x; c < k; c += blockDim.x) out[c * ntiles + tile] = hist[c];
}

// Copy of the bucketed rows: xs[b][pos][0..d) = x row i of problem b, so the
// sums read each cluster's members as one contiguous, row-ordered block.
struct RowCopy {
    const float* x;
    uint64_t ldx;
    uint32_t col_stride, d;
    float* out;      // [B][n][d]
    bool vec;        // float4 path (d, ldx, col_stride and x 16-byte aligned)
};

// One CTA per (tile, problem), W warps, warp w owning rows [w*T/W, (w+1)*T/W)
// of the tile.  Pass 1 counts each warp's keys, pass 2 turns the counts into
// per-warp bases (tile base from the scan + the earlier warps' counts), pass 3
// re-walks the rows in order: __match_any_sync ranks equal keys within 32
// rows and the per-warp cursor keeps order across rounds, so members land in
// ascending row order.  Output: the row permutation or (ROWS) the rows
// themselves; tile 0 also writes the problem's cluster offsets.  (The
// minimum-blocks hint keeps ptxas from sinking the row loads of the copy into
// their stores, which serialises them.)
// Lanes holding the same key (valid lanes only): NB > 0 compares the low NB
// key bits with NB ballots (r2e: ALU votes instead of the MIO-bound MATCH
// instruction, which throttled the scatter -- ncu: mio_throttle and
// short_scoreboard stalls); NB == 0 is __match_any_sync.  Invalid lanes get
// an arbitrary mask and must not use it.
template <int NB>
__device__ __forceinline__ uint32_t key_peers(uint32_t c, bool valid) {
    if constexpr (NB == 0) {
        return __match_any_sync(0xffffffffu, valid ? c : 0xFFFFFFFFu);
    } else {
        uint32_t peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            const bool bit = (c >> i) & 1u;
            const uint32_t b = __ballot_sync(0xffffffffu, bit);
            peers &= bit ? b : ~b;
        }
        return peers;
    }
}

template <bool ROWS, int NB = 0>
__global__ void __launch_bounds__(256, 1) scatter_kernel(const uint32_t* keys, uint64_t n, uint64_t k, uint32_t ntiles, uint32_t T,
                               const uint64_t* tile_base, uint32_t* perm, RowCopy rc, uint64_t* offsets,
                               const uint64_t* nb) {
    extern __shared__ uint32_t wc[];  // [W][k]
    const uint32_t W = blockDim.x >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t tile = blockIdx.x, b = blockIdx.y;
    const uint64_t* tb = tile_base + uint64_t(b) * k * ntiles;
    const uint64_t first = tb[0];  // problem b's start in the all-problem scan
    for (uint64_t e = threadIdx.x; e < uint64_t(W) * k; e += blockDim.x) wc[e] = 0;
    __syncthreads();
    const uint64_t seg = T / W;
    const uint64_t wr0 = uint64_t(tile) * T + w * seg;
    const uint64_t wr1 = min64(n, wr0 + seg);
    const uint32_t* kb = keys + uint64_t(b) * n;
    uint32_t* mine = wc + uint64_t(w) * k;
    // rows go in batches of kRounds x 32: the batch's keys are loaded together
    constexpr int kRounds = 4;
    for (uint64_t i0 = wr0; i0 < wr1; i0 += 32 * kRounds) {
        uint32_t cs[kRounds];
#pragma unroll
        for (int r = 0; r < kRounds; ++r) {
            const uint64_t i = i0 + r * 32 + lane;
            cs[r] = i < wr1 ? __ldg(kb + i) : 0xFFFFFFFFu;
        }
#pragma unroll
        for (int r = 0; r < kRounds; ++r) {
            const uint64_t i = i0 + r * 32 + lane;
            const uint32_t c = cs[r];
            const bool ok = i < wr1 && c < k;
            const uint32_t peers = key_peers<NB>(c, ok);
            if (ok && (peers & lanemask_lt()) == 0) mine[c] += __popc(peers);
            __syncwarp();
        }
    }
    __syncthreads();
    for (uint64_t c = threadIdx.x; c < k; c += blockDim.x) {
        const uint64_t start = tb[c * ntiles] - first;
        uint64_t base = tb[c * ntiles + tile] - first;
        for (uint32_t v = 0; v < W; ++v) {
            const uint32_t t = wc[uint64_t(v) * k + c];
            wc[uint64_t(v) * k + c] = uint32_t(base);
            base += t;
        }
        if (tile == 0 && offsets) offsets[uint64_t(b) * (k + 1) + c] = start;
    }
    if (tile == 0 && offsets && threadIdx.x == 0) offsets[uint64_t(b) * (k + 1) + k] = nb ? nb[b] : n;
    __syncthreads();
    for (uint64_t i0 = wr0; i0 < wr1; i0 += 32 * kRounds) {
        uint32_t cs[kRounds], pos[kRounds];
        bool valid[kRounds];
#pragma unroll
        for (int r = 0; r < kRounds; ++r) {
            const uint64_t i = i0 + r * 32 + lane;
            cs[r] = i < wr1 ? __ldg(kb + i) : 0xFFFFFFFFu;
        }
#pragma unroll
        for (int r = 0; r < kRounds; ++r) {
            const uint64_t i = i0 + r * 32 + lane;
            const uint32_t c = cs[r];
            valid[r] = i < wr1 && c < k;
            const uint32_t peers = key_peers<NB>(c, valid[r]);
            const uint32_t rank = __popc(peers & lanemask_lt());
            pos[r] = valid[r] ? mine[c] + rank : 0u;
            __syncwarp();
            if (valid[r] && rank == 0) mine[c] += __popc(peers);
            __syncwarp();
        }
        if (!ROWS) {
#pragma unroll
            for (int r = 0; r < kRounds; ++r)
                if (valid[r]) perm[uint64_t(b) * n + pos[r]] = uint32_t(i0 + r * 32 + lane);
        } else {
            // each lane copies its rows: whole 16-byte pieces (full sectors);
            // the batch's (row, piece) units go eight at a time, all loads
            // (unpredicated, clamped) issued before the stores
            const uint32_t Q = rc.vec ? rc.d / 4 : rc.d;
            const uint32_t U = kRounds * Q;
            const float* xb = rc.x + uint64_t(b) * rc.col_stride;
            float* ob = rc.out + uint64_t(b) * n * rc.d;
            for (uint32_t e0 = 0; e0 < U; e0 += 8) {
                float4 v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint32_t e = min(e0 + u, U - 1);
                    const uint32_t r = e / Q, t = e - r * Q;
                    const uint64_t i = min64(i0 + r * 32 + lane, wr1 - 1);
                    if (rc.vec) v[u] = __ldg(reinterpret_cast<const float4*>(xb + i * rc.ldx) + t);
                    else v[u].x = __ldg(xb + i * rc.ldx + t);
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint32_t e = e0 + u;
                    if (e >= U) break;
                    const uint32_t r = e / Q, t = e - r * Q;
                    bool ok = false;
                    uint32_t ps = 0;
#pragma unroll
                    for (int rr = 0; rr < kRounds; ++rr)
                        if (uint32_t(rr) == r) { ok = valid[rr]; ps = pos[rr]; }
                    if (!ok) continue;
                    if (rc.vec) reinterpret_cast<float4*>(ob + uint64_t(ps) * rc.d)[t] = v[u];
                    else ob[uint64_t(ps) * rc.d + t] = v[u].x;
                }
            }
        }
    }
}

// ---- exclusive scan u32 -> u64 (three phase, 4096 elements per block) ----
constexpr int kScanThreads = 1024, kScanItems = 4;
constexpr int kScanBlock = kScanThreads * kScanItems;

template <typename T>
__device__ uint64_t block_exclusive(T (&v)[kScanItems], uint64_t (&out)[kScanItems]) {
    __shared__ uint64_t warp_tot[32];
    uint64_t s = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) { out[j] = s; s += v[j]; }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint64_t incl = s;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint64_t o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += o;
    }
    if (lane == 31) warp_tot[w] = incl;
    __syncthreads();
    if (w == 0) {
        uint64_t t = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
        uint64_t ti = t;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint64_t o = __shfl_up_sync(0xffffffffu, ti, off);
            if (lane >= off) ti += o;
        }
        warp_tot[lane] = ti - t;  // exclusive warp prefix
    }
    __syncthreads();
    const uint64_t pre = warp_tot[w] + (incl - s);
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) out[j] += pre;
    __shared__ uint64_t total;
    if (threadIdx.x == blockDim.x - 1) total = pre + s;
    __syncthreads();
    const uint64_t t = total;
    __syncthreads();
    return t;
}

template <typename T>
__global__ void scan_reduce_kernel(const T* in, uint64_t count, uint64_t* block_sums) {
    const uint64_t base = uint64_t(blockIdx.x) * kScanBlock;
    T v[kScanItems];
    uint64_t o[kScanItems];
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        const uint64_t e = base + uint64_t(threadIdx.x) * kScanItems + j;
        v[j] = e < count ? in[e] : T(0);
    }
    const uint64_t tot = block_exclusive(v, o);
    if (threadIdx.x == 0) block_sums[blockIdx.x] = tot;
}

template <typename T>
__global__ void scan_apply_kernel(const T* in, uint64_t count, const uint64_t* block_pre,
                                  uint64_t* out) {
    const uint64_t base = uint64_t(blockIdx.x) * kScanBlock;
    T v[kScanItems];
    uint64_t o[kScanItems];
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        const uint64_t e = base + uint64_t(threadIdx.x) * kScanItems + j;
        v[j] = e < count ? in[e] : T(0);
    }
    block_exclusive(v, o);
    const uint64_t pre = block_pre ? block_pre[blockIdx.x] : 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        const uint64_t e = base + uint64_t(threadIdx.x) * kScanItems + j;
        if (e < count) out[e] = o[j] + pre;
    }
}

template <typename T>
void exclusive_scan(pqg_ctx* ctx, const T* in, uint64_t* out, uint64_t count) {
    if (count == 0) return;
    const uint64_t nb = (count + kScanBlock - 1) / kScanBlock;
    if (nb == 1) {
        launch(ctx, "scan", scan_apply_kernel<T>, dim3(1), dim3(kScanThreads), 0, in, count,
               (const uint64_t*)nullptr, out);
        return;
    }
    uint64_t* sums = scratch<uint64_t>(ctx, nb);
    uint64_t* pre = scratch<uint64_t>(ctx, nb);
    launch(ctx, "scan", scan_reduce_kernel<T>, dim3(unsigned(nb)), dim3(kScanThreads), 0, in,
           count, sums);
    exclusive_scan<uint64_t>(ctx, sums, pre, nb);
    launch(ctx, "scan", scan_apply_kernel<T>, dim3(unsigned(nb)), dim3(kScanThreads), 0, in,
           count, (const uint64_t*)pre, out);
}

__global__ void gather_kernel(const float* x, uint64_t ldx, uint32_t B, uint32_t d,
                              uint32_t col_stride, const uint64_t* rows, uint64_t k,
                              float* table) {
    const uint64_t total = uint64_t(B) * k * d;
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t bc = e / d, t = e - bc * d;
        const uint64_t b = bc / k;
        table[e] = x[rows[bc] * ldx + b * col_stride + t];
    }
}

// ---- inertia (deterministic fixed-shape tree) and the stop rule ----------
constexpr int kRedThreads = 256;

__device__ double block_sum(double v) {
    __shared__ double sh[kRedThreads];
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int s = kRedThreads / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) sh[threadIdx.x] = __dadd_rn(sh[threadIdx.x], sh[threadIdx.x + s]);
        __syncthreads();
    }
    const double r = sh[0];
    __syncthreads();
    return r;
}

// The fixed reduction shape (chunking of n rows) shared by the in-loop
// inertia and pqg_rows_sum_f64, so sharded and single-process fits see
// identical sums; a problem with fewer rows (nb) uses its own shape, so a
// batched fit of unequal problems sums exactly like separate fits.
__host__ __device__ inline void inertia_parts(uint64_t n, uint64_t& nparts, uint64_t& chunk) {
    nparts = n == 0 ? 1 : min64(512, (n + 8191) / 8192);
    chunk = n == 0 ? 1 : (n + nparts - 1) / nparts;
    nparts = n == 0 ? 1 : (n + chunk - 1) / chunk;
}

__global__ void partial_sum_kernel(const double* v, uint64_t n, uint64_t chunk, double* parts,
                                   const int* active, const uint64_t* nb) {
    const uint32_t b = blockIdx.y;
    if (active && !active[b]) return;
    uint64_t nn = n;
    if (nb) {
        uint64_t np;
        nn = nb[b];
        inertia_parts(nn, np, chunk);
        if (blockIdx.x >= np) return;
    }
    const uint64_t c0 = uint64_t(blockIdx.x) * chunk;
    const uint64_t c1 = min64(nn, c0 + chunk);
    const double* vb = v + uint64_t(b) * n;
    double s = 0.0;
    for (uint64_t i = c0 + threadIdx.x; i < c1; i += kRedThreads) s = __dadd_rn(s, vb[i]);
    s = block_sum(s);
    if (threadIdx.x == 0) parts[uint64_t(b) * gridDim.x + blockIdx.x] = s;
}

// proj/src/kmeans.cpp:93-100 for problem b, every thread of a kRedThreads
// block calling it (parts read through L2: other blocks wrote them)
__device__ void stop_rule(const double* parts, uint32_t nparts, uint32_t b, uint32_t max_iters, double tol,
                          const KMeansState& st, const uint64_t* nb) {
    const uint32_t itd = st.iters[b] + 1;
    uint64_t cnt = nparts;
    if (nb) {
        uint64_t chunk;
        inertia_parts(nb[b], cnt, chunk);
    }
    double s = 0.0;
    for (uint32_t i = threadIdx.x; i < cnt; i += kRedThreads)
        s = __dadd_rn(s, __ldcg(parts + uint64_t(b) * nparts + i));
    s = block_sum(s);
    if (threadIdx.x != 0) return;
    st.inertia[b] = s;
    if (st.per_iter) st.per_iter[uint64_t(b) * max_iters + (itd - 1)] = s;
    st.iters[b] = itd;
    const double prev = st.prev[b];
    const double floor1 = prev > 1.0 ? prev : 1.0;
    if ((itd > 1 && prev - s < tol * floor1) || itd == max_iters) {
        st.active[b] = 0;
        return;
    }
    st.prev[b] = s;
}

// The inertia's partial sums with the stop rule fused (r2e): the block that
// completes a problem's parts (ticket) applies the rule; tickets re-armed.
__global__ void partial_sum_stop_kernel(const double* v, uint64_t n, uint64_t chunk, double* parts,
                                        const uint64_t* nb, uint32_t max_iters, double tol, KMeansState st) {
    const uint32_t b = blockIdx.y;
    if (!st.active[b]) return;
    uint64_t nn = n, np = gridDim.x;
    if (nb) {
        nn = nb[b];
        inertia_parts(nn, np, chunk);
        if (blockIdx.x >= np) return;
    }
    const uint64_t c0 = uint64_t(blockIdx.x) * chunk;
    const uint64_t c1 = min64(nn, c0 + chunk);
    const double* vb = v + uint64_t(b) * n;
    double s = 0.0;
    for (uint64_t i = c0 + threadIdx.x; i < c1; i += kRedThreads) s = __dadd_rn(s, vb[i]);
    s = block_sum(s);
    __shared__ unsigned last;
    if (threadIdx.x == 0) {
        parts[uint64_t(b) * gridDim.x + blockIdx.x] = s;
        __threadfence();
        last = atomicAdd(st.tickets + b, 1u) == unsigned(np - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    stop_rule(parts, gridDim.x, b, max_iters, tol, st, nb);
    if (threadIdx.x == 0) st.tickets[b] = 0u;
}

__global__ void stop_kernel(const double* parts, uint32_t nparts, uint32_t it, uint32_t max_iters,
                            double tol, KMeansState st, const uint64_t* nb) {
    const uint32_t b = blockIdx.x;
    if (!st.active[b]) return;
    // the pass number from the device state (an active problem has run every
    // pass so far), so the launch is the same for every pass
    (void)it;
    const uint32_t itd = st.iters[b] + 1;
    uint64_t cnt = nparts;
    if (nb) {
        uint64_t chunk;
        inertia_parts(nb[b], cnt, chunk);
    }
    double s = 0.0;
    for (uint32_t i = threadIdx.x; i < cnt; i += kRedThreads)
        s = __dadd_rn(s, parts[uint64_t(b) * nparts + i]);
    s = block_sum(s);
    if (threadIdx.x != 0) return;
    // proj/src/kmeans.cpp:93-100
    st.inertia[b] = s;
    if (st.per_iter) st.per_iter[uint64_t(b) * max_iters + (itd - 1)] = s;
    st.iters[b] = itd;
    const double prev = st.prev[b];
    const double floor1 = prev > 1.0 ? prev : 1.0;
    if ((itd > 1 && prev - s < tol * floor1) || itd == max_iters) {
        st.active[b] = 0;
        return;
    }
    st.prev[b] = s;
}

__global__ void final_parts_kernel(const double* parts, uint32_t nparts, double* out) {
    const uint32_t b = blockIdx.x;
    double s = 0.0;
    for (uint32_t i = threadIdx.x; i < nparts; i += kRedThreads)
        s = __dadd_rn(s, parts[uint64_t(b) * nparts + i]);
    s = block_sum(s);
    if (threadIdx.x == 0) out[b] = s;
}

// Centroid means without a sequential chain.  The reference adds the members'
// fp32 values into an fp64 sum in row order (kmeans.cpp:103-111).  Every fp32
// value is an integer multiple of the smallest member's ulp; when the largest
// magnitude is within 2^(28 - ceil(log2 count)) of that ulp scale, every
// partial sum of any order fits in fp64's 53-bit significand, so all orders
// give the same exact sum and the members can be added in parallel.  A
// (cluster, dim) outside that range (values spanning > ~20 binades, or
// non-finite) is summed sequentially in row order as the reference does.
// One CTA per (problem, cluster): threads = (member group, dim), rows read
// through the stable member permutation (no gathered copy).
constexpr int kMeanThreads = 256;
constexpr int kMeanStage = 4096;  // members staged per step of the row-order fallback

// Row-order fp64 sum (kmeans.cpp:103-111) of the staged values col[mi*nf+f],
// mi < nm, continuing from s; every thread of a kMeanThreads block calls it
// and gets the same result.  The members go in chunks of kMeanThreads: a
// chunk whose additions are all exact -- every partial sum is a multiple of
// q = min(ulp(s), ulp of its smallest value) and below 2^lb, lb - log2 q <= 53
// -- is added as one parallel exact sum; only a chunk that can round is walked
// sequentially.  (A rejected (cluster, dim) typically holds one tiny value,
// so one chunk in a thousand-member cluster runs the serial chain.)  s is a
// normal double here (sums of fp32 values never reach the fp64 subnormals).
struct SeqScratch {
    double rsum[2][kMeanThreads / 32];
    int rmax[2][kMeanThreads / 32], rmin[2][kMeanThreads / 32];
    double bc;
};
__device__ double staged_row_order_sum(double s, const float* col, uint32_t nf, uint32_t f, uint32_t nm,
                                       SeqScratch& sc, uint32_t& par) {
    const uint32_t tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    for (uint32_t c0 = 0; c0 < nm; c0 += kMeanThreads) {
        const uint32_t mi = c0 + tid;
        const float v = mi < nm ? col[mi * nf + f] : 0.f;
        const int eb = int((__float_as_uint(v) >> 23) & 0xFFu);
        int ehi = v != 0.f ? eb : -1;
        int elo = v != 0.f ? max(eb, 1) : (1 << 30);
        double ds = (double)v;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            ds = __dadd_rn(ds, __shfl_xor_sync(0xffffffffu, ds, o));
            ehi = max(ehi, __shfl_xor_sync(0xffffffffu, ehi, o));
            elo = min(elo, __shfl_xor_sync(0xffffffffu, elo, o));
        }
        if (lane == 0) {
            sc.rsum[par][w] = ds;
            sc.rmax[par][w] = ehi;
            sc.rmin[par][w] = elo;
        }
        __syncthreads();
        double tot = 0.0;
        ehi = -1;
        elo = 1 << 30;
#pragma unroll
        for (int u = 0; u < kMeanThreads / 32; ++u) {
            tot = __dadd_rn(tot, sc.rsum[par][u]);
            ehi = max(ehi, sc.rmax[par][u]);
            elo = min(elo, sc.rmin[par][u]);
        }
        par ^= 1u;
        bool exact;
        if (ehi < 0) {
            exact = true;  // all zeros
        } else if (ehi == 255 || !isfinite(s)) {
            exact = false;
        } else {
            int lq = elo - 150;  // log2 ulp of the smallest nonzero value
            if (s != 0.0) {
                // s = mant * 2^(E-1075): its lowest set bit, not its ulp, bounds
                // the granularity (a running sum of fp32 values is usually a
                // multiple of a much coarser power of two than its ulp)
                const unsigned long long sb = __double_as_longlong(s);
                const int E = int((sb >> 52) & 0x7FF);
                const unsigned long long mant = (sb & ((1ull << 52) - 1)) | (1ull << 52);
                lq = min(lq, E - 1075 + (__ffsll((long long)mant) - 1));
            }
            // every partial sum is at most |s| + kMeanThreads values below
            // 2^(ehi-126) each, rounded up: below 2^lb
            const double bound = __dadd_ru(fabs(s), ldexp(1.0, ehi - 118));
            const int lb = int((__double_as_longlong(bound) >> 52) & 0x7FF) - 1022;
            exact = lb - lq <= 53;
        }
        if (exact) {
            s = __dadd_rn(s, tot);
        } else {
            if (tid == 0) {
                const uint32_t me = min(nm - c0, uint32_t(kMeanThreads));
                double q = s;
#pragma unroll 8
                for (uint32_t i = 0; i < me; ++i) q = __dadd_rn(q, (double)col[(c0 + i) * nf + f]);
                sc.bc = q;
            }
            __syncthreads();
            s = sc.bc;
        }
    }
    return s;
}

__global__ void __launch_bounds__(kMeanThreads) mean_exact_kernel(
    const float* x, uint64_t ldx, uint32_t col_stride, uint64_t n, uint32_t d, uint64_t k,
    const uint64_t* offsets, const uint32_t* perm, float* table, int* has_empty, const int* active) {
    __shared__ double ps[kMeanThreads];
    __shared__ int pmax[kMeanThreads], pmin[kMeanThreads];
    __shared__ float col[kMeanStage];  // one dim of the members, row order (fallback)
    __shared__ uint32_t nfail;
    __shared__ uint32_t failed[kMeanThreads];
    __shared__ SeqScratch sc;
    __shared__ double sres[kMeanThreads];
    const uint64_t bc = blockIdx.x;
    const uint64_t b = bc / k, c = bc - b * k;
    if (active && !active[b]) return;
    const uint64_t* off = offsets + b * (k + 1);
    const uint64_t beg = off[c], end = off[c + 1];
    if (beg == end) {
        if (threadIdx.x == 0) has_empty[b] = 1;
        return;
    }
    const uint64_t cnt = end - beg;
    const uint32_t* pb = perm ? perm + b * n : nullptr;  // null: x is the bucketed copy
    const float* xb = x + b * col_stride;
    const uint32_t DG = d < kMeanThreads ? d : kMeanThreads;
    const uint32_t G = kMeanThreads / DG;
    const uint32_t g = threadIdx.x / DG, tl = threadIdx.x - g * DG;
    int lg = 0;
    while ((uint64_t(1) << lg) < cnt) ++lg;
    const double inv = __ddiv_rn(1.0, (double)cnt);
    for (uint32_t t0 = 0; t0 < d; t0 += DG) {
        const uint32_t t = t0 + tl;
        double s = 0.0;
        int emax = -1, emin = 1 << 30;
        if (g < G && t < d) {
            auto acc = [&](float v) {
                s = __dadd_rn(s, (double)v);
                const int e = int((__float_as_uint(v) >> 23) & 0xFFu);
                if (v != 0.f) {
                    emax = max(emax, e);
                    emin = min(emin, max(e, 1));
                }
            };
            uint64_t m = beg + g;
            // four members in flight per thread: the permutation and row loads of
            // one step are independent of the adds
            for (; m + 3 * uint64_t(G) < end; m += 4 * uint64_t(G)) {
                uint32_t r[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) r[u] = pb ? __ldg(pb + m + u * G) : uint32_t(m + u * G);
                float v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = __ldg(xb + uint64_t(r[u]) * ldx + t);
#pragma unroll
                for (int u = 0; u < 4; ++u) acc(v[u]);
            }
            for (; m < end; m += G) acc(__ldg(xb + uint64_t(pb ? __ldg(pb + m) : uint32_t(m)) * ldx + t));
        }
        ps[threadIdx.x] = s;
        pmax[threadIdx.x] = emax;
        pmin[threadIdx.x] = emin;
        if (threadIdx.x == 0) nfail = 0;
        __syncthreads();
        if (g == 0 && t < d) {
            for (uint32_t h = 1; h < G; ++h) {
                s = __dadd_rn(s, ps[h * DG + tl]);
                emax = max(emax, pmax[h * DG + tl]);
                emin = min(emin, pmin[h * DG + tl]);
            }
            const bool exact = emax < 0 || (emax < 255 && emax - emin + lg <= 28);
            if (exact) table[bc * d + t] = __double2float_rn(__dmul_rn(s, inv));  // kmeans.cpp:112-118
            else failed[atomicAdd(&nfail, 1u)] = t;
        }
        __syncthreads();
        // row-order sums (kmeans.cpp:103-111) for the dims the exactness test
        // rejects: the block stages a chunk of members x failing dims, then one
        // thread per failing dim adds its column in row order (dims in parallel)
        const uint32_t nf = nfail;
        if (nf > 0) {
            const uint64_t mchunk = kMeanStage / nf;
            uint32_t par = 0;
            if (threadIdx.x < nf) sres[threadIdx.x] = 0.0;
            for (uint64_t m0 = beg; m0 < end; m0 += mchunk) {
                const uint64_t m1 = m0 + mchunk < end ? m0 + mchunk : end;
                const uint32_t nm = uint32_t(m1 - m0);
                for (uint32_t e = threadIdx.x; e < nm * nf; e += blockDim.x) {
                    const uint32_t mi = e / nf, f = e - mi * nf;
                    col[e] = __ldg(xb + uint64_t(pb ? __ldg(pb + m0 + mi) : uint32_t(m0 + mi)) * ldx + failed[f]);
                }
                __syncthreads();
                for (uint32_t f = 0; f < nf; ++f) {
                    const double sf = staged_row_order_sum(sres[f], col, nf, f, nm, sc, par);
                    __syncthreads();
                    if (threadIdx.x == 0) sres[f] = sf;
                }
                __syncthreads();
            }
            if (threadIdx.x < nf)
                table[bc * d + failed[threadIdx.x]] = __double2float_rn(__dmul_rn(sres[threadIdx.x], inv));
        }
        __syncthreads();
    }
}


// ---- Piece-parallel exact means -------------------------------------------
// A cluster's members (row order after the stable bucketing) are cut into
// pieces of R = 8*G rows; one warp per piece accumulates fp64 sums and the
// exponent range per dim (lane (g, q): float4 column group q of rows g, g+G,
// ...; eight row loads in flight), writes them as PieceStats, and the warp
// that completes a cluster's last piece finalizes it: if the whole cluster
// passes the exactness test the piece sums are added in any order; otherwise
// the pieces are replayed in row order -- a piece whose additions are
// provably exact given the running sum is added whole, any other one member
// by member (the reference's sequential fp64 chain, kmeans.cpp:103-111).
// Big clusters therefore spread over many warps, and the serial fallback is
// confined to the pieces that can actually round.
struct PieceStat {
    double s;
    int emax, emin;
};
struct PieceGeom {
    uint32_t DG, G, R, lR;  // lanes per row, row groups, rows per piece, log2 R
    uint64_t PP;            // piece slots per problem
};
__host__ __device__ inline PieceGeom piece_geom(uint32_t d, uint64_t n, uint64_t k) {
    PieceGeom g;
    g.DG = d / 4;
    g.G = 32 / g.DG;
    g.R = 8 * g.G;
    g.lR = 0;
    while ((1u << g.lR) < g.R) ++g.lR;
    g.PP = (n + g.R - 1) / g.R + k;
    return g;
}

// A piece: rows [r0, r0 + rows) of its problem's bucketed order (rows == 0:
// unused slot).
struct PieceDesc {
    uint64_t r0;
    uint32_t rows, c;
};

// Per problem: piece counts -> piece_start (exclusive scan), the piece
// descriptors, the empty-cluster flag.
__global__ void __launch_bounds__(1024) pieces_setup_kernel(const uint64_t* offsets, uint64_t k, uint32_t R,
                                                            uint64_t PP, uint32_t* piece_start,
                                                            PieceDesc* pieces, int* has_empty,
                                                            const int* active, uint32_t d, double* csum,
                                                            int* cmax, int* cmin,
                                                            unsigned long long* work_count) {
    __shared__ uint32_t wsum[32];
    __shared__ int any_empty;
    const uint32_t b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (tid == 0) any_empty = 0;
    (void)d; (void)csum; (void)cmax; (void)cmin;  // zeroed by the histogram launch (SumInit)
    const uint64_t* off = offsets + uint64_t(b) * (k + 1);
    const uint64_t per = (k + blockDim.x - 1) / blockDim.x;
    const uint64_t c0 = min64(k, tid * per), c1 = min64(k, c0 + per);
    uint32_t local = 0;
    bool empty = false;
    for (uint64_t c = c0; c < c1; ++c) {
        const uint64_t cnt = off[c + 1] - off[c];
        local += uint32_t((cnt + R - 1) / R);
        empty |= cnt == 0;
    }
    uint32_t incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= uint32_t(o)) incl += v;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (empty) any_empty = 1;
    if (w == 0) {
        const uint32_t nw = blockDim.x >> 5;
        uint32_t t = lane < nw ? wsum[lane] : 0u, ti = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, ti, o);
            if (lane >= uint32_t(o)) ti += v;
        }
        if (lane < nw) wsum[lane] = ti - t;
    }
    __syncthreads();
    uint32_t base = wsum[w] + incl - local;
    for (uint64_t c = c0; c < c1; ++c) {
        const uint64_t cnt = off[c + 1] - off[c];
        const uint32_t np = uint32_t((cnt + R - 1) / R);
        piece_start[uint64_t(b) * k + c] = base;
        for (uint32_t i = 0; i < np; ++i) {
            const uint64_t r0 = off[c] + uint64_t(i) * R;
            pieces[uint64_t(b) * PP + base + i] = PieceDesc{r0, uint32_t(min64(R, off[c + 1] - r0)), uint32_t(c)};
        }
        base += np;
    }
    __syncthreads();
    // the last thread's end is the total: mark the unused slots
    __shared__ uint32_t total;
    if (tid == blockDim.x - 1) total = base;
    __syncthreads();
    for (uint64_t p = total + tid; p < PP; p += blockDim.x) pieces[uint64_t(b) * PP + p] = PieceDesc{0, 0u, 0u};
    if (tid == 0) has_empty[b] = (active && !active[b]) ? 0 : any_empty;
    if (b == 0 && tid == 0) *work_count = 0;
}

// Row m of problem b's bucketed order: the copy (xs) or the permutation.
struct MemberRows {
    const float* x;      // copy: [B][n][d]; permutation: the rows
    uint64_t ldx;
    uint32_t col_stride;
    const uint32_t* perm;  // null: x is the bucketed copy
};
__device__ __forceinline__ const float* member_row(const MemberRows& mr, uint64_t n, uint32_t d, uint64_t b,
                                                   uint64_t m) {
    if (!mr.perm) return mr.x + (b * n + m) * d;
    return mr.x + uint64_t(__ldg(mr.perm + b * n + m)) * mr.ldx + b * mr.col_stride;
}

__global__ void __launch_bounds__(kMeanThreads, 4) mean_pieces_kernel(
    MemberRows mr, uint64_t n, uint32_t d, uint64_t k, uint32_t B, const PieceDesc* pieces, PieceStat* stats,
    const int* active, double* csum, int* cmax, int* cmin) {
    const uint32_t lane = threadIdx.x & 31;
    const PieceGeom pg = piece_geom(d, n, k);
    const uint64_t wgl = uint64_t(blockIdx.x) * (kMeanThreads / 32) + (threadIdx.x >> 5);
    if (wgl >= uint64_t(B) * pg.PP) return;
    const uint64_t b = wgl / pg.PP;
    if (active && !active[b]) return;
    const PieceDesc pd = pieces[wgl];
    if (pd.rows == 0) return;
    const uint64_t r0 = pd.r0;
    const uint32_t rows = pd.rows;
    const uint32_t DG = pg.DG, G = pg.G;
    const uint32_t g = lane / DG, q = lane - g * DG;
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    int emax[4] = {-1, -1, -1, -1}, emin[4] = {1 << 30, 1 << 30, 1 << 30, 1 << 30};
    // r2e: the exponent range from the magnitude bits a = bits << 1 (sign
    // dropped, biased exponent in bits 31..24): max a, and min (a - 1), which
    // wraps zeros to 0xFFFFFFFF -- two integer min/max per value instead of
    // the extract / test / clamp chain (the kernel was ALU-bound, ncu r2e 65%)
    uint32_t amax[4] = {0u, 0u, 0u, 0u}, amin1[4] = {~0u, ~0u, ~0u, ~0u};
    if (g < G) {
        float4 v[8];
        if (!mr.perm) {
#pragma unroll
            for (int u = 0; u < 8; ++u)
                v[u] = __ldg(reinterpret_cast<const float4*>(mr.x + (b * n + r0 + min(g + u * G, rows - 1)) * d) + q);
        } else {
            uint32_t rid[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) rid[u] = __ldg(mr.perm + b * n + r0 + min(g + u * G, rows - 1));
#pragma unroll
            for (int u = 0; u < 8; ++u)
                v[u] = __ldg(reinterpret_cast<const float4*>(mr.x + uint64_t(rid[u]) * mr.ldx + b * mr.col_stride) + q);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const bool in = g + u * G < rows;  // rows past the end count as zeros: exact, no exponent
            const float e4[4] = {in ? v[u].x : 0.f, in ? v[u].y : 0.f, in ? v[u].z : 0.f, in ? v[u].w : 0.f};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                s[j] = __dadd_rn(s[j], (double)e4[j]);
                const uint32_t a2 = __float_as_uint(e4[j]) * 2u;
                amax[j] = max(amax[j], a2);
                amin1[j] = min(amin1[j], a2 - 1u);
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (amax[j] != 0u) emax[j] = int(amax[j] >> 24);
            if (amin1[j] != ~0u) emin[j] = max(int((amin1[j] + 1u) >> 24), 1);
        }
    }
    for (uint32_t h = 1; h < G; ++h) {  // groups into group 0 (exact: any order)
        const uint32_t src = h * DG + q;
        const uint32_t sl = (g == 0 && src < 32) ? src : lane;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const double os = __shfl_sync(0xffffffffu, s[j], sl);
            const int oa = __shfl_sync(0xffffffffu, emax[j], sl);
            const int oi = __shfl_sync(0xffffffffu, emin[j], sl);
            if (g == 0) {
                s[j] = __dadd_rn(s[j], os);
                emax[j] = max(emax[j], oa);
                emin[j] = min(emin[j], oi);
            }
        }
    }
    // the piece's stats (for a row-order replay) and the cluster totals:
    // atomic fp64 adds of exact partial sums are exact in any order whenever
    // the cluster passes the test; the finalize checks that
    PieceStat* st = stats + wgl * d;
    if (g == 0) {
        const uint64_t cb = (b * k + pd.c) * d + q * 4;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            st[q * 4 + j] = PieceStat{s[j], emax[j], emin[j]};
            atomicAdd(csum + cb + j, s[j]);
            if (emax[j] >= 0) {
                atomicMax(cmax + cb + j, emax[j]);
                atomicMin(cmin + cb + j, emin[j]);
            }
        }
    }
}

// One warp per cluster: combine its pieces' stats (see above).
__global__ void __launch_bounds__(kMeanThreads) mean_finalize_kernel(
    MemberRows mr, uint64_t n, uint32_t d, uint64_t k, uint32_t B, const uint64_t* offsets,
    const uint32_t* piece_start, const PieceStat* stats, float* table, const int* active, const double* csum,
    const int* cmax, const int* cmin, unsigned long long* work_count, uint64_t* work) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t bc = uint64_t(blockIdx.x) * (kMeanThreads / 32) + (threadIdx.x >> 5);
    if (bc >= uint64_t(B) * k) return;
    const uint64_t b = bc / k, c = bc - b * k;
    if (active && !active[b]) return;
    const uint64_t beg = offsets[b * (k + 1) + c], end = offsets[b * (k + 1) + c + 1];
    if (beg == end) return;  // empty: the reseed fills it
    const uint64_t cnt = end - beg;
    (void)piece_start;
    (void)stats;
    (void)mr;
    int lg = 0;
    while ((uint64_t(1) << lg) < cnt) ++lg;
    const double inv = __ddiv_rn(1.0, (double)cnt);
    // (1) lane t: the cluster's total and exponent range of dim t
    uint32_t need = 0;  // bit: dim lane + 32*bit rejected by the exactness test
    for (uint32_t t = lane, bit = 0; t < d; t += 32, ++bit) {
        const int ea = cmax[bc * d + t], ei = cmin[bc * d + t];
        if (ea < 0 || (ea < 255 && ea - ei + lg <= 28))
            table[bc * d + t] = __double2float_rn(__dmul_rn(csum[bc * d + t], inv));  // any order is exact
        else
            need |= 1u << bit;
    }
    // (2) rejected dims go to the replay worklist (a warp each, below)
    for (uint32_t bit = 0; 32 * bit < d; ++bit) {
        if ((need >> bit) & 1u) {
            const unsigned long long slot = atomicAdd(work_count, 1ull);
            work[slot] = (uint64_t(bc) << 16) | (32 * bit + lane);
        }
    }
}

// Row-order replay of one rejected (cluster, dim) per warp: the pieces in
// row order, 32 at a time -- a batch whose additions provably cannot round
// (every partial sum a multiple of 2^lq below 2^(lq+53), lq from the running
// sum's lowest set bit and the batch's smallest ulp) is added as one sum,
// otherwise piece by piece: a piece that cannot round is added whole, any
// other member by member (the reference's chain, kmeans.cpp:103-111).
__device__ __forceinline__ int lowbit_exp(double r) {  // log2 of r's lowest set bit (r normal, != 0)
    const unsigned long long sb = __double_as_longlong(r);
    const int E = int((sb >> 52) & 0x7FF);
    const unsigned long long mant = (sb & ((1ull << 52) - 1)) | (1ull << 52);
    return E - 1075 + (__ffsll((long long)mant) - 1);
}
__device__ __forceinline__ int mag_exp(double r) {  // |r| < 2^mag_exp
    return int((__double_as_longlong(r) >> 52) & 0x7FF) - 1022;
}

__global__ void __launch_bounds__(kMeanThreads) mean_replay_kernel(
    MemberRows mr, uint64_t n, uint32_t d, uint64_t k, const uint64_t* offsets, const uint32_t* piece_start,
    const PieceStat* stats, float* table, const unsigned long long* work_count, const uint64_t* work) {
    __shared__ float wbuf[kMeanThreads / 32][256];  // a piece's members, for the serial chain
    const uint32_t lane = threadIdx.x & 31;
    float* buf = wbuf[threadIdx.x >> 5];
    const PieceGeom pg = piece_geom(d, n, k);
    const unsigned long long cntw = *work_count;
    for (uint64_t wi = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; wi < cntw;
         wi += (uint64_t(gridDim.x) * blockDim.x) >> 5) {
        const uint64_t item = work[wi];
        const uint64_t bc = item >> 16;
        const uint32_t t = uint32_t(item & 0xFFFFu);
        const uint64_t b = bc / k, c = bc - b * k;
        const uint64_t beg = offsets[b * (k + 1) + c], end = offsets[b * (k + 1) + c + 1];
        const uint64_t cnt = end - beg;
        const uint32_t np = uint32_t((cnt + pg.R - 1) / pg.R);
        const PieceStat* cs = stats + (b * pg.PP + piece_start[bc]) * d;
        double r = 0.0;
        uint64_t wbeg = 0, wend = 0;  // members cached in buf
        for (uint32_t i0 = 0; i0 < np; i0 += 32) {
            const uint32_t nb = min(32u, np - i0);
            const bool in = lane < nb;
            const PieceStat* e = &cs[uint64_t(i0 + (in ? lane : 0)) * d + t];
            const double ls = in ? __ldcg(&e->s) : 0.0;
            const int la = in ? __ldcg(&e->emax) : -1, lm = in ? __ldcg(&e->emin) : (1 << 30);
            // batch test
            int ehi = la, elo = lm;
            double tot = ls;
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) {
                ehi = max(ehi, __shfl_xor_sync(0xffffffffu, ehi, o));
                elo = min(elo, __shfl_xor_sync(0xffffffffu, elo, o));
                tot = __dadd_rn(tot, __shfl_xor_sync(0xffffffffu, tot, o));
            }
            bool batch_exact;
            if (ehi < 0) {
                batch_exact = true;
            } else if (ehi == 255 || !isfinite(r)) {
                batch_exact = false;
            } else {
                // every partial sum is a multiple of 2^lq and at most
                // |r| + (32 R values below 2^(ehi-126)) < 2^lb
                int lq = elo - 150;
                if (r != 0.0) lq = min(lq, lowbit_exp(r));
                const double bound = __dadd_ru(fabs(r), ldexp(1.0, ehi - 126 + int(pg.lR) + 5));
                batch_exact = mag_exp(bound) - lq <= 53;
            }
            if (batch_exact) {
                r = __dadd_rn(r, tot);
                continue;
            }
            for (uint32_t ii = 0; ii < nb; ++ii) {
                const double ss = __shfl_sync(0xffffffffu, ls, ii);
                const int a = __shfl_sync(0xffffffffu, la, ii), m = __shfl_sync(0xffffffffu, lm, ii);
                bool exact;
                if (a < 0) {
                    exact = true;
                } else if (a == 255 || !isfinite(r)) {
                    exact = false;
                } else {
                    int lq = m - 150;
                    if (r != 0.0) lq = min(lq, lowbit_exp(r));
                    const double bound = __dadd_ru(fabs(r), ldexp(1.0, a - 126 + int(pg.lR)));
                    exact = mag_exp(bound) - lq <= 53;
                }
                if (exact) {
                    r = __dadd_rn(r, ss);
                    continue;
                }
                // this piece can round: the reference's chain, member by member;
                // members come through a 256-member window in shared memory
                // (runs of such pieces share one load round trip)
                const uint64_t m0 = beg + uint64_t(i0 + ii) * pg.R;
                const uint32_t mn = uint32_t(min64(pg.R, end - m0));  // <= 256
                if (m0 < wbeg || m0 + mn > wend) {
                    wbeg = m0;
                    wend = min64(end, m0 + 256);
                    const uint32_t wn = uint32_t(wend - wbeg);
                    float v[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        v[u] = __ldg(member_row(mr, n, d, b, wbeg + min(uint32_t(u * 32) + lane, wn - 1)) + t);
                    __syncwarp();
#pragma unroll
                    for (int u = 0; u < 8; ++u) buf[u * 32 + lane] = v[u];
                    __syncwarp();
                }
                // r2e: in batches of 32 members -- a batch whose additions
                // provably cannot round given r (the piece test at member
                // granularity) is added as one warp sum; only the others walk
                // the chain (ncu r2e at configs[3] scale: the member-by-member
                // walk of whole pieces was the kernel's tail, 10% occupancy)
                const float* wv = buf + (m0 - wbeg);
                for (uint32_t j0 = 0; j0 < mn; j0 += 32) {
                    const uint32_t nm = min(32u, mn - j0);
                    const float v = lane < nm ? wv[j0 + lane] : 0.f;
                    const int eb = int((__float_as_uint(v) >> 23) & 0xFFu);
                    int bhi = v != 0.f ? eb : -1, blo = v != 0.f ? max(eb, 1) : (1 << 30);
                    double ws = (double)v;
#pragma unroll
                    for (int o = 16; o >= 1; o >>= 1) {
                        ws = __dadd_rn(ws, __shfl_xor_sync(0xffffffffu, ws, o));
                        bhi = max(bhi, __shfl_xor_sync(0xffffffffu, bhi, o));
                        blo = min(blo, __shfl_xor_sync(0xffffffffu, blo, o));
                    }
                    bool bex;
                    if (bhi < 0) {
                        bex = true;
                    } else if (bhi == 255 || !isfinite(r)) {
                        bex = false;
                    } else {
                        int lq = blo - 150;
                        if (r != 0.0) lq = min(lq, lowbit_exp(r));
                        // 32 values below 2^(bhi-126) each
                        const double bound = __dadd_ru(fabs(r), ldexp(1.0, bhi - 121));
                        bex = mag_exp(bound) - lq <= 53;
                    }
                    if (bex) {
                        r = __dadd_rn(r, ws);
                        continue;
                    }
                    if (lane == 0) {
                        double q = r;
#pragma unroll 8
                        for (uint32_t l = 0; l < nm; ++l) q = __dadd_rn(q, (double)wv[j0 + l]);
                        r = q;
                    }
                    r = __shfl_sync(0xffffffffu, r, 0);
                }
            }
        }
        if (lane == 0) table[bc * d + t] = __double2float_rn(__dmul_rn(r, __ddiv_rn(1.0, (double)cnt)));
    }
}

// The same sums for small sub-dimensions (d <= 32, the PQ fits): one warp per
// (problem, cluster), lanes = (member group, dim); eight clusters per CTA, so
// batched fits with many small clusters do not pay one CTA launch each.
constexpr int kMeanWarpStage = 512;  // members staged per step of the row-order fallback

__global__ void __launch_bounds__(kMeanThreads) mean_exact_warp_kernel(
    const float* x, uint64_t ldx, uint32_t col_stride, uint64_t n, uint32_t d, uint64_t k,
    uint64_t nclusters, const uint64_t* offsets, const uint32_t* perm, float* table,
    int* has_empty, const int* active) {
    __shared__ float col_all[kMeanThreads / 32][kMeanWarpStage];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    float* col = col_all[wid];
    const uint64_t bc = uint64_t(blockIdx.x) * (kMeanThreads / 32) + wid;
    if (bc >= nclusters) return;
    const uint64_t b = bc / k, c = bc - b * k;
    if (active && !active[b]) return;
    const uint64_t* off = offsets + b * (k + 1);
    const uint64_t beg = off[c], end = off[c + 1];
    if (beg == end) {
        if (lane == 0) has_empty[b] = 1;
        return;
    }
    const uint64_t cnt = end - beg;
    const uint32_t* pb = perm ? perm + b * n : nullptr;  // null: x is the bucketed copy
    const float* xb = x + b * col_stride;
    const uint32_t G = 32 / d;  // member groups
    const uint32_t g = uint32_t(lane) / d, t = uint32_t(lane) - g * d;
    double s = 0.0;
    int emax = -1, emin = 1 << 30;
    if (g < G) {
        auto acc = [&](float v) {
            s = __dadd_rn(s, (double)v);
            const int e = int((__float_as_uint(v) >> 23) & 0xFFu);
            if (v != 0.f) {
                emax = max(emax, e);
                emin = min(emin, max(e, 1));
            }
        };
        uint64_t m = beg + g;
        for (; m + 3 * uint64_t(G) < end; m += 4 * uint64_t(G)) {
            uint32_t r[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) r[u] = pb ? __ldg(pb + m + u * G) : uint32_t(m + u * G);
            float v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = __ldg(xb + uint64_t(r[u]) * ldx + t);
#pragma unroll
            for (int u = 0; u < 4; ++u) acc(v[u]);
        }
        for (; m < end; m += G) acc(__ldg(xb + uint64_t(pb ? __ldg(pb + m) : uint32_t(m)) * ldx + t));
    }
    // combine the member groups of each dim (lanes t, t+d, t+2d, ...): exact
    // sums, so the combination order does not matter
    for (uint32_t h = 1; h < G; ++h) {
        const uint32_t src = h * d + t;
        const double os = __shfl_sync(0xffffffffu, s, src < 32 ? src : 0);
        const int oxa = __shfl_sync(0xffffffffu, emax, src < 32 ? src : 0);
        const int oxi = __shfl_sync(0xffffffffu, emin, src < 32 ? src : 0);
        if (g == 0) {
            s = __dadd_rn(s, os);
            emax = max(emax, oxa);
            emin = min(emin, oxi);
        }
    }
    int lg = 0;
    while ((uint64_t(1) << lg) < cnt) ++lg;
    const double inv = __ddiv_rn(1.0, (double)cnt);
    const bool mine = g == 0;
    const bool exact = emax < 0 || (emax < 255 && emax - emin + lg <= 28);
    if (mine && exact) table[bc * d + t] = __double2float_rn(__dmul_rn(s, inv));  // kmeans.cpp:112-118
    uint32_t todo = __ballot_sync(0xffffffffu, mine && !exact);
    while (todo) {  // row-order sums (kmeans.cpp:103-111) of the rejected dims
        const int src = __ffs(todo) - 1;
        todo &= todo - 1;
        const uint32_t tf = uint32_t(src);  // lane src has g == 0, so t == src
        double sf = 0.0;
        for (uint64_t m0 = beg; m0 < end; m0 += kMeanWarpStage) {
            const uint64_t m1 = m0 + kMeanWarpStage < end ? m0 + kMeanWarpStage : end;
            for (uint64_t m = m0 + lane; m < m1; m += 32)
                col[m - m0] = __ldg(xb + uint64_t(pb ? __ldg(pb + m) : uint32_t(m)) * ldx + tf);
            __syncwarp();
            if (lane == 0)
                for (uint64_t m = m0; m < m1; ++m) sf = __dadd_rn(sf, (double)col[m - m0]);
            __syncwarp();
        }
        if (lane == 0) table[bc * d + tf] = __double2float_rn(__dmul_rn(sf, inv));
    }
}

// Empty-cluster repair, proj/src/kmeans.cpp:122-130: for each empty cluster in
// ascending order take the row with the largest pre-update distance (first
// such row on ties), copy it, zero its distance.
__device__ void reseed_problem(const float* x, uint64_t ldx, uint32_t col_stride, uint64_t n,
                               uint32_t d, uint64_t k, const uint64_t* offsets, double* dist,
                               float* table, const uint64_t* nb);

// The next pass's centroid norms (cnorm non-null, r2e): norms_kernel's
// values -- ||c||^2 in fp64 in t order rounded to fp32, and the problem's max
// ||c|| rounded up -- computed by the problem's reseed block once its table
// is final, instead of a separate launch at the head of every pass.
__device__ void problem_norms(const float* table, uint32_t b, uint64_t k, uint32_t d, float* cnorm,
                              float* cmax);

// table_norms for small tables (r2e): a block per problem, no memset and no
// atomics (the PQ encode and fit heads; the wide kernel stays for coarse tables)
__global__ void __launch_bounds__(256) norms_block_kernel(const float* table, uint64_t k, uint32_t d, float* cnorm,
                                                          float* cmax) {
    problem_norms(table, blockIdx.x, k, d, cnorm, cmax);
}

__device__ void problem_norms(const float* table, uint32_t b, uint64_t k, uint32_t d, float* cnorm,
                              float* cmax) {
    __shared__ unsigned wmax[32];
    unsigned mx = 0u;
    for (uint64_t c = threadIdx.x; c < k; c += blockDim.x) {
        const float* cp = table + (uint64_t(b) * k + c) * d;
        double s = 0.0;
        for (uint32_t t0 = 0; t0 < d; t0 += 8) {
            float v[8];  // the row's loads issued together (clamped, unpredicated)
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = cp[min(t0 + u, d - 1)];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (t0 + u < d) s = __dadd_rn(s, __dmul_rn((double)v[u], (double)v[u]));
        }
        cnorm[uint64_t(b) * k + c] = __double2float_rn(s);
        mx = max(mx, __float_as_uint(__double2float_ru(sqrt(s))));
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (uint32_t w = 1; w < (blockDim.x >> 5); ++w) mx = max(mx, wmax[w]);
        cmax[b] = __uint_as_float(mx);
    }
}

__global__ void reseed_kernel(const float* x, uint64_t ldx, uint32_t col_stride, uint64_t n,
                              uint32_t d, uint64_t k, const uint64_t* offsets, double* dist,
                              float* table, const int* has_empty, const int* active,
                              const uint64_t* nb, float* cnorm, float* cmax) {
    const uint32_t b = blockIdx.x;
    if (active && !active[b]) return;
    if (has_empty[b]) reseed_problem(x, ldx, col_stride, n, d, k, offsets, dist, table, nb);
    if (cnorm) {
        __syncthreads();
        problem_norms(table, b, k, d, cnorm, cmax);
    }
}

__device__ void reseed_problem(const float* x, uint64_t ldx, uint32_t col_stride, uint64_t n,
                               uint32_t d, uint64_t k, const uint64_t* offsets, double* dist,
                               float* table, const uint64_t* nb) {
    const uint32_t b = blockIdx.x;
    const uint64_t nn = nb ? nb[b] : n;
    __shared__ double sv[32];
    __shared__ uint64_t si[32];
    const uint64_t* off = offsets + uint64_t(b) * (k + 1);
    double* db = dist + uint64_t(b) * n;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (uint64_t c = 0; c < k; ++c) {
        if (off[c] != off[c + 1]) continue;
        double bv = -1.0;
        uint64_t bi = ~uint64_t(0);
        for (uint64_t i = threadIdx.x; i < nn; i += blockDim.x) {
            const double v = db[i];
            if (bi == ~uint64_t(0) || v > bv) { bv = v; bi = i; }
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const uint64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (oi != ~uint64_t(0) && (bi == ~uint64_t(0) || ov > bv || (ov == bv && oi < bi))) {
                bv = ov;
                bi = oi;
            }
        }
        if (lane == 0) { sv[w] = bv; si[w] = bi; }
        __syncthreads();
        if (w == 0) {
            const int nw = blockDim.x >> 5;
            bv = lane < nw ? sv[lane] : -1.0;
            bi = lane < nw ? si[lane] : ~uint64_t(0);
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const uint64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (oi != ~uint64_t(0) && (bi == ~uint64_t(0) || ov > bv || (ov == bv && oi < bi))) {
                    bv = ov;
                    bi = oi;
                }
            }
            if (lane == 0) si[0] = bi;
        }
        __syncthreads();
        const uint64_t far = si[0];
        for (uint32_t t = threadIdx.x; t < d; t += blockDim.x)
            table[(uint64_t(b) * k + c) * d + t] = x[far * ldx + uint64_t(b) * col_stride + t];
        __syncthreads();
        if (threadIdx.x == 0) db[far] = 0.0;
        __syncthreads();
    }
}

// Rows i >= nb[b] of a shorter problem get key k: no cluster, skipped by the
// bucketing, the sums and the reseed.
__global__ void pad_keys_kernel(uint32_t* keys, uint64_t n, uint64_t k, const uint64_t* nb) {
    const uint32_t b = blockIdx.y;
    const uint64_t nn = nb[b];
    for (uint64_t i = nn + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        keys[uint64_t(b) * n + i] = uint32_t(k);
}

}  // namespace

void kmeans_pad_keys(pqg_ctx* ctx, uint32_t* keys, uint64_t n, uint32_t B, uint64_t k,
                     const uint64_t* nb, uint64_t max_pad) {
    if (max_pad == 0) return;
    launch(ctx, "pad_keys", pad_keys_kernel, dim3(unsigned((max_pad + 255) / 256), B), dim3(256), 0,
           keys, n, k, nb);
}

void exclusive_scan_u32(pqg_ctx* ctx, const uint32_t* in, uint64_t* out, uint64_t count) {
    exclusive_scan<uint32_t>(ctx, in, out, count);
}

static void bucket_impl(pqg_ctx* ctx, const uint32_t* keys, uint64_t n, uint32_t B, uint64_t k,
                        Bucketing out, const RowCopy* rows, const uint64_t* nb, SumInit zi = SumInit{}) {
    if (k > 16384) fail(PQG_EUNSUPPORTED, "bucketing supports at most 16384 lists/clusters");
    if (n == 0) {
        PQG_CUDA(cudaMemsetAsync(out.offsets, 0, sizeof(uint64_t) * B * (k + 1), ctx->stream));
        if (zi.count) {
            PQG_CUDA(cudaMemsetAsync(zi.csum, 0, sizeof(double) * zi.count, ctx->stream));
            PQG_CUDA(cudaMemsetAsync(zi.cmax, 0xff, sizeof(int) * zi.count, ctx->stream));
            std::vector<int> big(zi.count, 1 << 30);
            PQG_CUDA(cudaMemcpyAsync(zi.cmin, big.data(), sizeof(int) * zi.count, cudaMemcpyHostToDevice,
                                     ctx->stream));
            PQG_CUDA(cudaStreamSynchronize(ctx->stream));
        }
        return;
    }
    const BucketGeom g = bucket_geom(n, k);
    uint32_t* tile_counts = scratch<uint32_t>(ctx, uint64_t(B) * k * g.ntiles);
    uint64_t* tile_base = scratch<uint64_t>(ctx, uint64_t(B) * k * g.ntiles);
    const size_t hsmem = sizeof(uint32_t) * k;
    set_smem(hist_kernel, hsmem);
    launch(ctx, "bucket", hist_kernel, dim3(g.ntiles, B), dim3(256), hsmem, keys, n, k, g.ntiles, g.T,
           tile_counts, zi);
    exclusive_scan<uint32_t>(ctx, tile_counts, tile_base, uint64_t(B) * k * g.ntiles);
    const size_t ssmem = sizeof(uint32_t) * k * g.W;
    if (rows) {
        set_smem(scatter_kernel<true>, ssmem);
        launch(ctx, "bucket", scatter_kernel<true>, dim3(g.ntiles, B), dim3(32 * g.W), ssmem, keys, n, k,
               g.ntiles, g.T, (const uint64_t*)tile_base, (uint32_t*)nullptr, *rows, out.offsets, nb);
    } else {
        const char* me = std::getenv("PQG_BUCKET_MATCH");
        // keys 0..k (k = padding), so NB bits must cover k itself
        auto kern = scatter_kernel<false, 0>;
        if (!(me && me[0] == '1')) {
            if (k < 512) kern = scatter_kernel<false, 9>;
            else if (k < 2048) kern = scatter_kernel<false, 11>;
            else if (k < 8192) kern = scatter_kernel<false, 13>;
            else if (k < 32768) kern = scatter_kernel<false, 15>;
        }
        set_smem(kern, ssmem);
        launch(ctx, "bucket", kern, dim3(g.ntiles, B), dim3(32 * g.W), ssmem, keys, n, k,
               g.ntiles, g.T, (const uint64_t*)tile_base, out.perm, RowCopy{}, out.offsets, nb);
    }
}

void stable_bucket(pqg_ctx* ctx, const uint32_t* keys, uint64_t n, uint32_t B, uint64_t k,
                   const int* active, Bucketing out, const uint64_t* nb) {
    (void)active;
    bucket_impl(ctx, keys, n, B, k, out, nullptr, nb);
}

namespace {
// out[b][i][t] = x[i*ldx + b*col_stride + t]: reads each row once, coalesced
__global__ void transpose_blocks_kernel(const float* x, uint64_t n, uint64_t ldx, uint32_t B,
                                        uint32_t d, uint32_t col_stride, float* out) {
    const uint64_t per_row = uint64_t(B) * d, total = n * per_row;
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i = e / per_row, r = e - i * per_row;
        const uint64_t b = r / d, t = r - b * d;
        out[(b * n + i) * d + t] = __ldg(x + i * ldx + b * col_stride + t);
    }
}
}  // namespace

void transpose_blocks(pqg_ctx* ctx, const float* x, uint64_t n, uint64_t ldx, uint32_t B, uint32_t d,
                      uint32_t col_stride, float* out) {
    launch(ctx, "gather", transpose_blocks_kernel, dim3(grid1d(n * B * d, 256, ctx->num_sms * 32)),
           dim3(256), 0, x, n, ldx, B, d, col_stride, out);
}

void gather_rows(pqg_ctx* ctx, const float* x, uint64_t ldx, uint32_t B, uint32_t d,
                 uint32_t col_stride, const uint64_t* rows, uint64_t k, float* table) {
    launch(ctx, "gather", gather_kernel, dim3(grid1d(uint64_t(B) * k * d, 256, 8192)), dim3(256), 0,
           x, ldx, B, d, col_stride, rows, k, table);
}

void kmeans_inertia_and_stop(pqg_ctx* ctx, const double* dist, uint64_t n, uint32_t B,
                             uint32_t it, uint32_t max_iters, double tol, KMeansState st,
                             const uint64_t* nb) {
    uint64_t nparts, chunk;
    inertia_parts(n, nparts, chunk);
    double* parts = scratch<double>(ctx, uint64_t(B) * nparts);
    if (st.tickets) {
        launch(ctx, "inertia", partial_sum_stop_kernel, dim3(unsigned(nparts), B), dim3(kRedThreads), 0,
               dist, n, chunk, parts, nb, max_iters, tol, st);
        return;
    }
    launch(ctx, "inertia", partial_sum_kernel, dim3(unsigned(nparts), B), dim3(kRedThreads), 0,
           dist, n, chunk, parts, (const int*)st.active, nb);
    launch(ctx, "inertia", stop_kernel, dim3(B), dim3(kRedThreads), 0, (const double*)parts,
           uint32_t(nparts), it, max_iters, tol, st, nb);
}

void rows_sum_f64(pqg_ctx* ctx, const double* v, uint64_t n, uint32_t B, double* out) {
    uint64_t nparts, chunk;
    inertia_parts(n, nparts, chunk);
    double* parts = scratch<double>(ctx, uint64_t(B) * nparts);
    launch(ctx, "inertia", partial_sum_kernel, dim3(unsigned(nparts), B), dim3(kRedThreads), 0,
           v, n, chunk, parts, (const int*)nullptr, (const uint64_t*)nullptr);
    launch(ctx, "inertia", final_parts_kernel, dim3(B), dim3(kRedThreads), 0, (const double*)parts,
           uint32_t(nparts), out);
}

void table_norms_small(pqg_ctx* ctx, const float* table, uint32_t B, uint64_t k, uint32_t d, float* cnorm,
                       float* cmax) {
    launch(ctx, "norms", norms_block_kernel, dim3(B), dim3(256), 0, table, k, d, cnorm, cmax);
}

void kmeans_update(pqg_ctx* ctx, const RowSrc& src, uint64_t n, uint32_t B, uint32_t d,
                   float* table, uint64_t k, const uint32_t* assign, double* dist,
                   const int* active, const uint64_t* nb, float* cnorm, float* cmax) {
    if (uint64_t(B) * k > 0x7FFFFFFFull) fail(PQG_EUNSUPPORTED, "kmeans: too many clusters");
    // Default: the stable permutation, the sums gathering rows through it.
    // PQG_KM_COPY=1 buckets a copy of the rows instead (measured r1 at 100k x
    // 128, M=8: 6.8 ms per 25-pass fit with the copy vs 6.1 ms without --
    // the copy's scattered 64-byte writes cost more than the gather saves).
    const char* ce = std::getenv("PQG_KM_COPY");
    const bool copy = ce && ce[0] == '1' && uint64_t(n) * d <= 0xFFFFFFFFull;
    Bucketing bk{scratch<uint64_t>(ctx, uint64_t(B) * (k + 1)), nullptr};
    const uint64_t ncl = uint64_t(B) * k;
    const char* mean_env = std::getenv("PQG_KM_MEAN");
    const bool pieces = d % 4 == 0 && d <= 128 && !(mean_env && mean_env[0] != 'p') &&
                        (copy ? true
                              : ((src.ldx | src.col_stride) & 3u) == 0 &&
                                    (reinterpret_cast<uintptr_t>(src.x) & 15u) == 0);
    SumInit zi;
    if (pieces) {
        zi.csum = scratch<double>(ctx, ncl * d);
        zi.cmax = scratch<int>(ctx, ncl * d);
        zi.cmin = scratch<int>(ctx, ncl * d);
        zi.count = ncl * d;
    }
    const float* mx = src.x;
    uint64_t mldx = src.ldx;
    uint32_t mcs = src.col_stride;
    if (copy) {
        RowCopy rc;
        rc.x = src.x;
        rc.ldx = src.ldx;
        rc.col_stride = src.col_stride;
        rc.d = d;
        rc.out = scratch<float>(ctx, uint64_t(B) * n * d);
        rc.vec = (d % 4) == 0 && (src.ldx % 4) == 0 && (src.col_stride % 4) == 0 &&
                 (reinterpret_cast<uintptr_t>(src.x) & 15u) == 0;
        bucket_impl(ctx, assign, n, B, k, bk, &rc, nb, zi);
        mx = rc.out;
        mldx = d;
        mcs = uint32_t(n * d);
    } else {
        bk.perm = scratch<uint32_t>(ctx, uint64_t(B) * n);
        bucket_impl(ctx, assign, n, B, k, bk, nullptr, nb, zi);
    }
    int* has_empty = scratch<int>(ctx, B);
    if (pieces) {
        const PieceGeom pg = piece_geom(d, n, k);
        if (uint64_t(B) * pg.PP > 0xFFFFFFFFull) fail(PQG_EUNSUPPORTED, "kmeans: too many pieces");
        uint32_t* piece_start = scratch<uint32_t>(ctx, uint64_t(B) * k);
        PieceDesc* pieces_d = scratch<PieceDesc>(ctx, uint64_t(B) * pg.PP);
        PieceStat* stats = scratch<PieceStat>(ctx, uint64_t(B) * pg.PP * d);
        double* csum = zi.csum;
        int* cmax = zi.cmax;
        int* cmin = zi.cmin;
        unsigned long long* work_count = scratch<unsigned long long>(ctx, 1);
        uint64_t* work = scratch<uint64_t>(ctx, ncl * d);
        launch(ctx, "kmeans_sum", pieces_setup_kernel, dim3(B), dim3(1024), 0, (const uint64_t*)bk.offsets, k,
               pg.R, pg.PP, piece_start, pieces_d, has_empty, active, d, csum, cmax, cmin, work_count);
        MemberRows mr;
        mr.x = mx;
        mr.ldx = mldx;
        mr.col_stride = mcs;
        mr.perm = bk.perm;
        const uint64_t warps = uint64_t(B) * pg.PP;
        launch(ctx, "kmeans_sum", mean_pieces_kernel, dim3(unsigned((warps + 7) / 8)), dim3(kMeanThreads), 0, mr,
               n, d, k, B, (const PieceDesc*)pieces_d, stats, active, csum, cmax, cmin);
        launch(ctx, "kmeans_sum", mean_finalize_kernel, dim3(unsigned((ncl + 7) / 8)), dim3(kMeanThreads), 0,
               mr, n, d, k, B, (const uint64_t*)bk.offsets, (const uint32_t*)piece_start,
               (const PieceStat*)stats, table, active, (const double*)csum, (const int*)cmax, (const int*)cmin,
               work_count, work);
        launch(ctx, "kmeans_sum", mean_replay_kernel, dim3(ctx->num_sms * 4), dim3(kMeanThreads), 0, mr, n, d, k,
               (const uint64_t*)bk.offsets, (const uint32_t*)piece_start, (const PieceStat*)stats, table,
               (const unsigned long long*)work_count, (const uint64_t*)work);
    } else {
        PQG_CUDA(cudaMemsetAsync(has_empty, 0, sizeof(int) * B, ctx->stream));
        // small clusters (batched chunk fits): a warp each; large ones: a CTA each
        if (d <= 32 && n <= 128 * k) {
            const uint64_t blocks = (ncl + kMeanThreads / 32 - 1) / (kMeanThreads / 32);
            launch(ctx, "kmeans_sum", mean_exact_warp_kernel, dim3(unsigned(blocks)), dim3(kMeanThreads), 0,
                   mx, mldx, mcs, n, d, k, ncl, (const uint64_t*)bk.offsets, (const uint32_t*)bk.perm, table,
                   has_empty, active);
        } else {
            launch(ctx, "kmeans_sum", mean_exact_kernel, dim3(unsigned(ncl)), dim3(kMeanThreads), 0,
                   mx, mldx, mcs, n, d, k, (const uint64_t*)bk.offsets, (const uint32_t*)bk.perm, table,
                   has_empty, active);
        }
    }
    launch(ctx, "reseed", reseed_kernel, dim3(B), dim3(1024), 0, src.x, src.ldx, src.col_stride, n,
           d, k, (const uint64_t*)bk.offsets, dist, table, (const int*)has_empty, active, nb, cnorm, cmax);
}

// ---- one rank's side of a row-sharded fit (kmshard.cu, pqg_kmshard_*) -----
// The stable bucketing of the rank's rows by cluster and the exact piece sums
// with their exponent ranges (csum / cmax / cmin per (problem, cluster,
// dim)), exactly as kmeans_update computes them before its finalize.
bool kmeans_partials_supported(const RowSrc& src, uint32_t d) {
    return d % 4 == 0 && d <= 128 && ((src.ldx | src.col_stride) & 3u) == 0 &&
           (reinterpret_cast<uintptr_t>(src.x) & 15u) == 0 && !src.codes;
}

void kmeans_local_partials(pqg_ctx* ctx, const RowSrc& src, uint64_t n, uint32_t B, uint32_t d,
                           uint64_t k, const uint32_t* assign, const int* active, uint64_t* offsets,
                           uint32_t* perm, double* csum, int* cmax, int* cmin) {
    Bucketing bk{offsets, perm};
    SumInit zi;
    zi.csum = csum;
    zi.cmax = cmax;
    zi.cmin = cmin;
    zi.count = uint64_t(B) * k * d;
    bucket_impl(ctx, assign, n, B, k, bk, nullptr, nullptr, zi);
    const PieceGeom pg = piece_geom(d, n, k);
    if (uint64_t(B) * pg.PP > 0xFFFFFFFFull) fail(PQG_EUNSUPPORTED, "kmeans: too many pieces");
    uint32_t* piece_start = scratch<uint32_t>(ctx, uint64_t(B) * k);
    PieceDesc* pieces_d = scratch<PieceDesc>(ctx, uint64_t(B) * pg.PP);
    PieceStat* stats = scratch<PieceStat>(ctx, uint64_t(B) * pg.PP * d);
    unsigned long long* work_count = scratch<unsigned long long>(ctx, 1);
    int* has_empty = scratch<int>(ctx, B);
    launch(ctx, "kmeans_sum", pieces_setup_kernel, dim3(B), dim3(1024), 0, (const uint64_t*)offsets, k, pg.R,
           pg.PP, piece_start, pieces_d, has_empty, active, d, csum, cmax, cmin, work_count);
    MemberRows mr;
    mr.x = src.x;
    mr.ldx = src.ldx;
    mr.col_stride = src.col_stride;
    mr.perm = perm;
    const uint64_t warps = uint64_t(B) * pg.PP;
    launch(ctx, "kmeans_sum", mean_pieces_kernel, dim3(unsigned((warps + 7) / 8)), dim3(kMeanThreads), 0, mr, n,
           d, k, B, (const PieceDesc*)pieces_d, stats, active, csum, cmax, cmin);
}

// The stop rule (kmeans.cpp:93-100) on an already reduced per-problem inertia.
void kmeans_stop_global(pqg_ctx* ctx, const double* inertia, uint32_t B, uint32_t max_iters, double tol,
                        KMeansState st) {
    launch(ctx, "inertia", stop_kernel, dim3(B), dim3(kRedThreads), 0, inertia, 1u, 0u, max_iters, tol, st,
           (const uint64_t*)nullptr);
}

}  // namespace pqg
