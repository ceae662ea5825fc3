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

namespace pqg {

namespace {

constexpr int kTile = 2048;  // rows per bucketing tile (one warp walks a tile)

__global__ void hist_kernel(const uint32_t* keys, uint64_t n, uint64_t k, uint32_t ntiles,
                            uint32_t* tile_counts) {
    extern __shared__ uint32_t hist[];
    const uint32_t tile = blockIdx.x, b = blockIdx.y;
    for (uint64_t c = threadIdx.x; c < k; c += blockDim.x) hist[c] = 0;
    __syncthreads();
    const uint64_t r0 = uint64_t(tile) * kTile;
    const uint64_t r1 = min64(n, r0 + kTile);
    const uint32_t* kb = keys + uint64_t(b) * n;
    for (uint64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
        const uint32_t c = kb[i];
        if (c < k) atomicAdd(&hist[c], 1u);  // key k marks a padding row (no cluster)
    }
    __syncthreads();
    uint32_t* out = tile_counts + uint64_t(b) * k * ntiles;
    for (uint64_t c = threadIdx.x; c < k; c += blockDim.x) out[c * ntiles + tile] = hist[c];
}

__global__ void offsets_kernel(const uint64_t* tile_base, uint64_t n, uint32_t B, uint64_t k,
                               uint32_t ntiles, uint64_t* offsets, const uint64_t* nb) {
    const uint64_t total = uint64_t(B) * (k + 1);
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t b = e / (k + 1), c = e - b * (k + 1);
        // tile_base is one scan over all problems: problem b starts at its own
        // first entry (b*n only when every problem has n keys)
        offsets[e] = (c == k) ? (nb ? nb[b] : n)
                              : tile_base[(b * k + c) * ntiles] - tile_base[b * k * ntiles];
    }
}

// One warp per (tile, problem): walks its tile in row order 32 rows at a
// time; __match_any_sync ranks equal keys inside the 32, the per-warp running
// cursor keeps order across rounds, and tiles start at their scanned base.
__global__ void scatter_kernel(const uint32_t* keys, uint64_t n, uint64_t k, uint32_t ntiles,
                               const uint64_t* tile_base, uint32_t* perm, int warps_per_block) {
    extern __shared__ uint32_t running_all[];
    const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t tile = blockIdx.x * warps_per_block + wib;
    const uint32_t b = blockIdx.y;
    if (tile >= ntiles) return;
    uint32_t* running = running_all + uint64_t(wib) * k;
    const uint64_t* tb = tile_base + uint64_t(b) * k * ntiles;
    const uint64_t base_b = uint64_t(b) * n;
    const uint64_t first = tb[0];  // problem b's start in the all-problem scan
    for (uint64_t c = lane; c < k; c += 32) running[c] = uint32_t(tb[c * ntiles + tile] - first);
    __syncwarp();
    const uint64_t r0 = uint64_t(tile) * kTile;
    const uint64_t r1 = min64(n, r0 + kTile);
    const uint32_t* kb = keys + base_b;
    uint32_t* pb = perm + base_b;
    // keys of the tile prefetched 32 rounds at a time (one register per round)
    for (uint64_t c0 = r0; c0 < r1; c0 += 32 * 32) {
        uint32_t key[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) {
            const uint64_t i = c0 + uint64_t(q) * 32 + lane;
            key[q] = i < r1 ? __ldg(kb + i) : 0xFFFFFFFFu;
        }
#pragma unroll
        for (int q = 0; q < 32; ++q) {
            const uint64_t i = c0 + uint64_t(q) * 32 + lane;
            const uint32_t c = key[q];
            const bool valid = i < r1 && c < k;
            const uint32_t peers = __match_any_sync(0xffffffffu, c);
            const uint32_t rank = __popc(peers & lanemask_lt());
            uint32_t pos = 0;
            if (valid) pos = running[c] + rank;
            __syncwarp();
            if (valid && rank == 0) running[c] += __popc(peers);
            __syncwarp();
            if (valid) pb[pos] = uint32_t(i);
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

__global__ void stop_kernel(const double* parts, uint32_t nparts, uint32_t it, uint32_t max_iters,
                            double tol, KMeansState st, const uint64_t* nb) {
    const uint32_t b = blockIdx.x;
    if (!st.active[b]) return;
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
    if (st.per_iter) st.per_iter[uint64_t(b) * max_iters + (it - 1)] = s;
    st.iters[b] = it;
    const double prev = st.prev[b];
    const double floor1 = prev > 1.0 ? prev : 1.0;
    if ((it > 1 && prev - s < tol * floor1) || it == max_iters) {
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

__global__ void __launch_bounds__(kMeanThreads) mean_exact_kernel(
    const float* x, uint64_t ldx, uint32_t col_stride, uint64_t n, uint32_t d, uint64_t k,
    const uint64_t* offsets, const uint32_t* perm, float* table, int* has_empty, const int* active) {
    __shared__ double ps[kMeanThreads];
    __shared__ int pmax[kMeanThreads], pmin[kMeanThreads];
    __shared__ float col[kMeanStage];  // one dim of the members, row order (fallback)
    __shared__ uint32_t nfail;
    __shared__ uint32_t failed[kMeanThreads];
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
    const uint32_t* pb = perm + b * n;
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
                for (int u = 0; u < 4; ++u) r[u] = __ldg(pb + m + u * G);
                float v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = __ldg(xb + uint64_t(r[u]) * ldx + t);
#pragma unroll
                for (int u = 0; u < 4; ++u) acc(v[u]);
            }
            for (; m < end; m += G) acc(__ldg(xb + uint64_t(__ldg(pb + m)) * ldx + t));
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
            double sf = 0.0;
            for (uint64_t m0 = beg; m0 < end; m0 += mchunk) {
                const uint64_t m1 = m0 + mchunk < end ? m0 + mchunk : end;
                const uint32_t nm = uint32_t(m1 - m0);
                for (uint32_t e = threadIdx.x; e < nm * nf; e += blockDim.x) {
                    const uint32_t mi = e / nf, f = e - mi * nf;
                    col[e] = __ldg(xb + uint64_t(__ldg(pb + m0 + mi)) * ldx + failed[f]);
                }
                __syncthreads();
                if (threadIdx.x < nf)
                    for (uint32_t mi = 0; mi < nm; ++mi) sf = __dadd_rn(sf, (double)col[mi * nf + threadIdx.x]);
                __syncthreads();
            }
            if (threadIdx.x < nf) table[bc * d + failed[threadIdx.x]] = __double2float_rn(__dmul_rn(sf, inv));
        }
        __syncthreads();
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
    const uint32_t* pb = perm + b * n;
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
            for (int u = 0; u < 4; ++u) r[u] = __ldg(pb + m + u * G);
            float v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = __ldg(xb + uint64_t(r[u]) * ldx + t);
#pragma unroll
            for (int u = 0; u < 4; ++u) acc(v[u]);
        }
        for (; m < end; m += G) acc(__ldg(xb + uint64_t(__ldg(pb + m)) * ldx + t));
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
                col[m - m0] = __ldg(xb + uint64_t(__ldg(pb + m)) * ldx + tf);
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
__global__ void reseed_kernel(const float* x, uint64_t ldx, uint32_t col_stride, uint64_t n,
                              uint32_t d, uint64_t k, const uint64_t* offsets, double* dist,
                              float* table, const int* has_empty, const int* active,
                              const uint64_t* nb) {
    const uint32_t b = blockIdx.x;
    if ((active && !active[b]) || !has_empty[b]) return;
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

void stable_bucket(pqg_ctx* ctx, const uint32_t* keys, uint64_t n, uint32_t B, uint64_t k,
                   const int* active, Bucketing out, const uint64_t* nb) {
    (void)active;
    if (k > 16384) fail(PQG_EUNSUPPORTED, "bucketing supports at most 16384 lists/clusters");
    const uint32_t ntiles = uint32_t((n + kTile - 1) / kTile);
    uint32_t* tile_counts = scratch<uint32_t>(ctx, uint64_t(B) * k * ntiles);
    uint64_t* tile_base = scratch<uint64_t>(ctx, uint64_t(B) * k * ntiles);
    const size_t hsmem = sizeof(uint32_t) * k;
    set_smem(hist_kernel, hsmem);
    launch(ctx, "bucket", hist_kernel, dim3(ntiles, B), dim3(256), hsmem, keys, n, k, ntiles,
           tile_counts);
    exclusive_scan<uint32_t>(ctx, tile_counts, tile_base, uint64_t(B) * k * ntiles);
    launch(ctx, "bucket", offsets_kernel, dim3(grid1d(uint64_t(B) * (k + 1), 256, 4096)),
           dim3(256), 0, (const uint64_t*)tile_base, n, B, k, ntiles, out.offsets, nb);
    int wpb = int(std::max<uint64_t>(1, std::min<uint64_t>(8, (96 * 1024) / (4 * k))));
    const size_t ssmem = sizeof(uint32_t) * k * wpb;
    set_smem(scatter_kernel, ssmem);
    launch(ctx, "bucket", scatter_kernel, dim3((ntiles + wpb - 1) / wpb, B), dim3(32 * wpb), ssmem,
           keys, n, k, ntiles, (const uint64_t*)tile_base, out.perm, wpb);
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

void kmeans_update(pqg_ctx* ctx, const RowSrc& src, uint64_t n, uint32_t B, uint32_t d,
                   float* table, uint64_t k, const uint32_t* assign, double* dist,
                   const int* active, const uint64_t* nb) {
    Bucketing bk{scratch<uint64_t>(ctx, uint64_t(B) * (k + 1)), scratch<uint32_t>(ctx, uint64_t(B) * n)};
    stable_bucket(ctx, assign, n, B, k, active, bk, nb);
    int* has_empty = scratch<int>(ctx, B);
    PQG_CUDA(cudaMemsetAsync(has_empty, 0, sizeof(int) * B, ctx->stream));
    if (uint64_t(B) * k > 0x7FFFFFFFull) fail(PQG_EUNSUPPORTED, "kmeans: too many clusters");
    const uint64_t ncl = uint64_t(B) * k;
    // small clusters (batched chunk fits): a warp each; large ones: a CTA each
    if (d <= 32 && n <= 128 * k) {
        const uint64_t blocks = (ncl + kMeanThreads / 32 - 1) / (kMeanThreads / 32);
        launch(ctx, "kmeans_sum", mean_exact_warp_kernel, dim3(unsigned(blocks)), dim3(kMeanThreads), 0,
               src.x, src.ldx, src.col_stride, n, d, k, ncl, (const uint64_t*)bk.offsets,
               (const uint32_t*)bk.perm, table, has_empty, active);
    } else {
        launch(ctx, "kmeans_sum", mean_exact_kernel, dim3(unsigned(ncl)), dim3(kMeanThreads), 0,
               src.x, src.ldx, src.col_stride, n, d, k, (const uint64_t*)bk.offsets,
               (const uint32_t*)bk.perm, table, has_empty, active);
    }
    launch(ctx, "reseed", reseed_kernel, dim3(B), dim3(1024), 0, src.x, src.ldx, src.col_stride, n,
           d, k, (const uint64_t*)bk.offsets, dist, table, (const int*)has_empty, active, nb);
}

}  // namespace pqg
