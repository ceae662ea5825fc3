// pq.cu -- K4 decode + squared-error reduction and K7 ADC tables.
//
//  pq_decode / pq_decode_row   proj/src/pq.cpp:113-130
//  rmse numerator              proj/src/pq.cpp:169-177
//  reconstruction_rmse         proj/src/pq.cpp:179-181 (decode fused into the SSE)
//  adc_table                   proj/src/pq.cpp:132-151 (float(fp64 squared_l2))
//  adc_lookup                  proj/src/pq.cpp:153-167 (fp64 sum of float entries)
//
// The SSE is reduced in a fixed-shape fp64 tree (deterministic, independent of
// timing); the reference sums sequentially, so the two agree to ~1e-15
// relative, far inside the 1e-4 RMSE tolerance of BASELINE.json.
#include <algorithm>

#include "kernels.cuh"

namespace pqg {

namespace {

__device__ __forceinline__ uint32_t code_at(const uint8_t* codes, uint64_t i, uint32_t m,
                                            uint32_t M, uint32_t w) {
    const uint8_t* p = codes + (i * M + m) * w;
    return w == 1 ? uint32_t(p[0]) : (uint32_t(p[0]) | (uint32_t(p[1]) << 8));
}

// (row, column) of flat element e of a row-major n x D array; 32-bit division
// whenever the index fits (a 64-bit division costs ~5x more and dominated the
// element loops below).
__device__ __forceinline__ void split_elem(uint64_t e, uint64_t D, uint64_t& i, uint64_t& col) {
    if ((e | D) <= 0xFFFFFFFFull) {
        const uint32_t i32 = uint32_t(e) / uint32_t(D);
        i = i32;
        col = uint32_t(e) - i32 * uint32_t(D);
    } else {
        i = e / D;
        col = e - i * D;
    }
}

__global__ void decode_kernel(const uint8_t* codes, uint64_t n, uint32_t M, uint32_t ks,
                              uint32_t ds, const float* tables, float* out, int* err) {
    const uint32_t w = ks <= 256 ? 1 : 2;
    const uint64_t D = uint64_t(M) * ds, total = n * D;
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t i, col;
        split_elem(e, D, i, col);
        const uint32_t m = uint32_t(col) / ds, t = uint32_t(col) - m * ds;
        const uint32_t code = code_at(codes, i, m, M, w);
        if (code >= ks) {
            atomicExch(err, 1);
            out[e] = 0.f;
            continue;
        }
        out[e] = __ldg(tables + (uint64_t(m) * ks + code) * ds + t);
    }
}

constexpr int kThreads = 256;

__device__ double block_sum256(double v) {
    __shared__ double sh[kThreads];
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int s = kThreads / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) sh[threadIdx.x] = __dadd_rn(sh[threadIdx.x], sh[threadIdx.x + s]);
        __syncthreads();
    }
    const double r = sh[0];
    __syncthreads();
    return r;
}

// a - b squared, summed over [chunk*blk, chunk*(blk+1)) in a fixed tree.
__global__ void sse_kernel(const float* a, const float* b, uint64_t count, uint64_t chunk,
                           double* parts) {
    const uint64_t c0 = uint64_t(blockIdx.x) * chunk, c1 = min64(count, c0 + chunk);
    double s = 0.0;
    for (uint64_t e = c0 + threadIdx.x; e < c1; e += kThreads) {
        const double diff = __dsub_rn((double)a[e], (double)b[e]);
        s = __dadd_rn(s, __dmul_rn(diff, diff));
    }
    s = block_sum256(s);
    if (threadIdx.x == 0) parts[blockIdx.x] = s;
}

// Streamed rows bypass L1 (r2e): the codeword gathers are the kernel's L1
// working set (M x Ks x Ds fp32, 128 KB at D = 128, Ks = 256) and the rows,
// read once, would evict it.
__device__ __forceinline__ float4 ldg_stream(const float4* p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}

// Squared error of one (row, subspace) pair: ds elements of x against the
// codeword, accumulated in fp64 (vector loads when both are 16-byte aligned).
__device__ __forceinline__ double pair_sse(const float* xp, const float* cw, uint32_t ds, bool vec,
                                           double s) {
    if (vec) {
        for (uint32_t t = 0; t < ds; t += 4) {
            const float4 a = ldg_stream(reinterpret_cast<const float4*>(xp + t));
            const float4 c = __ldg(reinterpret_cast<const float4*>(cw + t));
            const double d0 = __dsub_rn((double)a.x, (double)c.x), d1 = __dsub_rn((double)a.y, (double)c.y);
            const double d2 = __dsub_rn((double)a.z, (double)c.z), d3 = __dsub_rn((double)a.w, (double)c.w);
            s = __dadd_rn(s, __dmul_rn(d0, d0));
            s = __dadd_rn(s, __dmul_rn(d1, d1));
            s = __dadd_rn(s, __dmul_rn(d2, d2));
            s = __dadd_rn(s, __dmul_rn(d3, d3));
        }
    } else {
        for (uint32_t t = 0; t < ds; ++t) {
            const double diff = __dsub_rn((double)__ldg(xp + t), (double)__ldg(cw + t));
            s = __dadd_rn(s, __dmul_rn(diff, diff));
        }
    }
    return s;
}

// x vs decode(codes) without materialising the decode: one (row, subspace)
// pair per thread step, one code load per pair; block b sums the pairs
// [b*chunk, (b+1)*chunk) in a fixed order (deterministic).
__global__ void recon_sse_kernel(const float* x, const uint8_t* codes, uint64_t n, uint32_t M,
                                 uint32_t ks, uint32_t ds, const float* tables, uint64_t chunk,
                                 double* parts, int* err, bool vec) {
    const uint32_t w = ks <= 256 ? 1 : 2;
    const uint64_t D = uint64_t(M) * ds, total = n * M;
    const uint64_t c0 = uint64_t(blockIdx.x) * chunk, c1 = min64(total, c0 + chunk);
    double s = 0.0;
    for (uint64_t p = c0 + threadIdx.x; p < c1; p += kThreads) {
        uint64_t i, m;
        split_elem(p, M, i, m);
        uint32_t code = code_at(codes, i, uint32_t(m), M, w);
        if (code >= ks) {
            atomicExch(err, 1);
            code = 0;
        }
        s = pair_sse(x + i * D + m * ds, tables + (m * ks + code) * ds, ds, vec, s);
    }
    s = block_sum256(s);
    if (threadIdx.x == 0) parts[blockIdx.x] = s;
}

// The same sum for Ds in {4, 8, 16, 32} with aligned rows (r2), software-
// pipelined: the code of the thread's NEXT pair is loaded one step ahead, so
// the dependent codeword gather (L2) no longer waits behind the code's HBM
// latency (ncu r2: the one-pair loop stalled on long scoreboard, 0.57 of
// HBM).  Every addition happens in recon_sse_kernel's order, so the two are
// bit-identical (the chunked pipeline's local RMSE, chunk_sse_kernel, relies
// on that order too).
template <int DS>
__global__ void __launch_bounds__(kThreads, DS <= 4 ? 8 : 4) recon_sse_vec_kernel(const float* x, const uint8_t* codes, uint64_t n,
                                                                    uint32_t M, uint32_t ks, const float* tables,
                                                                    uint64_t chunk, double* parts, int* err) {
    const uint64_t D = uint64_t(M) * DS, total = n * M;
    const uint64_t c0 = uint64_t(blockIdx.x) * chunk, c1 = min64(total, c0 + chunk);
    double s = 0.0;
    auto code_of = [&](uint64_t p) -> uint32_t {
        if (p >= c1) return 0u;
        uint32_t c = ks <= 256 ? uint32_t(__ldg(codes + p)) : uint32_t(__ldg(reinterpret_cast<const uint16_t*>(codes) + p));
        if (c >= ks) {
            atomicExch(err, 1);
            c = 0;
        }
        return c;
    };
    uint64_t p = c0 + threadIdx.x;
    uint32_t code = code_of(p);
    for (; p < c1; p += kThreads) {
        uint64_t i, m;
        split_elem(p, M, i, m);
        const float4* xp = reinterpret_cast<const float4*>(x + i * D + m * DS);
        const float4* cp = reinterpret_cast<const float4*>(tables + (m * ks + code) * DS);
        float4 xv[DS / 4], cv[DS / 4];
#pragma unroll
        for (int q = 0; q < DS / 4; ++q) {
            xv[q] = ldg_stream(xp + q);
            cv[q] = __ldg(cp + q);
        }
        code = code_of(p + kThreads);  // next step's code, in flight during this one
#pragma unroll
        for (int q = 0; q < DS / 4; ++q) {
            const float4 a = xv[q], c = cv[q];
            const double d0 = __dsub_rn((double)a.x, (double)c.x), d1 = __dsub_rn((double)a.y, (double)c.y);
            const double d2 = __dsub_rn((double)a.z, (double)c.z), d3 = __dsub_rn((double)a.w, (double)c.w);
            s = __dadd_rn(s, __dmul_rn(d0, d0));
            s = __dadd_rn(s, __dmul_rn(d1, d1));
            s = __dadd_rn(s, __dmul_rn(d2, d2));
            s = __dadd_rn(s, __dmul_rn(d3, d3));
        }
    }
    s = block_sum256(s);
    if (threadIdx.x == 0) parts[blockIdx.x] = s;
}

__global__ void final_sum_kernel(const double* parts, uint64_t count, double* out) {
    double s = 0.0;
    for (uint64_t i = threadIdx.x; i < count; i += kThreads) s = __dadd_rn(s, parts[i]);
    s = block_sum256(s);
    if (threadIdx.x == 0) *out = s;
}

// Batched LUT build (r2) for the search: entries[q][m][j] =
// float(sum_t (double(q_t) - double(c_jt))^2) in t order, exactly adc_table
// (proj/src/pq.cpp:132-151).  Block = (subspace m, block of 32 queries),
// thread = codeword j: the codeword is converted to fp64 ONCE and kept in
// registers, the 32 queries' sub-vectors sit in shared memory as fp64, so an
// entry costs Ds x (dsub, dmul, dadd) + one conversion back; the search
// kernel then loads its query's table instead of building it (the in-kernel
// build was 16.5% of the scan's instructions, r1h).
constexpr uint32_t kLutQB = 32;
template <int DS>
__global__ void __launch_bounds__(256) adc_luts_kernel(const float* tables, uint32_t M, uint32_t ks,
                                                       const float* queries, uint64_t nq, float* entries) {
    __shared__ double qs[kLutQB][DS];
    const uint32_t m = blockIdx.y;
    const uint64_t q0 = uint64_t(blockIdx.x) * kLutQB;
    const uint64_t D = uint64_t(M) * DS;
    for (uint32_t e = threadIdx.x; e < kLutQB * DS; e += blockDim.x) {
        const uint32_t qi = e / DS, t = e - qi * DS;
        qs[qi][t] = q0 + qi < nq ? (double)__ldg(queries + (q0 + qi) * D + uint64_t(m) * DS + t) : 0.0;
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < ks; j += blockDim.x) {
        double c[DS];
#pragma unroll
        for (int t = 0; t < DS; ++t) c[t] = (double)__ldg(tables + (uint64_t(m) * ks + j) * DS + t);
        const uint32_t nqb = uint32_t(min64(uint64_t(kLutQB), nq - q0));
        // four queries per step: four independent fp64 chains in flight
        for (uint32_t qb = 0; qb < kLutQB; qb += 4) {
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int t = 0; t < DS; ++t) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const double diff = __dsub_rn(qs[qb + u][t], c[t]);
                    acc[u] = __dadd_rn(acc[u], __dmul_rn(diff, diff));
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (qb + u < nqb) entries[((q0 + qb + u) * M + m) * ks + j] = __double2float_rn(acc[u]);
        }
    }
}

__global__ void adc_tables_kernel(const float* tables, uint32_t M, uint32_t ks, uint32_t ds,
                                  const float* queries, uint64_t nq, float* entries) {
    const uint64_t D = uint64_t(M) * ds, per_q = uint64_t(M) * ks, total = nq * per_q;
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t q = e / per_q, mj = e - q * per_q;
        const uint32_t m = uint32_t(mj / ks);
        entries[e] = __double2float_rn(
            exact_sq_l2(queries + q * D + uint64_t(m) * ds, tables + mj * ds, int(ds)));
    }
}

__global__ void adc_lookup_kernel(const float* entries, uint32_t M, uint32_t ks,
                                  const uint8_t* codes, uint64_t n, double* out, int* err) {
    const uint32_t w = ks <= 256 ? 1 : 2;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        double acc = 0.0;
        for (uint32_t m = 0; m < M; ++m) {
            const uint32_t code = code_at(codes, i, m, M, w);
            if (code >= ks) {
                atomicExch(err, 1);
                break;
            }
            acc = __dadd_rn(acc, (double)__ldg(entries + uint64_t(m) * ks + code));
        }
        out[i] = acc;
    }
}

__host__ __device__ inline uint64_t nparts_for(uint64_t count) {
    const uint64_t p = (count + 65535) / 65536;
    return p < 1 ? 1 : (p > 4096 ? 4096 : p);
}

// ---- the paper's chunked pipeline (proj/src/pipeline.cpp) -----------------
// Chunk c of chunk_rows(n, C) (proj/src/dataset_io.cpp:322-339) starts at
// c*base + min(c, extra) and holds base + (c < extra) rows.
__device__ __forceinline__ void chunk_range(uint64_t c, uint64_t base, uint64_t extra,
                                            uint64_t& r0, uint64_t& nc) {
    r0 = c * base + (c < extra ? c : extra);
    nc = base + (c < extra ? 1 : 0);
}

// Y[i][c*D + j] = x[r0_c + i][j]: the C chunks side by side, so the C*M
// local PQ fits become C*M column-block problems over n_max shared rows.
// Rows past a chunk's end repeat its last row (finite; their keys are
// padded out of every update).
__global__ void interleave_chunks_kernel(const float* x, uint64_t D, uint64_t C, uint64_t base,
                                         uint64_t extra, uint64_t n_max, float* y) {
    const uint64_t W = C * D, total = n_max * W;
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i = e / W, cj = e - i * W;
        const uint64_t c = cj / D, j = cj - c * D;
        uint64_t r0, nc;
        chunk_range(c, base, extra, r0, nc);
        y[e] = __ldg(x + (r0 + (i < nc ? i : nc - 1)) * D + j);
    }
}

// Representative j of chunk c = local codeword j of every subspace,
// concatenated (pipeline.cpp:95-103): reps[c*ks + j][m*ds + t].
__global__ void representatives_kernel(const float* tables, uint64_t C, uint32_t M, uint32_t ks,
                                       uint32_t ds, float* reps) {
    const uint64_t D = uint64_t(M) * ds, total = C * ks * D;
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t cj = e / D, col = e - cj * D;
        const uint64_t c = cj / ks, j = cj - c * ks;
        const uint64_t m = col / ds, t = col - m * ds;
        reps[e] = __ldg(tables + (((c * M + m) * ks) + j) * ds + t);
    }
}

// Per-chunk reconstruction SSE of the chunk against its own local codebook,
// codes taken from the fit's final assignments (the last pass has no update
// after it, kmeans.cpp:93-101, so they are the chunk's encode).  Same pair
// order and reduction shape as recon_sse_kernel on that chunk alone.
__global__ void chunk_sse_kernel(const float* x, uint32_t M, uint32_t ks, uint32_t ds,
                                 uint64_t base, uint64_t extra, const uint32_t* assign,
                                 uint64_t n_max, const float* tables, double* parts, bool vec) {
    const uint64_t c = blockIdx.y;
    const uint64_t D = uint64_t(M) * ds;
    uint64_t r0, nc;
    chunk_range(c, base, extra, r0, nc);
    const uint64_t total = nc * M, np = nparts_for(nc * D);
    if (blockIdx.x >= np) return;
    const uint64_t chunk = (total + np - 1) / np;
    const uint64_t c0 = uint64_t(blockIdx.x) * chunk, c1 = min64(total, c0 + chunk);
    const float* xc = x + r0 * D;
    double s = 0.0;
    for (uint64_t p = c0 + threadIdx.x; p < c1; p += kThreads) {
        uint64_t i, m;
        split_elem(p, M, i, m);
        const uint64_t b = c * M + m;
        const uint32_t code = __ldg(assign + b * n_max + i);
        s = pair_sse(xc + i * D + m * ds, tables + (b * ks + code) * ds, ds, vec, s);
    }
    s = block_sum256(s);
    if (threadIdx.x == 0) parts[c * gridDim.x + blockIdx.x] = s;
}

__global__ void chunk_sse_final_kernel(const double* parts, uint64_t stride, uint32_t M,
                                       uint32_t ds, uint64_t base, uint64_t extra, double* sse) {
    const uint64_t c = blockIdx.x;
    uint64_t r0, nc;
    chunk_range(c, base, extra, r0, nc);
    const uint64_t np = nparts_for(nc * M * ds);
    double s = 0.0;
    for (uint64_t i = threadIdx.x; i < np; i += kThreads) s = __dadd_rn(s, parts[c * stride + i]);
    s = block_sum256(s);
    if (threadIdx.x == 0) sse[c] = s;
}

}  // namespace

void interleave_chunks(pqg_ctx* ctx, const float* x, uint64_t D, uint64_t C, uint64_t base,
                       uint64_t extra, uint64_t n_max, float* y) {
    launch(ctx, "pipeline", interleave_chunks_kernel, dim3(grid1d(n_max * C * D, 256, ctx->num_sms * 32)),
           dim3(256), 0, x, D, C, base, extra, n_max, y);
}

void chunk_representatives(pqg_ctx* ctx, const float* tables, uint64_t C, uint32_t M, uint32_t ks,
                           uint32_t ds, float* reps) {
    launch(ctx, "pipeline", representatives_kernel,
           dim3(grid1d(C * ks * uint64_t(M) * ds, 256, ctx->num_sms * 32)), dim3(256), 0, tables, C, M,
           ks, ds, reps);
}

void chunk_sse(pqg_ctx* ctx, const float* x, uint64_t C, uint32_t M, uint32_t ks, uint32_t ds,
               uint64_t base, uint64_t extra, const uint32_t* assign, uint64_t n_max,
               const float* tables, double* sse) {
    const uint64_t np_max = nparts_for(n_max * M * ds);
    double* parts = scratch<double>(ctx, C * np_max);
    const bool vec = ds % 4 == 0 && ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(tables)) & 15u) == 0;
    launch(ctx, "recon_sse", chunk_sse_kernel, dim3(unsigned(np_max), unsigned(C)), dim3(kThreads), 0,
           x, M, ks, ds, base, extra, assign, n_max, tables, parts, vec);
    launch(ctx, "reduce", chunk_sse_final_kernel, dim3(unsigned(C)), dim3(kThreads), 0,
           (const double*)parts, np_max, M, ds, base, extra, sse);
}

void reduce_sum_f64(pqg_ctx* ctx, const double* parts, uint64_t count, double* out) {
    launch(ctx, "reduce", final_sum_kernel, dim3(1), dim3(kThreads), 0, parts, count, out);
}

void pq_decode_dev(pqg_ctx* ctx, const uint8_t* codes, uint64_t n, uint32_t M, uint32_t ks,
                   uint32_t ds, const float* tables, float* out, int* err) {
    launch(ctx, "decode", decode_kernel, dim3(grid1d(n * M * ds, 256, ctx->num_sms * 32)),
           dim3(256), 0, codes, n, M, ks, ds, tables, out, err);
}

void sq_error_dev(pqg_ctx* ctx, const float* a, const float* b, uint64_t count, double* sse) {
    const uint64_t np = nparts_for(count);
    const uint64_t chunk = (count + np - 1) / np;
    double* parts = scratch<double>(ctx, np);
    launch(ctx, "sse", sse_kernel, dim3(unsigned(np)), dim3(kThreads), 0, a, b, count, chunk, parts);
    reduce_sum_f64(ctx, parts, np, sse);
}

void recon_sse_dev(pqg_ctx* ctx, const float* x, const uint8_t* codes, uint64_t n, uint32_t M,
                   uint32_t ks, uint32_t ds, const float* tables, double* sse, int* err) {
    const uint64_t np = nparts_for(n * M * ds);
    const uint64_t chunk = (n * M + np - 1) / np;  // (row, subspace) pairs per part
    double* parts = scratch<double>(ctx, np);
    const bool vec = ds % 4 == 0 && ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(tables)) & 15u) == 0;
    auto go = [&](auto kern) {
        launch(ctx, "recon_sse", kern, dim3(unsigned(np)), dim3(kThreads), 0, x, codes, n, M, ks, tables, chunk,
               parts, err);
    };
    // measured r2 (tools/sse_bench.py, 4M rows): the pipelined kernel wins at
    // Ds <= 8 (D=128 M=16 0.57 -> 0.53 ms), the generic one at Ds = 16
    if (vec && ds == 4) go(recon_sse_vec_kernel<4>);
    else if (vec && ds == 8) go(recon_sse_vec_kernel<8>);
    else
        launch(ctx, "recon_sse", recon_sse_kernel, dim3(unsigned(np)), dim3(kThreads), 0, x, codes, n, M,
               ks, ds, tables, chunk, parts, err, vec);
    reduce_sum_f64(ctx, parts, np, sse);
}

void adc_tables_dev(pqg_ctx* ctx, const float* tables, uint32_t M, uint32_t ks, uint32_t ds,
                    const float* queries, uint64_t nq, float* entries) {
    launch(ctx, "adc_tables", adc_tables_kernel, dim3(grid1d(nq * M * ks, 256, 1u << 20)), dim3(256), 0,
           tables, M, ks, ds, queries, nq, entries);
}

bool adc_luts_dev(pqg_ctx* ctx, const float* tables, uint32_t M, uint32_t ks, uint32_t ds,
                  const float* queries, uint64_t nq, float* entries) {
    if (!(ds == 4 || ds == 8 || ds == 16 || ds == 32) || nq == 0 || M > 65535) return false;
    const dim3 grid(unsigned((nq + kLutQB - 1) / kLutQB), M);
    const unsigned th = std::min<unsigned>(256, (ks + 31) / 32 * 32);
    if (ds == 4) launch(ctx, "adc_luts", adc_luts_kernel<4>, grid, dim3(th), 0, tables, M, ks, queries, nq, entries);
    else if (ds == 8) launch(ctx, "adc_luts", adc_luts_kernel<8>, grid, dim3(th), 0, tables, M, ks, queries, nq, entries);
    else if (ds == 16) launch(ctx, "adc_luts", adc_luts_kernel<16>, grid, dim3(th), 0, tables, M, ks, queries, nq, entries);
    else launch(ctx, "adc_luts", adc_luts_kernel<32>, grid, dim3(th), 0, tables, M, ks, queries, nq, entries);
    return true;
}

void adc_lookup_dev(pqg_ctx* ctx, const float* entries, uint32_t M, uint32_t ks,
                    const uint8_t* codes, uint64_t n, double* out, int* err) {
    launch(ctx, "adc_lookup", adc_lookup_kernel, dim3(grid1d(n, 256, 1u << 20)), dim3(256), 0, entries,
           M, ks, codes, n, out, err);
}

}  // namespace pqg
