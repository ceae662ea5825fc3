// formats.cu -- device side of the on-disk formats:
// the PQII posting-list section (proj/src/ivf.cpp:264-355) converted between
// its interleaved file layout and the device CSR, plus the validation scans
// of load_codes / load_codebook / load_index (code range, finite codewords).
//
// PQII list section: for every list l in order, u64 len_l then len_l entries
// of (u64 id, row_bytes code bytes), little endian (ivf.cpp:283-291).  With
// CSR offsets off[] the position of list l's header is 8 l + off[l] (8 + rb)
// and entry i of the CSR (list l) starts at 8 (l + 1) + i (8 + rb): both are
// closed forms, so packing and unpacking are embarrassingly parallel byte
// moves (HBM-bound; one thread per entry, byte-granular because entries of
// 8 + rb bytes are not word aligned in general).
#include "kernels.cuh"

namespace pqg {

namespace {

__device__ __forceinline__ uint64_t list_of(const uint64_t* off, uint64_t nl, uint64_t i) {
    // last l with off[l] <= i and off[l + 1] > i (empty lists share offsets)
    uint64_t lo = 0, hi = nl;
    while (hi - lo > 1) {
        const uint64_t mid = (lo + hi) >> 1;
        if (off[mid] <= i) lo = mid; else hi = mid;
    }
    while (lo + 1 < nl && off[lo + 1] <= i) ++lo;
    return lo;
}

__device__ __forceinline__ void put_u64(uint8_t* p, uint64_t v) {
#pragma unroll
    for (int b = 0; b < 8; ++b) p[b] = uint8_t(v >> (8 * b));
}

__device__ __forceinline__ uint64_t get_u64(const uint8_t* p) {
    uint64_t v = 0;
#pragma unroll
    for (int b = 7; b >= 0; --b) v = (v << 8) | p[b];
    return v;
}

__global__ void pqii_pack_kernel(const uint64_t* off, const uint64_t* ids, const uint8_t* codes, uint64_t nl,
                                 uint64_t n, uint64_t rb, uint8_t* out) {
    const uint64_t es = 8 + rb;
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n + nl;
         e += uint64_t(gridDim.x) * blockDim.x) {
        if (e >= n) {  // list header
            const uint64_t l = e - n;
            put_u64(out + 8 * l + off[l] * es, off[l + 1] - off[l]);
            continue;
        }
        const uint64_t l = list_of(off, nl, e);
        uint8_t* p = out + 8 * (l + 1) + e * es;
        put_u64(p, ids[e]);
        const uint8_t* c = codes + e * rb;
        for (uint64_t j = 0; j < rb; ++j) p[8 + j] = c[j];
    }
}

// src_off[l]: byte offset (within the section) of list l's first entry;
// off[]: CSR offsets of the parsed lists (nl of them), n entries in all
__global__ void pqii_unpack_kernel(const uint8_t* sec, const uint64_t* src_off, const uint64_t* off, uint64_t nl,
                                   uint64_t n, uint64_t rb, uint64_t* ids, uint8_t* codes) {
    const uint64_t es = 8 + rb;
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
         e += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t l = list_of(off, nl, e);
        const uint8_t* p = sec + src_off[l] + (e - off[l]) * es;
        ids[e] = get_u64(p);
        uint8_t* c = codes + e * rb;
        for (uint64_t j = 0; j < rb; ++j) c[j] = p[8 + j];
    }
}

// first row (lowest index) holding a code >= ks
__global__ void first_bad_code_kernel(const uint8_t* codes, uint64_t n, uint32_t M, uint32_t ks, uint32_t w,
                                      unsigned long long* first) {
    const uint64_t total = n * M;
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += uint64_t(gridDim.x) * blockDim.x) {
        const uint8_t* p = codes + e * w;
        const uint32_t c = w == 1 ? p[0] : (uint32_t(p[0]) | (uint32_t(p[1]) << 8));
        if (c >= ks) atomicMin(first, (unsigned long long)(e / M));
    }
}

__global__ void first_nonfinite_kernel(const float* v, uint64_t count, unsigned long long* first) {
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < count;
         e += uint64_t(gridDim.x) * blockDim.x)
        if (!isfinite(v[e])) atomicMin(first, (unsigned long long)e);
}

}  // namespace

void pqii_pack(pqg_ctx* ctx, const uint64_t* off, const uint64_t* ids, const uint8_t* codes, uint64_t nlist,
               uint64_t n, uint64_t rb, uint8_t* out) {
    launch(ctx, "pqii_pack", pqii_pack_kernel, dim3(grid1d(n + nlist, 256, ctx->num_sms * 16)), dim3(256), 0,
           off, ids, codes, nlist, n, rb, out);
}

void pqii_unpack(pqg_ctx* ctx, const uint8_t* sec, const uint64_t* src_off, const uint64_t* off, uint64_t nl,
                 uint64_t n, uint64_t rb, uint64_t* ids, uint8_t* codes) {
    if (n == 0) return;
    launch(ctx, "pqii_unpack", pqii_unpack_kernel, dim3(grid1d(n, 256, ctx->num_sms * 16)), dim3(256), 0, sec,
           src_off, off, nl, n, rb, ids, codes);
}

void first_bad_code(pqg_ctx* ctx, const uint8_t* codes, uint64_t n, uint32_t M, uint32_t ks, uint32_t w,
                    unsigned long long* first) {
    PQG_CUDA(cudaMemsetAsync(first, 0xFF, sizeof(unsigned long long), ctx->stream));
    if (n == 0 || M == 0) return;
    launch(ctx, "codes_check", first_bad_code_kernel, dim3(grid1d(n * M, 256, ctx->num_sms * 16)), dim3(256), 0,
           codes, n, M, ks, w, first);
}

void first_nonfinite(pqg_ctx* ctx, const float* v, uint64_t count, unsigned long long* first) {
    PQG_CUDA(cudaMemsetAsync(first, 0xFF, sizeof(unsigned long long), ctx->stream));
    if (count == 0) return;
    launch(ctx, "finite_check", first_nonfinite_kernel, dim3(grid1d(count, 256, ctx->num_sms * 16)), dim3(256), 0,
           v, count, first);
}

}  // namespace pqg
