// common.cuh -- shared device helpers, the context object, the scratch arena
// and the launch wrapper of libpqg (B200 / sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/pqg.h"

namespace pqg {

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
struct Error {
    int code;
    std::string msg;
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error{code, msg}; }

inline void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(PQG_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define PQG_CUDA(x) ::pqg::check_cuda((x), #x)

// ---------------------------------------------------------------------------
// exact reference arithmetic (proj/src/kmeans.cpp:11-18): fp64, left to right,
// separate multiply and add (no FMA contraction), as the x86-64 reference.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double exact_sq_l2(const float* a, const float* b, int d) {
    double acc = 0.0;
    for (int t = 0; t < d; ++t) {
        const double diff = __dsub_rn((double)a[t], (double)b[t]);
        acc = __dadd_rn(acc, __dmul_rn(diff, diff));
    }
    return acc;
}

constexpr float kU = 5.9604644775390625e-08f;  // fp32 unit roundoff 2^-24

__host__ __device__ __forceinline__ uint64_t min64(uint64_t a, uint64_t b) { return a < b ? a : b; }

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ---------------------------------------------------------------------------
// scratch arena: stream-ordered bump allocator reused across calls
// ---------------------------------------------------------------------------
struct Arena {
    std::vector<std::pair<char*, size_t>> blocks;  // (base, capacity)
    size_t cur_block = 0, cur_off = 0;
    int depth = 0;
    size_t peak_total = 0, used_total = 0;

    void* alloc(size_t bytes) {
        bytes = (bytes + 255) & ~size_t(255);
        if (bytes == 0) bytes = 256;
        while (cur_block < blocks.size()) {
            if (cur_off + bytes <= blocks[cur_block].second) {
                void* p = blocks[cur_block].first + cur_off;
                cur_off += bytes;
                used_total += bytes;
                if (used_total > peak_total) peak_total = used_total;
                return p;
            }
            ++cur_block;
            cur_off = 0;
        }
        size_t cap = bytes;
        size_t have = 0;
        for (auto& b : blocks) have += b.second;
        if (cap < have) cap = have;
        if (cap < (size_t(64) << 20)) cap = size_t(64) << 20;
        char* p = nullptr;
        cudaError_t e = cudaMalloc(&p, cap);
        if (e != cudaSuccess) {
            cudaGetLastError();
            fail(PQG_ENOMEM, "device scratch allocation of " + std::to_string(cap) + " bytes failed");
        }
        blocks.push_back({p, cap});
        cur_block = blocks.size() - 1;
        cur_off = bytes;
        used_total += bytes;
        if (used_total > peak_total) peak_total = used_total;
        return p;
    }
    // Stream-ordered reuse inside one call: everything allocated after mark()
    // is handed out again after reset_to(mark) (later kernels on the same
    // stream run after the earlier ones finished with it).
    std::pair<size_t, size_t> mark() const { return {cur_block, cur_off}; }
    void reset_to(std::pair<size_t, size_t> m) {
        cur_block = m.first;
        cur_off = m.second;
    }
    // Called when the outermost scope closes: rewind; consolidate fragments.
    void rewind() {
        cur_block = 0;
        cur_off = 0;
        used_total = 0;
        if (blocks.size() > 1) {
            cudaDeviceSynchronize();
            size_t total = 0;
            for (auto& b : blocks) {
                total += b.second;
                cudaFree(b.first);
            }
            blocks.clear();
            char* p = nullptr;
            if (cudaMalloc(&p, total) == cudaSuccess) blocks.push_back({p, total});
            else cudaGetLastError();
        }
    }
    void release() {
        for (auto& b : blocks) cudaFree(b.first);
        blocks.clear();
        cur_block = cur_off = 0;
    }
};

struct ProfRec {
    int cls;
    cudaEvent_t a, b;
};

}  // namespace pqg

struct pqg_ctx {
    int device = 0;
    int num_sms = 148;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    uint64_t launches = 0;
    pqg::Arena arena;
    // profiling
    bool profiling = false;
    std::vector<std::string> prof_names;
    std::vector<pqg::ProfRec> prof_recs;
    std::vector<cudaEvent_t> event_pool;
    // device flag word for kernel-side error reports (range errors)
    int* d_err = nullptr;
    // copy stream + events for host-input pipelines (created on first use)
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t pipe_ev[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t handoff_ev = nullptr;  // pqg_ctx_set_stream: new stream waits for the old
    bool err_pending = false;          // d_err not yet read (device-output searches)
    pqg_ctx* shard_ws = nullptr;       // cached workspace context of pqg_kmshard handles
};

namespace pqg {

// RAII: rewinds the arena when the outermost API call returns.
struct Scope {
    pqg_ctx* ctx;
    explicit Scope(pqg_ctx* c) : ctx(c) {
        PQG_CUDA(cudaSetDevice(c->device));
        ++ctx->arena.depth;
    }
    ~Scope() {
        if (--ctx->arena.depth == 0) ctx->arena.rewind();
    }
};

template <class T>
T* scratch(pqg_ctx* ctx, size_t count) {
    return static_cast<T*>(ctx->arena.alloc(count * sizeof(T)));
}

inline int prof_class(pqg_ctx* ctx, const char* name) {
    for (size_t i = 0; i < ctx->prof_names.size(); ++i)
        if (ctx->prof_names[i] == name) return int(i);
    ctx->prof_names.push_back(name);
    return int(ctx->prof_names.size() - 1);
}

inline cudaEvent_t take_event(pqg_ctx* ctx) {
    if (!ctx->event_pool.empty()) {
        cudaEvent_t e = ctx->event_pool.back();
        ctx->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    PQG_CUDA(cudaEventCreate(&e));
    return e;
}

// Launch wrapper: counts launches and, when profiling, brackets the kernel
// with CUDA events on the context stream.
template <typename Kernel, typename... Args>
void launch(pqg_ctx* ctx, const char* cls, Kernel kernel, dim3 grid, dim3 block, size_t smem,
            Args... args) {
    if (grid.x == 0 || grid.y == 0 || grid.z == 0) return;
    cudaEvent_t a = nullptr, b = nullptr;
    if (ctx->profiling) {
        a = take_event(ctx);
        b = take_event(ctx);
        PQG_CUDA(cudaEventRecord(a, ctx->stream));
    }
    kernel<<<grid, block, smem, ctx->stream>>>(args...);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fail(PQG_ECUDA, std::string("launch ") + cls + ": " + cudaGetErrorString(e));
    ++ctx->launches;
    if (ctx->profiling) {
        PQG_CUDA(cudaEventRecord(b, ctx->stream));
        ctx->prof_recs.push_back({prof_class(ctx, cls), a, b});
    }
}

template <typename Kernel>
void set_smem(Kernel k, size_t bytes) {
    static_assert(sizeof(Kernel) > 0, "");
    if (bytes > 48 * 1024)
        PQG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
}

inline unsigned grid1d(uint64_t n, unsigned block, unsigned cap = 1u << 30) {
    uint64_t g = (n + block - 1) / block;
    if (g > cap) g = cap;
    return unsigned(g ? g : 1);
}

}  // namespace pqg
