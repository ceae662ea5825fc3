// kmnccl.cu -- the native (C++) host of the row-sharded k-means fit
// (SURVEY.md 8(e)), NCCL underneath: one rank per GPU, each rank calls
// pqg_kmeans_fit_sharded with its own communicator and its contiguous block
// of the global row-ordered sample.  Per iteration, on the context's stream:
//   pqg_kmshard_partials -> ncclAllReduce SUM (fp64 sums | counts | inertia)
//                         + ncclAllReduce MAX (u8 exponent ranges), grouped
//   pqg_kmshard_apply    -> the one host synchronisation (replay / reseed sizes)
//   inexact columns      -> ncclRecv(run) from rank r-1, replay_step,
//                           ncclSend(run) to rank r+1, ncclBroadcast from the
//                           last rank, replay_finish (no member values move)
//   empty clusters       -> ncclAllGather of every rank's reseed candidates
// -- the same protocol as paper_2604_21645_b200/dist.py, without Python and
// torch.distributed in the loop.  kmeans.cpp:61-133 / pq.cpp:63-93 bit for
// bit at any world size.
//
// libnccl.so.2 is opened at run time (dlopen): the library keeps no link-time
// NCCL dependency, and inside a process that already loaded NCCL (torch) the
// same copy is used.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/pqg.h"
#include "common.cuh"

namespace pqg {
void set_last_error(const std::string& m);  // capi.cu
namespace {

template <class F>
int guard(F&& f) {
    try {
        f();
        return PQG_OK;
    } catch (const Error& e) {
        set_last_error(e.msg);
        return e.code;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return PQG_ECUDA;
    } catch (...) {
        set_last_error("unknown error");
        return PQG_ECUDA;
    }
}

void inval(const std::string& m) { fail(PQG_EINVAL, m); }

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            api.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (api.h) break;
        }
        if (!api.h) return;
        auto sym = [](const char* s) { return dlsym(api.h, s); };
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
        api.CommInitAll = reinterpret_cast<decltype(api.CommInitAll)>(sym("ncclCommInitAll"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
        api.CommCount = reinterpret_cast<decltype(api.CommCount)>(sym("ncclCommCount"));
        api.CommUserRank = reinterpret_cast<decltype(api.CommUserRank)>(sym("ncclCommUserRank"));
        api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
        api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
        api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(sym("ncclBroadcast"));
        api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
        api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    });
    if (!api.h || !api.AllReduce || !api.Send || !api.CommInitRank)
        fail(PQG_EUNSUPPORTED, "NCCL (libnccl.so.2) is not available");
    return api;
}

void nccheck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        const char* s = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
        fail(PQG_ECUDA, std::string("nccl ") + what + ": " + s);
    }
}

// A pqg_* call's status as an exception (the C ABI reports, guard rethrows).
void check_rc(int rc) {
    if (rc != PQG_OK) fail(rc, pqg_last_error());
}

template <class T>
T* dev_alloc(uint64_t count) {
    T* p = nullptr;
    if (cudaMalloc(&p, std::max<uint64_t>(count, 1) * sizeof(T)) != cudaSuccess) {
        cudaGetLastError();
        fail(PQG_ENOMEM, "device allocation of " + std::to_string(count * sizeof(T)) + " bytes failed");
    }
    return p;
}

struct DevBufs {  // freed on every exit path
    std::vector<void*> p;
    template <class T>
    T* get(uint64_t count) {
        T* q = dev_alloc<T>(count);
        p.push_back(q);
        return q;
    }
    ~DevBufs() {
        for (void* q : p) cudaFree(q);
    }
};

}  // namespace
}  // namespace pqg

using namespace pqg;

extern "C" {

int pqg_nccl_get_unique_id(void* id) {
    return guard([&] {
        if (!id) inval("nccl: null id");
        ncclUniqueId u;
        nccheck(nccl().GetUniqueId(&u), "GetUniqueId");
        std::memcpy(id, &u, sizeof(u));
    });
}

int pqg_nccl_comm_init(int device, int world, int rank, const void* id, void** comm) {
    return guard([&] {
        if (!id || !comm) inval("nccl: null argument");
        if (world < 1 || rank < 0 || rank >= world) inval("nccl: rank out of range");
        PQG_CUDA(cudaSetDevice(device));
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof(u));
        ncclComm_t c = nullptr;
        nccheck(nccl().CommInitRank(&c, world, u, rank), "CommInitRank");
        *comm = c;
    });
}

int pqg_nccl_comm_init_all(int ndev, const int* devices, void** comms) {
    return guard([&] {
        if (ndev < 1 || !comms) inval("nccl: bad device list");
        std::vector<ncclComm_t> c(ndev);
        nccheck(nccl().CommInitAll(c.data(), ndev, devices), "CommInitAll");
        for (int i = 0; i < ndev; ++i) comms[i] = c[i];
    });
}

void pqg_nccl_comm_destroy(void* comm) {
    if (comm) (void)guard([&] { nccl().CommDestroy(static_cast<ncclComm_t>(comm)); });
}

int pqg_kmeans_fit_sharded(pqg_ctx* ctx, void* comm, const float* rows, uint64_t n_local, uint64_t ld,
                           uint32_t B, uint32_t d, uint32_t col_stride, uint64_t k, uint32_t max_iters,
                           const uint64_t* seeds, double tol, float* tables_out, uint32_t* iterations_run,
                           double* inertia, double* inertia_per_iter, uint32_t* assignments_local,
                           uint64_t* stats) {
    pqg_kmshard* h = nullptr;
    const int rc = guard([&] {
        if (!ctx || !comm || !seeds) inval("kmeans_fit_sharded: null argument");
        const NcclApi& nc = nccl();
        ncclComm_t cm = static_cast<ncclComm_t>(comm);
        int world = 1, rank = 0;
        nccheck(nc.CommCount(cm, &world), "CommCount");
        nccheck(nc.CommUserRank(cm, &rank), "CommUserRank");
        PQG_CUDA(cudaSetDevice(ctx->device));
        cudaStream_t st = ctx->stream;
        DevBufs bufs;
        // every rank's row count (kmeans.cpp:65-71 checks are on the global n)
        uint64_t* dcnt = bufs.get<uint64_t>(world + 1);
        PQG_CUDA(cudaMemcpyAsync(dcnt + world, &n_local, sizeof(uint64_t), cudaMemcpyHostToDevice, st));
        nccheck(nc.AllGather(dcnt + world, dcnt, 1, ncclUint64, cm, st), "AllGather(counts)");
        std::vector<uint64_t> counts(world);
        PQG_CUDA(cudaMemcpyAsync(counts.data(), dcnt, sizeof(uint64_t) * world, cudaMemcpyDeviceToHost, st));
        PQG_CUDA(cudaStreamSynchronize(st));
        uint64_t n = 0, row0 = 0;
        for (int r = 0; r < world; ++r) {
            if (r < rank) row0 += counts[r];
            n += counts[r];
        }
        if (k == 0) inval("kmeans_fit: k must be >= 1");
        if (k > n) inval("kmeans_fit: k (" + std::to_string(k) + ") exceeds number of points (" + std::to_string(n) + ")");
        if (max_iters < 1) inval("kmeans_fit: max_iters must be >= 1");
        if (tol < 0.0) inval("kmeans_fit: tol must be >= 0");
        check_rc(pqg_kmshard_create(ctx, rows, n_local, ld, B, d, col_stride, k, max_iters, tol, &h));
        uint64_t nf = 0, nu = 0;
        check_rc(pqg_kmshard_sizes(h, &nf, &nu));
        double* f64 = bufs.get<double>(nf);
        uint8_t* u8 = bufs.get<uint8_t>(nu);
        const uint64_t nkd = uint64_t(B) * k * d;
        float* tables = bufs.get<float>(nkd);
        // the init rows (kmeans.cpp:73-85, seed per problem) assembled by an
        // integer SUM of the owners' bit patterns (zeros elsewhere): exact
        std::vector<uint64_t> init(uint64_t(B) * k);
        for (uint32_t b = 0; b < B; ++b) check_rc(pqg_kmeans_init_rows(n, k, seeds[b], init.data() + uint64_t(b) * k));
        uint32_t* bits = reinterpret_cast<uint32_t*>(tables);
        check_rc(pqg_kmshard_init_table(ctx, h, init.data(), row0, bits));
        nccheck(nc.AllReduce(bits, bits, nkd, ncclUint32, ncclSum, cm, st), "AllReduce(init)");
        double* run = nullptr;
        uint64_t run_cap = 0;
        uint64_t iters = 0, replay_cols = 0, reseeds = 0;
        for (uint32_t it = 0; it < max_iters; ++it) {
            check_rc(pqg_kmshard_partials(ctx, h, tables, f64, u8));
            nccheck(nc.GroupStart(), "GroupStart");
            nccheck(nc.AllReduce(f64, f64, nf, ncclFloat64, ncclSum, cm, st), "AllReduce(partials)");
            nccheck(nc.AllReduce(u8, u8, nu, ncclUint8, ncclMax, cm, st), "AllReduce(exponents)");
            nccheck(nc.GroupEnd(), "GroupEnd");
            ++iters;
            uint64_t n_fail = 0, stride = 0;
            uint32_t max_empty = 0;
            int any_active = 0;
            check_rc(pqg_kmshard_apply(ctx, h, tables, f64, u8, &n_fail, &stride, &max_empty, &any_active));
            if (n_fail) {  // the row-order chains, rank to rank
                if (n_fail > run_cap) {
                    run = bufs.get<double>(n_fail);
                    run_cap = n_fail;
                }
                PQG_CUDA(cudaMemsetAsync(run, 0, sizeof(double) * n_fail, st));
                if (rank > 0) nccheck(nc.Recv(run, n_fail, ncclFloat64, rank - 1, cm, st), "Recv(chain)");
                check_rc(pqg_kmshard_replay_step(ctx, h, run));
                if (rank < world - 1) nccheck(nc.Send(run, n_fail, ncclFloat64, rank + 1, cm, st), "Send(chain)");
                nccheck(nc.Broadcast(run, run, n_fail, ncclFloat64, world - 1, cm, st), "Broadcast(chain)");
                check_rc(pqg_kmshard_replay_finish(ctx, h, tables, f64, run));
                replay_cols += n_fail;
            }
            if (max_empty) {  // every rank's best candidates, merged identically everywhere
                const uint64_t slots = uint64_t(B) * (max_empty + 1);
                double* cd = bufs.get<double>(slots * (world + 1));
                uint64_t* ci = bufs.get<uint64_t>(slots * (world + 1));
                float* cr = bufs.get<float>(slots * d * (world + 1));
                double* my_d = cd + slots * world;
                uint64_t* my_i = ci + slots * world;
                float* my_r = cr + slots * d * world;
                check_rc(pqg_kmshard_reseed_candidates(ctx, h, row0, max_empty, my_d, my_i, my_r));
                nccheck(nc.GroupStart(), "GroupStart");
                nccheck(nc.AllGather(my_d, cd, slots, ncclFloat64, cm, st), "AllGather(cand d)");
                nccheck(nc.AllGather(my_i, ci, slots, ncclUint64, cm, st), "AllGather(cand i)");
                nccheck(nc.AllGather(my_r, cr, slots * d, ncclFloat32, cm, st), "AllGather(cand rows)");
                nccheck(nc.GroupEnd(), "GroupEnd");
                check_rc(pqg_kmshard_reseed_apply(ctx, h, tables, f64, max_empty, uint32_t(world), cd, ci, cr));
                ++reseeds;
            }
            if (!any_active) break;
        }
        check_rc(pqg_kmshard_result(ctx, h, iterations_run, inertia, inertia_per_iter, assignments_local));
        PQG_CUDA(cudaMemcpyAsync(tables_out, tables, sizeof(float) * nkd, cudaMemcpyDefault, st));
        PQG_CUDA(cudaStreamSynchronize(st));
        if (stats) {  // iterations, replay columns, reseeds, all-reduce bytes per iteration
            stats[0] = iters;
            stats[1] = replay_cols;
            stats[2] = reseeds;
            stats[3] = nf * 8 + nu;
        }
    });
    if (h) pqg_kmshard_destroy(h);
    return rc;
}

}  // extern "C"
