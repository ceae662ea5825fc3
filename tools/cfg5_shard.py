"""One GPU's shard of BASELINE configs[4] (100M x 128 over 8 GPUs), end to end:
12.5M rows generated on the device from seed + rank (1024-component mixture),
PQ fit (M=16, Ks=256) and coarse fit (nlist=4096) with 20 iterations on a
seeded 2M-row sample, encode of the shard, inverted-index build of the shard,
and batched ADC search of 100k queries (nprobe 32, k 10).  Prints one JSON
line of phase timings (CUDA events on the library stream).

  python tools/cfg5_shard.py [--rows 12500000] [--rank 0]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=12_500_000)
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--queries", type=int, default=100_000)
    args = ap.parse_args()
    import torch

    import paper_2604_21645_b200._lib as L
    from paper_2604_21645_b200 import pqii
    from paper_2604_21645_b200.datagen import mixture_params
    D, COMP, SEED = 128, 1024, 2604
    M, KS, NLIST, ITERS = 16, 256, 4096, 20
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    ctx = pqii.Context(0)
    ctx.set_stream(s.cuda_stream)
    lib = ctx.lib
    vp = C.c_void_p
    out = {"rows": args.rows, "rank": args.rank}

    def timed(name, fn):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record(s)
        r = fn()
        b.record(s)
        torch.cuda.synchronize()
        out[name + "_ms"] = a.elapsed_time(b)
        out[name + "_wall_ms"] = (time.perf_counter() - t0) * 1e3
        return r

    # ---- data: mixture parameters from the base seed, rows from seed + rank
    means, sigmas = mixture_params(D, COMP, SEED)
    mu = torch.from_numpy(means.astype(np.float64)).cuda()
    sg = torch.from_numpy(sigmas.astype(np.float64)).cuda()
    g = torch.Generator(device="cuda")
    g.manual_seed(SEED + args.rank)
    x = torch.empty((args.rows, D), dtype=torch.float32, device="cuda")

    def gen():
        for r0 in range(0, args.rows, 1 << 20):
            r1 = min(args.rows, r0 + (1 << 20))
            comp = torch.randint(0, COMP, (r1 - r0,), generator=g, device="cuda")
            z = torch.randn((r1 - r0, D), generator=g, device="cuda", dtype=torch.float64)
            x[r0:r1] = (mu[comp] + sg[comp, None] * z).float()
    timed("generate", gen)
    n_train = 2_000_000
    stride = args.rows // n_train
    train = x[(SEED % stride)::stride][:n_train].contiguous()

    tables = torch.empty((M, KS, D // M), dtype=torch.float32, device="cuda")
    it = (C.c_uint32 * M)()
    # one-iteration warm-up fits of the same shapes (module load, scratch arena
    # growth by cudaMalloc) so the timed fits measure the fits alone
    L.check(lib.pqg_pq_fit(ctx.h, vp(train.data_ptr()), n_train, D, M, KS, 1, SEED, vp(tables.data_ptr()),
                           it, None))
    warm_c = torch.empty((NLIST, D), dtype=torch.float32, device="cuda")
    L.check(lib.pqg_kmeans_fit(ctx.h, vp(train.data_ptr()), n_train, D, NLIST, 1, SEED + M, 1e-4,
                               vp(warm_c.data_ptr()), None, None, None, None))
    timed("pq_fit", lambda: L.check(lib.pqg_pq_fit(ctx.h, vp(train.data_ptr()), n_train, D, M, KS, ITERS,
                                                   SEED, vp(tables.data_ptr()), it, None)))
    out["pq_fit_iters"] = list(it)
    coarse = torch.empty((NLIST, D), dtype=torch.float32, device="cuda")
    inertia, citers = C.c_double(), C.c_uint32()
    timed("coarse_fit", lambda: L.check(lib.pqg_kmeans_fit(ctx.h, vp(train.data_ptr()), n_train, D, NLIST,
                                                           ITERS, SEED + M, 1e-4, vp(coarse.data_ptr()),
                                                           None, C.byref(inertia), C.byref(citers), None)))
    out["coarse_fit_iters"] = citers.value
    if os.environ.get("CFG5_PROFILE"):  # per-kernel-class breakdown of one more coarse fit
        ctx.profile(True)
        L.check(lib.pqg_kmeans_fit(ctx.h, vp(train.data_ptr()), n_train, D, NLIST, ITERS, SEED + M, 1e-4,
                                   vp(coarse.data_ptr()), None, C.byref(inertia), C.byref(citers), None))
        out["coarse_fit_classes_ms"] = {c: ctx.profile_read(c)[1] for c in (
            "nearest_big_tc", "big_split", "fixup", "norms", "inertia", "bucket", "scan", "kmeans_sum",
            "reseed", "gather")}
        ctx.profile(False)
    codes = torch.empty((args.rows, M), dtype=torch.uint8, device="cuda")
    timed("encode", lambda: L.check(lib.pqg_pq_encode(ctx.h, vp(x.data_ptr()), args.rows, M, KS, D // M,
                                                      vp(tables.data_ptr()), vp(codes.data_ptr()))))
    sse = C.c_double()
    timed("recon_sse", lambda: L.check(lib.pqg_pq_recon_sse(ctx.h, vp(x.data_ptr()), vp(codes.data_ptr()),
                                                            args.rows, M, KS, D // M, vp(tables.data_ptr()),
                                                            C.byref(sse))))
    out["rmse"] = (sse.value / (args.rows * D)) ** 0.5
    ids = torch.arange(args.rows, dtype=torch.int64, device="cuda") + args.rank * args.rows
    h = C.c_void_p()
    timed("ivf_build", lambda: L.check(lib.pqg_ivf_build_with_centroids(
        ctx.h, vp(tables.data_ptr()), M, KS, D // M, vp(codes.data_ptr()), vp(ids.data_ptr()), args.rows,
        vp(coarse.data_ptr()), NLIST, C.byref(h))))
    gq = torch.Generator(device="cuda")
    gq.manual_seed(SEED + 1000003)
    comp = torch.randint(0, COMP, (args.queries,), generator=gq, device="cuda")
    q = (mu[comp] + sg[comp, None] * torch.randn((args.queries, D), generator=gq, device="cuda",
                                                 dtype=torch.float64)).float().contiguous()
    oi = torch.empty((args.queries, 10), dtype=torch.int64, device="cuda")
    od = torch.empty((args.queries, 10), dtype=torch.float64, device="cuda")
    oc = torch.empty((args.queries,), dtype=torch.int32, device="cuda")
    search = lambda: L.check(lib.pqg_index_search(ctx.h, h, vp(q.data_ptr()), args.queries, 10, 32, 0, 0.0,  # noqa: E731
                                                  vp(oi.data_ptr()), vp(od.data_ptr()), vp(oc.data_ptr())))
    search()
    timed("search", search)
    out["search_queries_per_s"] = args.queries / (out["search_ms"] / 1e3)
    off = torch.empty(NLIST + 1, dtype=torch.int64)
    L.check(lib.pqg_index_export(ctx.h, h, vp(off.data_ptr()), None, None, None, None))
    sizes = (off[1:] - off[:-1]).numpy()
    out["list_len_mean"], out["list_len_max"] = float(sizes.mean()), int(sizes.max())
    out["candidates_per_query_est"] = float(sizes.mean() * 32)
    lib.pqg_index_destroy(h)
    out["encode_vectors_per_s"] = args.rows / (out["encode_ms"] / 1e3)
    out["gpu_mem_peak_gb"] = torch.cuda.max_memory_allocated() / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
