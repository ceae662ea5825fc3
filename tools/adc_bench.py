"""ADC scan timing on configs[2]-shaped indexes (1M x 128, Ks=256, nlist
1024, 10k queries, nprobe 16, k 10) for several M; kernel time from the
library's CUDA-event launch profiling, plus the candidates actually scanned.
Prints one JSON line per M.

  python tools/adc_bench.py [--rows 1000000] [--queries 10000] [--nprobe 16] [--m 16]
"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--queries", type=int, default=10_000)
    ap.add_argument("--nprobe", type=int, default=16)
    ap.add_argument("--nlist", type=int, default=1024)
    ap.add_argument("--m", default="16,8,32")
    ap.add_argument("--k", type=int, default=10)
    args = ap.parse_args()
    import torch

    import paper_2604_21645_b200._lib as L
    from paper_2604_21645_b200 import pqii
    from paper_2604_21645_b200.datagen import gaussian_mixture
    D, SEED = 128, 2604
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    ctx = pqii.Context(0)
    ctx.set_stream(s.cuda_stream)
    lib, vp = ctx.lib, C.c_void_p
    x = torch.from_numpy(gaussian_mixture(args.rows, D, 256, SEED)).cuda()
    train = x[:100_000].contiguous()
    q = torch.from_numpy(gaussian_mixture(args.queries, D, 256, SEED, stream=1)).cuda()
    coarse = torch.empty((args.nlist, D), dtype=torch.float32, device="cuda")
    L.check(lib.pqg_kmeans_fit(ctx.h, vp(train.data_ptr()), 100_000, D, args.nlist, 10, SEED, 1e-4,
                               vp(coarse.data_ptr()), None, None, None, None))
    for M in [int(v) for v in args.m.split(",")]:
        tables = torch.empty((M, 256, D // M), dtype=torch.float32, device="cuda")
        L.check(lib.pqg_pq_fit(ctx.h, vp(train.data_ptr()), 100_000, D, M, 256, 10, SEED,
                               vp(tables.data_ptr()), None, None))
        codes = torch.empty((args.rows, M), dtype=torch.uint8, device="cuda")
        L.check(lib.pqg_pq_encode(ctx.h, vp(x.data_ptr()), args.rows, M, 256, D // M,
                                  vp(tables.data_ptr()), vp(codes.data_ptr())))
        ids = torch.arange(args.rows, dtype=torch.int64, device="cuda")
        h = C.c_void_p()
        L.check(lib.pqg_ivf_build_with_centroids(ctx.h, vp(tables.data_ptr()), M, 256, D // M,
                                                 vp(codes.data_ptr()), vp(ids.data_ptr()), args.rows,
                                                 vp(coarse.data_ptr()), args.nlist, C.byref(h)))
        out = {"M": M, "rows": args.rows, "queries": args.queries, "nprobe": args.nprobe}
        oi = torch.empty((args.queries, args.k), dtype=torch.int64, device="cuda")
        od = torch.empty((args.queries, args.k), dtype=torch.float64, device="cuda")
        oc = torch.empty((args.queries,), dtype=torch.int32, device="cuda")

        def run():
            L.check(lib.pqg_index_search(ctx.h, h, vp(q.data_ptr()), args.queries, args.k,
                                         args.nprobe, 0, 0.0, vp(oi.data_ptr()),
                                         vp(od.data_ptr()), vp(oc.data_ptr())))
        run()  # warm-up (builds the cached decoded operand of the tensor-core path)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(s)
        for _ in range(5):
            run()
        ev1.record(s)
        torch.cuda.synchronize()
        out["search_ms"] = ev0.elapsed_time(ev1) / 5
        out["queries_per_s"] = args.queries / (out["search_ms"] / 1e3)
        ctx.profile(True)
        for _ in range(5):
            run()
        per = {}
        for cls in ("adc_scan", "adc_scan_tc", "tc_tasks", "bucket", "scan", "topk_merge",
                    "probe_select", "distance_matrix_tc", "big_split"):
            n, ms = ctx.profile_read(cls)
            if n:
                per[cls] = ms / 5
        ctx.profile(False)
        out["kernel_ms"] = per
        out["scan_ms"] = per.get("adc_scan", 0.0) + per.get("adc_scan_tc", 0.0)
        off = torch.empty(args.nlist + 1, dtype=torch.int64)
        L.check(lib.pqg_index_export(ctx.h, h, vp(off.data_ptr()), None, None, None, None))
        probes = torch.empty((args.queries, args.nprobe), dtype=torch.int32, device="cuda")
        L.check(lib.pqg_index_probe(ctx.h, h, vp(q.data_ptr()), args.queries, args.nprobe,
                                    vp(probes.data_ptr())))
        cand = int((off[1:] - off[:-1]).cuda()[probes.long()].sum())
        out["candidates_per_query"] = cand / args.queries
        out["scan_code_GBps"] = cand * M / (out["scan_ms"] / 1e3) / 1e9
        lib.pqg_index_destroy(h)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
