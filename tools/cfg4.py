"""BASELINE configs[3] on one GPU (its N=1 point): 10M x 96 fp32 rows from a
64-component mixture generated on the device, PQ fit (M=12, Ds=8, Ks=256, 20
iterations) on a seeded 1M-row strided sample, encode of all 10M rows and the
global RMSE.  Prints one JSON line of phase timings (CUDA events on the
library stream).  At N GPUs the rows shard by chunk_rows and the encode / SSE
are shard-local (paper_2604_21645_b200/dist.py).

  python tools/cfg4.py [--rows 10000000]
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
    ap.add_argument("--rows", type=int, default=10_000_000)
    args = ap.parse_args()
    import torch

    import paper_2604_21645_b200._lib as L
    from paper_2604_21645_b200 import pqii
    from paper_2604_21645_b200.datagen import mixture_params
    D, COMP, SEED = 96, 64, 2604
    M, KS, ITERS, SAMPLE = 12, 256, 20, 1_000_000
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    ctx = pqii.Context(0)
    ctx.set_stream(s.cuda_stream)
    lib, vp = ctx.lib, C.c_void_p
    out = {"config": "BASELINE configs[3]", "rows": args.rows, "dims": D, "M": M, "Ks": KS,
           "sample_rows": SAMPLE, "iters": ITERS, "data": "synthetic mixture, generated on device"}

    def timed(name, fn):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        r = fn()
        b.record(s)
        torch.cuda.synchronize()
        out[name + "_ms"] = a.elapsed_time(b)
        return r

    means, sigmas = mixture_params(D, COMP, SEED)
    mu = torch.from_numpy(means.astype(np.float64)).cuda()
    sg = torch.from_numpy(sigmas.astype(np.float64)).cuda()
    g = torch.Generator(device="cuda")
    g.manual_seed(SEED)
    x = torch.empty((args.rows, D), dtype=torch.float32, device="cuda")
    for r0 in range(0, args.rows, 1 << 20):
        r1 = min(args.rows, r0 + (1 << 20))
        comp = torch.randint(0, COMP, (r1 - r0,), generator=g, device="cuda")
        z = torch.randn((r1 - r0, D), generator=g, device="cuda", dtype=torch.float64)
        x[r0:r1] = (mu[comp] + sg[comp, None] * z).float()
    stride = args.rows // SAMPLE
    train = x[(SEED % stride)::stride][:SAMPLE].contiguous()

    tables = torch.empty((M, KS, D // M), dtype=torch.float32, device="cuda")
    it = (C.c_uint32 * M)()

    def fit():
        L.check(lib.pqg_pq_fit(ctx.h, vp(train.data_ptr()), SAMPLE, D, M, KS, ITERS, SEED,
                               vp(tables.data_ptr()), it, None))
    fit()  # warm-up (module load, scratch growth)
    timed("pq_fit", fit)
    out["pq_fit_iters"] = list(it)
    out["kmeans_iters_per_s"] = max(it) / (out["pq_fit_ms"] / 1e3)
    codes = torch.empty((args.rows, M), dtype=torch.uint8, device="cuda")
    enc = lambda: L.check(lib.pqg_pq_encode(ctx.h, vp(x.data_ptr()), args.rows, M, KS, D // M,  # noqa: E731
                                            vp(tables.data_ptr()), vp(codes.data_ptr())))
    enc()
    timed("encode", enc)
    out["encode_vectors_per_s"] = args.rows / (out["encode_ms"] / 1e3)
    sse = C.c_double()
    rs = lambda: L.check(lib.pqg_pq_recon_sse(ctx.h, vp(x.data_ptr()), vp(codes.data_ptr()),  # noqa: E731
                                              args.rows, M, KS, D // M, vp(tables.data_ptr()), C.byref(sse)))
    rs()  # warm-up (scratch growth)
    timed("recon_sse", rs)
    out["recon_sse_hbm_frac"] = (args.rows * D * 4 + args.rows * M) / (out["recon_sse_ms"] / 1e3) / 6.4546e12
    out["rmse"] = (sse.value / (args.rows * D)) ** 0.5
    out["gpu_mem_peak_gb"] = torch.cuda.max_memory_allocated() / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
