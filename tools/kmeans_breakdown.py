"""Per-kernel-class device time of one PQ fit (default: configs[0]/[1] shape,
100k x 128, M=8, Ks=256, 25 iterations) and one coarse fit (100k x 128,
k=1024, 20 iterations), from the library's CUDA-event launch profiling.  One
JSON line.

  python tools/kmeans_breakdown.py [--rows 100000] [--dims 128] [--m 8] [--no-coarse]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CLASSES = ("nearest_tc", "nearest", "nearest_big_tc", "big_split", "fixup", "norms", "pad_keys", "inertia",
           "bucket", "scan", "kmeans_sum", "reseed", "gather")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=100_000)
    ap.add_argument("--dims", type=int, default=128)
    ap.add_argument("--m", type=int, default=8)
    ap.add_argument("--no-coarse", action="store_true")
    args = ap.parse_args()
    import torch

    import paper_2604_21645_b200._lib as L
    from paper_2604_21645_b200 import pqii
    from paper_2604_21645_b200.datagen import gaussian_mixture
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    ctx = pqii.Context(0)
    ctx.set_stream(s.cuda_stream)
    lib, vp = ctx.lib, C.c_void_p
    N, D, M = args.rows, args.dims, args.m
    x = torch.from_numpy(gaussian_mixture(N, D, 64, 2604)).cuda()
    out = {}
    t = torch.empty((M, 256, D // M), dtype=torch.float32, device="cuda")
    it = (C.c_uint32 * M)()

    def pq():
        L.check(lib.pqg_pq_fit(ctx.h, vp(x.data_ptr()), N, D, M, 256, 25, 7,
                               vp(t.data_ptr()), it, None))
    coarse = torch.empty((1024, D), dtype=torch.float32, device="cuda")
    ci = C.c_uint32()

    def km():
        L.check(lib.pqg_kmeans_fit(ctx.h, vp(x.data_ptr()), N, D, 1024, 20, 7, 0.0,
                                   vp(coarse.data_ptr()), None, None, C.byref(ci), None))
    for name, fn in (("pq_fit", pq),) + (() if args.no_coarse else (("coarse_fit", km),)):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        ctx.profile(True)
        fn()
        per = {}
        for c in CLASSES:
            n, ms = ctx.profile_read(c)
            if n:
                per[c] = {"launches": n, "ms": ms}
        ctx.profile(False)
        passes = max(it) if name == "pq_fit" else ci.value
        out[name] = {"wall_ms": wall * 1e3, "passes": passes, "iters_per_s": passes / wall,
                     "classes": per}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
