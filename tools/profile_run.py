"""Short fixed workload for ncu captures: encode 1M x 128 (M=8, Ks=256) three
times, one k-means fit and one config-3 ADC search batch.

  ncu ... python tools/profile_run.py [encode|kmeans|adc|all]
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(what="all"):
    import torch

    import paper_2604_21645_b200._lib as L
    from paper_2604_21645_b200 import pqii
    from paper_2604_21645_b200.datagen import gaussian_mixture, strided_sample
    ctx = pqii.Context(0)
    lib = ctx.lib
    vp = C.c_void_p
    N, D = 1_000_000, 128
    x = torch.from_numpy(gaussian_mixture(N, D, 256, 2604)).cuda()
    train = x.index_select(0, torch.from_numpy(strided_sample(N, 100_000, 2604)).cuda()).contiguous()
    torch.cuda.synchronize()
    if what in ("encode", "all", "kmeans"):
        M, ks = 8, 256
        t = torch.empty((M, ks, D // M), dtype=torch.float32, device="cuda")
        L.check(lib.pqg_pq_fit(ctx.h, vp(train.data_ptr()), 100_000, D, M, ks, 25 if what != "encode" else 2,
                               2604, vp(t.data_ptr()), None, None))
        codes = torch.empty((N, M), dtype=torch.uint8, device="cuda")
        for _ in range(3):
            L.check(lib.pqg_pq_encode(ctx.h, vp(x.data_ptr()), N, M, ks, D // M, vp(t.data_ptr()),
                                      vp(codes.data_ptr())))
    if what in ("adc", "all"):
        M, ks, nlist = 16, 256, 1024
        t = torch.empty((M, ks, D // M), dtype=torch.float32, device="cuda")
        L.check(lib.pqg_pq_fit(ctx.h, vp(train.data_ptr()), 100_000, D, M, ks, 4, 2604,
                               vp(t.data_ptr()), None, None))
        coarse = torch.empty((nlist, D), dtype=torch.float32, device="cuda")
        inertia, it = C.c_double(), C.c_uint32()
        L.check(lib.pqg_kmeans_fit(ctx.h, vp(train.data_ptr()), 100_000, D, nlist, 4, 7, 1e-4,
                                   vp(coarse.data_ptr()), None, C.byref(inertia), C.byref(it), None))
        codes = torch.empty((N, M), dtype=torch.uint8, device="cuda")
        L.check(lib.pqg_pq_encode(ctx.h, vp(x.data_ptr()), N, M, ks, D // M, vp(t.data_ptr()),
                                  vp(codes.data_ptr())))
        ids = torch.arange(N, dtype=torch.int64, device="cuda")
        h = C.c_void_p()
        L.check(lib.pqg_ivf_build_with_centroids(ctx.h, vp(t.data_ptr()), M, ks, D // M,
                                                 vp(codes.data_ptr()), vp(ids.data_ptr()), N,
                                                 vp(coarse.data_ptr()), nlist, C.byref(h)))
        q = torch.from_numpy(gaussian_mixture(10_000, D, 256, 2604, stream=1)).cuda()
        oi = torch.empty((10_000, 10), dtype=torch.int64, device="cuda")
        od = torch.empty((10_000, 10), dtype=torch.float64, device="cuda")
        oc = torch.empty((10_000,), dtype=torch.int32, device="cuda")
        for _ in range(2):
            L.check(lib.pqg_index_search(ctx.h, h, vp(q.data_ptr()), 10_000, 10, 16, 0, 0.0,
                                         vp(oi.data_ptr()), vp(od.data_ptr()), vp(oc.data_ptr())))
        lib.pqg_index_destroy(h)
    ctx.sync()
    print("profile_run ok", what, ctx.launches)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all")
