"""k-means fit workloads for the launch list: PQ fit (100k x 128, M=8, Ks=256,
25 iters) and a coarse fit (100k x 128, k=1024, 20 iters)."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_2604_21645_b200._lib as L
    from paper_2604_21645_b200 import pqii
    from paper_2604_21645_b200.datagen import gaussian_mixture
    ctx = pqii.Context(0)
    lib = ctx.lib
    vp = C.c_void_p
    x = torch.from_numpy(gaussian_mixture(100_000, 128, 256, 2604)).cuda()
    t = torch.empty((8, 256, 16), dtype=torch.float32, device="cuda")
    it = (C.c_uint32 * 8)()
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        L.check(lib.pqg_pq_fit(ctx.h, vp(x.data_ptr()), 100_000, 128, 8, 256, 25, 7, vp(t.data_ptr()), it, None))
        torch.cuda.synchronize()
        print("pq_fit", time.perf_counter() - t0, list(it))
    coarse = torch.empty((1024, 128), dtype=torch.float32, device="cuda")
    inertia, iters = C.c_double(), C.c_uint32()
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        L.check(lib.pqg_kmeans_fit(ctx.h, vp(x.data_ptr()), 100_000, 128, 1024, 20, 7, 1e-4,
                                   vp(coarse.data_ptr()), None, C.byref(inertia), C.byref(iters), None))
        torch.cuda.synchronize()
        print("coarse kmeans", time.perf_counter() - t0, iters.value)


if __name__ == "__main__":
    main()
