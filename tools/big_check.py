"""tcgen05 coarse path vs FP32 screen: identical assignments / probes, timing."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_2604_21645_b200._lib as L
    from paper_2604_21645_b200 import pqii
    from paper_2604_21645_b200.datagen import gaussian_mixture
    ctx = pqii.Context(0)
    lib = ctx.lib
    vp = C.c_void_p
    n = 1_000_000
    x = torch.from_numpy(gaussian_mixture(n, 128, 256, 5)).cuda()
    for nlist in (1024, 4096):
        cent = x[:: n // nlist][:nlist].contiguous()
        res = {}
        for mode in ("fp32", "tc"):
            os.environ["PQG_SCREEN"] = mode
            idx = torch.empty(n, dtype=torch.int32, device="cuda")
            dist = torch.empty(n, dtype=torch.float64, device="cuda")
            for rep in range(2):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                L.check(lib.pqg_nearest_batch(ctx.h, vp(x.data_ptr()), n, 128, vp(cent.data_ptr()), nlist,
                                              vp(idx.data_ptr()), vp(dist.data_ptr())))
                torch.cuda.synchronize()
                dt = time.perf_counter() - t0
            res[mode] = (idx.cpu().numpy(), dist.cpu().numpy())
            print(f"nlist={nlist} {mode}: {dt*1e3:.2f} ms for {n} rows", flush=True)
        same = np.array_equal(res["fp32"][0], res["tc"][0]) and np.array_equal(res["fp32"][1].view(np.uint64), res["tc"][1].view(np.uint64))
        print("  identical:", same, flush=True)
    # coarse k-means fit 100k x 1024
    coarse = torch.empty((1024, 128), dtype=torch.float32, device="cuda")
    inertia, iters = C.c_double(), C.c_uint32()
    for mode in ("fp32", "tc"):
        os.environ["PQG_SCREEN"] = mode
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        L.check(lib.pqg_kmeans_fit(ctx.h, vp(x.data_ptr()), 100_000, 128, 1024, 20, 7, 1e-4,
                                   vp(coarse.data_ptr()), None, C.byref(inertia), C.byref(iters), None))
        torch.cuda.synchronize()
        print(f"coarse kmeans {mode}: {time.perf_counter()-t0:.4f} s iters={iters.value} inertia={inertia.value!r}", flush=True)


if __name__ == "__main__":
    main()
