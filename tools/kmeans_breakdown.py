"""Per-kernel-class device time of one PQ fit (configs[0]/[1] shape: 100k x
128, M=8, Ks=256, 25 iterations) and one coarse fit (100k x 128, k=1024, 20
iterations), from the library's CUDA-event launch profiling.  One JSON line.

  python tools/kmeans_breakdown.py
"""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CLASSES = ("nearest_tc", "nearest", "nearest_big_tc", "big_split", "fixup", "norms", "pad_keys", "inertia",
           "bucket", "scan", "kmeans_sum", "reseed", "gather")


def main():
    import torch

    import paper_2604_21645_b200._lib as L
    from paper_2604_21645_b200 import pqii
    from paper_2604_21645_b200.datagen import gaussian_mixture
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    ctx = pqii.Context(0)
    ctx.set_stream(s.cuda_stream)
    lib, vp = ctx.lib, C.c_void_p
    x = torch.from_numpy(gaussian_mixture(100_000, 128, 64, 2604)).cuda()
    out = {}
    t = torch.empty((8, 256, 16), dtype=torch.float32, device="cuda")
    it = (C.c_uint32 * 8)()

    def pq():
        L.check(lib.pqg_pq_fit(ctx.h, vp(x.data_ptr()), 100_000, 128, 8, 256, 25, 7,
                               vp(t.data_ptr()), it, None))
    coarse = torch.empty((1024, 128), dtype=torch.float32, device="cuda")
    ci = C.c_uint32()

    def km():
        L.check(lib.pqg_kmeans_fit(ctx.h, vp(x.data_ptr()), 100_000, 128, 1024, 20, 7, 0.0,
                                   vp(coarse.data_ptr()), None, None, C.byref(ci), None))
    for name, fn in (("pq_fit", pq), ("coarse_fit", km)):
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
