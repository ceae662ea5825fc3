"""Phase breakdown of the sharded k-means iteration at world 1 (NCCL) vs the
single-process fit: host wall time per phase with a device sync after each.

  python tools/shard_profile.py
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import torch.distributed as tdist

    from paper_2604_21645_b200 import dist as D
    from paper_2604_21645_b200 import pqii
    from paper_2604_21645_b200.datagen import gaussian_mixture, strided_sample
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    tdist.init_process_group("nccl", store=tdist.HashStore(), rank=0, world_size=1,
                             device_id=torch.device("cuda", 0))
    x = gaussian_mixture(1_000_000, 128, 256, 2604)
    train = torch.from_numpy(np.ascontiguousarray(x[strided_sample(1_000_000, 100_000, 2604)])).cuda()
    comm, be = D.Comm(), D.CudaBackend(0)
    be.ctx.set_stream(s.cuda_stream)
    seeds = [2604 + m for m in range(8)]
    phases = {}

    class Timed:
        def __init__(self, obj):
            self.o = obj

        def __getattr__(self, name):
            f = getattr(self.o, name)
            if not callable(f):
                return f

            def g(*a, **k):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                r = f(*a, **k)
                torch.cuda.synchronize()
                phases[name] = phases.get(name, 0.0) + time.perf_counter() - t0
                return r
            return g

    D.kmeans_fit_sharded(comm, be, train, 8, 16, 16, 256, 3, seeds)
    for rep in range(2):
        phases.clear()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = {}
        D.kmeans_fit_sharded(Timed(comm), Timed(be), train, 8, 16, 16, 256, 25, seeds, 1e-4, stats=st)
        torch.cuda.synchronize()
        tot = time.perf_counter() - t0
    print({k: round(v * 1e3, 3) for k, v in sorted(phases.items(), key=lambda kv: -kv[1])}, "total ms", tot * 1e3, st)
    t0 = time.perf_counter()
    D.kmeans_fit_sharded(comm, be, train, 8, 16, 16, 256, 25, seeds, 1e-4)
    torch.cuda.synchronize()
    print("untimed sharded ms", (time.perf_counter() - t0) * 1e3)
    ctx = pqii.Context(0)
    ctx.set_stream(s.cuda_stream)
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pqii.pq_fit(train, 8, 256, 25, 2604, ctx=ctx)
        torch.cuda.synchronize()
    print("single-process ms", (time.perf_counter() - t0) * 1e3)
    be.ctx.profile(True)
    D.kmeans_fit_sharded(comm, be, train, 8, 16, 16, 256, 25, seeds, 1e-4)
    torch.cuda.synchronize()
    for c in ("nearest_tc", "nearest", "fixup", "norms", "bucket", "scan", "kmeans_sum", "kmshard", "inertia",
              "reseed", "gather"):
        print(c, be.ctx.profile_read(c))
    tdist.destroy_process_group()


if __name__ == "__main__":
    main()
