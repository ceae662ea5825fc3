"""Sharded coarse k-means at world 1 with the exchange forced: device time of
the row-order replay (class "kmshard") for the chained protocol vs the r2
all-gather protocol, on N x D device rows (default configs[4]'s coarse fit:
2M x 128, nlist 4096).  One JSON line per protocol.

  python tools/replay_bench.py [--n 2000000] [--k 4096] [--iters 6]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2_000_000)
    ap.add_argument("--d", type=int, default=128)
    ap.add_argument("--k", type=int, default=4096)
    ap.add_argument("--iters", type=int, default=6)
    args = ap.parse_args()
    import torch
    import torch.distributed as tdist

    from paper_2604_21645_b200 import dist as D
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    tdist.init_process_group("nccl", store=tdist.HashStore(), rank=0, world_size=1,
                             device_id=torch.device("cuda", 0))
    g = torch.Generator(device="cuda")
    g.manual_seed(2604)
    mu = torch.randn((256, args.d), generator=g, device="cuda") * 2
    x = (mu[torch.randint(0, 256, (args.n,), generator=g, device="cuda")] +
         torch.randn((args.n, args.d), generator=g, device="cuda")).contiguous()
    comm, be = D.Comm(), D.CudaBackend(0)
    be.ctx.set_stream(s.cuda_stream)
    for replay in ("chain", "gather", "chain"):
        st = {}
        D.kmeans_fit_sharded(comm, be, x, 1, args.d, 0, args.k, 1, [7], 0.0, force_exchange=True, replay=replay)
        torch.cuda.synchronize()
        be.ctx.profile(True)
        t0 = time.perf_counter()
        f = D.kmeans_fit_sharded(comm, be, x, 1, args.d, 0, args.k, args.iters, [7], 0.0, stats=st,
                                 force_exchange=True, replay=replay)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        cls = {}
        for c in ("kmshard", "kmeans_sum", "bucket", "scan", "nearest_big_tc", "fixup", "reseed", "big_split"):
            nl, ms = be.ctx.profile_read(c)
            if nl:
                cls[c] = round(ms, 3)
        be.ctx.profile(False)
        print(json.dumps({"replay": replay, "wall_ms": wall * 1e3, "iters": int(f.iterations_run[0]),
                          "replay_columns": st["replay_columns"], "allgather_bytes": st["allgather_bytes"],
                          "classes_ms": cls}), flush=True)
    tdist.destroy_process_group()


if __name__ == "__main__":
    main()
