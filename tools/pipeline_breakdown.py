"""Per-kernel-class device time of the batched chunk fits of the paper's
pipeline (train_chunks: criterion-4 shape, 500k x 48, C=32, M=8, Ks=256, 20
iterations), from the library's CUDA-event launch profiling.

  python tools/pipeline_breakdown.py [--rows 500000] [--dims 48] [--chunks 32] [--m 8] [--ks 256]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=500_000)
    ap.add_argument("--dims", type=int, default=48)
    ap.add_argument("--chunks", type=int, default=32)
    ap.add_argument("--m", type=int, default=8)
    ap.add_argument("--ks", type=int, default=256)
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    import torch

    from paper_2604_21645_b200 import pqii
    from paper_2604_21645_b200.datagen import gaussian_mixture
    x = torch.from_numpy(gaussian_mixture(args.rows, args.dims, 64, 2604)).cuda()
    ctx = pqii.get_context()
    run = lambda: pqii.train_chunks(x, args.chunks, args.m, args.ks, args.iters, 1, ctx=ctx)  # noqa: E731
    run()
    ctx.profile(True)
    t0 = time.perf_counter()
    run()
    print("wall_s", round(time.perf_counter() - t0, 5))
    for c in ("pipeline", "gather", "nearest_tc", "nearest", "fixup", "norms", "pad_keys", "inertia",
              "bucket", "scan", "kmeans_sum", "reseed", "recon_sse", "reduce"):
        n, ms = ctx.profile_read(c)
        if n:
            print(f"{c:12s} {n:4d} launches {ms:9.3f} ms  {ms / n * 1000:8.1f} us/launch")
    ctx.profile(False)


if __name__ == "__main__":
    main()
