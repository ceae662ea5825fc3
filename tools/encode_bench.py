"""pq_encode of 1M x 128 device rows at (M, Ks) points: time per launch (CUDA
events), vectors/s, the screen kernel that ran, and a sampled check against
the oracle.  --ncu: one encode per point (for an ncu capture).

  python tools/encode_bench.py [--points 32x16,16x16,4x16] [--ncu]
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
    ap.add_argument("--points", default="4x16,8x16,16x16,32x16,4x64,8x64,16x64,32x64")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--ncu", action="store_true")
    ap.add_argument("--rows", type=int, default=1_000_000)
    args = ap.parse_args()
    import torch

    import oracle
    import paper_2604_21645_b200._lib as L
    from paper_2604_21645_b200 import pqii
    from paper_2604_21645_b200.datagen import gaussian_mixture, strided_sample
    ctx = pqii.Context(0)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    ctx.set_stream(s.cuda_stream)
    lib = ctx.lib
    vp = C.c_void_p
    N, D = args.rows, 128
    xh = gaussian_mixture(N, D, 256, 2604)
    x = torch.from_numpy(xh).cuda()
    train = x.index_select(0, torch.from_numpy(strided_sample(N, 100_000, 2604)).cuda()).contiguous()
    orc = oracle.c_oracle()
    rng = np.random.default_rng(1)
    sel = np.sort(rng.choice(N, min(N, 3000), replace=False))
    out = []
    for p in args.points.split(","):
        M, ks = (int(v) for v in p.split("x"))
        t = torch.empty((M, ks, D // M), dtype=torch.float32, device="cuda")
        L.check(lib.pqg_pq_fit(ctx.h, vp(train.data_ptr()), 100_000, D, M, ks, 3, 7, vp(t.data_ptr()), None, None))
        codes = torch.empty((N, M), dtype=torch.uint8, device="cuda")
        enc = lambda: L.check(lib.pqg_pq_encode(ctx.h, vp(x.data_ptr()), N, M, ks, D // M, vp(t.data_ptr()),  # noqa
                                                vp(codes.data_ptr())))
        enc()
        torch.cuda.synchronize()
        if args.ncu:  # one profiled encode (ncu --profile-from-start off)
            torch.cuda.cudart().cudaProfilerStart()
            enc()
            torch.cuda.synchronize()
            torch.cuda.cudart().cudaProfilerStop()
            continue
        ctx.profile(True)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(args.reps):
            enc()
        b.record(s)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / args.reps
        kern = {c: ctx.profile_read(c) for c in ("nearest_small", "nearest_narrow", "nearest_tc", "nearest", "fixup",
                                                   "norms")}
        ctx.profile(False)
        got = codes.cpu().numpy()[sel]
        want = orc.pq_encode(xh[sel], t.cpu().numpy())
        rec = {"M": M, "Ks": ks, "ms": ms, "G_vec_s": N / ms / 1e6, "exact": bool(np.array_equal(got, want)),
               "kernels_ms": {k: v[1] / max(1, v[0]) for k, v in kern.items() if v[0]},
               "hbm_frac": (N * (4 * D + M) / (ms / 1e3)) / 6.5546e12}
        out.append(rec)
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
