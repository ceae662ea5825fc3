"""Decode + squared-error (recon SSE) timing: pqg_pq_recon_sse over N x D
device rows (configs[3] shape by default: D=96, M=12, Ks=256).  --ncu: one
profiled call (ncu --profile-from-start off).

  python tools/sse_bench.py [--n 4000000] [--d 96] [--m 12] [--ncu]
"""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4_000_000)
    ap.add_argument("--d", type=int, default=96)
    ap.add_argument("--m", type=int, default=12)
    ap.add_argument("--ks", type=int, default=256)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--ncu", action="store_true")
    args = ap.parse_args()
    import torch

    import paper_2604_21645_b200._lib as L
    from paper_2604_21645_b200 import pqii
    ctx = pqii.Context(0)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    ctx.set_stream(s.cuda_stream)
    lib, vp = ctx.lib, C.c_void_p
    N, D, M, ks = args.n, args.d, args.m, args.ks
    x = torch.randn(N, D, device="cuda")
    t = torch.randn(M, ks, D // M, device="cuda")
    codes = torch.randint(0, ks, (N, M), dtype=torch.uint8, device="cuda")
    sse = C.c_double()
    run = lambda: L.check(lib.pqg_pq_recon_sse(ctx.h, vp(x.data_ptr()), vp(codes.data_ptr()), N, M, ks, D // M,  # noqa
                                               vp(t.data_ptr()), C.byref(sse)))
    run()
    torch.cuda.synchronize()
    if args.ncu:
        torch.cuda.cudart().cudaProfilerStart()
        run()
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
        return
    ctx.profile(True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(args.reps):
        run()
    b.record(s)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.reps
    n_k, k_ms = ctx.profile_read("recon_sse")
    byts = N * D * 4 + N * M
    print(json.dumps({"N": N, "D": D, "M": M, "ms": ms, "kernel_ms": k_ms / max(1, n_k),
                      "GBps": byts / (k_ms / max(1, n_k) / 1e3) / 1e9,
                      "hbm_frac": byts / (k_ms / max(1, n_k) / 1e3) / 6.4546e12}))


if __name__ == "__main__":
    main()
