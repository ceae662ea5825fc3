"""Compare the tcgen05 and FP32 screens: equal codes (and vs the oracle on a
sample), timing of pq_encode for 1M x 128 at several (M, Ks)."""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
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
    N, D = 1_000_000, 128
    xh = gaussian_mixture(N, D, 256, 2604)
    x = torch.from_numpy(xh).cuda()
    train = x.index_select(0, torch.from_numpy(strided_sample(N, 100_000, 2604)).cuda()).contiguous()
    orc = oracle.c_oracle()
    rng = np.random.default_rng(1)
    sel = np.sort(rng.choice(N, 4000, replace=False))
    for M, ks in [(8, 256), (16, 256), (4, 256), (32, 256), (8, 64), (16, 16), (32, 16)]:
        t = torch.empty((M, ks, D // M), dtype=torch.float32, device="cuda")
        os.environ["PQG_SCREEN"] = "fp32"
        L.check(lib.pqg_pq_fit(ctx.h, vp(train.data_ptr()), 100_000, D, M, ks, 3, 7, vp(t.data_ptr()), None, None))
        res = {}
        modes = ("fp32", "tc1", "tc1s", "tc8", "tc16", "tcdef", "auto")
        for mode in modes:
            # tc1: 1-pass v1; tc1s: v1 in two 128-codeword passes; tc8/tc16: the
            # pipelined kernel with 8/16 warps; tcdef: the library's own choice
            os.environ["PQG_SCREEN"] = "fp32" if mode == "fp32" else "tc"
            os.environ["PQG_UMMA"] = {"tc1": "1", "tc1s": "1", "tc8": "2", "tc16": "2"}.get(mode, "0")
            os.environ["PQG_UMMA_WARPS"] = "16" if mode == "tc16" else "8"
            os.environ["PQG_UMMA_SPLIT"] = "1" if mode == "tc1s" else "0"
            if mode in ("tcdef", "auto"):
                del os.environ["PQG_UMMA_SPLIT"]
            if mode == "auto":  # the library's own choice of screen
                del os.environ["PQG_SCREEN"]
            codes = torch.empty((N, M), dtype=torch.uint8, device="cuda")
            enc = lambda: L.check(lib.pqg_pq_encode(ctx.h, vp(x.data_ptr()), N, M, ks, D // M,
                                                     vp(t.data_ptr()), vp(codes.data_ptr())))
            for _ in range(3):
                enc()
            ctx.profile(True)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            for _ in range(10):
                enc()
            b.record(s)
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / 10
            kname = "nearest" if mode == "fp32" else "nearest_tc"
            n1, k1 = ctx.profile_read(kname)
            if mode == "auto" and n1 == 0:
                n1, k1 = ctx.profile_read("nearest_small")
            n2, k2 = ctx.profile_read("fixup")
            ctx.profile(False)
            res[mode] = codes.cpu().numpy()
            print(f"M={M:2d} Ks={ks:3d} {mode:4s}: {ms:7.3f} ms/encode  {N/ms/1e6:8.2f} Mvec/s  "
                  f"screen {k1/max(n1,1):.3f} ms  fixup {k2/max(n2,1):.3f} ms", flush=True)
        same = all(np.array_equal(res["fp32"], res[m]) for m in modes[1:])
        ref = orc.pq_encode(xh[sel], t.cpu().numpy())
        ok = np.array_equal(res["tc16"][sel], ref)
        print(f"   codes tc==fp32: {same}  tc==oracle(sample): {ok}", flush=True)
        if not same:
            diff = np.argwhere(res["fp32"] != res["tc16"])
            print("   first diffs", diff[:5].tolist(), flush=True)


if __name__ == "__main__":
    main()
