"""Per-kernel-class device time of one ivf_build_with_centroids (2M rows, M=16, Ks=256, nlist 4096)."""
import ctypes as C, sys, os, json, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2604_21645_b200._lib as L
from paper_2604_21645_b200 import pqii
from paper_2604_21645_b200.datagen import gaussian_mixture
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
ctx = pqii.Context(0); ctx.set_stream(s.cuda_stream); lib, vp = ctx.lib, C.c_void_p
N, D, M, KS, NL = 2_000_000, 128, 16, 256, 4096
x = torch.from_numpy(gaussian_mixture(N, D, 1024, 7)).cuda()
tr = x[::10].contiguous()
t = torch.empty((M, KS, D // M), dtype=torch.float32, device='cuda')
L.check(lib.pqg_pq_fit(ctx.h, vp(tr.data_ptr()), tr.shape[0], D, M, KS, 4, 7, vp(t.data_ptr()), None, None))
coarse = tr[:NL].contiguous()
codes = torch.empty((N, M), dtype=torch.uint8, device='cuda')
L.check(lib.pqg_pq_encode(ctx.h, vp(x.data_ptr()), N, M, KS, D // M, vp(t.data_ptr()), vp(codes.data_ptr())))
ids = torch.arange(N, dtype=torch.int64, device='cuda')
def build():
    h = C.c_void_p()
    L.check(lib.pqg_ivf_build_with_centroids(ctx.h, vp(t.data_ptr()), M, KS, D // M, vp(codes.data_ptr()), vp(ids.data_ptr()), N, vp(coarse.data_ptr()), NL, C.byref(h)))
    return h
lib.pqg_index_destroy(build()); torch.cuda.synchronize()
t0 = time.perf_counter(); h = build(); torch.cuda.synchronize(); wall = time.perf_counter() - t0
lib.pqg_index_destroy(h)
ctx.profile(True); h = build(); torch.cuda.synchronize()
out = {'wall_ms': wall * 1e3}
for c in ("nearest_big_tc", "big_split", "fixup", "norms", "bucket", "scan", "dup_check", "csr_scatter", "gather", "nearest_tc", "nearest", "decode"):
    n, ms = ctx.profile_read(c)
    if n: out[c] = (n, round(ms, 3))
ctx.profile(False)
print(json.dumps(out))
