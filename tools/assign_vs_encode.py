import ctypes as C, json, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2604_21645_b200._lib as L
from paper_2604_21645_b200 import pqii
from paper_2604_21645_b200.datagen import gaussian_mixture
ctx = pqii.get_context(0); lib = ctx.lib; vp = C.c_void_p
s = torch.cuda.Stream(); torch.cuda.set_stream(s); ctx.set_stream(s.cuda_stream)
N, D, M, KS = 100000, 128, 8, 256
x = torch.from_numpy(gaussian_mixture(N, D, 64, 2604)).cuda()
t = torch.empty((M, KS, D // M), dtype=torch.float32, device="cuda")
it = (C.c_uint32 * M)()
L.check(lib.pqg_pq_fit(ctx.h, vp(x.data_ptr()), N, D, M, KS, 5, 7, vp(t.data_ptr()), it, None))
codes = torch.empty((N, M), dtype=torch.uint8, device="cuda")
a = torch.empty((M, N), dtype=torch.int32, device="cuda"); dist = torch.empty((M, N), dtype=torch.float64, device="cuda")
def enc(): L.check(lib.pqg_pq_encode(ctx.h, vp(x.data_ptr()), N, M, KS, D // M, vp(t.data_ptr()), vp(codes.data_ptr())))
def asg(): L.check(lib.pqg_assign_pass(ctx.h, vp(x.data_ptr()), N, D, M, D // M, D // M, vp(t.data_ptr()), KS, vp(a.data_ptr()), vp(dist.data_ptr())))
for name, fn in (("encode", enc), ("assign_pass", asg)):
    fn(); torch.cuda.synchronize()
    ctx.profile(True)
    for _ in range(20): fn()
    torch.cuda.synchronize()
    out = {c: ctx.profile_read(c) for c in ("nearest_tc", "fixup", "norms", "inertia", "bucket", "kmeans_sum", "reseed")}
    ctx.profile(False)
    print(name, {k: round(v[1] / max(1, v[0]) * 1e3, 2) for k, v in out.items() if v[0]})
