"""Single-query search latency through the C ABI (pqg_index_search, host
buffers) on a configs[2]-shaped index (1M items, D=128, M=16, Ks=256, nlist
1024, nprobe 16, k 10), with the per-class device time of one call from the
library's launch profiling.  One JSON line.

  python tools/query_latency.py [--calls 300]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CLASSES = ("adc_scan", "adc_luts", "probe_select", "distance_matrix_tc", "distance_matrix", "big_split",
           "probe", "topk", "norms")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--calls", type=int, default=300)
    ap.add_argument("--nq", type=int, default=1)
    args = ap.parse_args()
    import paper_2604_21645_b200._lib as L
    from paper_2604_21645_b200 import pqii
    rng = np.random.default_rng(2604)
    N, D, M, KS, NL = 1_000_000, 128, 16, 256, 1024
    tables = rng.standard_normal((M, KS, D // M)).astype(np.float32)
    coarse = rng.standard_normal((NL, D)).astype(np.float32)
    lists = np.sort(rng.integers(0, NL, N))
    offsets = np.zeros(NL + 1, np.uint64)
    np.add.at(offsets, lists + 1, 1)
    offsets = np.cumsum(offsets).astype(np.uint64)
    ids = np.arange(N, dtype=np.uint64)
    codes = rng.integers(0, KS, (N, M)).astype(np.uint8)
    ctx = pqii.get_context(0)
    lib, vp = ctx.lib, C.c_void_p
    h = C.c_void_p()
    L.check(lib.pqg_index_create(ctx.h, tables.ctypes.data_as(vp), M, KS, D // M, coarse.ctypes.data_as(vp), NL,
                                 offsets.ctypes.data_as(vp), ids.ctypes.data_as(vp), codes.ctypes.data_as(vp),
                                 C.byref(h)), "create")
    q = rng.standard_normal((args.calls + 1, args.nq, D)).astype(np.float32)
    oi = np.zeros((args.nq, 10), np.uint64)
    od = np.zeros((args.nq, 10), np.float64)
    oc = np.zeros(args.nq, np.uint32)

    def call(i):
        L.check(lib.pqg_index_search(ctx.h, h, q[i].ctypes.data_as(vp), args.nq, 10, 16, 0, 0.0,
                                     oi.ctypes.data_as(vp), od.ctypes.data_as(vp), oc.ctypes.data_as(vp)), "search")
    call(0)
    t0 = time.perf_counter()
    for i in range(1, args.calls + 1):
        call(i)
    per = (time.perf_counter() - t0) / args.calls
    ctx.profile(True)
    l0 = ctx.launches
    call(1)
    launches = ctx.launches - l0
    cls = {}
    for c in CLASSES:
        n, ms = ctx.profile_read(c)
        if n:
            cls[c] = {"launches": n, "us": round(ms * 1e3, 2)}
    ctx.profile(False)
    print(json.dumps({"nq": args.nq, "us_per_call": per * 1e6, "launches_per_call": launches, "classes": cls}))
    lib.pqg_index_destroy(h)


if __name__ == "__main__":
    main()
