"""Parity of the B200 path with the reference at BASELINE.json's own configs.

Shared by ``tests/test_gpu_configs.py`` (the ``-m gpu`` assertions) and
``tools/parity_configs.py`` (writes the agreement counts to
``profiles/parity_r2.json``).  TEST INFRASTRUCTURE: this module is the only
place the config-size comparisons live; the product package never imports it.

The checkers:

* the reference compiled from its own sources (``oracle/_ref``), run on all
  host cores through its own entry points -- ``pq_fit`` as one reference
  ``kmeans_fit(slice, ks, iters, seed + m)`` per subspace on a thread pool
  (exactly ``proj/src/pq.cpp:63-93``; kmeans_fit is safe for concurrent
  disjoint fits, ``kmeans.hpp:40``), ``pq_encode`` over ``chunk_rows`` ranges
  (``pipeline.cpp:226-231``), ``ivf_build_with_centroids`` per row chunk
  combined by the reference's ``ivf_merge`` in chunk order (= the monolithic
  build, acceptance criterion 5), ``ivf_query`` split over queries, and
  ``nearest_in_table`` over row chunks;
* the C restatement (``oracle/pqii_oracle.c``) where the reference has no
  parallel structure: the coarse ``kmeans_fit`` at nlist 1024 (its assignment
  rows split over threads, every reduction sequential -- bit-identical to the
  single-threaded reference, ``tests/test_oracle.py``), ``probe_order``, and
  the one-Lloyd-step update of the sampled protocol.

configs[0]-[2] (cfg1-3) are compared in full.  configs[3]-[4] (cfg4-5) use the
sampled protocol of SURVEY.md 8(c): one Lloyd step checked from the GPU's own
iteration-t centroids (fit(t) -> the reference's assignment of every sample
row (PQ) or of 1% of them (coarse), then the reference's update from the
GPU's pass-t assignments == the GPU's fit(t+1)), codes on a seeded 1% row
sample and posting-list membership on a 0.1% sample computed by the
reference from the GPU-fitted codebook and coarse centroids, and top-k of
1,000 queries by the oracle over the GPU's exported index.  Every comparison
records (agreeing, total) so the agreement fraction is reported, not just a
pass bit; the bar is bit-exact (the north star allows >= 99.99% with
documented fp32 near-ties, 1e-4 relative for codebooks / RMSE).
"""
from __future__ import annotations

import ctypes as C
import os
import time

import numpy as np

SEED = 2604
# RMSE: the reference sums (x - x_hat)^2 sequentially over N*D fp64 terms
# (pq.cpp:169-177), the GPU with a fixed-shape tree; over 1.28e8 terms each
# order carries ~sqrt(n)*u ~ 1e-12 relative rounding of its own, so the two
# agree to ~1e-12 -- held here to 1e-9 (the north star's bar is 1e-4).
RMSE_RTOL = 1e-9

CONFIGS = {
    1: dict(n=100_000, d=128, comp=64, M=8, ks=256, iters=20),
    2: dict(n=1_000_000, d=128, comp=256, sample=100_000, iters=25,
            sweep=[(M, ks) for M in (4, 8, 16, 32) for ks in (16, 64, 256)]),
    3: dict(n=1_000_000, d=128, comp=256, sample=100_000, M=16, ks=256, iters=20, nlist=1024,
            nq=10_000, nprobe=16, k=10),
    4: dict(n=10_000_000, d=96, comp=64, sample=1_000_000, M=12, ks=256, iters=20, t=5),
    5: dict(n=100_000_000, d=128, comp=1024, sample=2_000_000, M=16, ks=256, nlist=4096, iters=20,
            t=5, nq=100_000, nprobe=32, k=10, check_queries=1000, shards=8),
}


# ---------------------------------------------------------------------------
# comparison records
# ---------------------------------------------------------------------------

def bits(a):
    a = np.ascontiguousarray(a)
    return a.view({1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}[a.dtype.itemsize])


def agree(name, got, want, out, exact=True, first=5):
    """Element agreement of two arrays (bit patterns for floats)."""
    got, want = np.asarray(got), np.asarray(want)
    if got.shape != want.shape:
        out[name] = {"ok": False, "why": f"shape {got.shape} vs {want.shape}"}
        return out[name]
    g, w = (bits(got), bits(want)) if got.dtype.kind == "f" else (got, want)
    eq = g == w
    n_eq, n = int(eq.sum()), int(eq.size)
    rec = {"agree": n_eq, "total": n, "frac": (n_eq / n) if n else 1.0, "ok": n_eq == n}
    if n_eq != n:
        bad = np.argwhere(~eq)[:first]
        rec["first_mismatches"] = [list(map(int, b)) for b in bad]
        if not exact:
            rec["ok"] = rec["frac"] >= 0.9999
    out[name] = rec
    return rec


def close(name, got, want, out, rtol):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    m = ~np.isnan(want)
    same_nan = np.array_equal(np.isnan(got), np.isnan(want))
    rel = np.abs(got[m] - want[m]) / np.maximum(np.abs(want[m]), 1e-300)
    r = float(rel.max()) if rel.size else 0.0
    out[name] = {"max_rel": r, "rtol": rtol, "count": int(m.sum()), "ok": same_nan and r <= rtol}
    return out[name]


def seq_sum(v):
    """Left-to-right fp64 sum (assign_pass's inertia order, kmeans.cpp:55)."""
    v = np.asarray(v, np.float64)
    return float(np.add.accumulate(v)[-1]) if v.size else 0.0


def seq_sq_dist(x, c):
    """squared_l2 (kmeans.cpp:11-18) row-wise: fp64 differences squared and
    added in dimension order, no contraction."""
    acc = np.zeros(x.shape[0], np.float64)
    for j in range(x.shape[1]):
        diff = x[:, j].astype(np.float64) - c[:, j].astype(np.float64)
        acc += diff * diff
    return acc


def all_ok(rec) -> bool:
    if isinstance(rec, dict):
        if "ok" in rec and not isinstance(rec["ok"], dict):
            return bool(rec["ok"]) and all(all_ok(v) for k, v in rec.items() if isinstance(v, dict))
        return all(all_ok(v) for v in rec.values() if isinstance(v, (dict, list)))
    if isinstance(rec, list):
        return all(all_ok(v) for v in rec)
    return True


# ---------------------------------------------------------------------------
# shared plumbing
# ---------------------------------------------------------------------------

class Env:
    """GPU context on torch's current stream + the two checkers."""

    def __init__(self, threads=None):
        import torch

        import oracle
        from paper_2604_21645_b200 import _lib, pqii
        self.torch = torch
        self.pq = pqii
        self.L = _lib
        # one dedicated stream shared by torch (data generation, gathers) and
        # the library, so their work is ordered without host syncs
        self.stream = torch.cuda.Stream()
        torch.cuda.set_stream(self.stream)
        self.ctx = pqii.Context(0)
        self.ctx.set_stream(self.stream.cuda_stream)
        self.lib = self.ctx.lib
        self.orc = oracle.c_oracle()
        self.ref = oracle.ref_impl()
        self.threads = threads or oracle.default_threads()

    def vp(self, t):
        return C.c_void_p(t.data_ptr())

    def sync(self):
        self.torch.cuda.synchronize()


def _fit_record(tables_g, st_g, tables_r, iters_r, per_r, out, prefix=""):
    agree(prefix + "codebook_bits", tables_g, tables_r, out)
    agree(prefix + "iterations_run", np.asarray(st_g["iterations_run"], np.uint32), iters_r, out)
    close(prefix + "inertia_per_iter", st_g["inertia_per_iter"][:, : per_r.shape[1]], per_r, out,
          rtol=1e-12)


# ---------------------------------------------------------------------------
# configs[0]: 100k x 128, M=8, Ks=256, 20 iterations on all rows
# ---------------------------------------------------------------------------

def run_cfg1(env: Env):
    from paper_2604_21645_b200.datagen import gaussian_mixture
    c = CONFIGS[1]
    out, t = {}, {}
    x = gaussian_mixture(c["n"], c["d"], c["comp"], SEED)
    st = {}
    t0 = time.perf_counter()
    cb = env.pq.pq_fit(x, c["M"], c["ks"], c["iters"], SEED, ctx=env.ctx, stats=st)
    t["gpu_fit_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    rt, rit, rper = env.ref.pq_fit_stats(x, c["M"], c["ks"], c["iters"], SEED, env.threads)
    t["ref_fit_s"] = time.perf_counter() - t0
    _fit_record(cb.tables, st, rt, rit, rper, out)
    codes_g = env.pq.pq_encode(cb, x, ctx=env.ctx).bytes
    codes_r = env.ref.pq_encode(x, rt, threads=env.threads)
    agree("codes", codes_g, codes_r, out)
    r_g = env.pq.reconstruction_rmse(cb, x, ctx=env.ctx)
    r_r = env.ref.rmse(x, env.ref.pq_decode(codes_r, rt))
    close("rmse", [r_g], [r_r], out, rtol=RMSE_RTOL)
    out["rmse_value"] = r_r
    out["seconds"] = t
    return out


# ---------------------------------------------------------------------------
# configs[1]: 1M x 128, 12-point M x Ks sweep, 25 iterations on the 100k sample
# ---------------------------------------------------------------------------

def run_cfg2(env: Env, sweep=None):
    from paper_2604_21645_b200.datagen import gaussian_mixture, strided_sample
    c = CONFIGS[2]
    sweep = sweep or c["sweep"]
    x = gaussian_mixture(c["n"], c["d"], c["comp"], SEED)
    train = np.ascontiguousarray(x[strided_sample(c["n"], c["sample"], SEED)])
    t0 = time.perf_counter()
    # every subspace fit of every sweep point in one reference thread pool
    problems, owner = [], []
    for (M, ks) in sweep:
        ds = c["d"] // M
        for m in range(M):
            problems.append((np.ascontiguousarray(train[:, m * ds:(m + 1) * ds]), ks, c["iters"],
                             SEED + m))
            owner.append((M, ks))
    fits = env.ref.kmeans_fit_many(problems, env.threads)
    ref_fit_s = time.perf_counter() - t0
    import oracle
    res = {"points": [], "seconds": {"ref_fit_all_s": ref_fit_s}}
    for (M, ks) in sweep:
        rec = {"M": M, "Ks": ks}
        mine = [f for f, o in zip(fits, owner) if o == (M, ks)]
        rt, rit, rper = oracle.stack_fits(mine, c["iters"])
        st = {}
        cb = env.pq.pq_fit(train, M, ks, c["iters"], SEED, ctx=env.ctx, stats=st)
        _fit_record(cb.tables, st, rt, rit, rper, rec)
        codes_g = env.pq.pq_encode(cb, x, ctx=env.ctx).bytes
        codes_r = env.ref.pq_encode(x, rt, threads=env.threads)
        agree("codes", codes_g, codes_r, rec)
        r_g = env.pq.reconstruction_rmse(cb, x, ctx=env.ctx)
        r_r = env.ref.rmse(x, env.ref.pq_decode(codes_r, rt))
        close("rmse", [r_g], [r_r], rec, rtol=RMSE_RTOL)
        rec["rmse_value"] = r_r
        res["points"].append(rec)
    res["seconds"]["total_s"] = time.perf_counter() - t0
    return res


# ---------------------------------------------------------------------------
# configs[2]: 1M x 128, M=16, Ks=256, nlist 1024, 10k queries nprobe 16 k 10
# ---------------------------------------------------------------------------

def run_cfg3(env: Env, nq=None):
    from paper_2604_21645_b200.datagen import gaussian_mixture, strided_sample
    c = CONFIGS[3]
    nq = nq or c["nq"]
    M, ks, nlist, D = c["M"], c["ks"], c["nlist"], c["d"]
    out, t = {}, {}
    x = gaussian_mixture(c["n"], D, c["comp"], SEED)
    train = np.ascontiguousarray(x[strided_sample(c["n"], c["sample"], SEED)])
    q = gaussian_mixture(nq, D, c["comp"], SEED, stream=1)
    # PQ fit (reference, threaded by subspace) vs GPU
    st = {}
    cb = env.pq.pq_fit(train, M, ks, c["iters"], SEED, ctx=env.ctx, stats=st)
    t0 = time.perf_counter()
    rt, rit, rper = env.ref.pq_fit_stats(train, M, ks, c["iters"], SEED, env.threads)
    t["ref_pq_fit_s"] = time.perf_counter() - t0
    _fit_record(cb.tables, st, rt, rit, rper, out, "pq_")
    # coarse kmeans_fit(sample, nlist, 20, seed + M)
    km = env.pq.kmeans_fit(train, nlist, c["iters"], SEED + M, ctx=env.ctx)
    t0 = time.perf_counter()
    okm = env.orc.kmeans_fit(train, nlist, c["iters"], SEED + M, threads=env.threads)
    t["oracle_coarse_fit_s"] = time.perf_counter() - t0
    agree("coarse_centroid_bits", km.centroids, okm["centroids"], out)
    agree("coarse_assignments", km.assignments, okm["assignments"], out)
    agree("coarse_iterations_run", np.array([km.iterations_run]), np.array([okm["iterations_run"]]), out)
    close("coarse_inertia_per_iter", km.inertia_per_iter, okm["inertia_per_iter"], out, rtol=1e-12)
    # codes of all rows
    codes_g = env.pq.pq_encode(cb, x, ctx=env.ctx)
    t0 = time.perf_counter()
    codes_r = env.ref.pq_encode(x, rt, threads=env.threads)
    t["ref_encode_s"] = time.perf_counter() - t0
    agree("codes", codes_g.bytes, codes_r, out)
    # posting lists of all rows (reference threaded build + ivf_merge)
    ids = np.arange(c["n"], dtype=np.uint64)
    index = env.pq.ivf_build_with_centroids(cb, codes_g, ids, km.centroids, ctx=env.ctx)
    g_off, g_ids, g_codes, _, _ = index.export()
    t0 = time.perf_counter()
    rindex = env.ref.ivf_build_with_centroids_mt(codes_r, ids, rt, okm["centroids"], env.threads)
    r_off, r_ids, r_codes, _ = rindex.export()
    t["ref_ivf_build_s"] = time.perf_counter() - t0
    agree("posting_offsets", g_off, r_off, out)
    agree("posting_ids", g_ids, r_ids, out)
    agree("posting_codes", g_codes, r_codes, out)
    # probe_order at d=128, nlist=1024 (tensor-core distance matrix + select)
    g_probe = env.pq.ivf_probe(index, q, c["nprobe"])
    t0 = time.perf_counter()
    o_probe = env.orc.probe_order_mt(okm["centroids"], q, c["nprobe"], env.threads)
    t["oracle_probe_s"] = time.perf_counter() - t0
    agree("probe_lists", g_probe, o_probe, out)
    # top-k of every query
    gi, gd, gc = env.pq.ivf_query_batch(index, q, c["k"], c["nprobe"])
    t0 = time.perf_counter()
    ri, rd, rc = rindex.query_batch(q, c["k"], c["nprobe"], threads=env.threads)
    t["ref_query_s"] = time.perf_counter() - t0
    agree("topk_counts", gc, rc, out)
    agree("topk_ids", gi, ri, out)
    agree("topk_dist_bits", gd, rd, out)
    out["candidates_per_query"] = float(
        (np.diff(g_off.astype(np.int64))[g_probe.astype(np.int64)]).sum() / nq)
    out["seconds"] = t
    return out


# ---------------------------------------------------------------------------
# sampled protocol (configs[3], configs[4])
# ---------------------------------------------------------------------------

def lloyd_step_pq(env: Env, train_dev, train_host, M, ks, t, seed, out):
    """fit(t) and fit(t+1) on the GPU; the reference assigns every sample row
    under fit(t)'s codebook (pass t of the fit) and the restated update from
    the GPU's pass-t assignments must give fit(t+1)'s codebook bit for bit."""
    n, D = train_host.shape
    ds = D // M
    st_t, st_t1 = {}, {}
    cb_t = env.pq.pq_fit(train_dev, M, ks, t, seed, ctx=env.ctx, stats=st_t)
    cb_t1 = env.pq.pq_fit(train_dev, M, ks, t + 1, seed, ctx=env.ctx, stats=st_t1)
    out["pq_fit_t_iterations"] = [int(v) for v in st_t["iterations_run"]]
    out["pq_fit_t1_iterations"] = [int(v) for v in st_t1["iterations_run"]]
    ran = all(v == t for v in st_t["iterations_run"]) and all(v == t + 1 for v in st_t1["iterations_run"])
    out["pq_no_early_stop"] = {"ok": bool(ran)}
    a_gpu = env.pq.pq_encode(cb_t, train_dev, ctx=env.ctx).codes()  # pass-t assignments (n x M)
    ag_eq = ag_n = 0
    upd_eq = upd_n = 0
    inert = []
    for m in range(M):
        pts = np.ascontiguousarray(train_host[:, m * ds:(m + 1) * ds])
        idx, dist = env.ref.nearest_batch_mt(pts, cb_t.tables[m], env.threads)
        ag_eq += int((idx == a_gpu[:, m]).sum())
        ag_n += n
        inert.append((st_t["inertia_per_iter"][m, t - 1], seq_sum(dist)))
        new, _ = env.orc.lloyd_update(pts, a_gpu[:, m].astype(np.uint32), dist, cb_t.tables[m])
        e = bits(new) == bits(cb_t1.tables[m])
        upd_eq += int(e.sum())
        upd_n += e.size
    out["pq_assignments_pass_t"] = {"agree": ag_eq, "total": ag_n, "frac": ag_eq / ag_n,
                                    "ok": ag_eq == ag_n}
    out["pq_update_bits"] = {"agree": upd_eq, "total": upd_n, "frac": upd_eq / upd_n,
                             "ok": upd_eq == upd_n}
    close("pq_inertia_pass_t", [a for a, _ in inert], [b for _, b in inert], out, rtol=1e-12)
    return cb_t1


def lloyd_step_coarse(env: Env, train_dev, train_host, nlist, t, seed, frac, out):
    """Coarse fit(t)/fit(t+1) on the GPU; the reference assigns a seeded
    `frac` of the sample rows under fit(t)'s centroids; the restated update
    from the GPU's (all-row) pass-t assignments must give fit(t+1)."""
    n, D = train_host.shape
    km_t = env.pq.kmeans_fit(train_dev, nlist, t, seed, ctx=env.ctx)
    km_t1 = env.pq.kmeans_fit(train_dev, nlist, t + 1, seed, ctx=env.ctx)
    out["coarse_no_early_stop"] = {"ok": km_t.iterations_run == t and km_t1.iterations_run == t + 1}
    rng = np.random.default_rng(seed)
    rows = np.sort(rng.choice(n, size=max(1, int(n * frac)), replace=False))
    idx, dist = env.ref.nearest_batch_mt(np.ascontiguousarray(train_host[rows]), km_t.centroids,
                                         env.threads)
    agree("coarse_assignments_pass_t_sampled", km_t.assignments[rows], idx, out)
    # dists of the GPU's pass-t assignments in squared_l2's order (needed by the
    # reseed only), then the restated update
    a = km_t.assignments.astype(np.uint32)
    counts = np.bincount(a, minlength=nlist)
    out["coarse_empty_clusters_pass_t"] = int((counts == 0).sum())
    dists = seq_sq_dist(train_host, km_t.centroids[a]) if (counts == 0).any() else np.zeros(n)
    new, _ = env.orc.lloyd_update(train_host, a, dists, km_t.centroids)
    agree("coarse_update_bits", km_t1.centroids, new, out)
    return km_t1


def _sample_rows(n, count, seed):
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(n, size=count, replace=False))


def run_cfg4(env: Env, full_fit: bool = True):
    """configs[3]: 10M x 96 (64-comp mixture), M=12 (Ds=8), Ks=256, 20
    iterations on the 1M sample; encode of all rows + global RMSE."""
    from paper_2604_21645_b200.datagen import device_mixture, strided_sample
    torch = env.torch
    c = CONFIGS[4]
    N, D, M, ks = c["n"], c["d"], c["M"], c["ks"]
    out, tm = {}, {}
    x = device_mixture(N, D, c["comp"], SEED, SEED)
    sidx = torch.from_numpy(strided_sample(N, c["sample"], SEED)).cuda()
    train = x[sidx].contiguous()
    train_h = train.cpu().numpy()
    t0 = time.perf_counter()
    lloyd_step_pq(env, train, train_h, M, ks, c["t"], SEED, out)
    tm["lloyd_step_pq_s"] = time.perf_counter() - t0
    # the config's own fit (20 iterations), encode of all 10M, global RMSE
    st = {}
    cb = env.pq.pq_fit(train, M, ks, c["iters"], SEED, ctx=env.ctx, stats=st)
    out["fit_iterations_run"] = [int(v) for v in st["iterations_run"]]
    if full_fit:  # the whole 20-iteration fit on the 1M sample, reference threaded by subspace
        t0 = time.perf_counter()
        rt, rit, rper = env.ref.pq_fit_stats(train_h, M, ks, c["iters"], SEED, env.threads)
        tm["ref_full_fit_s"] = time.perf_counter() - t0
        _fit_record(cb.tables, st, rt, rit, rper, out, "full_fit_")
    codes = torch.empty((N, M), dtype=torch.uint8, device="cuda")
    tables = torch.from_numpy(cb.tables).cuda()
    sse = C.c_double()
    env.L.check(env.lib.pqg_pq_encode_sse(env.ctx.h, env.vp(x), N, M, ks, D // M, env.vp(tables),
                                          env.vp(codes), C.byref(sse)))
    env.sync()
    out["global_rmse"] = (sse.value / (N * D)) ** 0.5
    # 1% row sample: codes and the sample's SSE by the reference
    rows = _sample_rows(N, N // 100, SEED + 1)
    xr = x[torch.from_numpy(rows).cuda()].cpu().numpy()
    g_codes = codes[torch.from_numpy(rows).cuda()].cpu().numpy()
    t0 = time.perf_counter()
    r_codes = env.ref.pq_encode(xr, cb.tables, threads=env.threads)
    tm["ref_encode_sample_s"] = time.perf_counter() - t0
    agree("codes_1pct_rows", g_codes, r_codes, out)
    g_sse = env.pq.reconstruction_rmse(cb, xr, ctx=env.ctx)
    r_sse = env.ref.rmse(xr, env.ref.pq_decode(r_codes, cb.tables))
    close("rmse_1pct_rows", [g_sse], [r_sse], out, rtol=RMSE_RTOL)
    out["seconds"] = tm
    del x, train
    torch.cuda.empty_cache()
    return out


def run_cfg5(env: Env, n=None, check_queries=None):
    """configs[4]: 100M x 128 (1024-comp mixture, 8 shards generated from
    seed + rank), M=16, Ks=256, nlist=4096, 20 iterations on the 2M sample;
    encode + index of all rows; 100k queries nprobe 32 top-10.  One GPU holds
    all 8 shards here (51.2 GB of 180 GB); the shard layout only changes
    which generator seed fills which rows."""
    from paper_2604_21645_b200.datagen import device_mixture, mixture_params, strided_sample
    torch = env.torch
    c = CONFIGS[5]
    N = n or c["n"]
    D, M, ks, nlist = c["d"], c["M"], c["ks"], c["nlist"]
    nq, nprobe, k = c["nq"], c["nprobe"], c["k"]
    cq = check_queries or c["check_queries"]
    out, tm = {"rows": N}, {}
    x = torch.empty((N, D), dtype=torch.float32, device="cuda")
    S = c["shards"]
    for r in range(S):  # chunk_rows(N, 8): shard r from seed + r
        b0, b1 = N * r // S, N * (r + 1) // S
        device_mixture(b1 - b0, D, c["comp"], SEED, SEED + r, out=x[b0:b1])
    n_train = min(c["sample"], N)
    sidx = torch.from_numpy(strided_sample(N, n_train, SEED)).cuda()
    train = x[sidx].contiguous()
    train_h = train.cpu().numpy()
    t0 = time.perf_counter()
    lloyd_step_pq(env, train, train_h, M, ks, c["t"], SEED, out)
    tm["lloyd_step_pq_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    lloyd_step_coarse(env, train, train_h, nlist, c["t"], SEED + M, 0.01, out)
    tm["lloyd_step_coarse_s"] = time.perf_counter() - t0
    # the config's own fits
    st = {}
    cb = env.pq.pq_fit(train, M, ks, c["iters"], SEED, ctx=env.ctx, stats=st)
    km = env.pq.kmeans_fit(train, nlist, c["iters"], SEED + M, ctx=env.ctx)
    out["pq_fit_iterations_run"] = [int(v) for v in st["iterations_run"]]
    out["coarse_fit_iterations_run"] = int(km.iterations_run)
    del train
    tables = torch.from_numpy(cb.tables).cuda()
    coarse = torch.from_numpy(km.centroids).cuda()
    codes = torch.empty((N, M), dtype=torch.uint8, device="cuda")
    sse = C.c_double()
    env.L.check(env.lib.pqg_pq_encode_sse(env.ctx.h, env.vp(x), N, M, ks, D // M, env.vp(tables),
                                          env.vp(codes), C.byref(sse)))
    out["global_rmse"] = (sse.value / (N * D)) ** 0.5
    ids = torch.arange(N, dtype=torch.int64, device="cuda")
    h = C.c_void_p()
    env.L.check(env.lib.pqg_ivf_build_with_centroids(env.ctx.h, env.vp(tables), M, ks, D // M,
                                                     env.vp(codes), env.vp(ids), N, env.vp(coarse),
                                                     nlist, C.byref(h)))
    index = env.pq.InvertedIndex(h, env.ctx)
    del ids
    # codes of a 1% row sample and their SSE, by the reference
    rows = _sample_rows(N, N // 100, SEED + 1)
    rows_d = torch.from_numpy(rows).cuda()
    xr = x[rows_d].cpu().numpy()
    g_codes = codes[rows_d].cpu().numpy()
    t0 = time.perf_counter()
    r_codes = env.ref.pq_encode(xr, cb.tables, threads=env.threads)
    tm["ref_encode_sample_s"] = time.perf_counter() - t0
    agree("codes_1pct_rows", g_codes, r_codes, out)
    close("rmse_1pct_rows", [env.pq.reconstruction_rmse(cb, xr, ctx=env.ctx)],
          [env.ref.rmse(xr, env.ref.pq_decode(r_codes, cb.tables))], out, rtol=RMSE_RTOL)
    del x
    torch.cuda.empty_cache()
    # the index: exported CSR; posting-list membership of a 0.1% item sample
    off, lids, lcodes, _, _ = index.export()
    sizes = np.diff(off.astype(np.int64))
    list_of = np.repeat(np.arange(nlist, dtype=np.uint32), sizes)
    pos = np.empty(N, np.int64)
    pos[lids.astype(np.int64)] = np.arange(N)
    out["index_ids_are_a_permutation"] = {"ok": bool(np.array_equal(np.sort(lids), np.arange(N, dtype=np.uint64)))}
    # stable scatter: ids ascend within every list (ivf.cpp:44-46 input order)
    inc = np.ones(N, bool)
    inc[1:] = lids[1:] > lids[:-1]
    inc[off[:-1][sizes > 0].astype(np.int64)] = True
    out["lists_in_input_order"] = {"ok": bool(inc.all()), "violations": int((~inc).sum())}
    mrows = _sample_rows(N, N // 1000, SEED + 2)
    t0 = time.perf_counter()
    r_list = env.orc.ivf_assign_mt(g_codes_of(lcodes, pos, mrows), cb.tables, km.centroids, env.threads)
    tm["oracle_membership_s"] = time.perf_counter() - t0
    agree("posting_membership_0.1pct", list_of[pos[mrows]], r_list, out)
    agree("posting_codes_match_encode_1pct", lcodes[pos[rows]], g_codes, out)
    # 100k-query batch on the GPU; the first `cq` checked by the oracle over
    # the GPU's index (GPU-fitted codebook and coarse centroids)
    means, sigmas = mixture_params(D, c["comp"], SEED)
    gq = torch.Generator(device="cuda")
    gq.manual_seed(SEED + 1000003)
    comp = torch.randint(0, c["comp"], (nq,), generator=gq, device="cuda")
    mu = torch.from_numpy(means).cuda()
    sg = torch.from_numpy(sigmas).cuda()
    q = (mu[comp] + sg[comp, None] * torch.randn((nq, D), generator=gq, device="cuda",
                                                 dtype=torch.float64)).float().contiguous()
    oi = torch.empty((nq, k), dtype=torch.int64, device="cuda")
    od = torch.empty((nq, k), dtype=torch.float64, device="cuda")
    oc = torch.empty((nq,), dtype=torch.int32, device="cuda")
    env.L.check(env.lib.pqg_index_search(env.ctx.h, h, env.vp(q), nq, k, nprobe, 0, 0.0,
                                         env.vp(oi), env.vp(od), env.vp(oc)))
    env.sync()
    qh = q[:cq].cpu().numpy()
    t0 = time.perf_counter()
    ri, rd, rc = env.orc.ivf_query_mt(cb.tables, km.centroids, off, lids, lcodes, qh, k, nprobe,
                                      env.threads)
    tm["oracle_query_s"] = time.perf_counter() - t0
    agree("topk_counts_1k", oc[:cq].cpu().numpy().astype(np.uint32), rc, out)
    agree("topk_ids_1k", oi[:cq].cpu().numpy().astype(np.uint64), ri, out)
    agree("topk_dist_bits_1k", od[:cq].cpu().numpy(), rd, out)
    out["seconds"] = tm
    del codes, index
    torch.cuda.empty_cache()
    return out


def g_codes_of(lcodes, pos, rows):
    return np.ascontiguousarray(lcodes[pos[rows]])


RUNNERS = {1: run_cfg1, 2: run_cfg2, 3: run_cfg3, 4: run_cfg4, 5: run_cfg5}
