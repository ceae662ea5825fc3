"""Writes tests/golden/golden.npz from the REFERENCE compiled from its own
sources (oracle/_ref/libpqii_ref.so, built by `make -C oracle` in the
container where /root/reference exists).

Every array in the file is an output of the reference's own functions on a
small seeded input; inputs come from the reference's test helper
random_matrix (proj/tests/test_helpers.cpp:26-33) or from the package's
seeded Gaussian-mixture generator.  The fixtures pin the C restatement
(oracle/pqii_oracle.c) and the CUDA path when oracle/_ref is unavailable.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2604_21645_b200.datagen import gaussian_mixture  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def main() -> None:
    R = oracle.ref_impl()
    g: dict[str, np.ndarray] = {}

    # -- kmeans_fit (proj/src/kmeans.cpp:61-133) --------------------------
    cases = [
        ("km_rand", R.random_matrix(300, 6, 41), 12, 15, 9, 1e-4),       # test_kmeans.cpp:146
        ("km_1d", np.array([[0], [1], [9], [10]], np.float32), 2, 20, 3, 1e-4),  # :80-96
        ("km_dup", np.full((6, 2), 1.5, np.float32), 3, 10, 0, 1e-4),     # :174-179 (empties)
        ("km_mix", gaussian_mixture(3000, 16, 24, 7), 64, 20, 11, 1e-4),
        ("km_mix_tol0", gaussian_mixture(2000, 8, 16, 8), 40, 12, 5, 0.0),
        ("km_k1", R.random_matrix(50, 4, 21), 1, 20, 3, 1e-4),            # :48-64
    ]
    for name, pts, k, iters, seed, tol in cases:
        r = R.kmeans_fit(pts, k, iters, seed, tol)
        g[f"{name}/points"] = pts
        g[f"{name}/params"] = np.array([k, iters, seed], np.uint64)
        g[f"{name}/tol"] = np.array([tol], np.float64)
        g[f"{name}/centroids"] = r["centroids"]
        g[f"{name}/assignments"] = r["assignments"]
        g[f"{name}/inertia_per_iter"] = r["inertia_per_iter"]
        g[f"{name}/iterations_run"] = np.array([r["iterations_run"]], np.uint32)

    # init draws of uniform_int_distribution (proj/src/kmeans.cpp:74-80)
    g["init_draws/seed1234_n1000_k256"] = R.uniform_indices(1234, 1000, 256)

    # random_matrix bytes (proj/tests/test_helpers.cpp:26-33)
    g["random_matrix/120x8_s57"] = R.random_matrix(120, 8, 57)

    # -- pq_fit / encode / decode / rmse (proj/src/pq.cpp) -----------------
    data = gaussian_mixture(2500, 32, 32, 21)
    tables = R.pq_fit(data, 4, 16, 25, 5)
    g["pq/data"] = data
    g["pq/params"] = np.array([4, 16, 25, 5], np.uint64)
    g["pq/tables"] = tables
    codes = R.pq_encode(data, tables)
    g["pq/codes"] = codes
    g["pq/decoded"] = R.pq_decode(codes, tables)
    g["pq/rmse"] = np.array([R.reconstruction_rmse(data, tables)], np.float64)
    small = R.random_matrix(64, 4, 17)
    g["pq_m1/data"] = small
    g["pq_m1/tables"] = R.pq_fit(small, 1, 8, 10, 42)              # test_pq.cpp:47-51
    g["pq_ds2/tables"] = R.pq_fit(small, 2, 8, 10, 1)              # test_pq.cpp:41-46

    # wide codes (Ks > 256 -> 2-byte little-endian codes, pq.hpp:45)
    wide = gaussian_mixture(1200, 8, 16, 4)
    wt = R.pq_fit(wide, 2, 300, 6, 2)
    g["pq_wide/data"] = wide
    g["pq_wide/tables"] = wt
    g["pq_wide/codes"] = R.pq_encode(wide, wt)

    # -- ADC (proj/src/pq.cpp:132-167) ---------------------------------------
    q = gaussian_mixture(5, 32, 32, 21, stream=1)
    g["adc/queries"] = q
    g["adc/tables"] = np.stack([R.adc_table(tables, qi) for qi in q])
    g["adc/lookup"] = np.stack([R.adc_lookup_all(R.adc_table(tables, qi), codes) for qi in q])

    # -- IVF (proj/src/ivf.cpp) ---------------------------------------------
    ids = (np.arange(data.shape[0], dtype=np.uint64) * 7 + 3)
    coarse = R.kmeans_fit(R.pq_decode(codes, tables), 40, 10, 99)["centroids"]
    h = R.ivf_build_with_centroids(codes, ids, tables, coarse)
    off, lid, lcodes, _ = h.export()
    g["ivf/ids"] = ids
    g["ivf/coarse"] = coarse
    g["ivf/offsets"] = off
    g["ivf/list_ids"] = lid
    g["ivf/list_codes"] = lcodes
    qs = gaussian_mixture(25, 32, 32, 21, stream=1)
    g["ivf/queries"] = qs
    for nprobe in (1, 4, 40):
        oi, od, oc = h.query_batch(qs, 10, nprobe)
        g[f"ivf/q_np{nprobe}_ids"] = oi
        g[f"ivf/q_np{nprobe}_dist"] = od
        g[f"ivf/q_np{nprobe}_count"] = oc
    oi, od, oc = h.query_batch(qs, 10, 4, max_sq_dist=60.0)
    g["ivf/q_max_ids"], g["ivf/q_max_dist"], g["ivf/q_max_count"] = oi, od, oc
    subset = ids[::3].copy()  # every third item (sorted ascending)
    sub = [h.query_subset(qi, 10, subset, 6) for qi in qs]
    g["ivf/subset"] = subset
    g["ivf/q_sub_ids"] = np.stack([np.pad(s_[0], (0, 10 - len(s_[0]))) for s_ in sub])
    g["ivf/q_sub_count"] = np.array([len(s_[0]) for s_ in sub], np.uint32)
    g["ivf/q_sub_dist"] = np.stack([np.pad(s_[1], (0, 10 - len(s_[1]))) for s_ in sub])
    fl = [R.flat_scan(tables, codes, ids, qi, 10) for qi in qs]
    g["ivf/flat_ids"] = np.stack([f[0] for f in fl])
    g["ivf/flat_dist"] = np.stack([f[1] for f in fl])

    # ivf_build (coarse k-means over decoded codes, proj/src/ivf.cpp:123-149)
    hb = R.ivf_build(codes[:800], ids[:800], tables, 20, 17, 8)
    boff, bid, bcodes, bcoarse = hb.export()
    g["ivf_build/offsets"], g["ivf_build/list_ids"] = boff, bid
    g["ivf_build/list_codes"], g["ivf_build/coarse"] = bcodes, bcoarse

    # -- the chunked pipeline (proj/src/pipeline.cpp:84-266) -----------------
    # pipe: uneven chunks (3001 = 5 x 600 + 1); pipe_dup: tiny chunks of
    # rounded (duplicate-heavy) rows, so local fits reseed empty clusters.
    pipe_cases = [
        ("pipe", gaussian_mixture(3001, 16, 12, 5), 5, 4, 16, 0, 8, 3),
        ("pipe_dup", np.round(gaussian_mixture(203, 8, 3, 6)), 6, 2, 16, 9, 6, 1),
    ]
    for name, pdata, C_, M_, ks_, nl_, it_, sd_ in pipe_cases:
        g[f"{name}/data"] = pdata.astype(np.float32)
        g[f"{name}/params"] = np.array([C_, M_, ks_, nl_, it_, sd_], np.uint64)
        bounds = R.chunk_rows(pdata.shape[0], C_)
        g[f"{name}/local_rmse"] = np.array(
            [R.train_chunk(pdata[bounds[c]:bounds[c + 1]], M_, ks_, it_, sd_ + c)[1]
             for c in range(C_)])
        for mode in ("single", "parallel_pq", "parallel_pq_index"):
            r = R.run_pipeline(pdata, C_, M_, ks_, nl_, it_, sd_, mode, threads=3)
            key = f"{name}/{mode}"
            g[f"{key}/tables"] = r["tables"]
            g[f"{key}/rmse"] = np.array([r["rmse"]])
            g[f"{key}/nlist"] = np.array([r["nlist"]], np.uint64)
            for extra in ("representatives", "offsets", "list_ids", "list_codes", "coarse"):
                if extra in r:
                    g[f"{key}/{extra}"] = r[extra]

    g["chunk_rows/10_3"] = R.chunk_rows(10, 3)
    g["default_nlist"] = np.array([R.default_nlist(n) for n in (1, 2, 10, 100, 1000, 12345)],
                                  np.uint64)

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes, {len(g)} arrays)")


if __name__ == "__main__":
    main()
