"""Pins the C restatement (oracle/pqii_oracle.c) before it is trusted as the
checker: against the golden fixtures written by the compiled reference,
against the compiled reference itself (oracle/_ref) and against the
reference's own known-answer tests."""
import numpy as np
import pytest


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


def test_random_matrix_matches_libstdcxx(golden, orc):
    # proj/tests/test_helpers.cpp:26-33
    assert np.array_equal(bits(orc.random_matrix(120, 8, 57)), bits(golden["random_matrix/120x8_s57"]))


def test_init_draws_match_libstdcxx(golden, orc):
    # proj/src/kmeans.cpp:74-80 (uniform_int_distribution is implementation-defined)
    assert np.array_equal(orc.uniform_indices(1234, 1000, 256), golden["init_draws/seed1234_n1000_k256"])


@pytest.mark.parametrize("name", ["km_rand", "km_1d", "km_dup", "km_mix", "km_mix_tol0", "km_k1"])
def test_kmeans_golden(golden, orc, name):
    k, iters, seed = (int(v) for v in golden[f"{name}/params"])
    tol = float(golden[f"{name}/tol"][0])
    r = orc.kmeans_fit(golden[f"{name}/points"], k, iters, seed, tol)
    assert np.array_equal(bits(r["centroids"]), bits(golden[f"{name}/centroids"]))
    assert np.array_equal(r["assignments"], golden[f"{name}/assignments"])
    assert np.array_equal(bits(r["inertia_per_iter"]), bits(golden[f"{name}/inertia_per_iter"]))
    assert r["iterations_run"] == int(golden[f"{name}/iterations_run"][0])


def test_kmeans_known_answers(orc):
    # proj/tests/test_kmeans.cpp:80-96: {0,1,9,10} -> {0.5, 9.5}, inertia 1.0
    pts = np.array([[0], [1], [9], [10]], np.float32)
    for seed in range(6):
        r = orc.kmeans_fit(pts, 2, 20, seed)
        assert abs(r["inertia"] - 1.0) < 1e-9
        assert sorted(r["centroids"].ravel().tolist()) == [0.5, 9.5]
    # :66-78 two separated points -> inertia 0
    r = orc.kmeans_fit(np.array([[0, 0], [10, 10]], np.float32), 2, 20, 5)
    assert r["inertia"] == 0.0
    # :174-179 duplicates never give non-finite centroids
    r = orc.kmeans_fit(np.full((6, 2), 1.5, np.float32), 3, 10, 0)
    assert r["inertia"] == 0.0 and np.isfinite(r["centroids"]).all()


def test_nearest_known_answers(orc):
    # proj/tests/test_kmeans.cpp:98-112
    table = orc.random_matrix(16, 8, 31)
    idx, dist = orc.nearest_batch(table[3:4], table)
    assert idx[0] == 3 and dist[0] == 0.0
    idx, _ = orc.nearest_batch(np.array([[2.0]], np.float32), np.array([[1.0], [3.0]], np.float32))
    assert idx[0] == 0  # equidistant -> lowest index


def test_pq_golden(golden, orc):
    M, ks, iters, seed = (int(v) for v in golden["pq/params"])
    tables, _, _ = orc.pq_fit(golden["pq/data"], M, ks, iters, seed)
    assert np.array_equal(bits(tables), bits(golden["pq/tables"]))
    codes = orc.pq_encode(golden["pq/data"], tables)
    assert np.array_equal(codes, golden["pq/codes"])
    dec = orc.pq_decode(codes, tables)
    assert np.array_equal(bits(dec), bits(golden["pq/decoded"]))
    assert orc.rmse(golden["pq/data"], dec) == float(golden["pq/rmse"][0])
    # M=1 degenerates to kmeans_fit(seed) bit-for-bit (test_pq.cpp:47-51)
    t1, _, _ = orc.pq_fit(golden["pq_m1/data"], 1, 8, 10, 42)
    assert np.array_equal(bits(t1), bits(golden["pq_m1/tables"]))
    t2, _, _ = orc.pq_fit(golden["pq_m1/data"], 2, 8, 10, 1)
    assert np.array_equal(bits(t2), bits(golden["pq_ds2/tables"]))


def test_pq_wide_codes_golden(golden, orc):
    codes = orc.pq_encode(golden["pq_wide/data"], golden["pq_wide/tables"])
    assert codes.shape[1] == 4  # 2 subspaces x 2 bytes
    assert np.array_equal(codes, golden["pq_wide/codes"])


def test_adc_golden(golden, orc):
    for i, q in enumerate(golden["adc/queries"]):
        t = orc.adc_table(golden["pq/tables"], q)
        assert np.array_equal(bits(t), bits(golden["adc/tables"][i]))
        lk = orc.adc_lookup_all(t, golden["pq/codes"])
        assert np.array_equal(bits(lk), bits(golden["adc/lookup"][i]))


def test_adc_known_answers(orc):
    # proj/tests/test_pq.cpp:163-214: (1-3)^2 == 4.0f
    tables = np.array([[[3.0]], [[0.0]]], np.float32).reshape(2, 1, 1)
    t = orc.adc_table(tables, np.array([1.0, 0.0], np.float32))
    assert t[0, 0] == 4.0 and t[1, 0] == 0.0


def test_ivf_golden(golden, orc):
    off, lid, lcodes = orc.ivf_build_with_centroids(golden["pq/codes"], golden["ivf/ids"],
                                                    golden["pq/tables"], golden["ivf/coarse"])
    assert np.array_equal(off, golden["ivf/offsets"])
    assert np.array_equal(lid, golden["ivf/list_ids"])
    assert np.array_equal(lcodes, golden["ivf/list_codes"])
    for nprobe in (1, 4, 40):
        for qi, q in enumerate(golden["ivf/queries"]):
            ids, dist = orc.ivf_query(golden["pq/tables"], golden["ivf/coarse"], off, lid, lcodes,
                                      q, 10, nprobe)
            c = int(golden[f"ivf/q_np{nprobe}_count"][qi])
            assert len(ids) == c
            assert np.array_equal(ids, golden[f"ivf/q_np{nprobe}_ids"][qi, :c])
            assert np.array_equal(bits(dist), bits(golden[f"ivf/q_np{nprobe}_dist"][qi, :c]))
    for qi, q in enumerate(golden["ivf/queries"]):
        ids, dist = orc.ivf_query(golden["pq/tables"], golden["ivf/coarse"], off, lid, lcodes,
                                  q, 10, 4, max_sq_dist=60.0)
        c = int(golden["ivf/q_max_count"][qi])
        assert np.array_equal(ids, golden["ivf/q_max_ids"][qi, :c])
        fi, fd = orc.flat_scan(golden["pq/tables"], golden["pq/codes"], golden["ivf/ids"], q, 10)
        assert np.array_equal(fi, golden["ivf/flat_ids"][qi])
        assert np.array_equal(bits(fd), bits(golden["ivf/flat_dist"][qi]))


def test_chunk_rows_golden(golden, orc):
    assert np.array_equal(orc.chunk_rows(10, 3), golden["chunk_rows/10_3"])


# --- live comparison against the compiled reference (oracle/_ref) -----------

@pytest.mark.parametrize("seed", [0, 3, 77])
def test_oracle_vs_ref_kmeans_random(orc, ref, seed):
    rng = np.random.default_rng(seed)
    n, d = int(rng.integers(50, 400)), int(rng.integers(1, 9))
    k = int(rng.integers(1, min(40, n)))
    pts = orc.random_matrix(n, d, seed + 100)
    a = orc.kmeans_fit(pts, k, 25, seed, 0.0)
    b = ref.kmeans_fit(pts, k, 25, seed, 0.0)
    assert np.array_equal(bits(a["centroids"]), bits(b["centroids"]))
    assert np.array_equal(a["assignments"], b["assignments"])
    assert np.array_equal(bits(a["inertia_per_iter"]), bits(b["inertia_per_iter"]))


def test_oracle_vs_ref_ivf_query(orc, ref, golden):
    h = ref.ivf_build_with_centroids(golden["pq/codes"], golden["ivf/ids"], golden["pq/tables"],
                                     golden["ivf/coarse"])
    off, lid, lcodes, _ = h.export()
    qs = golden["ivf/queries"]
    ri, rd, rc = h.query_batch(qs, 7, 9)
    for qi, q in enumerate(qs):
        ids, dist = orc.ivf_query(golden["pq/tables"], golden["ivf/coarse"], off, lid, lcodes,
                                  q, 7, 9)
        assert np.array_equal(ids, ri[qi, : rc[qi]])
        assert np.array_equal(bits(dist), bits(rd[qi, : rc[qi]]))


def test_ivf_query_subset_golden(golden, orc):
    off, lid, lcodes = golden["ivf/offsets"], golden["ivf/list_ids"], golden["ivf/list_codes"]
    for qi, q in enumerate(golden["ivf/queries"]):
        ids, dist = orc.ivf_query_subset(golden["pq/tables"], golden["ivf/coarse"], off, lid, lcodes,
                                         q, 10, golden["ivf/subset"], 6)
        c = int(golden["ivf/q_sub_count"][qi])
        assert np.array_equal(ids, golden["ivf/q_sub_ids"][qi, :c])
        assert np.array_equal(bits(dist), bits(golden["ivf/q_sub_dist"][qi, :c]))


# ---------------------------------------------------------------------------
# the chunked pipeline (proj/src/pipeline.cpp:84-266)
# ---------------------------------------------------------------------------
PIPE_MODES = ("single", "parallel_pq", "parallel_pq_index")


@pytest.mark.parametrize("case", ["pipe", "pipe_dup"])
def test_pipeline_golden(golden, orc, case):
    C_, M, ks, nl, it, sd = (int(v) for v in golden[f"{case}/params"])
    data = golden[f"{case}/data"]
    bounds = orc.chunk_rows(data.shape[0], C_)
    local = [orc.train_chunk(data[bounds[c]:bounds[c + 1]], M, ks, it, sd + c)[1]
             for c in range(C_)]
    assert np.array_equal(bits(np.array(local)), bits(golden[f"{case}/local_rmse"]))
    for mode in PIPE_MODES:
        key = f"{case}/{mode}"
        r = orc.run_pipeline(data, C_, M, ks, nl, it, sd, mode)
        assert np.array_equal(bits(r["tables"]), bits(golden[f"{key}/tables"])), mode
        assert r["rmse"] == golden[f"{key}/rmse"][0], mode
        assert r["nlist"] == golden[f"{key}/nlist"][0]
        for extra in ("representatives", "offsets", "list_ids", "list_codes", "coarse"):
            if f"{key}/{extra}" in golden:
                assert np.array_equal(r[extra], golden[f"{key}/{extra}"]), (mode, extra)


def test_oracle_vs_ref_pipeline(orc, ref):
    from paper_2604_21645_b200.datagen import gaussian_mixture
    data = gaussian_mixture(1207, 12, 9, 31)
    for mode in PIPE_MODES:
        a = orc.run_pipeline(data, 4, 3, 32, 0, 7, 11, mode)
        b = ref.run_pipeline(data, 4, 3, 32, 0, 7, 11, mode, threads=2)
        assert np.array_equal(a["tables"], b["tables"]) and a["rmse"] == b["rmse"]
        if mode == "parallel_pq_index":
            assert np.array_equal(a["list_ids"], b["list_ids"])
            assert np.array_equal(a["offsets"], b["offsets"])


# ---------------------------------------------------------------------------
# The threaded checkers used at BASELINE sizes (tests/config_parity.py) are
# bit-identical to the single-threaded reference for every thread count.
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("threads", [1, 3, 8])
def test_threaded_kmeans_equals_reference(orc, ref, threads):
    from paper_2604_21645_b200.datagen import gaussian_mixture
    x = gaussian_mixture(6000, 24, 16, seed=11)
    a = orc.kmeans_fit(x, 50, 12, 7, threads=threads)
    b = ref.kmeans_fit(x, 50, 12, 7)
    assert np.array_equal(a["centroids"].view(np.uint32), b["centroids"].view(np.uint32))
    assert np.array_equal(a["assignments"], b["assignments"])
    assert a["iterations_run"] == b["iterations_run"]
    assert np.array_equal(a["inertia_per_iter"].view(np.uint64), b["inertia_per_iter"].view(np.uint64))


def test_threaded_kmeans_reseed_equals_reference(orc, ref):
    # identical points force empty clusters and reseeds (test_kmeans.cpp:174-179)
    x = np.repeat(ref.random_matrix(40, 3, 5), 25, axis=0)
    a = orc.kmeans_fit(x, 60, 6, 3, threads=4)
    b = ref.kmeans_fit(x, 60, 6, 3)
    assert np.array_equal(a["centroids"].view(np.uint32), b["centroids"].view(np.uint32))
    assert np.array_equal(a["assignments"], b["assignments"])


def test_lloyd_update_is_one_reference_step(orc, ref):
    """fit(t+1)'s centroids == update(fit(t)'s assignment pass) -- the sampled
    protocol's step check (config_parity.lloyd_step_*)."""
    from paper_2604_21645_b200.datagen import gaussian_mixture
    x = gaussian_mixture(5000, 16, 8, seed=3)
    for t in (1, 2, 4):
        ft = ref.kmeans_fit(x, 40, t, 9, tol=0.0)
        ft1 = ref.kmeans_fit(x, 40, t + 1, 9, tol=0.0)
        idx, dist = ref.nearest_batch(x, ft["centroids"])
        assert np.array_equal(idx, ft["assignments"])
        new, _ = orc.lloyd_update(x, idx, dist, ft["centroids"])
        assert np.array_equal(new.view(np.uint32), ft1["centroids"].view(np.uint32))


def test_threaded_reference_entry_points(orc, ref):
    """pq_fit_stats (subspace fits on threads), nearest_batch_mt, threaded
    ivf_build (chunk builds + ivf_merge) and threaded queries equal the
    single-threaded reference calls."""
    from paper_2604_21645_b200.datagen import gaussian_mixture
    x = gaussian_mixture(4000, 32, 16, seed=21)
    tables, iters, per = ref.pq_fit_stats(x, 4, 32, 8, 5, threads=4)
    assert np.array_equal(tables.view(np.uint32), ref.pq_fit(x, 4, 32, 8, 5).view(np.uint32))
    for m in range(4):
        km = ref.kmeans_fit(np.ascontiguousarray(x[:, 8 * m:8 * m + 8]), 32, 8, 5 + m)
        assert iters[m] == km["iterations_run"]
        assert np.array_equal(per[m, : iters[m]], km["inertia_per_iter"])
    i1, d1 = ref.nearest_batch_mt(x, x[:50].copy(), 5)
    i0, d0 = ref.nearest_batch(x, x[:50].copy())
    assert np.array_equal(i0, i1) and np.array_equal(d0.view(np.uint64), d1.view(np.uint64))
    codes = ref.pq_encode(x, tables)
    assert np.array_equal(codes, ref.pq_encode(x, tables, threads=3))
    assert np.array_equal(codes, orc.pq_encode_mt(x, tables, 3))
    ids = np.arange(4000, dtype=np.uint64) * 3 + 1
    coarse = x[::200].copy()
    mono = ref.ivf_build_with_centroids(codes, ids, tables, coarse).export()
    par = ref.ivf_build_with_centroids_mt(codes, ids, tables, coarse, 5).export()
    for a, b in zip(mono, par):
        assert np.array_equal(a, b)
    assert np.array_equal(orc.ivf_assign_mt(codes, tables, coarse, 4),
                          orc.ivf_assign(codes, tables, coarse))
    q = gaussian_mixture(30, 32, 16, seed=21, stream=1)
    h = ref.ivf_build_with_centroids(codes, ids, tables, coarse)
    ri, rd, rc = h.query_batch(q, 7, 4, threads=4)
    oi, od, oc = orc.ivf_query_mt(tables, coarse, *mono[:3], q, 7, 4, 3)
    assert np.array_equal(ri, oi) and np.array_equal(rd.view(np.uint64), od.view(np.uint64))
    assert np.array_equal(rc, oc)
    po = orc.probe_order_mt(coarse, q, 5, 3)
    for j in range(q.shape[0]):
        assert np.array_equal(po[j], orc.probe_order(coarse, q[j], 5))
