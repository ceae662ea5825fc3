"""Parity of the CUDA path (through the C ABI) with the oracle and the golden
fixtures written by the compiled reference.  Mirrors the reference's own
tests (proj/tests/test_kmeans.cpp, test_pq.cpp, test_ivf.cpp); every
comparison is bit-exact unless the reference itself only promises a
tolerance (inertia / RMSE sums, whose fp64 summation order differs:
<= 1e-12 relative here, BASELINE.json allows 1e-4)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view({4: np.uint32, 8: np.uint64}[a.dtype.itemsize])


@pytest.fixture(scope="module")
def pq():
    from paper_2604_21645_b200 import pqii
    return pqii


@pytest.fixture(scope="module")
def mix():
    from paper_2604_21645_b200.datagen import gaussian_mixture
    return gaussian_mixture


# ---------------------------------------------------------------------------
# nearest_in_table (proj/src/kmeans.cpp:20-31)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("d,k", [(1, 2), (2, 7), (3, 5), (4, 16), (6, 33), (8, 64), (16, 256),
                                 (17, 100), (32, 256), (128, 1024), (96, 40), (5, 300)])
def test_nearest_batch_exact(pq, orc, d, k):
    pts = orc.random_matrix(3000, d, 1000 + d)
    table = orc.random_matrix(k, d, 2000 + k)
    gi, gd = pq.nearest_batch(pts, table)
    oi, od = orc.nearest_batch(pts, table)
    assert np.array_equal(gi, oi)
    assert np.array_equal(bits(gd), bits(od))


def test_nearest_ties_lowest_index(pq, orc):
    # proj/tests/test_kmeans.cpp:106-112 plus duplicated centroids (exact ties)
    gi, _ = pq.nearest_batch(np.array([[2.0]], np.float32), np.array([[1.0], [3.0]], np.float32))
    assert gi[0] == 0
    table = orc.random_matrix(64, 8, 5)
    table = np.concatenate([table, table, table])  # every row appears 3x
    pts = np.concatenate([table[:40], orc.random_matrix(500, 8, 6)])
    gi, gd = pq.nearest_batch(pts, table)
    oi, od = orc.nearest_batch(pts, table)
    assert np.array_equal(gi, oi) and (gi < 64).all()
    assert np.array_equal(bits(gd), bits(od))


@pytest.mark.parametrize("d,k", [(8, 64), (16, 256), (5, 40), (128, 1024), (8, 16), (32, 12), (4, 7)])
def test_nearest_nonfinite(pq, orc, d, k):
    """nearest_in_table's NaN rule (kmeans.cpp:20-31): the search starts from
    (0, d_0) and only a strictly smaller distance replaces it, so a NaN d_0
    is kept and NaN distances never win."""
    table = orc.random_matrix(k, d, 11).copy()
    pts = orc.random_matrix(600, d, 12).copy()
    table[0, 1] = np.nan          # d_0 is NaN for every point
    table[3, 0] = np.inf          # inf / NaN distances elsewhere
    table[5, :] = np.nan
    pts[7, 2] = np.nan            # every distance NaN for this point
    pts[9, 0] = np.inf
    gi, gd = pq.nearest_batch(pts, table)
    oi, od = orc.nearest_batch(pts, table)
    assert np.array_equal(gi, oi)
    assert np.array_equal(bits(gd), bits(od))
    t2 = table.copy()
    t2[0] = orc.random_matrix(1, d, 13)[0]   # finite d_0, NaN rows elsewhere
    gi, gd = pq.nearest_batch(pts, t2)
    oi, od = orc.nearest_batch(pts, t2)
    assert np.array_equal(gi, oi)
    assert np.array_equal(bits(gd), bits(od))


def test_nearest_exact_match_and_errors(pq, orc):
    table = orc.random_matrix(16, 8, 31)
    idx, dist = pq.nearest_centroid(table[3], table)
    assert idx == 3 and dist == 0.0
    with pytest.raises(ValueError, match="empty centroid set"):
        pq.nearest_centroid(np.zeros(1, np.float32), np.zeros((0, 1), np.float32))


# ---------------------------------------------------------------------------
# kmeans_fit (proj/src/kmeans.cpp:61-133)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", ["km_rand", "km_1d", "km_dup", "km_mix", "km_mix_tol0", "km_k1"])
def test_kmeans_golden(pq, golden, name):
    k, iters, seed = (int(v) for v in golden[f"{name}/params"])
    tol = float(golden[f"{name}/tol"][0])
    r = pq.kmeans_fit(golden[f"{name}/points"], k, iters, seed, tol)
    assert np.array_equal(bits(r.centroids), bits(golden[f"{name}/centroids"]))
    assert np.array_equal(r.assignments, golden[f"{name}/assignments"])
    assert r.iterations_run == int(golden[f"{name}/iterations_run"][0])
    np.testing.assert_allclose(r.inertia_per_iter, golden[f"{name}/inertia_per_iter"], rtol=1e-12)


def test_kmeans_known_answers(pq):
    pts = np.array([[0], [1], [9], [10]], np.float32)
    for seed in range(6):
        r = pq.kmeans_fit(pts, 2, 20, seed)
        assert abs(r.inertia - 1.0) < 1e-9
        assert sorted(r.centroids.ravel().tolist()) == [0.5, 9.5]
    r = pq.kmeans_fit(np.full((6, 2), 1.5, np.float32), 3, 10, 0)
    assert r.inertia == 0.0 and np.isfinite(r.centroids).all()


@pytest.mark.parametrize("seed", [0, 3, 77, 123])
def test_kmeans_random_vs_oracle(pq, orc, seed):
    rng = np.random.default_rng(seed)
    n, d = int(rng.integers(50, 3000)), int(rng.integers(1, 40))
    k = int(rng.integers(1, min(300, n)))
    pts = orc.random_matrix(n, d, seed + 100)
    a = pq.kmeans_fit(pts, k, 25, seed, 0.0)
    b = orc.kmeans_fit(pts, k, 25, seed, 0.0)
    assert a.iterations_run == b["iterations_run"]
    assert np.array_equal(bits(a.centroids), bits(b["centroids"]))
    assert np.array_equal(a.assignments, b["assignments"])
    np.testing.assert_allclose(a.inertia_per_iter, b["inertia_per_iter"], rtol=1e-12)


@pytest.mark.parametrize("scale", ["wide", "tiny", "mixed_sign"])
def test_kmeans_sum_order_paths(pq, orc, scale):
    """Centroid sums: the parallel path is taken only when every partial sum
    is exact; columns spanning many binades (or huge cancellations) must fall
    back to the reference's row order and still match bit for bit."""
    rng = np.random.default_rng(7)
    pts = orc.random_matrix(4000, 6, 31).astype(np.float32)
    if scale == "wide":      # values from 1e-30 to 1e4 in the same column
        pts[:, 0] *= np.float32(10.0) ** rng.integers(-30, 5, size=4000).astype(np.float32)
    elif scale == "tiny":    # subnormal and tiny magnitudes
        pts[:, 1] *= np.float32(1e-38)
        pts[::7, 2] = np.float32(1e-44)
    else:                    # large +/- pairs that cancel
        pts[:, 3] += np.where(rng.random(4000) < 0.5, 1e7, -1e7).astype(np.float32)
    a = pq.kmeans_fit(pts, 37, 15, 3, 0.0)
    b = orc.kmeans_fit(pts, 37, 15, 3, 0.0)
    assert np.array_equal(bits(a.centroids), bits(b["centroids"]))
    assert np.array_equal(a.assignments, b["assignments"])
    t = pq.pq_fit(pts[:, :6], 3, 16, 8, 5).tables
    ot, _, _ = orc.pq_fit(pts[:, :6], 3, 16, 8, 5)
    assert np.array_equal(bits(t), bits(ot))


@pytest.mark.parametrize("copy", ["1", "0"])
@pytest.mark.parametrize("pattern", ["tiny_sparse", "tiny_dense", "wide", "cancel", "nan"])
@pytest.mark.parametrize("d", [8, 6, 16])
def test_kmeans_large_cluster_sums(pq, orc, monkeypatch, d, pattern, copy):
    """Clusters of thousands of members (one CTA each): the chunked row-order
    fallback -- exact chunks added in parallel, a chunk that can round walked
    serially -- must reproduce the reference's sequential fp64 sums bit for
    bit, through the bucketed row copy and through the permutation."""
    monkeypatch.setenv("PQG_KM_COPY", copy)
    rng = np.random.default_rng(d * 100 + len(pattern))
    n = 20000
    pts = (orc.random_matrix(n, d, 41 + d) * 10.0).astype(np.float32)
    if pattern == "tiny_sparse":   # a few tiny values anywhere (one chunk each)
        pts[rng.choice(n, 12, replace=False), 0] = np.float32(3e-30)
        pts[rng.choice(n, 5, replace=False), 1] = np.float32(-7e-25)
    elif pattern == "tiny_dense":  # tiny values in many chunks of a cluster
        pts[rng.random(n) < 0.01, 1] *= np.float32(1e-20)
    elif pattern == "wide":        # every magnitude from 1e-20 to 1e5
        pts[:, 0] *= (np.float32(10.0) ** rng.integers(-20, 6, size=n)).astype(np.float32)
    elif pattern == "cancel":      # large +/- values that cancel
        pts[:, d - 1] += np.where(rng.random(n) < 0.5, 1e7, -1e7).astype(np.float32)
    else:                          # a NaN and an inf coordinate
        pts[123, 0] = np.nan
        pts[4567, 1] = np.inf
    a = pq.kmeans_fit(pts, 8, 6, 3, 0.0)
    b = orc.kmeans_fit(pts, 8, 6, 3, 0.0)
    ca, cb = np.asarray(a.centroids), np.asarray(b["centroids"])
    nan = np.isnan(ca)  # NaN payloads are platform-specific: positions must agree
    assert np.array_equal(nan, np.isnan(cb))
    assert np.array_equal(bits(np.where(nan, 0, ca)), bits(np.where(nan, 0, cb)))
    assert np.array_equal(a.assignments, b["assignments"])


@pytest.mark.parametrize("k", [3100, 4096, 5000])
def test_kmeans_many_clusters(pq, orc, k):
    """k > 3072: the bucketing runs fewer warps per tile (per-warp key
    counters in shared memory); every row must still land in its list."""
    pts = orc.random_matrix(12000, 4, 77 + k)
    a = pq.kmeans_fit(pts, k, 3, 5, 0.0)
    b = orc.kmeans_fit(pts, k, 3, 5, 0.0)
    assert np.array_equal(bits(a.centroids), bits(b["centroids"]))
    assert np.array_equal(a.assignments, b["assignments"])


def test_kmeans_validation(pq, orc):
    pts = orc.random_matrix(5, 2, 1)
    with pytest.raises(ValueError):
        pq.kmeans_fit(pts, 0, 10, 0)
    with pytest.raises(ValueError, match="exceeds"):
        pq.kmeans_fit(pts, 6, 10, 0)
    with pytest.raises(ValueError):
        pq.kmeans_fit(pts, 2, 0, 0)
    with pytest.raises(ValueError):
        pq.kmeans_fit(pts, 2, 10, 0, -1.0)


# ---------------------------------------------------------------------------
# pq_fit / encode / decode / rmse (proj/src/pq.cpp)
# ---------------------------------------------------------------------------

def test_pq_fit_golden(pq, golden):
    M, ks, iters, seed = (int(v) for v in golden["pq/params"])
    stats = {}
    cb = pq.pq_fit(golden["pq/data"], M, ks, iters, seed, stats=stats)
    assert np.array_equal(bits(cb.tables), bits(golden["pq/tables"]))
    codes = pq.pq_encode(cb, golden["pq/data"])
    assert np.array_equal(codes.bytes, golden["pq/codes"])
    dec = pq.pq_decode(cb, codes)
    assert np.array_equal(bits(dec), bits(golden["pq/decoded"]))
    r = pq.reconstruction_rmse(cb, golden["pq/data"])
    assert abs(r - float(golden["pq/rmse"][0])) <= 1e-12 * r
    assert abs(pq.rmse(golden["pq/data"], dec) - r) <= 1e-12 * r
    # M=1 degenerates to kmeans_fit(seed) bit-for-bit (test_pq.cpp:47-51)
    cb1 = pq.pq_fit(golden["pq_m1/data"], 1, 8, 10, 42)
    assert np.array_equal(bits(cb1.tables), bits(golden["pq_m1/tables"]))
    km = pq.kmeans_fit(golden["pq_m1/data"], 8, 10, 42)
    assert np.array_equal(bits(cb1.tables.reshape(8, -1)), bits(km.centroids))
    cb2 = pq.pq_fit(golden["pq_m1/data"], 2, 8, 10, 1)
    assert np.array_equal(bits(cb2.tables), bits(golden["pq_ds2/tables"]))


def test_pq_wide_codes(pq, golden):
    cb = pq.Codebook(2, 300, 4, golden["pq_wide/tables"])
    codes = pq.pq_encode(cb, golden["pq_wide/data"])
    assert codes.code_width() == 2
    assert np.array_equal(codes.bytes, golden["pq_wide/codes"])
    dec = pq.pq_decode(cb, codes)
    assert dec.shape == golden["pq_wide/data"].shape


@pytest.mark.parametrize("M,ks,ds", [(4, 16, 2), (8, 256, 16), (16, 256, 8), (32, 16, 4), (16, 16, 8), (4, 9, 32),
                                     (4, 64, 32), (3, 7, 5), (2, 1, 3), (12, 256, 8),
                                     (64, 256, 2), (128, 16, 1), (8, 100, 6), (6, 200, 12),
                                     (5, 256, 24)])
def test_pq_encode_vs_oracle(pq, orc, mix, M, ks, ds):
    x = mix(4000, M * ds, 32, seed=M * 100 + ks)
    tables = orc.random_matrix(M * ks, ds, 7 + ks).reshape(M, ks, ds) * 3.0
    tables = np.ascontiguousarray(tables, np.float32)
    cb = pq.Codebook(M, ks, ds, tables)
    codes = pq.pq_encode(cb, x)
    assert np.array_equal(codes.bytes, orc.pq_encode(x, tables))
    r = pq.reconstruction_rmse(cb, x)
    ro = orc.rmse(x, orc.pq_decode(codes.bytes, tables))
    assert abs(r - ro) <= 1e-12 * max(ro, 1e-30)


@pytest.mark.parametrize("M,ks,n,iters,D", [(8, 256, 20000, 20, 64), (16, 64, 8000, 25, 64),
                                            (4, 16, 6000, 25, 64), (8, 256, 12000, 15, 48),
                                            (32, 32, 5000, 12, 64), (6, 100, 7000, 12, 60)])
def test_pq_fit_vs_oracle(pq, orc, mix, M, ks, n, iters, D):
    x = mix(n, D, 64, seed=11 + M)
    stats = {}
    cb = pq.pq_fit(x, M, ks, iters, 9, stats=stats)
    t, it, _ = orc.pq_fit(x, M, ks, iters, 9)
    assert np.array_equal(stats["iterations_run"], it)
    assert np.array_equal(bits(cb.tables), bits(t))


def test_pq_fit_problem_major_copy(pq, orc, mix):
    """Batched fits over more than 64 MB of rows run on a problem-major copy
    of the column blocks (capi.cu run_kmeans); still bit-identical."""
    x = mix(140_000, 128, 64, seed=5)  # 71.7 MB
    stats = {}
    cb = pq.pq_fit(x, 8, 16, 3, 4, stats=stats)
    t, it, _ = orc.pq_fit(x, 8, 16, 3, 4)
    assert np.array_equal(stats["iterations_run"], it)
    assert np.array_equal(bits(cb.tables), bits(t))


def test_pq_code_semantics(pq, orc):
    data = orc.random_matrix(40, 8, 23)
    cb = pq.pq_fit(data, 4, 1, 5, 2)  # ks=1 encodes everything to zero
    assert (pq.pq_encode(cb, data).bytes == 0).all()
    cb = pq.pq_fit(data, 4, 8, 15, 2)
    probe = np.concatenate([cb.codeword(m, 5) for m in range(4)]).reshape(1, 8)
    assert (pq.pq_encode(cb, probe).bytes == 5).all()
    with pytest.raises(ValueError, match="not divisible"):
        pq.pq_fit(data, 3, 8, 10, 1)
    with pytest.raises(ValueError, match="exceeds"):
        pq.pq_fit(data, 2, 65, 10, 1)
    with pytest.raises(ValueError):
        pq.pq_encode(cb, orc.random_matrix(4, 6, 1))
    bad = pq.CodeMatrix.zeros(1, 4, 8)
    bad.set(0, 2, 9)  # code >= ks
    with pytest.raises(IndexError):
        pq.pq_decode(cb, bad)


def test_rmse_known_answers(pq):
    a = np.array([[0, 0]], np.float32)
    b = np.array([[3, 4]], np.float32)
    assert abs(pq.rmse(a, b) - np.sqrt(25 / 2)) < 1e-12
    with pytest.raises(ValueError):
        pq.rmse(np.zeros((2, 2), np.float32), np.zeros((2, 3), np.float32))


def test_exactly_representable_lossless(pq, orc):
    # test_pq.cpp:19-33, 62-66
    levels = orc.random_matrix(8, 8, 3, -5, 5)
    data = np.zeros((200, 8), np.float32)
    for i in range(200):
        for s in range(4):
            lv = (i + s) % 8
            data[i, s * 2:(s + 1) * 2] = levels[lv, s * 2:(s + 1) * 2]
    cb = pq.pq_fit(data, 4, 8, 25, 7)
    assert pq.reconstruction_rmse(cb, data) <= 1e-6


# ---------------------------------------------------------------------------
# ADC (proj/src/pq.cpp:132-167)
# ---------------------------------------------------------------------------

def test_adc_golden(pq, golden):
    tables = golden["pq/tables"]
    cb = pq.Codebook(*tables.shape, tables)
    codes = pq.CodeMatrix(golden["pq/codes"].shape[0], tables.shape[0], tables.shape[1],
                          golden["pq/codes"])
    for i, q in enumerate(golden["adc/queries"]):
        t = pq.adc_table(cb, q)
        assert np.array_equal(bits(t.entries), bits(golden["adc/tables"][i]))
        assert np.array_equal(bits(pq.adc_lookup_all(t, codes)), bits(golden["adc/lookup"][i]))


def test_adc_known_answers(pq):
    cb = pq.Codebook(2, 1, 1, np.array([[[3.0]], [[0.0]]], np.float32))
    t = pq.adc_table(cb, np.array([1.0, 0.0], np.float32))
    assert t.entry(0, 0) == 4.0 and t.entry(1, 0) == 0.0


# ---------------------------------------------------------------------------
# IVF (proj/src/ivf.cpp)
# ---------------------------------------------------------------------------

@pytest.fixture(scope="module")
def gidx(pq, golden):
    tables = golden["pq/tables"]
    cb = pq.Codebook(*tables.shape, tables)
    codes = pq.CodeMatrix(golden["pq/codes"].shape[0], tables.shape[0], tables.shape[1],
                          golden["pq/codes"])
    index = pq.ivf_build_with_centroids(cb, codes, golden["ivf/ids"], golden["ivf/coarse"])
    return cb, codes, index


def test_ivf_build_golden(gidx, golden):
    _, _, index = gidx
    off, ids, codes, coarse, _ = index.export()
    assert np.array_equal(off, golden["ivf/offsets"])
    assert np.array_equal(ids, golden["ivf/list_ids"])
    assert np.array_equal(codes, golden["ivf/list_codes"])
    assert np.array_equal(bits(coarse), bits(golden["ivf/coarse"]))


@pytest.mark.parametrize("nprobe", [1, 4, 40])
def test_ivf_query_golden(pq, gidx, golden, nprobe):
    _, _, index = gidx
    ids, dist, cnt = pq.ivf_query_batch(index, golden["ivf/queries"], 10, nprobe)
    assert np.array_equal(cnt, golden[f"ivf/q_np{nprobe}_count"])
    for q in range(len(cnt)):
        c = int(cnt[q])
        assert np.array_equal(ids[q, :c], golden[f"ivf/q_np{nprobe}_ids"][q, :c])
        assert np.array_equal(bits(dist[q, :c]), bits(golden[f"ivf/q_np{nprobe}_dist"][q, :c]))


def test_ivf_query_max_and_flat(pq, gidx, golden):
    cb, codes, index = gidx
    ids, dist, cnt = pq.ivf_query_batch(index, golden["ivf/queries"], 10, 4, max_sq_dist=60.0)
    assert np.array_equal(cnt, golden["ivf/q_max_count"])
    for q in range(len(cnt)):
        assert np.array_equal(ids[q, : cnt[q]], golden["ivf/q_max_ids"][q, : cnt[q]])
    fi, fd, fc = pq.flat_scan_batch(cb, codes, golden["ivf/ids"], golden["ivf/queries"], 10)
    assert np.array_equal(fi, golden["ivf/flat_ids"])
    assert np.array_equal(bits(fd), bits(golden["ivf/flat_dist"]))
    # nprobe == nlist equals flat_scan bit-for-bit (test_ivf.cpp:246-253)
    ai, ad, ac = pq.ivf_query_batch(index, golden["ivf/queries"], 10, index.nlist())
    assert np.array_equal(ai, fi) and np.array_equal(bits(ad), bits(fd))


def test_ivf_probe_vs_oracle(pq, orc, gidx, golden):
    _, _, index = gidx
    probes = pq.ivf_probe(index, golden["ivf/queries"], 7)
    for q, qv in enumerate(golden["ivf/queries"]):
        assert np.array_equal(probes[q], orc.probe_order(golden["ivf/coarse"], qv, 7))


def test_ivf_build_kmeans_golden(pq, golden):
    tables = golden["pq/tables"]
    cb = pq.Codebook(*tables.shape, tables)
    codes = pq.CodeMatrix(800, tables.shape[0], tables.shape[1], golden["pq/codes"][:800])
    index = pq.ivf_build(cb, codes, golden["ivf/ids"][:800], 20, 17, 8)
    off, ids, lcodes, coarse, _ = index.export()
    assert np.array_equal(bits(coarse), bits(golden["ivf_build/coarse"]))
    assert np.array_equal(off, golden["ivf_build/offsets"])
    assert np.array_equal(ids, golden["ivf_build/list_ids"])
    assert np.array_equal(lcodes, golden["ivf_build/list_codes"])


def test_ivf_add_merge_equivalence(pq, gidx, golden):
    cb, codes, full = gidx
    ids = golden["ivf/ids"]
    n = codes.rows
    half = n // 3
    a = pq.ivf_build_with_centroids(cb, pq.CodeMatrix(half, cb.m_subspaces, cb.ks, codes.bytes[:half]),
                                    ids[:half], golden["ivf/coarse"])
    b = pq.ivf_build_with_centroids(cb, pq.CodeMatrix(n - half, cb.m_subspaces, cb.ks, codes.bytes[half:]),
                                    ids[half:], golden["ivf/coarse"])
    m = pq.ivf_merge(a, b)
    fo, fi, fc, _, _ = full.export()
    mo, mi, mc, _, _ = m.export()
    assert np.array_equal(fo, mo) and np.array_equal(fi, mi) and np.array_equal(fc, mc)
    pq.ivf_add(a, pq.CodeMatrix(n - half, cb.m_subspaces, cb.ks, codes.bytes[half:]), ids[half:])
    ao, ai, ac, _, _ = a.export()
    assert np.array_equal(fo, ao) and np.array_equal(fi, ai) and np.array_equal(fc, ac)
    with pytest.raises(ValueError, match="id collision"):
        pq.ivf_add(a, pq.CodeMatrix(1, cb.m_subspaces, cb.ks, codes.bytes[:1]), ids[5:6])
    with pytest.raises(ValueError, match="id collision"):
        pq.ivf_merge(a, b)


def test_ivf_errors(pq, gidx, golden):
    cb, codes, index = gidx
    ids = golden["ivf/ids"].copy()
    ids[10] = ids[3]
    with pytest.raises(ValueError, match=f"duplicate id {int(ids[3])}"):
        pq.ivf_build_with_centroids(cb, codes, ids, golden["ivf/coarse"])
    with pytest.raises(ValueError, match="no items"):
        pq.ivf_build_with_centroids(cb, pq.CodeMatrix.zeros(0, cb.m_subspaces, cb.ks), [], golden["ivf/coarse"])
    with pytest.raises(ValueError, match="nprobe"):
        pq.ivf_query(index, golden["ivf/queries"][0], 10, 0)
    with pytest.raises(ValueError, match="nprobe"):
        pq.ivf_query(index, golden["ivf/queries"][0], 10, index.nlist() + 1)
    with pytest.raises(ValueError):
        pq.ivf_query(index, golden["ivf/queries"][0], 0, 1)


def test_ivf_empty_lists_and_k_saturation(pq, orc, mix):
    x = mix(3000, 16, 8, seed=2)
    cb = pq.pq_fit(x, 4, 16, 10, 1)
    codes = pq.pq_encode(cb, x)
    coarse = np.concatenate([x[:8], np.full((8, 16), 1e4, np.float32)])  # 8 empty lists
    ids = np.arange(3000, dtype=np.uint64) * 3
    index = pq.ivf_build_with_centroids(cb, codes, ids, coarse)
    off, lid, lcodes, _, _ = index.export()
    o_off, o_ids, o_codes = orc.ivf_build_with_centroids(codes.bytes, ids, cb.tables, coarse)
    assert np.array_equal(off, o_off) and np.array_equal(lid, o_ids)
    assert (np.diff(off)[8:] == 0).all()
    q = mix(20, 16, 8, seed=2, stream=1)
    gi, gd, gc = pq.ivf_query_batch(index, q, 32, 16)
    for i in range(20):
        ri, rd = orc.ivf_query(cb.tables, coarse, o_off, o_ids, o_codes, q[i], 32, 16)
        assert np.array_equal(gi[i, : gc[i]], ri) and np.array_equal(bits(gd[i, : gc[i]]), bits(rd))


@pytest.mark.parametrize("k", [1, 10, 32])
def test_search_duplicate_codes_ties(pq, orc, k):
    # many identical code rows -> exact distance ties broken by id
    rng = np.random.default_rng(4)
    tables = orc.random_matrix(8 * 16, 4, 9).reshape(8, 16, 4)
    base = rng.integers(0, 16, size=(50, 8), dtype=np.uint8)
    codes_b = base[rng.integers(0, 50, size=5000)]
    ids = rng.permutation(100000)[:5000].astype(np.uint64)
    cb = pq.Codebook(8, 16, 4, np.ascontiguousarray(tables, np.float32))
    codes = pq.CodeMatrix(5000, 8, 16, np.ascontiguousarray(codes_b))
    coarse = pq.pq_decode(cb, pq.CodeMatrix(12, 8, 16, np.ascontiguousarray(base[:12])))
    index = pq.ivf_build_with_centroids(cb, codes, ids, coarse)
    o_off, o_ids, o_codes = orc.ivf_build_with_centroids(codes.bytes, ids, cb.tables, coarse)
    q = orc.random_matrix(30, 32, 77)
    gi, gd, gc = pq.ivf_query_batch(index, q, k, 5)
    for i in range(30):
        ri, rd = orc.ivf_query(cb.tables, coarse, o_off, o_ids, o_codes, q[i], k, 5)
        assert np.array_equal(gi[i, : gc[i]], ri) and np.array_equal(bits(gd[i, : gc[i]]), bits(rd))


def test_topk_merge_is_monolithic(pq, gidx, golden):
    """Sharded search (rows split in contiguous ranges) merged by
    (dist, id) equals the monolithic query."""
    import ctypes as C
    from paper_2604_21645_b200 import _lib
    cb, codes, full = gidx
    ids = golden["ivf/ids"]
    q = golden["ivf/queries"]
    parts = []
    bounds = [0, 700, 1500, codes.rows]
    for s in range(3):
        a, b = bounds[s], bounds[s + 1]
        ix = pq.ivf_build_with_centroids(cb, pq.CodeMatrix(b - a, cb.m_subspaces, cb.ks, codes.bytes[a:b]),
                                         ids[a:b], golden["ivf/coarse"])
        parts.append(pq.ivf_query_batch(ix, q, 10, 6))
    si = np.ascontiguousarray(np.stack([p[0] for p in parts]))
    sd = np.ascontiguousarray(np.stack([p[1] for p in parts]))
    sc = np.ascontiguousarray(np.stack([p[2] for p in parts]))
    nq = q.shape[0]
    oi = np.zeros((nq, 10), np.uint64)
    od = np.zeros((nq, 10), np.float64)
    oc = np.zeros(nq, np.uint32)
    ctx = pq.get_context()
    v = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    _lib.check(ctx.lib.pqg_topk_merge(ctx.h, v(si), v(sd), v(sc), 3, nq, 10, v(oi), v(od), v(oc)))
    fi, fd, fc = pq.ivf_query_batch(full, q, 10, 6)
    assert np.array_equal(oc, fc) and np.array_equal(oi, fi) and np.array_equal(bits(od), bits(fd))


# ---------------------------------------------------------------------------
# full-size properties (BASELINE config 3 shapes, sampled oracle checks)
# ---------------------------------------------------------------------------

def test_encode_full_size_sampled(pq, orc, mix):
    n = 1_000_000
    x = mix(n, 128, 256, seed=42)
    train = x[::10]
    cb = pq.pq_fit(train[:20000], 16, 256, 6, 1)
    codes = pq.pq_encode(cb, x)
    rng = np.random.default_rng(0)
    sel = np.sort(rng.choice(n, 20000, replace=False))
    assert np.array_equal(codes.bytes[sel], orc.pq_encode(x[sel], cb.tables))
    # decode(encode(x)) is idempotent under encode (codewords are fixed points)
    dec = pq.pq_decode(cb, pq.CodeMatrix(20000, 16, 256, codes.bytes[sel]))
    assert np.array_equal(pq.pq_encode(cb, dec).bytes, codes.bytes[sel])


# ---------------------------------------------------------------------------
# both screens (tcgen05 default and the FP32 FFMA screen) on the coarse and
# PQ shapes that route to each kernel
# ---------------------------------------------------------------------------

@pytest.fixture(params=["tc", "fp32"])
def screen(request, monkeypatch):
    monkeypatch.setenv("PQG_SCREEN", request.param)
    return request.param


@pytest.mark.parametrize("n,d,k", [(5000, 32, 300), (3000, 128, 1024), (4000, 96, 520), (2500, 40, 64)])
def test_coarse_nearest_both_screens(pq, orc, mix, screen, n, d, k):
    x = mix(n, d, 64, seed=d + k)
    table = mix(k, d, 64, seed=d + k + 1)
    gi, gd = pq.nearest_batch(x, table)
    oi, od = orc.nearest_batch(x, table)
    assert np.array_equal(gi, oi)
    assert np.array_equal(bits(gd), bits(od))


def test_coarse_kmeans_both_screens(pq, orc, mix, screen):
    x = mix(6000, 32, 40, seed=77)
    a = pq.kmeans_fit(x, 150, 12, 4)
    b = orc.kmeans_fit(x, 150, 12, 4)
    assert a.iterations_run == b["iterations_run"]
    assert np.array_equal(bits(a.centroids), bits(b["centroids"]))
    assert np.array_equal(a.assignments, b["assignments"])


def test_ivf_large_nlist_both_screens(pq, orc, mix, screen):
    x = mix(8000, 32, 64, seed=5)
    cb = pq.pq_fit(x, 8, 64, 8, 2)
    codes = pq.pq_encode(cb, x)
    assert np.array_equal(codes.bytes, orc.pq_encode(x, cb.tables))
    coarse = pq.kmeans_fit(x, 300, 6, 9).centroids
    ids = np.arange(8000, dtype=np.uint64) + 10
    index = pq.ivf_build_with_centroids(cb, codes, ids, coarse)
    off, lid, lcodes, _, _ = index.export()
    o_off, o_ids, o_codes = orc.ivf_build_with_centroids(codes.bytes, ids, cb.tables, coarse)
    assert np.array_equal(off, o_off) and np.array_equal(lid, o_ids) and np.array_equal(lcodes, o_codes)
    q = mix(40, 32, 64, seed=5, stream=1)
    probes = pq.ivf_probe(index, q, 20)
    gi, gd, gc = pq.ivf_query_batch(index, q, 10, 20)
    for i in range(40):
        assert np.array_equal(probes[i], orc.probe_order(coarse, q[i], 20))
        ri, rd = orc.ivf_query(cb.tables, coarse, o_off, o_ids, o_codes, q[i], 10, 20)
        assert np.array_equal(gi[i, : gc[i]], ri) and np.array_equal(bits(gd[i, : gc[i]]), bits(rd))


def test_ivf_build_nlist_over_3072(pq, orc, mix):
    """Posting lists with nlist = 4500 (the bucketing's few-warps-per-tile
    geometry) equal the reference's, list by list and in insertion order."""
    x = mix(30000, 16, 64, seed=8)
    cb = pq.pq_fit(x, 4, 16, 4, 2)
    codes = pq.pq_encode(cb, x)
    coarse = np.ascontiguousarray(x[::6][:4500])
    ids = np.arange(30000, dtype=np.uint64) * 3 + 1
    index = pq.ivf_build_with_centroids(cb, codes, ids, coarse)
    off, lid, lcodes, _, _ = index.export()
    o_off, o_ids, o_codes = orc.ivf_build_with_centroids(codes.bytes, ids, cb.tables, coarse)
    assert np.array_equal(off, o_off) and np.array_equal(lid, o_ids) and np.array_equal(lcodes, o_codes)


@pytest.mark.parametrize("M,ks", [(8, 256), (16, 64), (4, 16)])
def test_pq_fit_both_screens(pq, orc, mix, screen, M, ks):
    x = mix(5000, 64, 32, seed=M * ks)
    t, it, _ = orc.pq_fit(x, M, ks, 10, 3)
    stats = {}
    cb = pq.pq_fit(x, M, ks, 10, 3, stats=stats)
    assert np.array_equal(stats["iterations_run"], it)
    assert np.array_equal(bits(cb.tables), bits(t))


def test_ivf_query_subset_golden_gpu(pq, gidx, golden):
    _, _, index = gidx
    for qi, q in enumerate(golden["ivf/queries"]):
        r = pq.ivf_query_subset(index, q, 10, golden["ivf/subset"], 6)
        c = int(golden["ivf/q_sub_count"][qi])
        assert [h.id for h in r.hits] == golden["ivf/q_sub_ids"][qi, :c].tolist()
        assert np.array_equal(bits(np.array([h.sq_dist for h in r.hits], np.float64)),
                              bits(golden["ivf/q_sub_dist"][qi, :c]))
    with pytest.raises(ValueError, match="not sorted"):
        pq.ivf_query_subset(index, golden["ivf/queries"][0], 10, golden["ivf/subset"][::-1], 6)
    assert pq.ivf_query_subset(index, golden["ivf/queries"][0], 10, [], 6).hits == []


@pytest.mark.parametrize("variant", ["v1", "v1split", "v2"])
@pytest.mark.parametrize("d,k", [(4, 256), (8, 256), (8, 200), (5, 144), (16, 256), (3, 129), (32, 256)])
def test_umma_screen_variants(pq, orc, mix, monkeypatch, variant, d, k):
    """Every tcgen05 screen variant (one pass, two 128-codeword passes, the
    pipelined kernel) returns nearest_in_table's index and distance bits."""
    monkeypatch.setenv("PQG_SCREEN", "tc")
    monkeypatch.setenv("PQG_UMMA", "2" if variant == "v2" else "1")
    monkeypatch.setenv("PQG_UMMA_SPLIT", "1" if variant == "v1split" else "0")
    pts = mix(5000, d, 32, seed=d * k)
    table = orc.random_matrix(k, d, 3000 + k) * 2.0
    gi, gd = pq.nearest_batch(pts, table)
    oi, od = orc.nearest_batch(pts, table)
    assert np.array_equal(gi, oi)
    assert np.array_equal(bits(gd), bits(od))


@pytest.mark.parametrize("M", [8, 16, 32])
@pytest.mark.parametrize("k", [1, 10, 32])
def test_search_ks256_ties_early_exit(pq, orc, M, k):
    """Ks = 256 byte codes take the scan's partial-sum early exit and the
    buffered survivor merge: many identical code rows (distance ties broken by
    id), the max_sq_dist filter, and a subset, all against the oracle."""
    rng = np.random.default_rng(M * 100 + k)
    ds = 4
    tables = orc.random_matrix(M * 256, ds, 11 + M).reshape(M, 256, ds)
    base = rng.integers(0, 256, size=(60, M), dtype=np.uint8)
    n = 6000
    codes_b = base[rng.integers(0, 60, size=n)]
    ids = rng.permutation(1_000_000)[:n].astype(np.uint64)
    cb = pq.Codebook(M, 256, ds, np.ascontiguousarray(tables, np.float32))
    codes = pq.CodeMatrix(n, M, 256, np.ascontiguousarray(codes_b))
    coarse = pq.pq_decode(cb, pq.CodeMatrix(10, M, 256, np.ascontiguousarray(base[:10])))
    index = pq.ivf_build_with_centroids(cb, codes, ids, coarse)
    o_off, o_ids, o_codes = orc.ivf_build_with_centroids(codes.bytes, ids, cb.tables, coarse)
    q = orc.random_matrix(24, M * ds, 5 + k)
    for max_sq in (None, float(M) * 0.9):
        gi, gd, gc = pq.ivf_query_batch(index, q, k, 4, max_sq_dist=max_sq)
        for i in range(q.shape[0]):
            ri, rd = orc.ivf_query(cb.tables, coarse, o_off, o_ids, o_codes, q[i], k, 4, max_sq_dist=max_sq)
            assert np.array_equal(gi[i, : gc[i]], ri) and np.array_equal(bits(gd[i, : gc[i]]), bits(rd))
    subset = np.sort(ids[rng.choice(n, n // 3, replace=False)])
    for i in range(8):
        r = pq.ivf_query_subset(index, q[i], k, subset, 4)
        ri, rd = orc.ivf_query_subset(cb.tables, coarse, o_off, o_ids, o_codes, q[i], k, subset, 4)
        assert [h.id for h in r.hits] == ri.tolist()
        assert np.array_equal(bits(np.array([h.sq_dist for h in r.hits], np.float64)), bits(rd))


# ---------------------------------------------------------------------------
# k > 32 (topk_large.cu): finalize_hits for any k (proj/src/ivf.cpp:58-68),
# saturating at the candidate count (proj/tests/test_ivf.cpp:255-259)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("k", [33, 100, 1000, 7000])
def test_search_large_k(pq, orc, k):
    rng = np.random.default_rng(k)
    M, ks, ds, n = 8, 256, 4, 6000
    tables = orc.random_matrix(M * ks, ds, 31).reshape(M, ks, ds)
    base = rng.integers(0, ks, size=(80, M), dtype=np.uint8)
    codes_b = base[rng.integers(0, 80, size=n)]  # duplicate rows: ties broken by id
    ids = rng.permutation(1_000_000)[:n].astype(np.uint64)
    cb = pq.Codebook(M, ks, ds, np.ascontiguousarray(tables, np.float32))
    codes = pq.CodeMatrix(n, M, ks, np.ascontiguousarray(codes_b))
    coarse = pq.pq_decode(cb, pq.CodeMatrix(10, M, ks, np.ascontiguousarray(base[:10])))
    index = pq.ivf_build_with_centroids(cb, codes, ids, coarse)
    o_off, o_ids, o_codes = orc.ivf_build_with_centroids(codes.bytes, ids, cb.tables, coarse)
    q = orc.random_matrix(12, M * ds, 3 + k)
    for nprobe in (3, 10):
        for max_sq in (None, float(M) * 0.8):
            gi, gd, gc = pq.ivf_query_batch(index, q, k, nprobe, max_sq_dist=max_sq)
            for i in range(q.shape[0]):
                ri, rd = orc.ivf_query(cb.tables, coarse, o_off, o_ids, o_codes, q[i], k, nprobe,
                                       max_sq_dist=max_sq)
                assert gc[i] == ri.size
                assert np.array_equal(gi[i, : gc[i]], ri) and np.array_equal(bits(gd[i, : gc[i]]), bits(rd))
                assert (gi[i, gc[i]:] == 0).all()
    subset = np.sort(ids[rng.choice(n, n // 4, replace=False)])
    for i in range(5):
        r = pq.ivf_query_subset(index, q[i], k, subset, 6)
        ri, rd = orc.ivf_query_subset(cb.tables, coarse, o_off, o_ids, o_codes, q[i], k, subset, 6)
        assert [h.id for h in r.hits] == ri.tolist() and r.k_requested == k
        assert np.array_equal(bits(np.array([h.sq_dist for h in r.hits], np.float64)), bits(rd))
    fi, fd, fc = pq.flat_scan_batch(cb, codes, ids, q, k)
    for i in range(q.shape[0]):
        ri, rd = orc.flat_scan(cb.tables, codes.bytes, ids, q[i], k)
        assert np.array_equal(fi[i, : fc[i]], ri) and np.array_equal(bits(fd[i, : fc[i]]), bits(rd))
    # nprobe = nlist == flat_scan for k > 32 as well (test_ivf.cpp:246-253)
    ai, ad, ac = pq.ivf_query_batch(index, q, k, index.nlist())
    assert np.array_equal(ac, fc) and np.array_equal(ai, fi) and np.array_equal(bits(ad), bits(fd))


def test_search_large_k_saturates_reference_case(pq, ref):
    """proj/tests/test_ivf.cpp:255-259 on the compiled reference's own index:
    400 items, k = 1000 at nprobe = nlist -> 400 hits, k_requested 1000."""
    x = ref.random_matrix(400, 16, 3, 0.0, 10.0)
    tables = ref.pq_fit(x, 4, 16, 10, 1)
    codes = ref.pq_encode(x, tables)
    ids = np.arange(400, dtype=np.uint64) + 7
    coarse = x[::50].copy()
    cb = pq.Codebook(4, 16, 4, tables)
    index = pq.ivf_build_with_centroids(cb, pq.CodeMatrix(400, 4, 16, codes), ids, coarse)
    q = ref.random_matrix(1, 16, 3)
    r = pq.ivf_query(index, q[0], 1000, index.nlist())
    assert len(r.hits) == 400 and r.k_requested == 1000
    h = ref.ivf_build_with_centroids(codes, ids, tables, coarse)
    ri, rd, rc = h.query_batch(q, 1000, index.nlist())
    assert rc[0] == 400
    assert [x.id for x in r.hits] == ri[0, :400].tolist()
    assert np.array_equal(bits(np.array([x.sq_dist for x in r.hits])), bits(rd[0, :400]))


def test_search_device_outputs_defer_range_error(pq):
    """An out-of-range code found by a search whose outputs stay on the device
    is reported by the next pqg_ctx_sync (adc_lookup's out_of_range)."""
    import ctypes as C

    import torch
    from paper_2604_21645_b200 import _lib
    M, ks, ds = 4, 16, 2
    tables = np.arange(M * ks * ds, dtype=np.float32).reshape(M, ks, ds) / 7
    codes = np.zeros((64, M), np.uint8)
    ctx = pq.Context(0)
    ids = np.arange(64, dtype=np.uint64)
    coarse = np.zeros((2, M * ds), np.float32)
    coarse[1] += 100
    offsets = np.array([0, 64, 64], np.uint64)
    h = C.c_void_p()
    v = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    codes[5, 2] = 20  # >= ks
    _lib.check(ctx.lib.pqg_index_create(ctx.h, v(tables), M, ks, ds, v(coarse), 2, v(offsets), v(ids),
                                        v(codes), C.byref(h)))
    q = torch.zeros((3, M * ds), dtype=torch.float32, device="cuda")
    oi = torch.empty((3, 5), dtype=torch.int64, device="cuda")
    od = torch.empty((3, 5), dtype=torch.float64, device="cuda")
    oc = torch.empty((3,), dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    assert ctx.lib.pqg_index_search(ctx.h, h, vp(q), 3, 5, 1, 0, 0.0, vp(oi), vp(od), vp(oc)) == 0
    assert ctx.lib.pqg_ctx_sync(ctx.h) == _lib.PQG_ERANGE
    assert ctx.lib.pqg_ctx_sync(ctx.h) == 0  # reported once
    ctx.lib.pqg_index_destroy(h)
    ctx.close()


def test_torch_inputs_ordered_on_torch_stream(pq, orc, mix):
    """Device inputs produced on torch's current stream are complete before
    the library's kernels read them, and device outputs before torch reads
    them (pqii orders its own stream against torch's with events)."""
    import torch
    x = mix(20000, 32, 16, seed=8)
    cb = pq.pq_fit(x, 4, 64, 6, 2)
    ref_codes = orc.pq_encode(x, cb.tables)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            xd = torch.zeros((20000, 32), dtype=torch.float32, device="cuda")
            torch.cuda._sleep(2_000_000)  # keep the stream busy before the data lands
            xd.copy_(torch.from_numpy(x).cuda(non_blocking=True))
            codes = pq.pq_encode(cb, xd)
            assert np.array_equal(codes.bytes, ref_codes)


# ---------------------------------------------------------------------------
# the register-resident narrow-codebook screen (nearest.cu narrow_kernel),
# forced on for every shape it accepts: encode and k-means fits (which also
# use its fp64 winner distances) bit-exact against the oracle
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("D,M,ks", [(128, 32, 16), (128, 16, 16), (128, 8, 16), (128, 4, 16), (96, 12, 16),
                                    (128, 32, 64), (128, 16, 64), (64, 8, 64), (64, 16, 12), (32, 8, 5),
                                    (128, 32, 32), (96, 24, 16), (128, 32, 256), (128, 16, 256),
                                    (128, 8, 256), (128, 8, 128), (64, 16, 100), (128, 16, 200)])
@pytest.mark.parametrize("kern", ["narrow", "rows"])
def test_narrow_screen_parity(pq, orc, mix, monkeypatch, D, M, ks, kern):
    monkeypatch.setenv("PQG_NARROW", "1")
    if kern == "narrow":  # the register-resident kernel (the row-blocked one owns Ks <= 32)
        monkeypatch.setenv("PQG_ROWSCREEN", "0")
    elif ks > 32:
        pytest.skip("row-blocked screen: Ks <= 32")
    x = mix(6000, D, 24, seed=D + M + ks)
    st = {}
    cb = pq.pq_fit(x, M, ks, 6, 3, stats=st)
    ref_t, ref_it, _ = orc.pq_fit(x, M, ks, 6, 3)
    assert np.array_equal(bits(cb.tables), bits(ref_t))
    assert np.array_equal(st["iterations_run"], ref_it)
    big = mix(40000, D, 24, seed=7)
    assert np.array_equal(pq.pq_encode(cb, big).bytes, orc.pq_encode_mt(big, ref_t, 8))
    # exact ties: duplicated codewords must resolve to the lowest index
    t2 = ref_t.copy()
    t2[:, ks - ks // 2:] = t2[:, : ks // 2]
    cb2 = pq.Codebook(M, ks, D // M, np.ascontiguousarray(t2))
    assert np.array_equal(pq.pq_encode(cb2, big[:5000]).bytes, orc.pq_encode(big[:5000], t2))


@pytest.mark.parametrize("nq", [1, 5, 40])
def test_probe_d128_small_and_batched_vs_oracle(pq, orc, nq):
    """probe_order (proj/src/ivf.cpp:91-101) at d=128, nlist 300: the exact
    small-batch probe (<= 16 queries, r2e) and the tensor-core batch path,
    plus a query whose distances all overflow to inf (every list ties: the
    lowest indices win, through the exact fallback)."""
    from paper_2604_21645_b200.datagen import gaussian_mixture
    x = gaussian_mixture(3000, 128, 24, seed=41)
    cb = pq.pq_fit(x, 16, 16, 4, 3)
    codes = pq.pq_encode(cb, x)
    coarse = np.ascontiguousarray(x[::10][:300])
    index = pq.ivf_build_with_centroids(cb, codes, np.arange(3000, dtype=np.uint64), coarse)
    qs = gaussian_mixture(nq, 128, 24, seed=41, stream=3)
    if nq > 1:
        qs[nq - 1, 7] = np.float32(1e30)  # squared distances overflow: all inf
    probes = pq.ivf_probe(index, qs, 9)
    for q in range(nq):
        assert np.array_equal(probes[q], orc.probe_order(coarse, qs[q], 9)), q
    # and the searches on top of them (split scan for < 64 queries)
    gi, gd, gc = pq.ivf_query_batch(index, qs, 7, 9)
    off, lid, lcodes, _, _ = index.export()
    for q in range(nq):  # the overflowing query too: every candidate at inf, ids ascending
        ri, rd = orc.ivf_query(cb.tables, coarse, off, lid, lcodes, qs[q], 7, 9)
        assert np.array_equal(gi[q, : gc[q]], ri) and np.array_equal(gd[q, : gc[q]], rd), q


@pytest.mark.parametrize("layout", ["mixture", "clustered_lanes", "duplicates"])
def test_probe_select_warp_nlist1024_vs_oracle(pq, orc, layout):
    """r2h warp-per-query probe select (nlist <= 1024, nprobe <= 32) against
    probe_order (proj/src/ivf.cpp:91-101) and the CTA radix select
    (PQG_PROBE_SEL=cta) at d=128, nlist 1024.  'clustered_lanes' puts the near
    lists in columns j % 32 < 10, so more than 128 keys lie below the lane-minimum
    bound and tau comes from the bisection; 'duplicates' repeats one centroid
    300 times (a band of > 256 lists: the exact fallback)."""
    import os
    from paper_2604_21645_b200.datagen import gaussian_mixture
    rng = np.random.default_rng(7)
    x = gaussian_mixture(4096, 128, 32, seed=43)
    cb = pq.pq_fit(x, 16, 16, 3, 3)
    codes = pq.pq_encode(cb, x)
    qs = gaussian_mixture(48, 128, 32, seed=43, stream=5)
    coarse = np.ascontiguousarray(x[::4][:1024]).copy()
    if layout == "clustered_lanes":
        near = np.array([j for j in range(1024) if j % 32 < 10])
        coarse = (rng.standard_normal((1024, 128)) * 30 + 100).astype(np.float32)
        coarse[near] = qs[0] + (rng.standard_normal((near.size, 128)) * 0.05).astype(np.float32)
    elif layout == "duplicates":
        coarse[100:400] = coarse[99]
        qs[1] = coarse[99]
    coarse = np.ascontiguousarray(coarse, dtype=np.float32)
    index = pq.ivf_build_with_centroids(cb, codes, np.arange(4096, dtype=np.uint64), coarse)
    for nprobe in (1, 16, 32):
        got = pq.ivf_probe(index, qs, nprobe)
        os.environ["PQG_PROBE_SEL"] = "cta"
        try:
            cta = pq.ivf_probe(index, qs, nprobe)
        finally:
            del os.environ["PQG_PROBE_SEL"]
        assert np.array_equal(got, cta), nprobe
        for q in range(0, 48, 3):
            assert np.array_equal(got[q], orc.probe_order(coarse, qs[q], nprobe)), (nprobe, q)
        assert np.array_equal(got[1], orc.probe_order(coarse, qs[1], nprobe)), nprobe
