"""Parity of the device pipeline (pqg_train_chunks / pqg_pipeline_run) with
the reference's run_pipeline (proj/src/pipeline.cpp:84-266), through the C
ABI.  Codebooks, representatives, coarse centroids and posting lists are
bit-exact; RMSE values are fp64 sums whose order differs from the
reference's sequential loop (fixed-shape tree here), so they are held to
1e-12 relative (BASELINE.json allows 1e-4)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

MODES = ("single", "parallel_pq", "parallel_pq_index")
RTOL = 1e-12


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view({4: np.uint32, 8: np.uint64}[a.dtype.itemsize])


@pytest.fixture(scope="module")
def pq():
    from paper_2604_21645_b200 import pqii
    return pqii


@pytest.mark.parametrize("case", ["pipe", "pipe_dup"])
def test_pipeline_golden_gpu(pq, golden, case):
    C_, M, ks, nl, it, sd = (int(v) for v in golden[f"{case}/params"])
    data = golden[f"{case}/data"]
    outs = pq.train_chunks(data, C_, M, ks, it, sd)
    assert [o.chunk_id for o in outs] == list(range(C_))
    np.testing.assert_allclose([o.local_rmse for o in outs], golden[f"{case}/local_rmse"],
                               rtol=RTOL, atol=0)
    for mode in MODES:
        key = f"{case}/{mode}"
        cfg = pq.PipelineConfig(n_chunks=C_, m_subspaces=M, ks=ks, nlist=nl, kmeans_iters=it,
                                seed=sd, n_threads=3, mode=mode)
        r = pq.run_pipeline(data, cfg)
        assert np.array_equal(bits(r.global_codebook.tables), bits(golden[f"{key}/tables"])), mode
        np.testing.assert_allclose(r.global_rmse, golden[f"{key}/rmse"][0], rtol=RTOL, atol=0)
        assert r.config.nlist == golden[f"{key}/nlist"][0]
        if mode == "single":
            assert r.single_rmse == r.global_rmse and r.representatives is None
            assert set(r.phase_seconds) == {"fit", "encode"}
            continue
        assert np.array_equal(bits(r.representatives), bits(golden[f"{key}/representatives"]))
        reps = pq.aggregate_representatives(list(reversed(outs)))
        assert np.array_equal(bits(reps), bits(golden[f"{key}/representatives"]))
        np.testing.assert_allclose(r.local_rmse, golden[f"{case}/local_rmse"], rtol=RTOL, atol=0)
        if mode == "parallel_pq":
            assert set(r.phase_seconds) == {"chunking", "local_fit", "global_fit", "encode"}
            assert r.merged_index is None
            continue
        assert set(r.phase_seconds) == {"chunking", "local_fit", "global_fit", "coarse_fit",
                                        "encode", "index_build", "merge"}
        off, ids, codes, coarse, cb = r.merged_index.export()
        assert np.array_equal(off, golden[f"{key}/offsets"])
        assert np.array_equal(ids, golden[f"{key}/list_ids"])
        assert np.array_equal(codes, golden[f"{key}/list_codes"])
        assert np.array_equal(bits(coarse), bits(golden[f"{key}/coarse"]))
        assert "index:" in r.summary()


@pytest.mark.parametrize("n,D,C_,M,ks,it,seed", [
    (5003, 32, 7, 4, 32, 10, 5),     # uneven chunks (5003 = 7 x 714 + 5), Ds=8
    (4096, 16, 16, 8, 16, 12, 2),    # Ds=2, even chunks
    (2000, 48, 3, 3, 64, 9, 8),      # Ds=16
    (1500, 8, 50, 1, 16, 6, 4),      # many small chunks, M=1
])
def test_train_chunks_vs_reference(pq, ref, n, D, C_, M, ks, it, seed):
    from paper_2604_21645_b200.datagen import gaussian_mixture
    data = gaussian_mixture(n, D, 20, seed)
    outs = pq.train_chunks(data, C_, M, ks, it, seed)
    bounds = ref.chunk_rows(n, C_)
    for c, o in enumerate(outs):
        reps, lr = ref.train_chunk(data[bounds[c]:bounds[c + 1]], M, ks, it, seed + c)
        assert np.array_equal(bits(o.representatives), bits(reps)), c
        np.testing.assert_allclose(o.local_rmse, lr, rtol=RTOL, atol=0)


def test_pipeline_vs_reference_index(pq, ref):
    from paper_2604_21645_b200.datagen import gaussian_mixture
    data = gaussian_mixture(20011, 32, 40, 17)
    cfg = pq.PipelineConfig(n_chunks=9, m_subspaces=8, ks=64, nlist=0, kmeans_iters=12, seed=21,
                            n_threads=4, mode="parallel_pq_index")
    r = pq.run_pipeline(data, cfg)
    b = ref.run_pipeline(data, 9, 8, 64, 0, 12, 21, "parallel_pq_index", threads=8)
    assert r.config.nlist == b["nlist"] == 141
    assert np.array_equal(bits(r.global_codebook.tables), bits(b["tables"]))
    np.testing.assert_allclose(r.global_rmse, b["rmse"], rtol=RTOL, atol=0)
    off, ids, codes, coarse, _ = r.merged_index.export()
    assert np.array_equal(off, b["offsets"]) and np.array_equal(ids, b["list_ids"])
    assert np.array_equal(codes, b["list_codes"]) and np.array_equal(coarse, b["coarse"])


def test_single_chunk_collapse(pq):
    # proj/tests/acceptance_main.cpp:296-340 (criterion 6), which holds exactly here
    from paper_2604_21645_b200.datagen import gaussian_mixture
    data = gaussian_mixture(4000, 16, 12, 23)
    single = pq.run_pipeline(data, pq.PipelineConfig(m_subspaces=4, ks=32, seed=5))
    one = pq.run_pipeline(data, pq.PipelineConfig(m_subspaces=4, ks=32, seed=5, n_chunks=1,
                                                  mode="parallel_pq"))
    assert abs(single.global_rmse - one.global_rmse) <= 1e-6


def test_pipeline_errors(pq):
    data = np.zeros((100, 8), np.float32)
    cfg = lambda **kw: pq.PipelineConfig(**{"m_subspaces": 2, "ks": 16, "mode": "parallel_pq",  # noqa: E731
                                            **kw})
    with pytest.raises(ValueError, match="empty dataset"):
        pq.run_pipeline(np.zeros((0, 8), np.float32), cfg(n_chunks=2))
    with pytest.raises(ValueError, match="n_threads"):
        pq.run_pipeline(data, cfg(n_chunks=2, n_threads=0))
    with pytest.raises(ValueError, match=r"chunk_rows: n_chunks \(101\) exceeds n_rows"):
        pq.run_pipeline(data, cfg(n_chunks=101))
    with pytest.raises(ValueError, match="n_chunks must be >= 1"):
        pq.run_pipeline(data, cfg(n_chunks=0))
    # chunk failures are runtime_errors naming the lowest failing chunk
    # (pipeline.cpp:30-62; proj/tests/test_pipeline.cpp:241-255).
    # 100 rows in 7 chunks: 15,15,14,... -> chunk 2 is the first with < 15 rows
    with pytest.raises(RuntimeError, match=r"^chunk 2: train_chunk: chunk has 14 rows, fewer than ks=15"):
        pq.run_pipeline(data, cfg(n_chunks=7, ks=15))
    with pytest.raises(RuntimeError, match=r"^chunk 0: train_chunk: chunk has 15 rows"):
        pq.run_pipeline(data, cfg(n_chunks=7, ks=16))
    with pytest.raises(RuntimeError, match=r"^chunk 0: pq_fit: D \(8\) is not divisible by M \(3\)"):
        pq.run_pipeline(data, cfg(n_chunks=2, m_subspaces=3))
    with pytest.raises(RuntimeError, match="fewer than ks"):
        pq.train_chunks(data[:10], 5, 2, 3)
    with pytest.raises(ValueError, match="not divisible"):
        pq.run_pipeline(data, cfg(n_chunks=2, m_subspaces=3, mode="single"))
    with pytest.raises(ValueError, match=r"kmeans_fit: k \(40\) exceeds number of points \(32\)"):
        pq.run_pipeline(data, cfg(n_chunks=2, nlist=40, mode="parallel_pq_index"))
