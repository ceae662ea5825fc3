"""Multi-rank (world_size 2, gloo, CPU) test of the row-sharded driver
(paper_2604_21645_b200/dist.py): sharded k-means / pq_fit equal the
single-process oracle bit-for-bit, sharded encode gives the global RMSE and
the merged shard search equals the monolithic ivf_query."""
import os
import socket

import numpy as np
import pytest


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_chunk_rows_matches_reference(orc):
    from paper_2604_21645_b200.dist import chunk_rows
    for n, c in [(10, 3), (1203, 2), (7, 7), (100, 8)]:
        b = orc.chunk_rows(n, c)
        assert [(int(b[i]), int(b[i + 1])) for i in range(c)] == chunk_rows(n, c)
    with pytest.raises(ValueError):
        chunk_rows(3, 4)


def test_sharded_pipeline_world2(tmp_path, orc):
    import torch.multiprocessing as mp

    from dist_workers import run_rank
    from paper_2604_21645_b200.datagen import gaussian_mixture
    port = free_port()
    mp.start_processes(run_rank, args=(2, port, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    r = [np.load(tmp_path / f"rank{i}.npz") for i in range(2)]
    x = gaussian_mixture(1203, 16, 12, seed=9)
    # k-means: identical on both ranks and equal to the single-process reference
    ref = orc.kmeans_fit(x, 24, 12, 5, 1e-4)
    for rr in r:
        assert np.array_equal(rr["km_tables"][0].view(np.uint32), ref["centroids"].view(np.uint32))
        assert np.array_equal(rr["km_assign"][0], ref["assignments"])
        assert int(rr["km_iters"][0]) == ref["iterations_run"]
    t, _, _ = orc.pq_fit(x, 4, 16, 10, 3)
    for rr in r:
        assert np.array_equal(rr["pq_tables"].view(np.uint32), t.view(np.uint32))
    codes = np.concatenate([r[0]["codes"], r[1]["codes"]])
    assert np.array_equal(codes, orc.pq_encode(x, t))
    ref_rmse = orc.rmse(x, orc.pq_decode(codes, t))
    assert abs(float(r[0]["rmse"][0]) - ref_rmse) <= 1e-12 * ref_rmse
    # merged shard search == monolithic query
    coarse = x[::100][:12].copy()
    ids = np.arange(1203, dtype=np.uint64) * 3 + 1
    off, lid, lcodes = orc.ivf_build_with_centroids(codes, ids, t, coarse)
    q = gaussian_mixture(9, 16, 12, seed=9, stream=1)
    for qi in range(9):
        ri, rd = orc.ivf_query(t, coarse, off, lid, lcodes, q[qi], 7, 4)
        c = int(r[0]["s_c"][qi])
        assert c == len(ri)
        assert np.array_equal(r[0]["s_ids"][qi, :c], ri)
        assert np.array_equal(r[0]["s_d"][qi, :c].view(np.uint64), rd.view(np.uint64))


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_kmeans_exchange_paths(tmp_path, orc, world):
    """The north-star exchange (all-reduce of sums / counts / exponent ranges,
    all-gathered row-order replay, reseed candidates) on rows that force the
    replay and the reseed, world 2 and 3 (uneven shards): equal to the
    single-process reference bit for bit."""
    import torch.multiprocessing as mp

    from dist_workers import run_rank_stress, stress_data
    port = free_port()
    mp.start_processes(run_rank_stress, args=(world, port, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    r = [np.load(tmp_path / f"stress{i}.npz") for i in range(world)]
    x = stress_data()
    ref = orc.kmeans_fit(x, 40, 9, 2, 0.0)
    for rr in r:
        assert np.array_equal(rr["km_tables"][0].view(np.uint32), ref["centroids"].view(np.uint32))
        assert np.array_equal(rr["km_assign"][0], ref["assignments"])
        assert int(rr["km_iters"][0]) == ref["iterations_run"]
    assert r[0]["stats"][0] > 0, "the row-order replay path was not exercised"
    assert r[0]["stats"][1] > 0, "the reseed path was not exercised"
    # the chained replay (default) moves one fp64 per column per hop and no
    # member values; the r2 all-gather protocol gives the identical fit
    assert r[0]["stats"][3] > 0 and r[0]["stats"][4] == 0
    assert r[0]["stats_g"][0] == r[0]["stats"][0] and r[0]["stats_g"][1] == 0 and r[0]["stats_g"][2] > 0
    for rr in r:
        assert np.array_equal(rr["kmg_tables"][0].view(np.uint32), ref["centroids"].view(np.uint32))
    t, _, _ = orc.pq_fit(x, 2, 32, 8, 7)
    for rr in r:
        assert np.array_equal(rr["pq_tables"].view(np.uint32), t.view(np.uint32))
