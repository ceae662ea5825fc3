"""Rank bodies for tests/test_dist_gloo.py (importable by spawned workers)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def run_rank(rank, world, port, outdir):
    import torch.distributed as dist

    from cpu_backend import OracleBackend, ShardOracleBackend
    from paper_2604_21645_b200 import dist as D
    from paper_2604_21645_b200.datagen import gaussian_mixture

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = D.Comm()
    be = ShardOracleBackend() if os.environ.get('PQG_TEST_SHARD', '1') == '1' else OracleBackend()
    import torch
    x = gaussian_mixture(1203, 16, 12, seed=9)  # odd size: uneven shards
    lo, hi = D.chunk_rows(x.shape[0], world)[rank]
    local = torch.from_numpy(np.ascontiguousarray(x[lo:hi]))
    res = {}
    fit = D.kmeans_fit_sharded(comm, be, local, 1, 16, 0, 24, 12, [5], 1e-4)
    res["km_tables"] = fit.tables.numpy()
    res["km_assign"] = fit.assignments.numpy().view(np.uint32)
    res["km_iters"] = fit.iterations_run
    tables = D.pq_fit_sharded(comm, be, local, 4, 16, 10, 3)
    res["pq_tables"] = tables.numpy()
    codes, rmse = D.encode_sharded(comm, be, local, tables)
    res["codes"], res["rmse"] = codes.numpy(), np.array([rmse])
    coarse = torch.from_numpy(x[::100][:12].copy())
    ids = torch.from_numpy((np.arange(lo, hi, dtype=np.uint64) * 3 + 1).view(np.int64))
    q = torch.from_numpy(gaussian_mixture(9, 16, 12, seed=9, stream=1))
    oi, od, oc = D.search_sharded(comm, be, tables, codes, ids, coarse, q, 7, 4)
    res["s_ids"], res["s_d"], res["s_c"] = oi.numpy().view(np.uint64), od.numpy(), oc.numpy().view(np.uint32)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), **res)
    dist.barrier()
    dist.destroy_process_group()


def stress_data():
    """Rows that exercise every exchange path of the sharded update: a column
    of tiny values next to large ones (exponent ranges beyond the exact-sum
    test -> the row-order replay), exact duplicates (empty clusters -> the
    reseed), 1-D subspaces of zeros (no nonzero members)."""
    from paper_2604_21645_b200.datagen import gaussian_mixture
    x = gaussian_mixture(901, 8, 6, seed=21)
    x[::7, 1] = np.float32(3e-9)
    x[::11, 2] *= np.float32(1e6)
    x[:, 3] = 0.0
    x[500:560] = x[10]  # duplicates
    return np.ascontiguousarray(x, np.float32)


def run_rank_stress(rank, world, port, outdir):
    import torch
    import torch.distributed as dist

    from cpu_backend import ShardOracleBackend
    from paper_2604_21645_b200 import dist as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = D.Comm()
    be = ShardOracleBackend()
    x = stress_data()
    lo, hi = D.chunk_rows(x.shape[0], world)[rank]
    local = torch.from_numpy(np.ascontiguousarray(x[lo:hi]))
    res = {}
    st = {}
    fit = D.kmeans_fit_sharded(comm, be, local, 1, 8, 0, 40, 9, [2], 0.0, stats=st)
    res["km_tables"], res["km_iters"] = fit.tables.numpy(), fit.iterations_run
    res["km_assign"] = fit.assignments.numpy().view(np.uint32)
    res["stats"] = np.array([st["replay_columns"], st["reseeds"], st["iterations"], st["chain_bytes"],
                             st["allgather_bytes"]])
    # the r2 protocol (members all-gathered) must give the same fit
    sg = {}
    fg = D.kmeans_fit_sharded(comm, be, local, 1, 8, 0, 40, 9, [2], 0.0, stats=sg, replay="gather")
    res["kmg_tables"] = fg.tables.numpy()
    res["stats_g"] = np.array([sg["replay_columns"], sg["chain_bytes"], sg["allgather_bytes"]])
    res["pq_tables"] = D.pq_fit_sharded(comm, be, local, 2, 32, 8, 7).numpy()
    np.savez(os.path.join(outdir, f"stress{rank}.npz"), **res)
    dist.barrier()
    dist.destroy_process_group()
