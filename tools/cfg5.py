"""BASELINE configs[4] end to end through the row-sharded path (dist.py), one
process per GPU:

  torchrun --nproc-per-node 8 --master-addr 127.0.0.1 tools/cfg5.py     # 100M rows on 8 GPUs
  python tools/cfg5.py --rows-per-rank 12500000                          # one GPU: a 1-rank group

Every rank generates its shard on the device from seed + rank (1024-component
mixture, mixture parameters from the base seed); the seeded 2M-row training
sample is the strided sample of the GLOBAL row range, each rank
holding the sample rows that fall in its shard.  Then:
  * PQ fit (M=16, Ks=256, 20 iterations) and coarse fit (nlist=4096, seed+M)
    with the exact sharded k-means (one all-reduce of sums / counts / inertia
    per iteration, dist.kmeans_fit_sharded);
  * shard encode + global RMSE (one all-reduce);
  * shard-local inverted index over global ids;
  * 100k queries (same on every rank), nprobe 32, k 10: local search,
    all-gather of the per-shard top-k, (dist, id) merge.
Phase times are CUDA-event times on the library stream, max over ranks; rank 0
prints one JSON line.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=100_000_000, help="global rows")
    ap.add_argument("--rows-per-rank", type=int, default=0, help="override: rows per rank")
    ap.add_argument("--queries", type=int, default=100_000)
    ap.add_argument("--sample", type=int, default=2_000_000)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--force-exchange", action="store_true",
                    help="run the exchange protocol even in a 1-rank group")
    ap.add_argument("--replay", default="chain", choices=["chain", "gather"],
                    help="row-order replay protocol of the sharded fits")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    from paper_2604_21645_b200 import dist as D
    from paper_2604_21645_b200.datagen import device_mixture, mixture_params, strided_sample
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if "RANK" in os.environ:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group("nccl", store=dist.HashStore(), rank=0, world_size=1,
                                device_id=torch.device("cuda", local))
    Dm, COMP, SEED = 128, 1024, 2604
    M, KS, NLIST, NPROBE, K = 16, 256, 4096, 32, 10
    n_local = args.rows_per_rank or args.rows // world
    n_global = n_local * world
    row0 = rank * n_local
    comm, be = D.Comm(), D.CudaBackend(local)
    stream = torch.cuda.current_stream()
    out = {"config": "BASELINE configs[4]", "world": world, "rows_per_rank": n_local, "global_rows": n_global}

    def timed(name, fn):
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record(stream)
        r = fn()
        b.record(stream)
        torch.cuda.synchronize()
        ms = torch.tensor([a.elapsed_time(b)], dtype=torch.float64, device="cuda")
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        out[name + "_ms"] = float(ms.item())
        out[name + "_wall_ms"] = (time.perf_counter() - t0) * 1e3
        return r

    x = torch.empty((n_local, Dm), dtype=torch.float32, device="cuda")
    timed("generate", lambda: device_mixture(n_local, Dm, COMP, SEED, SEED + rank, out=x))
    # the global strided sample, restricted to this shard's rows
    gs = strided_sample(n_global, args.sample, SEED)
    mine = gs[(gs >= row0) & (gs < row0 + n_local)] - row0
    train = x.index_select(0, torch.from_numpy(mine).cuda()).contiguous()
    out["sample_rows_global"] = int(len(gs))
    # warm-up of the fit shapes (module load, scratch arenas), then the timed fits
    D.pq_fit_sharded(comm, be, train, M, KS, 1, SEED)
    D.kmeans_fit_sharded(comm, be, train, 1, Dm, 0, NLIST, 1, [SEED + M], 1e-4)
    st_pq, st_co = {}, {}
    fx = dict(force_exchange=args.force_exchange, replay=args.replay)
    tables = timed("pq_fit", lambda: D.kmeans_fit_sharded(
        comm, be, train, M, Dm // M, Dm // M, KS, args.iters, [SEED + m for m in range(M)], 1e-4, stats=st_pq,
        **fx).tables)
    fit_c = timed("coarse_fit", lambda: D.kmeans_fit_sharded(
        comm, be, train, 1, Dm, 0, NLIST, args.iters, [SEED + M], 1e-4, stats=st_co, **fx))
    coarse = fit_c.tables.view(NLIST, Dm).contiguous()
    out["pq_fit_exchange"] = {k_: st_pq.get(k_) for k_ in ("allreduce_bytes", "allgather_bytes", "chain_bytes",
                                                            "replay_columns", "reseeds", "iterations", "replay")}
    out["coarse_fit_exchange"] = {k_: st_co.get(k_) for k_ in ("allreduce_bytes", "allgather_bytes", "chain_bytes",
                                                                "replay_columns", "reseeds", "iterations", "replay")}
    out["coarse_iters"] = int(np.max(fit_c.iterations_run))
    codes, rmse = timed("encode_rmse", lambda: D.encode_sharded(comm, be, x, tables))
    out["rmse"] = rmse
    ids = torch.arange(n_local, dtype=torch.int64, device="cuda") + row0
    # queries: identical on every rank (same generator seed)
    means, sigmas = mixture_params(Dm, COMP, SEED)
    gq = torch.Generator(device="cuda")
    gq.manual_seed(SEED + 1000003)
    mu = torch.from_numpy(means.astype(np.float64)).cuda()
    sg = torch.from_numpy(sigmas.astype(np.float64)).cuda()
    comp = torch.randint(0, COMP, (args.queries,), generator=gq, device="cuda")
    q = (mu[comp] + sg[comp, None] * torch.randn((args.queries, Dm), generator=gq, device="cuda",
                                                 dtype=torch.float64)).float().contiguous()
    res = timed("index_build_search", lambda: D.search_sharded(comm, be, tables, codes, ids, coarse, q, K, NPROBE))
    out["hits_per_query"] = float(res[2].float().mean().item())
    out["encode_vectors_per_s"] = n_global / (out["encode_rmse_ms"] / 1e3)
    out["fit_encode_ms"] = out["pq_fit_ms"] + out["coarse_fit_ms"] + out["encode_rmse_ms"]
    out["gpu_mem_peak_gb"] = torch.cuda.max_memory_allocated() / 1e9
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
