"""Rank body for tests/test_dist_gpu.py (launched by torchrun, NCCL, CUDA)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(outdir):
    import torch
    import torch.distributed as dist

    from paper_2604_21645_b200 import dist as D
    from paper_2604_21645_b200.datagen import gaussian_mixture
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = D.Comm()
    be = D.CudaBackend(local)
    x = gaussian_mixture(20011, 64, 32, seed=13)
    lo, hi = D.chunk_rows(x.shape[0], world)[rank]
    xl = torch.from_numpy(np.ascontiguousarray(x[lo:hi])).cuda()
    tables = D.pq_fit_sharded(comm, be, xl, 8, 64, 12, 4)
    codes, rmse = D.encode_sharded(comm, be, xl, tables)
    fit = D.kmeans_fit_sharded(comm, be, xl, 1, 64, 0, 128, 10, [3], 1e-4)
    coarse = fit.tables[0].contiguous()
    ids = torch.arange(lo, hi, dtype=torch.int64, device="cuda") * 5 + 2
    q = torch.from_numpy(gaussian_mixture(50, 64, 32, seed=13, stream=1)).cuda()
    oi, od, oc = D.search_sharded(comm, be, tables, codes, ids, coarse, q, 10, 8)
    if rank == 0:
        np.savez(os.path.join(outdir, "dist_gpu.npz"), tables=tables.cpu().numpy(),
                 codes=codes.cpu().numpy(), rmse=np.array([rmse]), coarse=coarse.cpu().numpy(),
                 assign=fit.assignments.cpu().numpy(), ids=oi.cpu().numpy(), d=od.cpu().numpy(),
                 c=oc.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
