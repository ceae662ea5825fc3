"""The native (C++) host of the row-sharded fit (pqg_kmeans_fit_sharded,
csrc/kmnccl.cu): the pqg_kmshard_* protocol with NCCL collectives issued by
the library.  One GPU here, so a 1-rank NCCL communicator: every exchange
(grouped all-reduces, the row-order chain's send / recv / broadcast, the
reseed all-gathers) runs with world 1 and the result must equal the
single-process fit and the oracle bit for bit.  The multi-rank protocol
itself is covered by tests/test_dist_gloo.py and tests/test_dist_threads_gpu.py."""
import types

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _one_rank(backend):
    from paper_2604_21645_b200 import dist as D
    comm = types.SimpleNamespace(rank=0, world=1, dist=None, group=None, broadcast_=lambda t, src: t)
    return D.NcclComm(comm, backend)


def test_native_sharded_coarse_matches_oracle(orc):
    import torch

    from paper_2604_21645_b200 import dist as D
    import os
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from dist_workers import stress_data
    x = stress_data()
    be = D.CudaBackend(0, private=True)
    nc = _one_rank(be)
    try:
        st = {}
        fit = D.kmeans_fit_sharded_native(nc, torch.from_numpy(x).cuda(), 1, 8, 0, 40, 9, [2], 0.0, stats=st)
    finally:
        nc.close()
    ref = orc.kmeans_fit(x, 40, 9, 2, 0.0)
    assert np.array_equal(fit.tables[0].cpu().numpy().view(np.uint32), ref["centroids"].view(np.uint32))
    assert np.array_equal(fit.assignments[0].cpu().numpy().view(np.uint32), ref["assignments"])
    assert int(fit.iterations_run[0]) == ref["iterations_run"]
    assert st["replay_columns"] > 0 and st["reseeds"] > 0, st


def test_native_sharded_pq_fit_matches_single_gpu():
    import torch

    from paper_2604_21645_b200 import dist as D
    from paper_2604_21645_b200 import pqii
    from paper_2604_21645_b200.datagen import gaussian_mixture
    x = gaussian_mixture(30011, 64, 32, seed=17)
    be = D.CudaBackend(0, private=True)
    nc = _one_rank(be)
    try:
        st = {}
        fit = D.kmeans_fit_sharded_native(nc, torch.from_numpy(x).cuda(), 8, 8, 8, 256, 12,
                                          [5 + m for m in range(8)], 1e-4, stats=st)
    finally:
        nc.close()
    stats = {}
    cb = pqii.pq_fit(x, 8, 256, 12, 5, stats=stats)
    assert np.array_equal(fit.tables.cpu().numpy().view(np.uint32), cb.tables.view(np.uint32))
    assert np.array_equal(np.asarray(fit.iterations_run), stats["iterations_run"])
    assert st["allreduce_bytes"] // st["iterations"] == 8 * 256 * 64 + 8 * 8 * 256 + 8 * 8 + 2 * 256 * 64


def test_native_sharded_errors():
    import torch

    from paper_2604_21645_b200 import dist as D
    be = D.CudaBackend(0, private=True)
    nc = _one_rank(be)
    try:
        x = torch.randn(10, 8, device="cuda")
        with pytest.raises(Exception, match="exceeds number of points"):
            D.kmeans_fit_sharded_native(nc, x, 1, 8, 0, 11, 5, [1], 0.0)
        with pytest.raises(Exception, match="max_iters"):
            D.kmeans_fit_sharded_native(nc, x, 1, 8, 0, 3, 0, [1], 0.0)
    finally:
        nc.close()
