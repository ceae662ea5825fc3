"""The sharded driver on a GPU with NCCL (torchrun, one rank per visible GPU,
world 1 on a single-GPU box): sharded pq_fit / k-means / encode / search
equal the single-process C ABI results bit-for-bit."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_sharded_pipeline_nccl(tmp_path):
    import torch
    from paper_2604_21645_b200 import pqii
    from paper_2604_21645_b200.datagen import gaussian_mixture
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    nproc = max(1, torch.cuda.device_count())
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={nproc}", "--master-addr", "127.0.0.1",
                        "--master-port", str(port), os.path.join(ROOT, "tests", "dist_gpu_worker.py"),
                        str(tmp_path)], capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    r = np.load(tmp_path / "dist_gpu.npz")
    x = gaussian_mixture(20011, 64, 32, seed=13)
    cb = pqii.pq_fit(x, 8, 64, 12, 4)
    assert np.array_equal(r["tables"].view(np.uint32), cb.tables.view(np.uint32))
    codes = pqii.pq_encode(cb, x)
    assert np.array_equal(r["codes"], codes.bytes)
    ref_rmse = pqii.reconstruction_rmse(cb, x)
    assert abs(float(r["rmse"][0]) - ref_rmse) <= 1e-12 * ref_rmse
    km = pqii.kmeans_fit(x, 128, 10, 3)
    assert np.array_equal(r["coarse"].view(np.uint32), km.centroids.view(np.uint32))
    assert np.array_equal(r["assign"][0].view(np.uint32), km.assignments)
    ids = np.arange(20011, dtype=np.uint64) * 5 + 2
    index = pqii.ivf_build_with_centroids(cb, codes, ids, km.centroids)
    q = gaussian_mixture(50, 64, 32, seed=13, stream=1)
    gi, gd, gc = pqii.ivf_query_batch(index, q, 10, 8)
    assert np.array_equal(r["c"].view(np.uint32), gc)
    assert np.array_equal(r["ids"].view(np.uint64), gi)
    assert np.array_equal(r["d"].view(np.uint64), gd.view(np.uint64))
