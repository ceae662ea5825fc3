"""The sharded k-means exchange at world 2 and 3 on ONE GPU, in-process: each
rank is a host thread with its own library context and CUDA stream, the
collectives are host-mediated (threading barrier + torch ops), so no rank's
kernels ever wait on another's.  This runs the device side of the north-star
exchange (pqg_kmshard_*: all-reduced partial sums / counts / exponent
ranges, the all-gathered row-order replay, the reseed candidates) with real
shards and checks it against the single-process fit and the oracle."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


class _ThreadDist:
    """The torch.distributed calls dist.Comm makes, between host threads."""

    class ReduceOp:
        SUM = "sum"
        MAX = "max"

    def __init__(self, rank, world, shared):
        self.rank, self.world, self.sh = rank, world, shared

    def get_rank(self, group=None):
        return self.rank

    def get_world_size(self, group=None):
        return self.world

    def _exchange(self, t):
        import torch
        torch.cuda.current_stream().synchronize()
        self.sh["slots"][self.rank] = t.clone()
        self.sh["bar"].wait()
        got = list(self.sh["slots"])
        self.sh["bar"].wait()
        return got

    def all_gather(self, outs, t, group=None):
        for o, g in zip(outs, self._exchange(t)):
            o.copy_(g.to(o.device))

    def send(self, t, dst, group=None):
        import torch
        torch.cuda.current_stream().synchronize()
        with self.sh["cv"]:
            self.sh["p2p"][(self.rank, dst)] = t.clone()
            self.sh["cv"].notify_all()

    def recv(self, t, src, group=None):
        with self.sh["cv"]:
            self.sh["cv"].wait_for(lambda: (src, self.rank) in self.sh["p2p"], timeout=120)
            t.copy_(self.sh["p2p"].pop((src, self.rank)).to(t.device))

    def broadcast(self, t, src, group=None):
        t.copy_(self._exchange(t)[src].to(t.device))

    def all_reduce(self, t, op="sum", group=None, async_op=False):
        import torch
        got = self._exchange(t)
        acc = got[0].clone()
        for g in got[1:]:
            acc = acc + g if op == "sum" else torch.maximum(acc, g)
        t.copy_(acc)

        class _Done:
            def wait(self):
                return True
        return _Done() if async_op else None


def _run_world(world, x, fn):
    import torch

    from paper_2604_21645_b200 import dist as D
    shared = {"slots": [None] * world, "bar": threading.Barrier(world), "cv": threading.Condition(), "p2p": {}}
    out, errs = [None] * world, []

    def body(rank):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                comm = D.Comm.__new__(D.Comm)
                comm.dist = _ThreadDist(rank, world, shared)
                comm.group, comm.rank, comm.world = None, rank, world
                be = D.CudaBackend(0, private=True)
                be.ctx.set_stream(s.cuda_stream)
                lo, hi = D.chunk_rows(x.shape[0], world)[rank]
                local = torch.from_numpy(np.ascontiguousarray(x[lo:hi])).cuda()
                out[rank] = fn(comm, be, local)
                s.synchronize()
        except Exception as e:  # surfaced below
            errs.append(e)
            shared["bar"].abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return out


def _stress():
    import sys
    import os
    sys.path.insert(0, os.path.dirname(__file__))
    from dist_workers import stress_data
    return stress_data()


@pytest.mark.parametrize("replay", ["chain", "gather"])
@pytest.mark.parametrize("world", [1, 2, 3])
def test_kmshard_coarse_exchange_paths(orc, world, replay):
    """Both replay protocols -- the chain handed rank to rank (r2e default)
    and the all-gathered members (r2) -- equal the oracle bit for bit."""
    from paper_2604_21645_b200 import dist as D
    x = _stress()
    st = [dict() for _ in range(world)]

    def fn(comm, be, local):
        return D.kmeans_fit_sharded(comm, be, local, 1, 8, 0, 40, 9, [2], 0.0, stats=st[comm.rank],
                                    force_exchange=True, replay=replay)
    res = _run_world(world, x, fn)
    ref = orc.kmeans_fit(x, 40, 9, 2, 0.0)
    for r in res:
        assert np.array_equal(r.tables[0].cpu().numpy().view(np.uint32), ref["centroids"].view(np.uint32))
        assert np.array_equal(r.assignments[0].cpu().numpy().view(np.uint32), ref["assignments"])
        assert int(r.iterations_run[0]) == ref["iterations_run"]
    assert st[0]["replay_columns"] > 0 and st[0]["reseeds"] > 0


@pytest.mark.parametrize("world", [2, 4])
def test_kmshard_pq_fit_matches_single_gpu(world):
    """Sharded pq_fit (M subspace problems per rank) == the single-process
    device fit, and the per-iteration all-reduce volume is the north star's
    8*Ks*D + 8*M*Ks (+ inertia) bytes, plus the u8 exponent ranges."""
    from paper_2604_21645_b200 import dist as D
    from paper_2604_21645_b200 import pqii
    from paper_2604_21645_b200.datagen import gaussian_mixture
    x = gaussian_mixture(30011, 64, 32, seed=17)
    st = [dict() for _ in range(world)]

    def fn(comm, be, local):
        return D.kmeans_fit_sharded(comm, be, local, 8, 8, 8, 256, 12, [5 + m for m in range(8)], 1e-4,
                                    stats=st[comm.rank])
    res = _run_world(world, x, fn)
    stats = {}
    cb = pqii.pq_fit(x, 8, 256, 12, 5, stats=stats)
    for r in res:
        assert np.array_equal(r.tables.cpu().numpy().view(np.uint32), cb.tables.view(np.uint32))
        assert np.array_equal(np.asarray(r.iterations_run), stats["iterations_run"])
    per_iter = st[0]["allreduce_bytes"] / st[0]["iterations"]
    assert per_iter == 8 * 256 * 64 + 8 * 8 * 256 + 8 * 8 + 2 * 256 * 64


@pytest.mark.parametrize("B,d,k", [(1, 8, 40), (8, 8, 256)])
def test_kmshard_one_rank_delegation(B, d, k):
    """A 1-rank group runs the single-process fit: same tables, assignments,
    iterations and inertia as the exchange protocol forced at world 1."""
    from paper_2604_21645_b200 import dist as D
    x = _stress() if B == 1 else __import__("paper_2604_21645_b200.datagen", fromlist=["x"]).gaussian_mixture(
        9001, 64, 32, seed=3)
    seeds = [2] if B == 1 else [5 + m for m in range(B)]
    tol = 0.0 if B == 1 else 1e-4
    st_d, st_f = {}, {}
    cs = 0 if B == 1 else d
    rd = _run_world(1, x, lambda comm, be, local: D.kmeans_fit_sharded(comm, be, local, B, d, cs, k, 9, seeds, tol,
                                                                       stats=st_d))[0]
    rf = _run_world(1, x, lambda comm, be, local: D.kmeans_fit_sharded(comm, be, local, B, d, cs, k, 9, seeds, tol,
                                                                       stats=st_f, force_exchange=True))[0]
    assert st_d.get("path", "").startswith("1-rank") and "path" not in st_f
    assert np.array_equal(rd.tables.cpu().numpy().view(np.uint32), rf.tables.cpu().numpy().view(np.uint32))
    assert np.array_equal(rd.assignments.cpu().numpy(), rf.assignments.cpu().numpy())
    assert np.array_equal(np.asarray(rd.iterations_run), np.asarray(rf.iterations_run))
    assert rd.inertia_per_iter == rf.inertia_per_iter
