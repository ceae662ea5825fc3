"""Row-sharded multi-GPU driver, one process per GPU.

GPU g owns the contiguous global rows ``chunk_rows(N, P)[g]``
(proj/src/dataset_io.cpp:322-339), the B200 replacement of the paper's CPU
row chunking.  ``torch.distributed`` carries the exchanges
(NCCL on GPUs, gloo in the CPU tests); the per-shard compute goes through a
*backend* -- ``CudaBackend`` (libpqg.so via the C ABI) in production.  The
exchange logic is backend-independent so it is tested on CPU with gloo and
an oracle-backed backend (tests/test_dist_gloo.py).

* ``kmeans_fit_sharded`` -- exact: each rank runs the assignment pass on its
  shard of the training sample, assignments + fp64 distances are
  all-gathered in global row order, and every rank runs the reference's
  ordered update (proj/src/kmeans.cpp:102-130) on the replicated sample, so
  the result is bit-identical to single-process ``kmeans_fit`` / ``pq_fit``.
* ``encode_sharded`` -- shard-local encode, global SSE by one all-reduce.
* ``search_sharded`` -- shard-local index + search, all-gather of the
  per-shard top-k lists, merge by (dist, id): equal to the monolithic
  ``ivf_query`` because shards are ascending id ranges and lists are stable.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np


def chunk_rows(n_rows: int, n_chunks: int) -> list[tuple[int, int]]:
    """proj/src/dataset_io.cpp:322-339: the first n % c ranges carry one extra row."""
    if n_chunks == 0:
        raise ValueError("chunk_rows: n_chunks must be >= 1")
    if n_chunks > n_rows:
        raise ValueError(f"chunk_rows: n_chunks ({n_chunks}) exceeds n_rows ({n_rows})")
    base, extra = divmod(n_rows, n_chunks)
    out, start = [], 0
    for i in range(n_chunks):
        ln = base + (1 if i < extra else 0)
        out.append((start, start + ln))
        start += ln
    return out


def kmeans_stop(it: int, max_iters: int, prev: float, inertia: float, tol: float) -> bool:
    """The stop rule of proj/src/kmeans.cpp:98-99 (IEEE double, as on the device)."""
    if it > 1 and prev - inertia < tol * max(1.0, prev):
        return True
    return it == max_iters


# ---------------------------------------------------------------------------
# collectives (torch.distributed); arrays travel as torch tensors
# ---------------------------------------------------------------------------
class Comm:
    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = "cuda" if dist.get_backend(group) == "nccl" else "cpu"

    _SIGNED = {np.dtype(np.uint32): np.int32, np.dtype(np.uint64): np.int64,
               np.dtype(np.uint16): np.int16}

    def _t(self, a):
        """numpy -> torch on the collective's device; unsigned dtypes travel as
        same-width signed views (gloo has no unsigned 32/64-bit types)."""
        import torch
        a = np.ascontiguousarray(a)
        if a.dtype in self._SIGNED:
            a = a.view(self._SIGNED[a.dtype])
        return torch.from_numpy(a).to(self.device)

    @staticmethod
    def _back(t, dtype):
        return t.cpu().numpy().view(dtype)

    def allgather_rows(self, a: np.ndarray, counts: list[int]) -> np.ndarray:
        """Concatenate per-rank arrays (first axis sizes ``counts``) in rank order."""
        import torch
        mx = max(counts)
        pad = np.zeros((mx,) + a.shape[1:], a.dtype)
        pad[: a.shape[0]] = a
        t = self._t(pad)
        outs = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(outs, t, group=self.group)
        return np.concatenate([self._back(o, a.dtype)[:c] for o, c in zip(outs, counts)])

    def allgather_cols(self, a: np.ndarray, counts: list[int]) -> np.ndarray:
        """a is [B, n_local]; returns [B, sum(counts)] in rank order."""
        g = self.allgather_rows(np.ascontiguousarray(a.T), counts)
        return np.ascontiguousarray(g.T)

    def allreduce_sum(self, x: float) -> float:
        import torch
        t = self._t(np.array([x], np.float64))
        self.dist.all_reduce(t, group=self.group)
        return float(t.cpu().numpy()[0])

    def allgather_equal(self, a: np.ndarray) -> np.ndarray:
        import torch
        a = np.ascontiguousarray(a)
        t = self._t(a)
        outs = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(outs, t, group=self.group)
        return np.stack([self._back(o, a.dtype) for o in outs])


# ---------------------------------------------------------------------------
# production backend: libpqg.so
# ---------------------------------------------------------------------------
class CudaBackend:
    """Shard-local compute through the C ABI (include/pqg.h)."""

    def __init__(self, device: int = 0):
        from . import _lib, pqii
        self.L = _lib
        self.pqii = pqii
        self.ctx = pqii.get_context(device)
        self.lib = self.ctx.lib

    def _v(self, a):
        return a.ctypes.data_as(C.c_void_p)

    def init_rows(self, n, k, seed):
        out = np.empty(k, np.uint64)
        self.L.check(self.lib.pqg_kmeans_init_rows(n, k, seed, self._v(out)), "init")
        return out

    def assign_pass(self, rows, B, d, col_stride, tables):
        rows = np.ascontiguousarray(rows, np.float32)
        n, ld = rows.shape
        k = tables.shape[1]
        a = np.empty((B, n), np.uint32)
        dist = np.empty((B, n), np.float64)
        self.L.check(self.lib.pqg_assign_pass(self.ctx.h, self._v(rows), n, ld, B, d, col_stride,
                                              self._v(np.ascontiguousarray(tables)), k, self._v(a),
                                              self._v(dist)), "assign_pass")
        return a, dist

    def rows_sum(self, v):
        v = np.ascontiguousarray(v, np.float64)
        B, n = v.shape
        out = np.empty(B, np.float64)
        self.L.check(self.lib.pqg_rows_sum_f64(self.ctx.h, self._v(v), n, B, self._v(out)), "sum")
        return out

    def update_pass(self, rows, B, d, col_stride, tables, assign, dist, active):
        rows = np.ascontiguousarray(rows, np.float32)
        n, ld = rows.shape
        k = tables.shape[1]
        act = np.ascontiguousarray(active, np.int32)
        self.L.check(self.lib.pqg_update_pass(self.ctx.h, self._v(rows), n, ld, B, d, col_stride,
                                              self._v(tables), k, self._v(np.ascontiguousarray(assign)),
                                              self._v(dist), self._v(act)), "update_pass")

    def encode_sse(self, rows, tables):
        rows = np.ascontiguousarray(rows, np.float32)
        M, ks, ds = tables.shape
        codes = np.empty((rows.shape[0], M * (1 if ks <= 256 else 2)), np.uint8)
        sse = C.c_double()
        self.L.check(self.lib.pqg_pq_encode_sse(self.ctx.h, self._v(rows), rows.shape[0], M, ks, ds,
                                                self._v(np.ascontiguousarray(tables)),
                                                self._v(codes), C.byref(sse)), "encode")
        return codes, sse.value

    def search_local(self, tables, codes, ids, coarse, queries, k, nprobe):
        pq = self.pqii
        M, ks, ds = tables.shape
        cb = pq.Codebook(M, ks, ds, np.ascontiguousarray(tables))
        cm = pq.CodeMatrix(codes.shape[0], M, ks, np.ascontiguousarray(codes))
        index = pq.ivf_build_with_centroids(cb, cm, ids, coarse)
        return pq.ivf_query_batch(index, queries, k, nprobe)

    def topk_merge(self, ids, dists, counts, k):
        S, nq, _ = ids.shape
        oi = np.zeros((nq, k), np.uint64)
        od = np.zeros((nq, k), np.float64)
        oc = np.zeros(nq, np.uint32)
        self.L.check(self.lib.pqg_topk_merge(
            self.ctx.h, self._v(np.ascontiguousarray(ids, np.uint64)),
            self._v(np.ascontiguousarray(dists, np.float64)),
            self._v(np.ascontiguousarray(counts, np.uint32)), S, nq, k, self._v(oi), self._v(od),
            self._v(oc)), "topk_merge")
        return oi, od, oc


# ---------------------------------------------------------------------------
# sharded algorithms
# ---------------------------------------------------------------------------
@dataclass
class ShardedFit:
    tables: np.ndarray          # [B, k, d]
    assignments: np.ndarray     # [B, N] (global row order)
    inertia: np.ndarray         # [B]
    iterations_run: np.ndarray  # [B]
    inertia_per_iter: list


def kmeans_fit_sharded(comm: Comm, backend, local_rows: np.ndarray, B: int, d: int,
                       col_stride: int, k: int, max_iters: int, seeds, tol: float = 1e-4) -> ShardedFit:
    """B batched k-means problems (B = M subspaces for pq_fit, B = 1 for the
    coarse quantizer) over rows sharded by rank; bit-identical to the
    single-process fit (see module docstring)."""
    counts = [int(c) for c in comm.allgather_equal(np.array([local_rows.shape[0]], np.int64))[:, 0]]
    n = sum(counts)
    if k == 0:
        raise ValueError("kmeans_fit: k must be >= 1")
    if k > n:
        raise ValueError(f"kmeans_fit: k ({k}) exceeds number of points ({n})")
    if max_iters < 1:
        raise ValueError("kmeans_fit: max_iters must be >= 1")
    full = comm.allgather_rows(np.ascontiguousarray(local_rows, np.float32), counts)
    offset = sum(counts[: comm.rank])
    tables = np.empty((B, k, d), np.float32)
    for b in range(B):  # init rows: the reference's draws, identical on every rank
        rows = backend.init_rows(n, k, int(seeds[b])).astype(np.int64)
        tables[b] = full[rows, b * col_stride: b * col_stride + d]
    active = np.ones(B, np.int32)
    prev = np.zeros(B)
    inertia = np.zeros(B)
    iters = np.zeros(B, np.uint32)
    per_iter = [[] for _ in range(B)]
    assign_full = np.zeros((B, n), np.uint32)
    for it in range(1, max_iters + 1):
        a_loc, d_loc = backend.assign_pass(local_rows, B, d, col_stride, tables)
        a_full = comm.allgather_cols(a_loc, counts)
        d_full = comm.allgather_cols(d_loc, counts)
        sums = backend.rows_sum(d_full)
        for b in range(B):
            if not active[b]:
                continue
            assign_full[b] = a_full[b]
            inertia[b] = sums[b]
            per_iter[b].append(float(sums[b]))
            iters[b] = it
            if kmeans_stop(it, max_iters, prev[b], sums[b], tol):
                active[b] = 0
            else:
                prev[b] = sums[b]
        if not active.any():
            break
        backend.update_pass(full, B, d, col_stride, tables, a_full, d_full, active)
    del offset
    return ShardedFit(tables, assign_full, inertia, iters, per_iter)


def pq_fit_sharded(comm: Comm, backend, local_rows: np.ndarray, M: int, ks: int,
                   max_iters: int = 20, seed: int = 0) -> np.ndarray:
    """pq_fit (proj/src/pq.cpp:63-93) over row shards: subspace m uses seed + m."""
    D = local_rows.shape[1]
    if M == 0 or D % M:
        raise ValueError(f"pq_fit: D ({D}) is not divisible by M ({M})")
    ds = D // M
    fit = kmeans_fit_sharded(comm, backend, local_rows, M, ds, ds, ks, max_iters,
                             [seed + m for m in range(M)], 1e-4)
    return fit.tables


def encode_sharded(comm: Comm, backend, local_rows: np.ndarray, tables: np.ndarray):
    """Shard-local codes and the GLOBAL reconstruction RMSE (one all-reduce)."""
    codes, sse = backend.encode_sse(local_rows, tables)
    n = comm.allreduce_sum(float(local_rows.shape[0]))
    total = comm.allreduce_sum(sse)
    return codes, float(np.sqrt(total / (n * local_rows.shape[1])))


def search_sharded(comm: Comm, backend, tables, local_codes, local_ids, coarse, queries, k: int,
                   nprobe: int):
    """Shard-local index + search, then all-gather and (dist, id) merge."""
    ids, dists, counts = backend.search_local(tables, local_codes, local_ids, coarse, queries, k,
                                              nprobe)
    all_ids = comm.allgather_equal(np.ascontiguousarray(ids, np.uint64))
    all_d = comm.allgather_equal(np.ascontiguousarray(dists, np.float64))
    all_c = comm.allgather_equal(np.ascontiguousarray(counts, np.uint32))
    return backend.topk_merge(all_ids, all_d, all_c, k)
