"""Row-sharded multi-GPU driver, one process per GPU.

GPU g owns the contiguous global rows ``chunk_rows(N, P)[g]``
(proj/src/dataset_io.cpp:322-339), the B200 replacement of the paper's CPU
row chunking.  ``torch.distributed`` carries the exchanges
(NCCL on GPUs, gloo in the CPU tests) on torch tensors that stay on the
device; the per-shard compute goes through a *backend* -- ``CudaBackend``
(libpqg.so via the C ABI, device pointers) in production.  The exchange
logic is backend-independent, so it is tested on CPU with gloo and an
oracle-backed backend (tests/test_dist_gloo.py) and on a GPU with NCCL
(tests/test_dist_gpu.py).

* ``kmeans_fit_sharded`` -- the north-star exchange, exact: per iteration
  each rank assigns its block of the training sample and computes its exact
  per-(problem, cluster, dim) fp64 sums, exponent ranges, counts and inertia
  on the device (``pqg_kmshard_partials``); ONE all-reduce SUM of the fp64
  partials (Ks x D sums + counts + inertia) and one all-reduce MAX of the u8
  exponent ranges carry the iteration; every rank then finalizes
  identically (``pqg_kmshard_apply``): sums whose global exponent range
  proves them exact are the reference's row-order sums
  (proj/src/kmeans.cpp:103-118), the rare rest are replayed in global row
  order from the members the ranks all-gather, and empty clusters are
  reseeded from every rank's best candidates (:122-130).  The result is
  bit-identical to single-process ``kmeans_fit`` / ``pq_fit``.  Shapes the
  device partials do not cover (d % 4 != 0, d > 128) use the replicated
  update: assignments + distances all-gathered, the ordered update on every
  rank.
* ``encode_sharded`` -- shard-local encode, global SSE by one all-reduce.
* ``search_sharded`` -- shard-local index + search, all-gather of the
  per-shard top-k lists, merge by (dist, id): equal to the monolithic
  ``ivf_query`` because shards are ascending id ranges and lists are stable.

Unsigned 32/64-bit values travel as same-width signed tensors (int32/int64
bit patterns): gloo and parts of torch have no unsigned types.
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
# collectives on torch tensors
# ---------------------------------------------------------------------------
class Comm:
    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def allgather_rows(self, t, counts: list[int]):
        """Concatenate per-rank tensors (first-axis sizes ``counts``) in rank order."""
        import torch
        mx = max(counts)
        pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
        outs = [torch.empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(outs, pad, group=self.group)
        return torch.cat([o[:c] for o, c in zip(outs, counts)])

    def allgather_cols(self, t, counts: list[int]):
        """t is [B, n_local]; returns [B, sum(counts)] in rank order."""
        return self.allgather_rows(t.t().contiguous(), counts).t().contiguous()

    def allreduce_sum(self, x: float, device) -> float:
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=device)
        self.dist.all_reduce(t, group=self.group)
        return float(t.item())

    def allreduce_(self, t, op="sum"):
        """In-place all-reduce of a tensor (SUM or MAX); a 1-rank group has
        nothing to exchange."""
        if self.world == 1:
            return t
        rop = self.dist.ReduceOp.SUM if op == "sum" else self.dist.ReduceOp.MAX
        self.dist.all_reduce(t, op=rop, group=self.group)
        return t

    def allreduce_pair_(self, a, b):
        """SUM-reduce a and MAX-reduce b, both in flight together."""
        if self.world == 1:
            return
        w1 = self.dist.all_reduce(a, op=self.dist.ReduceOp.SUM, group=self.group, async_op=True)
        w2 = self.dist.all_reduce(b, op=self.dist.ReduceOp.MAX, group=self.group, async_op=True)
        w1.wait()
        w2.wait()

    def allgather_padded(self, t):
        """1-D tensors of per-rank lengths -> ([world, stride] padded stack, stride)."""
        import torch
        n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
        sizes = [int(v) for v in self.allgather_equal(n).view(-1).tolist()]
        stride = max(1, max(sizes))
        pad = torch.zeros(stride, dtype=t.dtype, device=t.device)
        pad[: t.numel()] = t
        return self.allgather_equal(pad), stride

    def _peer(self, r: int) -> int:
        return r if self.group is None else self.dist.get_global_rank(self.group, r)

    def recv_prev_(self, t):
        """Rank r > 0 receives t (in place) from rank r - 1."""
        if self.rank > 0:
            self.dist.recv(t, src=self._peer(self.rank - 1), group=self.group)
        return t

    def send_next(self, t):
        """Rank r < world - 1 sends t to rank r + 1."""
        if self.rank < self.world - 1:
            self.dist.send(t.contiguous(), dst=self._peer(self.rank + 1), group=self.group)

    def broadcast_(self, t, src: int):
        if self.world > 1:
            self.dist.broadcast(t, src=self._peer(src), group=self.group)
        return t

    def allgather_equal(self, t):
        """[world, *t.shape]: every rank's equally shaped t, rank order."""
        import torch
        t = t.contiguous()
        if self.world == 1:
            return t.unsqueeze(0)
        out = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        if hasattr(self.dist, "all_gather_into_tensor") and t.is_cuda:
            self.dist.all_gather_into_tensor(out, t, group=self.group)
        else:
            self.dist.all_gather(list(out.unbind(0)), t, group=self.group)
        return out


# ---------------------------------------------------------------------------
# production backend: libpqg.so on device tensors
# ---------------------------------------------------------------------------
class CudaBackend:
    """Shard-local compute through the C ABI (include/pqg.h) on CUDA tensors."""

    def __init__(self, device: int = 0, private: bool = False):
        import torch

        from . import _lib, pqii
        self.torch = torch
        self.L = _lib
        self.pqii = pqii
        self.device = torch.device("cuda", device)
        # private: a context of its own (several backends driven from threads)
        self.ctx = pqii.Context(device) if private else pqii.get_context(device)
        self.lib = self.ctx.lib
        # libpqg runs on torch's current stream so collectives and kernels order;
        # torch's default stream is the legacy stream (handle 0 -> cudaStreamLegacy)
        self.ctx.set_stream(torch.cuda.current_stream(self.device).cuda_stream or 1)

    @staticmethod
    def _p(t):
        return C.c_void_p(t.data_ptr())

    def init_rows(self, n, k, seed):
        out = np.empty(k, np.uint64)
        self.L.check(self.lib.pqg_kmeans_init_rows(n, k, seed, out.ctypes.data_as(C.c_void_p)), "init")
        return out

    def assign_pass(self, rows, B, d, col_stride, tables):
        torch = self.torch
        n, ld = rows.shape
        k = tables.shape[1]
        a = torch.empty((B, n), dtype=torch.int32, device=rows.device)
        dist = torch.empty((B, n), dtype=torch.float64, device=rows.device)
        self.L.check(self.lib.pqg_assign_pass(self.ctx.h, self._p(rows), n, ld, B, d, col_stride,
                                              self._p(tables), k, self._p(a), self._p(dist)),
                     "assign_pass")
        return a, dist

    def rows_sum(self, v):
        B, n = v.shape
        out = np.empty(B, np.float64)
        self.L.check(self.lib.pqg_rows_sum_f64(self.ctx.h, self._p(v), n, B,
                                               out.ctypes.data_as(C.c_void_p)), "sum")
        return out

    def update_pass(self, rows, B, d, col_stride, tables, assign, dist, active):
        n, ld = rows.shape
        k = tables.shape[1]
        act = self.torch.as_tensor(np.ascontiguousarray(active, np.int32), device=rows.device)
        self.L.check(self.lib.pqg_update_pass(self.ctx.h, self._p(rows), n, ld, B, d, col_stride,
                                              self._p(tables), k, self._p(assign), self._p(dist),
                                              self._p(act)), "update_pass")

    def fit_local(self, rows, B, d, col_stride, k, max_iters, seeds, tol):
        """The single-process fit (pqg_kmeans_fit / pqg_pq_fit_ex) of a 1-rank
        group, or None where its seeds / layout are not those entry points'."""
        torch = self.torch
        n, ld = rows.shape
        iters = np.zeros(B, np.uint32)
        inertia = np.zeros(B, np.float64)
        per = np.zeros((B, max_iters), np.float64)
        v = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        tables = torch.empty((B, k, d), dtype=torch.float32, device=rows.device)
        if B == 1 and col_stride == 0 and ld == d:
            assign = torch.empty((1, n), dtype=torch.int32, device=rows.device)
            it, ine = C.c_uint32(), C.c_double()
            self.L.check(self.lib.pqg_kmeans_fit(self.ctx.h, self._p(rows), n, d, k, max_iters, int(seeds[0]), tol,
                                                 self._p(tables), self._p(assign), C.byref(ine), C.byref(it),
                                                 v(per)), "kmeans_fit")
            iters[0], inertia[0] = it.value, ine.value
            return tables, assign, inertia, iters, per
        if (col_stride == d and ld == B * d and tol == 1e-4 and
                all(int(seeds[b]) == int(seeds[0]) + b for b in range(B))):
            self.L.check(self.lib.pqg_pq_fit_ex(self.ctx.h, self._p(rows), n, ld, B, k, max_iters, int(seeds[0]),
                                                self._p(tables), v(iters), v(inertia), v(per)), "pq_fit")
            assign, _ = self.assign_pass(rows, B, d, col_stride, tables)  # the final pass's assignments
            return tables, assign, inertia, iters, per
        return None

    # -- one rank's side of the sharded fit (include/pqg.h pqg_kmshard_*) --
    def shard_create(self, rows, B, d, col_stride, k, max_iters, tol):
        """A device handle, or None where the sharded update does not apply."""
        h = C.c_void_p()
        n, ld = rows.shape
        rc = self.lib.pqg_kmshard_create(self.ctx.h, self._p(rows), n, ld, B, d, col_stride, k,
                                         max_iters, tol, C.byref(h))
        if rc == self.L.PQG_EUNSUPPORTED:
            return None
        self.L.check(rc, "kmshard_create")
        nf, nu = C.c_uint64(), C.c_uint64()
        self.L.check(self.lib.pqg_kmshard_sizes(h, C.byref(nf), C.byref(nu)), "kmshard_sizes")
        return {"h": h, "rows": rows, "B": B, "d": d, "k": k, "n": n, "max_iters": max_iters,
                "nf": nf.value, "nu": nu.value}

    def shard_destroy(self, s):
        self.lib.pqg_kmshard_destroy(s["h"])

    def shard_init_table(self, s, init_rows, row0):
        bits = self.torch.empty((s["B"], s["k"], s["d"]), dtype=self.torch.int32, device=s["rows"].device)
        init = np.ascontiguousarray(init_rows, np.uint64)
        self.L.check(self.lib.pqg_kmshard_init_table(self.ctx.h, s["h"], init.ctypes.data_as(C.c_void_p),
                                                     row0, self._p(bits)), "kmshard_init")
        return bits

    def shard_partials(self, s, tables):
        torch = self.torch
        dev = s["rows"].device
        if "f64" not in s:  # reused every iteration
            s["f64"] = torch.empty(s["nf"], dtype=torch.float64, device=dev)
            s["u8"] = torch.empty(s["nu"], dtype=torch.uint8, device=dev)
        f64, u8 = s["f64"], s["u8"]
        self.L.check(self.lib.pqg_kmshard_partials(self.ctx.h, s["h"], self._p(tables), self._p(f64),
                                                   self._p(u8)), "kmshard_partials")
        return f64, u8

    def shard_apply(self, s, tables, f64, u8):
        nf, stride, me, aa = C.c_uint64(), C.c_uint64(), C.c_uint32(), C.c_int()
        self.L.check(self.lib.pqg_kmshard_apply(self.ctx.h, s["h"], self._p(tables), self._p(f64), self._p(u8),
                                                C.byref(nf), C.byref(stride), C.byref(me), C.byref(aa)),
                     "kmshard_apply")
        s["stride"] = stride.value
        return nf.value, me.value, bool(aa.value)

    def shard_pack(self, s, n_fail):
        """(vals [stride] padded, offcnt [2*n_fail]): this rank's replay members."""
        torch = self.torch
        dev = s["rows"].device
        vals = torch.empty(s["stride"], dtype=torch.float32, device=dev)
        offcnt = torch.empty(2 * n_fail, dtype=torch.int64, device=dev)
        self.L.check(self.lib.pqg_kmshard_pack(self.ctx.h, s["h"], self._p(vals), vals.numel(), self._p(offcnt)),
                     "kmshard_pack")
        return vals, offcnt

    def shard_replay(self, s, tables, f64, all_vals, stride, all_offcnt, world):
        self.L.check(self.lib.pqg_kmshard_replay(self.ctx.h, s["h"], self._p(tables), self._p(f64),
                                                 self._p(all_vals.contiguous()), stride,
                                                 self._p(all_offcnt.contiguous()), world), "kmshard_replay")

    def shard_replay_step(self, s, run):
        self.L.check(self.lib.pqg_kmshard_replay_step(self.ctx.h, s["h"], self._p(run)), "kmshard_replay_step")

    def shard_replay_finish(self, s, tables, f64, run):
        self.L.check(self.lib.pqg_kmshard_replay_finish(self.ctx.h, s["h"], self._p(tables), self._p(f64),
                                                        self._p(run)), "kmshard_replay_finish")

    def shard_reseed_candidates(self, s, row0, E):
        torch = self.torch
        dev = s["rows"].device
        B, d = s["B"], s["d"]
        cd = torch.empty((B, E + 1), dtype=torch.float64, device=dev)
        ci = torch.empty((B, E + 1), dtype=torch.int64, device=dev)
        cr = torch.empty((B, E + 1, d), dtype=torch.float32, device=dev)
        self.L.check(self.lib.pqg_kmshard_reseed_candidates(self.ctx.h, s["h"], row0, E, self._p(cd), self._p(ci),
                                                            self._p(cr)), "kmshard_reseed")
        return cd, ci, cr

    def shard_reseed_apply(self, s, tables, f64, E, world, all_d, all_i, all_r):
        self.L.check(self.lib.pqg_kmshard_reseed_apply(self.ctx.h, s["h"], self._p(tables), self._p(f64), E, world,
                                                       self._p(all_d.contiguous()), self._p(all_i.contiguous()),
                                                       self._p(all_r.contiguous())), "kmshard_reseed")

    def shard_result(self, s):
        B, mi = s["B"], s["max_iters"]
        iters = np.empty(B, np.uint32)
        inertia = np.empty(B, np.float64)
        per = np.empty((B, mi), np.float64)
        assign = self.torch.empty((B, s["n"]), dtype=self.torch.int32, device=s["rows"].device)
        v = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        self.L.check(self.lib.pqg_kmshard_result(self.ctx.h, s["h"], v(iters), v(inertia), v(per),
                                                 self._p(assign)), "kmshard_result")
        return iters, inertia, per, assign

    def encode_sse(self, rows, tables):
        torch = self.torch
        M, ks, ds = tables.shape
        codes = torch.empty((rows.shape[0], M * (1 if ks <= 256 else 2)), dtype=torch.uint8,
                            device=rows.device)
        sse = C.c_double()
        self.L.check(self.lib.pqg_pq_encode_sse(self.ctx.h, self._p(rows), rows.shape[0], M, ks, ds,
                                                self._p(tables), self._p(codes), C.byref(sse)),
                     "encode")
        return codes, sse.value

    def search_local(self, tables, codes, ids, coarse, queries, k, nprobe):
        torch = self.torch
        M, ks, ds = tables.shape
        h = C.c_void_p()
        self.L.check(self.lib.pqg_ivf_build_with_centroids(
            self.ctx.h, self._p(tables), M, ks, ds, self._p(codes), self._p(ids), codes.shape[0],
            self._p(coarse), coarse.shape[0], C.byref(h)), "ivf_build")
        nq = queries.shape[0]
        oi = torch.zeros((nq, k), dtype=torch.int64, device=queries.device)
        od = torch.zeros((nq, k), dtype=torch.float64, device=queries.device)
        oc = torch.zeros(nq, dtype=torch.int32, device=queries.device)
        try:
            self.L.check(self.lib.pqg_index_search(self.ctx.h, h, self._p(queries), nq, k, nprobe,
                                                   0, 0.0, self._p(oi), self._p(od), self._p(oc)),
                         "search")
        finally:
            self.lib.pqg_index_destroy(h)
        return oi, od, oc

    def topk_merge(self, ids, dists, counts, k):
        torch = self.torch
        S, nq, _ = ids.shape
        oi = torch.zeros((nq, k), dtype=torch.int64, device=ids.device)
        od = torch.zeros((nq, k), dtype=torch.float64, device=ids.device)
        oc = torch.zeros(nq, dtype=torch.int32, device=ids.device)
        self.L.check(self.lib.pqg_topk_merge(self.ctx.h, self._p(ids.contiguous()),
                                             self._p(dists.contiguous()), self._p(counts.contiguous()),
                                             S, nq, k, self._p(oi), self._p(od), self._p(oc)),
                     "topk_merge")
        return oi, od, oc


# ---------------------------------------------------------------------------
# sharded algorithms
# ---------------------------------------------------------------------------
@dataclass
class ShardedFit:
    tables: object              # [B, k, d] float32 tensor
    assignments: object         # [B, N] int32 tensor (u32 bit patterns), global row order
    inertia: np.ndarray         # [B]
    iterations_run: np.ndarray  # [B]
    inertia_per_iter: list


def kmeans_fit_sharded(comm: Comm, backend, local_rows, B: int, d: int, col_stride: int, k: int,
                       max_iters: int, seeds, tol: float = 1e-4, stats: dict | None = None,
                       force_exchange: bool = False, replay: str | None = None) -> ShardedFit:
    """B batched k-means problems (B = M subspaces for pq_fit, B = 1 for the
    coarse quantizer) over rows sharded by rank; bit-identical to the
    single-process fit (see module docstring).  ``stats`` (optional) receives
    the exchange volume: bytes all-reduced / all-gathered per iteration.
    A 1-rank group has nothing to exchange: it runs the single-process fit
    (one device-resident graph per iteration, no host round trip) unless
    ``force_exchange`` (the tests drive the exchange protocol at world 1 too).
    ``replay``: "chain" (default; PQG_SHARD_REPLAY overrides) passes the
    row-order chains of the inexact columns rank to rank; "gather" is the r2
    protocol that all-gathers every rank's members of those columns."""
    import os

    import torch
    replay = replay or os.environ.get("PQG_SHARD_REPLAY", "chain")
    if replay not in ("chain", "gather"):
        raise ValueError(f"replay must be 'chain' or 'gather', not {replay!r}")
    dev = local_rows.device
    if comm.world == 1 and not force_exchange and hasattr(backend, "fit_local") and k >= 1 and \
            k <= local_rows.shape[0] and max_iters >= 1 and tol >= 0:
        r = backend.fit_local(local_rows.contiguous(), B, d, col_stride, k, max_iters, seeds, tol)
        if r is not None:
            tables, assign, inertia, iters, per = r
            if stats is not None:
                stats.update(allreduce_bytes=0, allgather_bytes=0, replay_columns=0, reseeds=0,
                             iterations=int(np.max(iters)), path="1-rank group: single-process fit")
            per_iter = [[float(v) for v in per[b, : iters[b]]] for b in range(B)]
            return ShardedFit(tables, assign, inertia, iters, per_iter)
    counts = [int(c) for c in comm.allgather_equal(
        torch.tensor([local_rows.shape[0]], dtype=torch.int64, device=dev)).view(-1).tolist()]
    n = sum(counts)
    if k == 0:
        raise ValueError("kmeans_fit: k must be >= 1")
    if k > n:
        raise ValueError(f"kmeans_fit: k ({k}) exceeds number of points ({n})")
    if max_iters < 1:
        raise ValueError("kmeans_fit: max_iters must be >= 1")
    if tol < 0:
        raise ValueError("kmeans_fit: tol must be >= 0")
    row0 = sum(counts[: comm.rank])
    s = backend.shard_create(local_rows.contiguous(), B, d, col_stride, k, max_iters, tol) \
        if hasattr(backend, "shard_create") and min(counts) > 0 else None
    if s is None:
        return _kmeans_fit_replicated(comm, backend, local_rows, counts, B, d, col_stride, k, max_iters,
                                      seeds, tol)
    st = stats if stats is not None else {}
    st.update(allreduce_bytes=0, allgather_bytes=0, chain_bytes=0, replay_columns=0, reseeds=0, iterations=0,
              replay=replay)
    try:
        init = np.concatenate([backend.init_rows(n, k, int(seeds[b])) for b in range(B)])
        bits = backend.shard_init_table(s, init, row0)
        comm.allreduce_(bits, "sum")  # owners' bit patterns, zeros elsewhere: exact
        tables = bits.view(torch.float32)
        for _ in range(max_iters):
            f64, u8 = backend.shard_partials(s, tables)
            comm.allreduce_pair_(f64, u8)
            st["allreduce_bytes"] += f64.numel() * 8 + u8.numel()
            st["iterations"] += 1
            n_fail, max_empty, any_active = backend.shard_apply(s, tables, f64, u8)
            if n_fail and replay == "chain":
                # columns whose sum may round: the row-order chain passes rank
                # to rank (one fp64 per column per hop), then the last rank's
                # sums are broadcast -- no member values cross ranks
                run = torch.zeros(n_fail, dtype=torch.float64, device=f64.device)
                comm.recv_prev_(run)
                backend.shard_replay_step(s, run)
                comm.send_next(run)
                comm.broadcast_(run, comm.world - 1)
                backend.shard_replay_finish(s, tables, f64, run)
                st["replay_columns"] += n_fail
                st["chain_bytes"] += 2 * run.numel() * 8 * (comm.world > 1)
            elif n_fail:  # r2 protocol: every rank's members all-gathered
                vals, offcnt = backend.shard_pack(s, n_fail)  # padded to the common stride
                all_vals, stride = comm.allgather_equal(vals), vals.numel()
                all_oc = comm.allgather_equal(offcnt)
                backend.shard_replay(s, tables, f64, all_vals, stride, all_oc, comm.world)
                st["replay_columns"] += n_fail
                st["allgather_bytes"] += all_vals.numel() * 4 + all_oc.numel() * 8
            if max_empty:
                cd, ci, cr = backend.shard_reseed_candidates(s, row0, max_empty)
                backend.shard_reseed_apply(s, tables, f64, max_empty, comm.world, comm.allgather_equal(cd),
                                           comm.allgather_equal(ci), comm.allgather_equal(cr))
                st["reseeds"] += 1
            if not any_active:
                break
        iters, inertia, per, assign = backend.shard_result(s)
    finally:
        backend.shard_destroy(s)
    per_iter = [[float(v) for v in per[b, : iters[b]]] for b in range(B)]
    return ShardedFit(tables, comm.allgather_cols(assign, counts), inertia, iters, per_iter)


class NcclComm:
    """The library's own NCCL communicator over the ranks of ``comm`` (one
    per GPU): rank 0 draws the unique id (``pqg_nccl_get_unique_id``), the
    torch group broadcasts it, every rank joins (``pqg_nccl_comm_init``).
    Used by :func:`kmeans_fit_sharded_native`, whose iteration loop runs in
    C++ (csrc/kmnccl.cu) with NCCL on the backend's stream."""

    def __init__(self, comm: Comm, backend):
        import torch
        self.backend, self.lib, self.L = backend, backend.lib, backend.L
        self.rank, self.world = comm.rank, comm.world
        on_gpu = comm.world > 1 and comm.dist.get_backend(comm.group) == "nccl"
        uid = torch.zeros(128, dtype=torch.uint8, device=backend.device if on_gpu else "cpu")
        host = np.zeros(128, np.uint8)
        if comm.rank == 0:
            self.L.check(self.lib.pqg_nccl_get_unique_id(host.ctypes.data_as(C.c_void_p)), "nccl_unique_id")
            uid.copy_(torch.from_numpy(host))
        comm.broadcast_(uid, 0)
        host = uid.cpu().numpy().copy()
        self.h = C.c_void_p()
        self.L.check(self.lib.pqg_nccl_comm_init(backend.device.index, comm.world, comm.rank,
                                                 host.ctypes.data_as(C.c_void_p), C.byref(self.h)),
                     "nccl_comm_init")

    def close(self):
        if self.h:
            self.lib.pqg_nccl_comm_destroy(self.h)
            self.h = C.c_void_p()


def kmeans_fit_sharded_native(ncomm: NcclComm, local_rows, B: int, d: int, col_stride: int, k: int,
                              max_iters: int, seeds, tol: float = 1e-4, stats: dict | None = None) -> ShardedFit:
    """kmeans_fit_sharded with the iteration loop in C++ (pqg_kmeans_fit_sharded):
    the same protocol and the same bit-exact result, NCCL collectives issued
    by the library on the backend's stream.  ``assignments`` are this rank's
    local rows (the caller gathers them if it needs the global vector)."""
    import torch
    be = ncomm.backend
    rows = local_rows.contiguous()
    n, ld = rows.shape
    tables = torch.empty((B, k, d), dtype=torch.float32, device=rows.device)
    assign = torch.empty((B, n), dtype=torch.int32, device=rows.device)
    iters = np.zeros(B, np.uint32)
    inertia = np.zeros(B, np.float64)
    per = np.zeros((B, max_iters), np.float64)
    st = np.zeros(4, np.uint64)
    sd = np.asarray([int(v) for v in seeds], np.uint64)
    vp = C.c_void_p
    be.L.check(be.lib.pqg_kmeans_fit_sharded(
        be.ctx.h, ncomm.h, vp(rows.data_ptr()), n, ld, B, d, col_stride, k, max_iters, sd.ctypes.data_as(vp), tol,
        vp(tables.data_ptr()), iters.ctypes.data_as(vp), inertia.ctypes.data_as(vp), per.ctypes.data_as(vp),
        vp(assign.data_ptr()), st.ctypes.data_as(vp)), "kmeans_fit_sharded")
    if stats is not None:
        stats.update(iterations=int(st[0]), replay_columns=int(st[1]), reseeds=int(st[2]),
                     allreduce_bytes=int(st[3]) * int(st[0]), host="C++ (pqg_kmeans_fit_sharded, NCCL)")
    per_iter = [[float(v) for v in per[b, : iters[b]]] for b in range(B)]
    return ShardedFit(tables, assign, inertia, iters, per_iter)


def _kmeans_fit_replicated(comm: Comm, backend, local_rows, counts, B, d, col_stride, k, max_iters, seeds,
                           tol) -> ShardedFit:
    """The replicated update for shapes the device partials do not cover:
    assignments + distances all-gathered in global row order, the reference's
    ordered update (kmeans.cpp:102-130) on every rank."""
    import torch
    dev = local_rows.device
    n = sum(counts)
    full = comm.allgather_rows(local_rows.contiguous(), counts)
    tables = torch.empty((B, k, d), dtype=torch.float32, device=dev)
    for b in range(B):  # init rows: the reference's draws, identical on every rank
        rows = torch.as_tensor(backend.init_rows(n, k, int(seeds[b])).astype(np.int64), device=dev)
        tables[b] = full.index_select(0, rows)[:, b * col_stride: b * col_stride + d]
    active = np.ones(B, np.int32)
    prev = np.zeros(B)
    inertia = np.zeros(B)
    iters = np.zeros(B, np.uint32)
    per_iter = [[] for _ in range(B)]
    assign_full = torch.zeros((B, n), dtype=torch.int32, device=dev)
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
    return ShardedFit(tables, assign_full, inertia, iters, per_iter)


def pq_fit_sharded(comm: Comm, backend, local_rows, M: int, ks: int, max_iters: int = 20,
                   seed: int = 0):
    """pq_fit (proj/src/pq.cpp:63-93) over row shards: subspace m uses seed + m."""
    D = local_rows.shape[1]
    if M == 0 or D % M:
        raise ValueError(f"pq_fit: D ({D}) is not divisible by M ({M})")
    ds = D // M
    fit = kmeans_fit_sharded(comm, backend, local_rows, M, ds, ds, ks, max_iters,
                             [seed + m for m in range(M)], 1e-4)
    return fit.tables


def encode_sharded(comm: Comm, backend, local_rows, tables):
    """Shard-local codes and the GLOBAL reconstruction RMSE (one all-reduce)."""
    codes, sse = backend.encode_sse(local_rows, tables)
    n = comm.allreduce_sum(float(local_rows.shape[0]), local_rows.device)
    total = comm.allreduce_sum(sse, local_rows.device)
    return codes, float(np.sqrt(total / (n * local_rows.shape[1])))


def search_sharded(comm: Comm, backend, tables, local_codes, local_ids, coarse, queries, k: int,
                   nprobe: int):
    """Shard-local index + search, then all-gather and (dist, id) merge."""
    ids, dists, counts = backend.search_local(tables, local_codes, local_ids, coarse, queries, k,
                                              nprobe)
    return backend.topk_merge(comm.allgather_equal(ids), comm.allgather_equal(dists),
                              comm.allgather_equal(counts), k)
