"""TEST INFRASTRUCTURE: a CPU shard backend for paper_2604_21645_b200.dist
built on the oracle, so the multi-rank exchange logic (sharding, all-gathers,
stop rule, merge) is exercised with gloo on CPU.  Numerics follow the
reference exactly (sequential fp64 sums), so a sharded fit must equal the
oracle's single-process fit bit-for-bit.  Tensors are torch CPU tensors
(u32/u64 values carried as int32/int64 bit patterns, as in dist.py)."""
import numpy as np
import torch

import oracle


def _np(t, dtype=None):
    a = t.numpy()
    return a.view(dtype) if dtype is not None else a


class OracleBackend:
    def __init__(self):
        self.orc = oracle.c_oracle()

    def init_rows(self, n, k, seed):
        draws = self.orc.uniform_indices(seed, n, k)
        perm = {}
        for i in range(k):
            j = int(draws[i])
            vi, vj = perm.get(i, i), perm.get(j, j)
            perm[i], perm[j] = vj, vi
        return np.array([perm.get(c, c) for c in range(k)], np.uint64)

    def assign_pass(self, rows, B, d, col_stride, tables):
        x = _np(rows)
        n = x.shape[0]
        a = np.empty((B, n), np.uint32)
        dist = np.empty((B, n), np.float64)
        for b in range(B):
            a[b], dist[b] = self.orc.nearest_batch(x[:, b * col_stride: b * col_stride + d], _np(tables)[b])
        return torch.from_numpy(a.view(np.int32)), torch.from_numpy(dist)

    def rows_sum(self, v):
        v = _np(v)
        out = np.zeros(v.shape[0])
        for b in range(v.shape[0]):
            s = 0.0
            for x in v[b].tolist():  # sequential, as proj/src/kmeans.cpp:51-55
                s += x
            out[b] = s
        return out

    def update_pass(self, rows, B, d, col_stride, tables, assign, dist, active):
        x_all = _np(rows)
        tab = _np(tables)
        asg = _np(assign, np.uint32)
        dd = _np(dist)
        k = tab.shape[1]
        for b in range(B):
            if not active[b]:
                continue
            x = x_all[:, b * col_stride: b * col_stride + d].astype(np.float64)
            sums = np.zeros((k, d))
            counts = np.zeros(k, np.int64)
            for i in range(x.shape[0]):  # row order, proj/src/kmeans.cpp:103-111
                c = asg[b, i]
                sums[c] += x[i]
                counts[c] += 1
            for c in range(k):
                if counts[c]:
                    tab[b, c] = (sums[c] * (1.0 / counts[c])).astype(np.float32)
            for c in range(k):  # :122-130
                if counts[c] == 0:
                    far = int(np.argmax(dd[b]))
                    tab[b, c] = x_all[far, b * col_stride: b * col_stride + d]
                    dd[b, far] = 0.0

    def encode_sse(self, rows, tables):
        x = _np(rows)
        codes = self.orc.pq_encode(x, _np(tables))
        dec = self.orc.pq_decode(codes, _np(tables))
        diff = x.astype(np.float64) - dec.astype(np.float64)
        s = 0.0
        for v in (diff * diff).ravel().tolist():
            s += v
        return torch.from_numpy(codes), s

    def search_local(self, tables, codes, ids, coarse, queries, k, nprobe):
        t = _np(tables)
        off, lid, lcodes = self.orc.ivf_build_with_centroids(_np(codes), _np(ids, np.uint64), t, _np(coarse))
        q = _np(queries)
        nq = q.shape[0]
        oi = np.zeros((nq, k), np.uint64)
        od = np.zeros((nq, k), np.float64)
        oc = np.zeros(nq, np.uint32)
        for i in range(nq):
            ii, dd = self.orc.ivf_query(t, _np(coarse), off, lid, lcodes, q[i], k, nprobe)
            oi[i, : len(ii)], od[i, : len(ii)], oc[i] = ii, dd, len(ii)
        return (torch.from_numpy(oi.view(np.int64)), torch.from_numpy(od),
                torch.from_numpy(oc.view(np.int32)))

    def topk_merge(self, ids, dists, counts, k):
        ids, dists, counts = _np(ids, np.uint64), _np(dists), _np(counts, np.uint32)
        S, nq, _ = ids.shape
        oi = np.zeros((nq, k), np.uint64)
        od = np.zeros((nq, k), np.float64)
        oc = np.zeros(nq, np.uint32)
        for q in range(nq):
            cand = sorted((dists[s, q, j], int(ids[s, q, j])) for s in range(S) for j in range(counts[s, q]))[:k]
            oc[q] = len(cand)
            for j, (dd, i) in enumerate(cand):
                oi[q, j], od[q, j] = i, dd
        return (torch.from_numpy(oi.view(np.int64)), torch.from_numpy(od),
                torch.from_numpy(oc.view(np.int32)))
