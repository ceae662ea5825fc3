"""TEST INFRASTRUCTURE: a CPU shard backend for paper_2604_21645_b200.dist
built on the oracle, so the multi-rank exchange logic (sharding, all-gathers,
stop rule, merge) is exercised with gloo on CPU.  Numerics follow the
reference exactly (sequential fp64 sums), so a sharded fit must equal the
oracle's single-process fit bit-for-bit."""
import numpy as np

import oracle


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
        n = rows.shape[0]
        a = np.empty((B, n), np.uint32)
        dist = np.empty((B, n), np.float64)
        for b in range(B):
            a[b], dist[b] = self.orc.nearest_batch(rows[:, b * col_stride: b * col_stride + d], tables[b])
        return a, dist

    def rows_sum(self, v):
        out = np.zeros(v.shape[0])
        for b in range(v.shape[0]):
            s = 0.0
            for x in v[b].tolist():  # sequential, as proj/src/kmeans.cpp:51-55
                s += x
            out[b] = s
        return out

    def update_pass(self, rows, B, d, col_stride, tables, assign, dist, active):
        k = tables.shape[1]
        for b in range(B):
            if not active[b]:
                continue
            x = rows[:, b * col_stride: b * col_stride + d].astype(np.float64)
            sums = np.zeros((k, d))
            counts = np.zeros(k, np.int64)
            for i in range(x.shape[0]):  # row order, proj/src/kmeans.cpp:103-111
                c = assign[b, i]
                sums[c] += x[i]
                counts[c] += 1
            for c in range(k):
                if counts[c]:
                    tables[b, c] = (sums[c] * (1.0 / counts[c])).astype(np.float32)
            for c in range(k):  # :122-130
                if counts[c] == 0:
                    far = int(np.argmax(dist[b]))
                    tables[b, c] = rows[far, b * col_stride: b * col_stride + d]
                    dist[b, far] = 0.0

    def encode_sse(self, rows, tables):
        codes = self.orc.pq_encode(rows, tables)
        dec = self.orc.pq_decode(codes, tables)
        diff = rows.astype(np.float64) - dec.astype(np.float64)
        s = 0.0
        for v in (diff * diff).ravel().tolist():
            s += v
        return codes, s

    def search_local(self, tables, codes, ids, coarse, queries, k, nprobe):
        off, lid, lcodes = self.orc.ivf_build_with_centroids(codes, ids, tables, coarse)
        nq = queries.shape[0]
        oi = np.zeros((nq, k), np.uint64)
        od = np.zeros((nq, k), np.float64)
        oc = np.zeros(nq, np.uint32)
        for q in range(nq):
            i, dd = self.orc.ivf_query(tables, coarse, off, lid, lcodes, queries[q], k, nprobe)
            oi[q, : len(i)], od[q, : len(i)], oc[q] = i, dd, len(i)
        return oi, od, oc

    def topk_merge(self, ids, dists, counts, k):
        S, nq, _ = ids.shape
        oi = np.zeros((nq, k), np.uint64)
        od = np.zeros((nq, k), np.float64)
        oc = np.zeros(nq, np.uint32)
        for q in range(nq):
            cand = [(dists[s, q, j], int(ids[s, q, j])) for s in range(S) for j in range(counts[s, q])]
            cand.sort()
            cand = cand[:k]
            oc[q] = len(cand)
            for j, (dd, i) in enumerate(cand):
                oi[q, j], od[q, j] = i, dd
        return oi, od, oc
