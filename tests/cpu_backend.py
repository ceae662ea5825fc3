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


class ShardOracleBackend(OracleBackend):
    """OracleBackend plus a numpy model of the device side of the sharded fit
    (pqg_kmshard_*: csrc/kmshard.cu, kmeans_local_partials).  It follows the
    device semantics step for step -- exact local sums with the u8 exponent
    encodings, the global exactness test, the ordered replay list, the
    member packs, the chained replay and the reseed candidates -- so the
    gloo tests exercise dist.kmeans_fit_sharded's exchange protocol exactly
    as the GPU runs it, against the single-process oracle."""

    def shard_create(self, rows, B, d, col_stride, k, max_iters, tol):
        if d % 4 or d > 128:
            return None
        x = _np(rows)
        return {"x": x, "n": x.shape[0], "B": B, "d": d, "cs": col_stride, "k": k, "max_iters": max_iters,
                "tol": tol, "active": np.ones(B, bool), "prev": np.zeros(B), "iters": np.zeros(B, np.uint32),
                "inertia": np.zeros(B), "per": np.zeros((B, max_iters)), "assign": None, "dist": None,
                "work": np.zeros(0, np.int64), "empties": np.zeros(B, np.uint32)}

    def shard_destroy(self, s):
        pass

    def _cols(self, s, b):
        return s["x"][:, b * s["cs"]: b * s["cs"] + s["d"]]

    def shard_init_table(self, s, init_rows, row0):
        B, k, d, n = s["B"], s["k"], s["d"], s["n"]
        bits = np.zeros((B, k, d), np.uint32)
        for b in range(B):
            for c in range(k):
                gi = int(init_rows[b * k + c])
                if row0 <= gi < row0 + n:
                    bits[b, c] = np.ascontiguousarray(self._cols(s, b)[gi - row0]).view(np.uint32)
        return torch.from_numpy(bits.view(np.int32))

    def shard_partials(self, s, tables):
        B, k, d, n = s["B"], s["k"], s["d"], s["n"]
        tab = _np(tables)
        nkd = B * k * d
        f64 = np.zeros(nkd + B * k + B)
        u8 = np.zeros(2 * nkd, np.uint8)
        if s["assign"] is None:  # persistent: a stopped problem keeps its last pass
            s["assign"] = np.zeros((B, n), np.uint32)
            s["dist"] = np.zeros((B, n))
        for b in range(B):
            if not s["active"][b]:
                continue
            xb = np.ascontiguousarray(self._cols(s, b))
            a, dd = self.orc.nearest_batch(xb, np.ascontiguousarray(tab[b]))
            s["assign"][b], s["dist"][b] = a, dd
            sums = np.zeros((k, d))
            np.add.at(sums, a, xb.astype(np.float64))
            e = ((xb.view(np.uint32) >> 23) & 0xFF).astype(np.int64)
            nz = xb != 0
            emax = np.full((k, d), -1, np.int64)
            emin = np.full((k, d), 1 << 30, np.int64)
            rows_c = np.broadcast_to(a[:, None], xb.shape)
            np.maximum.at(emax, (rows_c[nz], np.nonzero(nz)[1]), e[nz])
            np.minimum.at(emin, (rows_c[nz], np.nonzero(nz)[1]), np.maximum(e[nz], 1))
            sl = slice(b * k * d, (b + 1) * k * d)
            f64[sl] = sums.ravel()
            u8[sl] = np.where(emax < 0, 0, np.minimum(emax + 1, 255)).ravel()
            u8[nkd + b * k * d: nkd + (b + 1) * k * d] = np.where(emin > 255, 0, 256 - np.maximum(emin, 1)).ravel()
            f64[nkd + b * k: nkd + (b + 1) * k] = np.bincount(a, minlength=k)
            f64[nkd + B * k + b] = self.rows_sum(torch.from_numpy(dd[None, :]))[0]
        return torch.from_numpy(f64), torch.from_numpy(u8)

    def shard_apply(self, s, tables, f64t, u8t):
        B, k, d = s["B"], s["k"], s["d"]
        f64, u8, tab = _np(f64t), _np(u8t), _np(tables)
        nkd = B * k * d
        flags = np.zeros(nkd, bool)
        s["empties"][:] = 0
        for b in range(B):  # stop rule, kmeans.cpp:93-100
            if not s["active"][b]:
                continue
            v = f64[nkd + B * k + b]
            it = int(s["iters"][b]) + 1
            s["inertia"][b] = v
            s["per"][b, it - 1] = v
            s["iters"][b] = it
            prev = s["prev"][b]
            if (it > 1 and prev - v < s["tol"] * max(1.0, prev)) or it == s["max_iters"]:
                s["active"][b] = False
            else:
                s["prev"][b] = v
        for b in range(B):
            if not s["active"][b]:
                continue
            for c in range(k):
                cnt = f64[nkd + b * k + c]
                if cnt == 0:
                    s["empties"][b] += 1
                    continue
                lg = int(np.ceil(np.log2(cnt))) if cnt > 1 else 0
                for t in range(d):
                    e = (b * k + c) * d + t
                    ea = int(u8[e]) - 1
                    ei = 256 - int(u8[nkd + e]) if u8[nkd + e] else (1 << 30)
                    if ea < 0 or (ea < 254 and ea - ei + lg <= 28):
                        tab[b, c, t] = np.float32(f64[e] * (1.0 / cnt))
                    else:
                        flags[e] = True
        s["work"] = np.flatnonzero(flags)
        s["stride"] = max(1, int(sum(f64[nkd + int(e) // d] for e in s["work"])))
        me = max([int(s["empties"][b]) for b in range(B) if s["active"][b]] or [0])
        return int(s["work"].size), me, bool(s["active"].any())

    def shard_pack(self, s, n_fail):
        k, d = s["k"], s["d"]
        vals, offcnt = [], []
        off = 0
        for e in s["work"]:
            bc, t = divmod(int(e), d)
            b, c = divmod(bc, k)
            mem = np.flatnonzero(s["assign"][b] == c)  # local row order
            v = self._cols(s, b)[mem, t]
            vals.append(v)
            offcnt += [off, v.size]
            off += v.size
        vals = np.concatenate(vals).astype(np.float32) if vals else np.zeros(0, np.float32)
        padded = np.zeros(s["stride"], np.float32)  # common length on every rank (no size exchange)
        padded[: vals.size] = vals
        return torch.from_numpy(padded), torch.from_numpy(np.array(offcnt, np.int64))

    def shard_replay(self, s, tables, f64t, all_vals, stride, all_offcnt, world):
        B, k, d = s["B"], s["k"], s["d"]
        f64, tab = _np(f64t), _np(tables)
        av, ao = _np(all_vals), _np(all_offcnt)
        nkd = B * k * d
        for p, e in enumerate(s["work"]):
            acc = 0.0
            for r in range(world):
                o, c = int(ao[r, 2 * p]), int(ao[r, 2 * p + 1])
                for v in av[r, o:o + c].tolist():  # the reference's chain, kmeans.cpp:103-111
                    acc += v
            bc = int(e) // d
            tab.reshape(-1)[e] = np.float32(acc * (1.0 / f64[nkd + bc]))

    def shard_replay_step(self, s, run):
        k, d = s["k"], s["d"]
        r = _np(run)
        for p, e in enumerate(s["work"]):
            bc, t = divmod(int(e), d)
            b, c = divmod(bc, k)
            acc = float(r[p])
            for v in self._cols(s, b)[np.flatnonzero(s["assign"][b] == c), t].tolist():
                acc += v  # the reference's chain, kmeans.cpp:103-111, local row order
            r[p] = acc

    def shard_replay_finish(self, s, tables, f64t, run):
        B, k, d = s["B"], s["k"], s["d"]
        f64, tab, r = _np(f64t), _np(tables), _np(run)
        nkd = B * k * d
        for p, e in enumerate(s["work"]):
            tab.reshape(-1)[e] = np.float32(r[p] * (1.0 / f64[nkd + int(e) // d]))

    def shard_reseed_candidates(self, s, row0, E):
        B, d = s["B"], s["d"]
        cd = np.full((B, E + 1), -1.0)
        ci = np.full((B, E + 1), -1, np.int64)
        cr = np.zeros((B, E + 1, d), np.float32)
        for b in range(B):
            need = min(int(s["empties"][b]), E) if s["active"][b] else 0
            dd = s["dist"][b]
            pos = np.flatnonzero(dd > 0)
            order = pos[np.lexsort((pos, -dd[pos]))][:need]  # dist desc, index asc
            for j, i in enumerate(order):
                cd[b, j], ci[b, j], cr[b, j] = dd[i], row0 + i, self._cols(s, b)[i]
            cd[b, E], ci[b, E], cr[b, E] = -2.0, row0, self._cols(s, b)[0]
        return torch.from_numpy(cd), torch.from_numpy(ci), torch.from_numpy(cr)

    def shard_reseed_apply(self, s, tables, f64t, E, world, all_d, all_i, all_r):
        B, k, d = s["B"], s["k"], s["d"]
        f64, tab = _np(f64t), _np(tables)
        ad, ai, ar = _np(all_d), _np(all_i), _np(all_r)
        nkd = B * k * d
        for b in range(B):
            if not s["active"][b]:
                continue
            cands = sorted(((-ad[r, b, j], int(ai[r, b, j]), r, j) for r in range(world) for j in range(E)
                            if ad[r, b, j] > 0))
            q = 0
            for c in range(k):
                if f64[nkd + b * k + c] != 0:
                    continue
                if q < len(cands):
                    _, _, r, j = cands[q]
                    q += 1
                    tab[b, c] = ar[r, b, j]
                else:  # every distance is 0: the argmax is global row 0 (rank 0's slot E)
                    tab[b, c] = ar[0, b, E]

    def shard_result(self, s):
        return (s["iters"].copy(), s["inertia"].copy(), s["per"].copy(),
                torch.from_numpy(s["assign"].view(np.int32)))
