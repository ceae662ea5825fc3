"""Parity checkers for the PQ / IVF hot path -- TEST INFRASTRUCTURE ONLY.

Two CPU implementations live here, both built by ``oracle/Makefile``:

* ``C``   -- ``oracle/pqii_oracle.c``, a plain-C restatement of the reference's
  hot path (each function cites ``/root/reference/proj/<file>:<line>``).
* ``REF`` -- ``oracle/_ref/libpqii_ref.so``, the reference's own sources
  compiled as they lie plus ``oracle/ref_shim.cpp`` (extern "C" forwarding).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline and
``--impl reference``) may import this package.  The product package
``paper_2604_21645_b200`` never does: it fails loudly without its CUDA library.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
C_LIB_PATH = os.path.join(HERE, "build", "liboracle.so")
REF_LIB_PATH = os.path.join(HERE, "_ref", "libpqii_ref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_u64 = C.c_uint64
_u32 = C.c_uint32


def build() -> None:
    """Compile the checkers (the C restatement always; _ref when the
    reference sources are present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def code_width(ks: int) -> int:
    return 1 if ks <= 256 else 2


def default_threads() -> int:
    return max(1, os.cpu_count() or 1)


def pmap(fn, items, threads: int):
    """Run fn over items on `threads` Python threads.  ctypes drops the GIL for
    every call into the checkers, so independent calls (subspace fits, row
    chunks, queries) run in parallel; results come back in item order."""
    items = list(items)
    if threads <= 1 or len(items) <= 1:
        return [fn(it) for it in items]
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(threads, len(items))) as ex:
        return list(ex.map(fn, items))


def row_chunks(n: int, parts: int):
    parts = max(1, min(parts, n))
    return [(n * t // parts, n * (t + 1) // parts) for t in range(parts)]


class _Base:
    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing (run make -C oracle)")
        self.lib = C.CDLL(path)
        self.p = prefix

    def fn(self, name, restype, argtypes):
        # one prototype-bound callable per (name, signature): the CDLL's own
        # function objects are shared, and re-setting their argtypes while a
        # checker thread is inside a call raced (test_config3_full)
        key = (name, restype, tuple(argtypes))
        cache = self.__dict__.setdefault("_fn_cache", {})
        f = cache.get(key)
        if f is None:
            shared = getattr(self.lib, self.p + name)
            shared.restype = restype  # direct self.lib.<name> callers keep working
            shared.argtypes = argtypes
            f = C.CFUNCTYPE(restype, *argtypes)(C.cast(shared, C.c_void_p).value)
            cache[key] = f
        return f


class COracle(_Base):
    """The C restatement (``pqii_oracle.c``)."""

    def __init__(self, path: str = C_LIB_PATH):
        super().__init__(path, "orc_")

    def random_matrix(self, rows, dims, seed, lo=-1.0, hi=1.0):
        out = np.empty((rows, dims), np.float32)
        self.fn("random_matrix", None, [_u64, _u64, _u64, C.c_float, C.c_float, _f32p])(
            rows, dims, seed, lo, hi, out)
        return out

    def uniform_indices(self, seed, n, k):
        """The init index draws of kmeans_fit (kmeans.cpp:74-80)."""
        out = np.empty(k, np.uint64)
        self.fn("init_draws", None, [_u64, _u64, _u64, _u64p])(seed, n, k, out)
        return out

    def squared_l2(self, a, b):
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        return self.fn("squared_l2", C.c_double, [_f32p, _f32p, _u64])(a, b, a.size)

    def nearest_batch(self, points, table, threads=1):
        points = np.ascontiguousarray(points, np.float32)
        table = np.ascontiguousarray(table, np.float32)
        n, d = points.shape
        idx = np.empty(n, np.uint32)
        dist = np.empty(n, np.float64)
        self.fn("nearest_batch_mt", None,
                [_f32p, _u64, _u64, _f32p, _u64, _u32p, _f64p, C.c_int])(
            points, n, d, table, table.shape[0], idx, dist, int(threads))
        return idx, dist

    def lloyd_update(self, points, assignments, dists, centroids):
        """One update step (kmeans.cpp:102-130) from given assignments and
        fp64 distances: returns (new centroids, dists after the reseeds)."""
        points = np.ascontiguousarray(points, np.float32)
        n, d = points.shape
        cent = np.array(centroids, np.float32, copy=True, order="C")
        dist = np.array(dists, np.float64, copy=True, order="C")
        rc = self.fn("lloyd_update", C.c_int, [_f32p, _u64, _u64, _u64, _u32p, _f64p, _f32p])(
            points, n, d, cent.shape[0], np.ascontiguousarray(assignments, np.uint32), dist, cent)
        if rc:
            raise ValueError(f"lloyd_update rc={rc}")
        return cent, dist

    def kmeans_fit(self, points, k, max_iters=20, seed=0, tol=1e-4, threads=1):
        """kmeans_fit (kmeans.cpp:61-133); threads > 1 splits the assignment
        pass's rows only (bit-identical for every thread count)."""
        points = np.ascontiguousarray(points, np.float32)
        n, d = points.shape
        cent = np.empty((k, d), np.float32)
        assign = np.empty(n, np.uint32)
        inertia = C.c_double()
        iters = C.c_uint32()
        per = np.zeros(max(1, max_iters), np.float64)
        rc = self.fn("kmeans_fit_mt", C.c_int,
                     [_f32p, _u64, _u64, _u64, _u32, _u64, C.c_double, _f32p, _u32p,
                      C.POINTER(C.c_double), C.POINTER(C.c_uint32), _f64p, C.c_int])(
            points, n, d, k, max_iters, seed, tol, cent, assign, C.byref(inertia),
            C.byref(iters), per, int(threads))
        if rc:
            raise ValueError(f"kmeans_fit rc={rc}")
        return dict(centroids=cent, assignments=assign, inertia=inertia.value,
                    iterations_run=iters.value, inertia_per_iter=per[: iters.value].copy())

    def pq_fit(self, data, M, ks, max_iters=20, seed=0):
        data = np.ascontiguousarray(data, np.float32)
        n, D = data.shape
        if M == 0 or D % M:
            raise ValueError("not divisible")
        tables = np.empty((M, ks, D // M), np.float32)
        iters = np.empty(M, np.uint32)
        inert = np.empty(M, np.float64)
        rc = self.fn("pq_fit", C.c_int, [_f32p, _u64, _u64, _u32, _u32, _u32, _u64, _f32p,
                                         _u32p, _f64p])(
            data, n, D, M, ks, max_iters, seed, tables, iters, inert)
        if rc:
            raise ValueError(f"pq_fit rc={rc}")
        return tables, iters, inert

    def pq_encode(self, data, tables):
        data = np.ascontiguousarray(data, np.float32)
        tables = np.ascontiguousarray(tables, np.float32)
        M, ks, ds = tables.shape
        n = data.shape[0]
        codes = np.empty((n, M * code_width(ks)), np.uint8)
        self.fn("pq_encode", None, [_f32p, _u64, _u32, _u32, _u32, _f32p, _u8p])(
            data, n, M, ks, ds, tables, codes)
        return codes

    def pq_decode(self, codes, tables):
        tables = np.ascontiguousarray(tables, np.float32)
        codes = np.ascontiguousarray(codes, np.uint8)
        M, ks, ds = tables.shape
        n = codes.shape[0]
        out = np.empty((n, M * ds), np.float32)
        rc = self.fn("pq_decode", C.c_int, [_u8p, _u64, _u32, _u32, _u32, _f32p, _f32p])(
            codes, n, M, ks, ds, tables, out)
        if rc == -2:
            raise IndexError("pq_decode: code out of range")
        return out

    def rmse(self, a, b):
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        return self.fn("rmse", C.c_double, [_f32p, _f32p, _u64, _u64])(a, b, a.shape[0], a.shape[1])

    def adc_table(self, tables, query):
        tables = np.ascontiguousarray(tables, np.float32)
        M, ks, ds = tables.shape
        out = np.empty((M, ks), np.float32)
        self.fn("adc_table", None, [_f32p, _u32, _u32, _u32, _f32p, _f32p])(
            tables, M, ks, ds, np.ascontiguousarray(query, np.float32), out)
        return out

    def adc_lookup_all(self, entries, codes):
        entries = np.ascontiguousarray(entries, np.float32)
        codes = np.ascontiguousarray(codes, np.uint8)
        M, ks = entries.shape
        f = self.fn("adc_lookup", C.c_int, [_f32p, _u32, _u32, _u8p, _u64, C.POINTER(C.c_double)])
        out = np.empty(codes.shape[0], np.float64)
        v = C.c_double()
        for i in range(codes.shape[0]):
            if f(entries, M, ks, codes, i, C.byref(v)):
                raise IndexError("adc_lookup: code out of range")
            out[i] = v.value
        return out

    def ivf_assign(self, codes, tables, coarse):
        codes = np.ascontiguousarray(codes, np.uint8)
        tables = np.ascontiguousarray(tables, np.float32)
        coarse = np.ascontiguousarray(coarse, np.float32)
        M, ks, ds = tables.shape
        n = codes.shape[0]
        out = np.empty(n, np.uint32)
        rc = self.fn("ivf_assign", C.c_int,
                     [_u8p, _u64, _u32, _u32, _u32, _f32p, _f32p, _u64, _u32p])(
            codes, n, M, ks, ds, tables, coarse, coarse.shape[0], out)
        if rc:
            raise ValueError(f"ivf_assign rc={rc}")
        return out

    def ivf_assign_mt(self, codes, tables, coarse, threads):
        codes = np.ascontiguousarray(codes, np.uint8)
        parts = pmap(lambda r: self.ivf_assign(codes[r[0]:r[1]], tables, coarse),
                     row_chunks(codes.shape[0], 4 * threads), threads)
        return np.concatenate(parts) if parts else np.empty(0, np.uint32)

    def pq_encode_mt(self, data, tables, threads):
        parts = pmap(lambda r: self.pq_encode(data[r[0]:r[1]], tables),
                     row_chunks(data.shape[0], 4 * threads), threads)
        return np.concatenate(parts)

    def ivf_query_mt(self, tables, coarse, offsets, list_ids, list_codes, queries, k, nprobe,
                     threads, max_sq_dist=None):
        """ivf_query per query on `threads` threads: (ids nq x k, dists, counts)."""
        nq = queries.shape[0]
        ids = np.zeros((nq, k), np.uint64)
        dist = np.zeros((nq, k), np.float64)
        cnt = np.zeros(nq, np.uint32)
        tables = np.ascontiguousarray(tables, np.float32)
        coarse = np.ascontiguousarray(coarse, np.float32)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        list_ids = np.ascontiguousarray(list_ids, np.uint64)
        list_codes = np.ascontiguousarray(list_codes, np.uint8)

        def one(q):
            i, d = self.ivf_query(tables, coarse, offsets, list_ids, list_codes, queries[q], k,
                                  nprobe, max_sq_dist)
            ids[q, : i.size] = i
            dist[q, : i.size] = d
            cnt[q] = i.size
        pmap(one, range(nq), threads)
        return ids, dist, cnt

    def probe_order_mt(self, coarse, queries, nprobe, threads):
        out = np.empty((queries.shape[0], nprobe), np.uint32)

        def one(q):
            out[q] = self.probe_order(coarse, queries[q], nprobe)
        pmap(one, range(queries.shape[0]), threads)
        return out

    def ivf_csr(self, list_of, ids, codes, nlist):
        codes = np.ascontiguousarray(codes, np.uint8)
        n, rb = codes.shape
        offsets = np.empty(nlist + 1, np.uint64)
        out_ids = np.empty(n, np.uint64)
        out_codes = np.empty_like(codes)
        self.fn("ivf_csr", None, [_u32p, _u64p, _u8p, _u64, _u64, _u64, _u64p, _u64p, _u8p])(
            np.ascontiguousarray(list_of, np.uint32), np.ascontiguousarray(ids, np.uint64),
            codes, n, rb, nlist, offsets, out_ids, out_codes)
        return offsets, out_ids, out_codes

    def ivf_build_with_centroids(self, codes, ids, tables, coarse):
        lists = self.ivf_assign(codes, tables, coarse)
        return self.ivf_csr(lists, ids, codes, coarse.shape[0])

    def probe_order(self, coarse, query, nprobe):
        coarse = np.ascontiguousarray(coarse, np.float32)
        out = np.empty(nprobe, np.uint32)
        self.fn("probe_order", None, [_f32p, _u64, _u64, _f32p, _u64, _u32p])(
            coarse, coarse.shape[0], coarse.shape[1], np.ascontiguousarray(query, np.float32),
            nprobe, out)
        return out

    def ivf_query(self, tables, coarse, offsets, list_ids, list_codes, query, k, nprobe,
                  max_sq_dist=None):
        tables = np.ascontiguousarray(tables, np.float32)
        M, ks, ds = tables.shape
        ids = np.empty(k, np.uint64)
        dist = np.empty(k, np.float64)
        f = self.fn("ivf_query", C.c_int64,
                    [_f32p, _u32, _u32, _u32, _f32p, _u64, _u64p, _u64p, _u8p, _f32p, _u64, _u64,
                     C.c_int, C.c_double, _u64p, _f64p])
        cnt = f(tables, M, ks, ds, np.ascontiguousarray(coarse, np.float32), coarse.shape[0],
                np.ascontiguousarray(offsets, np.uint64), np.ascontiguousarray(list_ids, np.uint64),
                np.ascontiguousarray(list_codes, np.uint8), np.ascontiguousarray(query, np.float32),
                k, nprobe, int(max_sq_dist is not None),
                0.0 if max_sq_dist is None else float(max_sq_dist), ids, dist)
        if cnt < 0:
            raise ValueError(f"ivf_query rc={cnt}")
        return ids[:cnt], dist[:cnt]

    def ivf_query_subset(self, tables, coarse, offsets, list_ids, list_codes, query, k, subset,
                         nprobe, max_sq_dist=None):
        tables = np.ascontiguousarray(tables, np.float32)
        M, ks, ds = tables.shape
        subset = np.ascontiguousarray(subset, np.uint64)
        ids = np.empty(k, np.uint64)
        dist = np.empty(k, np.float64)
        f = self.fn("ivf_query_subset", C.c_int64,
                    [_f32p, _u32, _u32, _u32, _f32p, _u64, _u64p, _u64p, _u8p, _f32p, _u64,
                     C.c_void_p, _u64, _u64, C.c_int, C.c_double, _u64p, _f64p])
        cnt = f(tables, M, ks, ds, np.ascontiguousarray(coarse, np.float32), coarse.shape[0],
                np.ascontiguousarray(offsets, np.uint64), np.ascontiguousarray(list_ids, np.uint64),
                np.ascontiguousarray(list_codes, np.uint8), np.ascontiguousarray(query, np.float32),
                k, subset.ctypes.data if subset.size else None, subset.size, nprobe,
                int(max_sq_dist is not None), 0.0 if max_sq_dist is None else float(max_sq_dist),
                ids, dist)
        if cnt < 0:
            raise ValueError(f"ivf_query_subset rc={cnt}")
        return ids[:cnt], dist[:cnt]

    def flat_scan(self, tables, codes, ids, query, k, max_sq_dist=None):
        tables = np.ascontiguousarray(tables, np.float32)
        M, ks, ds = tables.shape
        out_ids = np.empty(k, np.uint64)
        dist = np.empty(k, np.float64)
        f = self.fn("flat_scan", C.c_int64,
                    [_f32p, _u32, _u32, _u32, _u8p, _u64p, _u64, _f32p, _u64, C.c_int,
                     C.c_double, _u64p, _f64p])
        codes = np.ascontiguousarray(codes, np.uint8)
        cnt = f(tables, M, ks, ds, codes, np.ascontiguousarray(ids, np.uint64), codes.shape[0],
                np.ascontiguousarray(query, np.float32), k, int(max_sq_dist is not None),
                0.0 if max_sq_dist is None else float(max_sq_dist), out_ids, dist)
        if cnt < 0:
            raise ValueError(f"flat_scan rc={cnt}")
        return out_ids[:cnt], dist[:cnt]

    def chunk_rows(self, n, c):
        b = np.empty(c + 1, np.uint64)
        if self.fn("chunk_rows", C.c_int, [_u64, _u64, _u64p])(n, c, b):
            raise ValueError("chunk_rows")
        return b


    # -- the chunked pipeline (proj/src/pipeline.cpp) -------------------------
    def train_chunk(self, chunk, M, ks, max_iters, chunk_seed):
        """train_chunk (pipeline.cpp:84-106): (representatives ks x D, local rmse)."""
        chunk = np.ascontiguousarray(chunk, np.float32)
        n, D = chunk.shape
        reps = np.empty((ks, D), np.float32)
        r = C.c_double()
        rc = self.fn("train_chunk", C.c_int, [_f32p, _u64, _u64, _u32, _u32, _u32, _u64, _f32p,
                                              C.POINTER(C.c_double)])(
            chunk, n, D, M, ks, max_iters, chunk_seed, reps, C.byref(r))
        if rc:
            raise ValueError(f"train_chunk rc={rc}")
        return reps, r.value

    def run_pipeline(self, data, n_chunks, M, ks, nlist=0, max_iters=20, seed=0, mode="single"):
        """run_pipeline (pipeline.cpp:142-266) composed from the restated pieces:
        chunk_rows -> train_chunk(seed + c) per chunk -> concatenation in chunk
        order (aggregate_representatives, :108-135) -> pq_fit(reps, seed)
        (fit_global, :137-140) -> reconstruction rmse on the data; index mode
        adds kmeans_fit(reps, nlist, iters, seed + M) for the shared coarse
        centroids, per-chunk ivf_build_with_centroids with ids [begin, end) and
        the per-list a-then-b merge (ivf.cpp:186-216)."""
        data = np.ascontiguousarray(data, np.float32)
        n, D = data.shape
        out = {}
        if nlist == 0:
            nlist = max(1, min(n, int(np.floor(np.sqrt(float(n)) + 0.5))))
            if mode == "parallel_pq_index":
                nlist = min(nlist, n_chunks * ks)
        out["nlist"] = nlist
        if mode == "single":
            tables, _, _ = self.pq_fit(data, M, ks, max_iters, seed)
            out["tables"] = tables
            out["rmse"] = self.rmse(data, self.pq_decode(self.pq_encode(data, tables), tables))
            return out
        bounds = self.chunk_rows(n, n_chunks)
        reps, local = [], []
        for c in range(n_chunks):
            r, lr = self.train_chunk(data[bounds[c]:bounds[c + 1]], M, ks, max_iters, seed + c)
            reps.append(r)
            local.append(lr)
        reps = np.concatenate(reps)
        tables, _, _ = self.pq_fit(reps, M, ks, max_iters, seed)
        codes = self.pq_encode(data, tables)
        out.update(tables=tables, representatives=reps, local_rmse=np.array(local),
                   rmse=self.rmse(data, self.pq_decode(codes, tables)))
        if mode == "parallel_pq_index":
            coarse = self.kmeans_fit(reps, nlist, max_iters, seed + M)["centroids"]
            lists_ids = [[] for _ in range(nlist)]
            lists_codes = [[] for _ in range(nlist)]
            for c in range(n_chunks):
                b0, b1 = int(bounds[c]), int(bounds[c + 1])
                ids = np.arange(b0, b1, dtype=np.uint64)
                off, lid, lcodes = self.ivf_build_with_centroids(codes[b0:b1], ids, tables, coarse)
                for l in range(nlist):
                    lists_ids[l].append(lid[off[l]:off[l + 1]])
                    lists_codes[l].append(lcodes[off[l]:off[l + 1]])
            sizes = [sum(len(a) for a in li) for li in lists_ids]
            out["coarse"] = coarse
            out["offsets"] = np.concatenate([[0], np.cumsum(sizes)]).astype(np.uint64)
            out["list_ids"] = np.concatenate([np.concatenate(li) for li in lists_ids])
            out["list_codes"] = np.concatenate([np.concatenate(li) for li in lists_codes])
        return out


class RefImpl(_Base):
    """The reference compiled from its own sources (``oracle/_ref``)."""

    def __init__(self, path: str = REF_LIB_PATH):
        super().__init__(path, "ref_")
        self.fn("ivf_build_with_centroids", C.c_void_p,
                [_f32p, _u32, _u32, _u32, _u8p, _u64p, _u64, _f32p, _u64, C.POINTER(C.c_int)])
        self.fn("ivf_build", C.c_void_p,
                [_f32p, _u32, _u32, _u32, _u8p, _u64p, _u64, _u64, _u64, _u32, C.POINTER(C.c_int)])
        self.fn("ivf_free", None, [C.c_void_p])
        self.fn("ivf_nlist", _u64, [C.c_void_p])
        self.fn("ivf_export", C.c_int, [C.c_void_p, _u64p, _u64p, _u8p, C.c_void_p])
        self.fn("ivf_add", C.c_int, [C.c_void_p, _u8p, _u64p, _u64])
        self.fn("ivf_merge", C.c_void_p, [C.c_void_p, C.c_void_p, C.POINTER(C.c_int)])
        self.fn("ivf_query_batch", C.c_int,
                [C.c_void_p, _f32p, _u64, _u64, _u64, C.c_int, C.c_double, _u64p, _f64p, _u32p,
                 C.c_int])
        self.fn("ivf_query_subset", C.c_int,
                [C.c_void_p, _f32p, _u64, _u64p, _u64, _u64, C.c_int, C.c_double, _u64p, _f64p,
                 _u32p])
        self.fn("hardware_concurrency", C.c_uint, [])
        self.fn("last_message", C.c_char_p, [])
        self.fn("save_index", C.c_int, [C.c_void_p, C.c_char_p])
        self.fn("load_index", C.c_void_p, [C.c_char_p, C.POINTER(C.c_int)])
        self.fn("save_codes", C.c_int, [_u8p, _u64, _u32, _u32, C.c_char_p])
        self.fn("load_codes", C.c_int, [C.c_char_p, C.POINTER(_u64), C.POINTER(_u32), C.POINTER(_u32),
                                        C.c_void_p, _u64])
        self.fn("save_codebook", C.c_int, [_f32p, _u32, _u32, _u32, C.c_char_p])
        self.fn("load_codebook", C.c_int, [C.c_char_p, C.POINTER(_u32), C.POINTER(_u32), C.POINTER(_u32),
                                           C.c_void_p, _u64])

    @staticmethod
    def _check(rc, what):
        if rc == -1:
            raise ValueError(f"{what}: invalid_argument")
        if rc == -2:
            raise IndexError(f"{what}: out_of_range")
        if rc:
            raise RuntimeError(f"{what}: rc={rc}")

    def random_matrix(self, rows, dims, seed, lo=-1.0, hi=1.0):
        out = np.empty((rows, dims), np.float32)
        self.fn("random_matrix", C.c_int, [_u64, _u64, _u64, C.c_float, C.c_float, _f32p])(
            rows, dims, seed, lo, hi, out)
        return out

    def uniform_indices(self, seed, n, k):
        out = np.empty(k, np.uint64)
        self.fn("uniform_indices", C.c_int, [_u64, _u64, _u64, _u64p])(seed, n, k, out)
        return out

    def nearest_batch(self, points, table):
        points = np.ascontiguousarray(points, np.float32)
        table = np.ascontiguousarray(table, np.float32)
        n, d = points.shape
        idx = np.empty(n, np.uint32)
        dist = np.empty(n, np.float64)
        rc = self.fn("nearest_batch", C.c_int, [_f32p, _u64, _u64, _f32p, _u64, _u32p, _f64p])(
            points, n, d, table, table.shape[0], idx, dist)
        self._check(rc, "nearest")
        return idx, dist

    def kmeans_fit(self, points, k, max_iters=20, seed=0, tol=1e-4):
        points = np.ascontiguousarray(points, np.float32)
        n, d = points.shape
        cent = np.empty((k, d), np.float32)
        assign = np.empty(n, np.uint32)
        inertia = C.c_double()
        iters = C.c_uint32()
        per = np.zeros(max(1, max_iters), np.float64)
        rc = self.fn("kmeans_fit", C.c_int,
                     [_f32p, _u64, _u64, _u64, _u32, _u64, C.c_double, _f32p, _u32p,
                      C.POINTER(C.c_double), C.POINTER(C.c_uint32), _f64p])(
            points, n, d, k, max_iters, seed, tol, cent, assign, C.byref(inertia),
            C.byref(iters), per)
        self._check(rc, "kmeans_fit")
        return dict(centroids=cent, assignments=assign, inertia=inertia.value,
                    iterations_run=iters.value, inertia_per_iter=per[: iters.value].copy())

    def pq_fit(self, data, M, ks, max_iters=20, seed=0, threads=1):
        data = np.ascontiguousarray(data, np.float32)
        n, D = data.shape
        tables = np.empty((M, ks, D // max(M, 1)), np.float32)
        if threads > 1:
            rc = self.fn("pq_fit_threads", C.c_int,
                         [_f32p, _u64, _u64, _u32, _u32, _u32, _u64, _f32p, C.c_int])(
                data, n, D, M, ks, max_iters, seed, tables, threads)
        else:
            rc = self.fn("pq_fit", C.c_int, [_f32p, _u64, _u64, _u32, _u32, _u32, _u64, _f32p])(
                data, n, D, M, ks, max_iters, seed, tables)
        self._check(rc, "pq_fit")
        return tables

    def pq_fit_stats(self, data, M, ks, max_iters=20, seed=0, threads=1):
        """pq_fit (pq.cpp:63-93) = one reference kmeans_fit(slice_m, ks,
        max_iters, seed + m) per subspace with the default tol, the M fits run
        on `threads` threads (kmeans_fit is safe for concurrent disjoint fits,
        kmeans.hpp:40).  Returns (tables, iterations_run[M],
        inertia_per_iter[M][max_iters] (NaN past iterations_run))."""
        fits = self.kmeans_fit_many([(np.ascontiguousarray(data[:, m * (data.shape[1] // M):
                                                                 (m + 1) * (data.shape[1] // M)]),
                                      ks, max_iters, seed + m) for m in range(M)], threads)
        return stack_fits(fits, max_iters)

    def kmeans_fit_many(self, problems, threads):
        """Independent reference kmeans_fit calls (points, k, iters, seed)
        spread over threads, biggest first."""
        order = sorted(range(len(problems)),
                       key=lambda i: -problems[i][0].shape[0] * problems[i][1] * problems[i][0].shape[1])
        res = pmap(lambda i: self.kmeans_fit(*problems[i]), order, threads)
        out = [None] * len(problems)
        for i, r in zip(order, res):
            out[i] = r
        return out

    def nearest_batch_mt(self, points, table, threads):
        parts = pmap(lambda r: self.nearest_batch(points[r[0]:r[1]], table),
                     row_chunks(points.shape[0], 4 * threads), threads)
        return np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts])

    def ivf_build_with_centroids_mt(self, codes, ids, tables, coarse, threads):
        """ivf_build_with_centroids over chunk_rows ranges on threads, the
        chunk indexes combined by the reference's own ivf_merge in chunk order
        (list l = chunk 0's then chunk 1's ..., ivf.cpp:203-211) -- the
        monolithic build (acceptance criterion 5)."""
        parts = pmap(lambda r: self.ivf_build_with_centroids(codes[r[0]:r[1]], ids[r[0]:r[1]],
                                                             tables, coarse),
                     row_chunks(codes.shape[0], threads), threads)
        while len(parts) > 1:  # pairwise, order preserving
            nxt = pmap(lambda i: parts[i].merge(parts[i + 1]), range(0, len(parts) - 1, 2), threads)
            if len(parts) % 2:
                nxt.append(parts[-1])
            parts = nxt
        return parts[0]

    def pq_encode(self, data, tables, threads=1):
        data = np.ascontiguousarray(data, np.float32)
        tables = np.ascontiguousarray(tables, np.float32)
        M, ks, ds = tables.shape
        n = data.shape[0]
        codes = np.empty((n, M * code_width(ks)), np.uint8)
        if threads > 1:
            rc = self.fn("pq_encode_threads", C.c_int,
                         [_f32p, _u64, _u32, _u32, _u32, _f32p, _u8p, C.c_int])(
                data, n, M, ks, ds, tables, codes, threads)
        else:
            rc = self.fn("pq_encode", C.c_int, [_f32p, _u64, _u32, _u32, _u32, _f32p, _u8p])(
                data, n, M, ks, ds, tables, codes)
        self._check(rc, "pq_encode")
        return codes

    def pq_decode(self, codes, tables):
        tables = np.ascontiguousarray(tables, np.float32)
        codes = np.ascontiguousarray(codes, np.uint8)
        M, ks, ds = tables.shape
        out = np.empty((codes.shape[0], M * ds), np.float32)
        rc = self.fn("pq_decode", C.c_int, [_u8p, _u64, _u32, _u32, _u32, _f32p, _f32p])(
            codes, codes.shape[0], M, ks, ds, tables, out)
        self._check(rc, "pq_decode")
        return out

    def rmse(self, a, b):
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        out = C.c_double()
        rc = self.fn("rmse", C.c_int, [_f32p, _f32p, _u64, _u64, C.POINTER(C.c_double)])(
            a, b, a.shape[0], a.shape[1], C.byref(out))
        self._check(rc, "rmse")
        return out.value

    def reconstruction_rmse(self, data, tables):
        data = np.ascontiguousarray(data, np.float32)
        tables = np.ascontiguousarray(tables, np.float32)
        M, ks, ds = tables.shape
        out = C.c_double()
        rc = self.fn("reconstruction_rmse", C.c_int,
                     [_f32p, _u64, _u32, _u32, _u32, _f32p, C.POINTER(C.c_double)])(
            data, data.shape[0], M, ks, ds, tables, C.byref(out))
        self._check(rc, "reconstruction_rmse")
        return out.value

    def adc_table(self, tables, query):
        tables = np.ascontiguousarray(tables, np.float32)
        M, ks, ds = tables.shape
        out = np.empty((M, ks), np.float32)
        rc = self.fn("adc_table", C.c_int, [_f32p, _u32, _u32, _u32, _f32p, _f32p])(
            tables, M, ks, ds, np.ascontiguousarray(query, np.float32), out)
        self._check(rc, "adc_table")
        return out

    def adc_lookup_all(self, entries, codes):
        entries = np.ascontiguousarray(entries, np.float32)
        codes = np.ascontiguousarray(codes, np.uint8)
        M, ks = entries.shape
        out = np.empty(codes.shape[0], np.float64)
        rc = self.fn("adc_lookup_all", C.c_int, [_f32p, _u32, _u32, _u8p, _u64, _f64p])(
            entries, M, ks, codes, codes.shape[0], out)
        self._check(rc, "adc_lookup")
        return out

    # -- index handles ---------------------------------------------------
    def ivf_build_with_centroids(self, codes, ids, tables, coarse):
        tables = np.ascontiguousarray(tables, np.float32)
        M, ks, ds = tables.shape
        codes = np.ascontiguousarray(codes, np.uint8)
        st = C.c_int()
        h = self.lib.ref_ivf_build_with_centroids(
            tables, M, ks, ds, codes, np.ascontiguousarray(ids, np.uint64), codes.shape[0],
            np.ascontiguousarray(coarse, np.float32), coarse.shape[0], C.byref(st))
        self._check(st.value, "ivf_build_with_centroids")
        return RefIndexHandle(self, h, codes.shape[1], M * ds)

    def ivf_build(self, codes, ids, tables, nlist, seed, iters=20):
        tables = np.ascontiguousarray(tables, np.float32)
        M, ks, ds = tables.shape
        codes = np.ascontiguousarray(codes, np.uint8)
        st = C.c_int()
        h = self.lib.ref_ivf_build(tables, M, ks, ds, codes, np.ascontiguousarray(ids, np.uint64),
                                   codes.shape[0], nlist, seed, iters, C.byref(st))
        self._check(st.value, "ivf_build")
        return RefIndexHandle(self, h, codes.shape[1], M * ds)

    def flat_scan(self, tables, codes, ids, query, k, max_sq_dist=None):
        tables = np.ascontiguousarray(tables, np.float32)
        M, ks, ds = tables.shape
        codes = np.ascontiguousarray(codes, np.uint8)
        out_ids = np.empty(k, np.uint64)
        dist = np.empty(k, np.float64)
        cnt = np.zeros(1, np.uint32)
        rc = self.fn("flat_scan", C.c_int,
                     [_f32p, _u32, _u32, _u32, _u8p, _u64p, _u64, _f32p, _u64, C.c_int,
                      C.c_double, _u64p, _f64p, _u32p])(
            tables, M, ks, ds, codes, np.ascontiguousarray(ids, np.uint64), codes.shape[0],
            np.ascontiguousarray(query, np.float32), k, int(max_sq_dist is not None),
            0.0 if max_sq_dist is None else float(max_sq_dist), out_ids, dist, cnt)
        self._check(rc, "flat_scan")
        return out_ids[: cnt[0]], dist[: cnt[0]]

    def default_nlist(self, n):
        return self.fn("default_nlist", _u64, [_u64])(n)

    # -- on-disk formats (the reference's own save_* / load_*) -------------
    # load_* return (status, message, value): status 0 ok, -1 invalid_argument,
    # -2 out_of_range, -4 runtime_error; message = the exception's what()
    def _msg(self):
        return self.lib.ref_last_message().decode()

    def save_index(self, handle, path):
        rc = self.lib.ref_save_index(handle.h, path.encode())
        return rc, self._msg()

    def load_index(self, path, row_bytes, dims):
        st = C.c_int()
        h = self.lib.ref_load_index(path.encode(), C.byref(st))
        if st.value:
            return st.value, self._msg(), None
        return 0, "", RefIndexHandle(self, h, row_bytes, dims)

    def save_codes(self, codes, M, ks, path):
        codes = np.ascontiguousarray(codes, np.uint8)
        return self.lib.ref_save_codes(codes, codes.shape[0], M, ks, path.encode()), self._msg()

    def load_codes(self, path):
        n, M, ks = _u64(), _u32(), _u32()
        rc = self.lib.ref_load_codes(path.encode(), C.byref(n), C.byref(M), C.byref(ks), None, 0)
        if rc:
            return rc, self._msg(), None
        out = np.empty((n.value, M.value * code_width(ks.value)), np.uint8)
        self.lib.ref_load_codes(path.encode(), C.byref(n), C.byref(M), C.byref(ks), out.ctypes.data, out.nbytes)
        return 0, "", (out, M.value, ks.value)

    def save_codebook(self, tables, path):
        tables = np.ascontiguousarray(tables, np.float32)
        M, ks, ds = tables.shape
        return self.lib.ref_save_codebook(tables, M, ks, ds, path.encode()), self._msg()

    def load_codebook(self, path):
        M, ks, ds = _u32(), _u32(), _u32()
        rc = self.lib.ref_load_codebook(path.encode(), C.byref(M), C.byref(ks), C.byref(ds), None, 0)
        if rc:
            return rc, self._msg(), None
        out = np.empty((M.value, ks.value, ds.value), np.float32)
        self.lib.ref_load_codebook(path.encode(), C.byref(M), C.byref(ks), C.byref(ds), out.ctypes.data,
                                   out.size)
        return 0, "", out

    def chunk_rows(self, n, c):
        b = np.empty(c + 1, np.uint64)
        self._check(self.fn("chunk_rows", C.c_int, [_u64, _u64, _u64p])(n, c, b), "chunk_rows")
        return b

    def hardware_concurrency(self):
        return self.lib.ref_hardware_concurrency()

    def train_chunk(self, chunk, M, ks, max_iters, chunk_seed):
        chunk = np.ascontiguousarray(chunk, np.float32)
        n, D = chunk.shape
        reps = np.empty((ks, D), np.float32)
        r = C.c_double()
        rc = self.fn("train_chunk", C.c_int, [_f32p, _u64, _u64, _u32, _u32, _u32, _u64, _f32p,
                                              C.POINTER(C.c_double)])(
            chunk, n, D, M, ks, max_iters, chunk_seed, reps, C.byref(r))
        self._check(rc, "train_chunk")
        return reps, r.value

    def run_pipeline(self, data, n_chunks, M, ks, nlist=0, max_iters=20, seed=0,
                     mode="single", threads=1):
        """The reference's own run_pipeline; returns a dict like
        COracle.run_pipeline plus "phases" (name -> seconds) and "total"."""
        data = np.ascontiguousarray(data, np.float32)
        n, D = data.shape
        m = {"single": 0, "parallel_pq": 1, "parallel_pq_index": 2}[mode]
        tables = np.empty((M, ks, D // max(M, 1)), np.float32)
        reps = np.empty((n_chunks * ks, D), np.float32) if m else None
        rm = C.c_double()
        nl = C.c_uint64()
        h = C.c_void_p()
        ph = np.empty(9, np.float64)
        err = C.create_string_buffer(512)
        rc = self.fn("run_pipeline", C.c_int,
                     [_f32p, _u64, _u64, _u64, _u32, _u32, _u64, _u32, _u64, _u64, C.c_int,
                      _f32p, C.POINTER(C.c_double), C.c_void_p, C.POINTER(C.c_uint64),
                      C.POINTER(C.c_void_p), _f64p, C.c_char_p, _u64])(
            data, n, D, n_chunks, M, ks, nlist, max_iters, seed, threads, m, tables, C.byref(rm),
            None if reps is None else reps.ctypes.data, C.byref(nl), C.byref(h), ph, err, 512)
        if rc:
            msg = err.value.decode()
            if rc == -1:
                raise ValueError(msg)
            raise RuntimeError(msg)
        names = ["fit", "chunking", "local_fit", "global_fit", "coarse_fit", "encode",
                 "index_build", "merge"]
        out = dict(tables=tables, rmse=rm.value, nlist=nl.value,
                   phases={k: float(v) for k, v in zip(names, ph[:8]) if v >= 0}, total=float(ph[8]))
        if reps is not None:
            out["representatives"] = reps
        if h.value:
            hd = RefIndexHandle(self, h.value, M * code_width(ks), D)
            off, lid, lcodes, coarse = hd.export()
            out.update(offsets=off, list_ids=lid, list_codes=lcodes, coarse=coarse)
        return out


def stack_fits(fits, max_iters):
    """Per-subspace kmeans_fit results -> (tables[M][ks][ds], iters[M],
    inertia_per_iter[M][max_iters] NaN-padded)."""
    tables = np.stack([f["centroids"] for f in fits])
    iters = np.array([f["iterations_run"] for f in fits], np.uint32)
    per = np.full((len(fits), max_iters), np.nan)
    for m, f in enumerate(fits):
        per[m, : f["iterations_run"]] = f["inertia_per_iter"]
    return tables, iters, per


class RefIndexHandle:
    def __init__(self, ref: RefImpl, h, row_bytes: int, dims: int):
        self.ref, self.h, self.row_bytes, self.dims = ref, h, row_bytes, dims

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_ivf_free(self.h)
            self.h = None

    @property
    def nlist(self):
        return self.ref.lib.ref_ivf_nlist(self.h)

    def export(self):
        """(offsets[nlist+1], ids[n], codes[n, row_bytes], coarse[nlist, D])."""
        nlist = self.nlist
        f = self.ref.lib.ref_ivf_n_items
        f.restype, f.argtypes = C.c_uint64, [C.c_void_p]
        n = int(f(self.h))
        offsets = np.empty(nlist + 1, np.uint64)
        ids = np.empty(max(n, 1), np.uint64)
        codes = np.empty((max(n, 1), self.row_bytes), np.uint8)
        coarse = np.empty((nlist, self.dims), np.float32)
        self.ref.lib.ref_ivf_export(self.h, offsets, ids, codes, coarse.ctypes.data)
        return offsets, ids[:n], codes[:n], coarse

    def add(self, codes, ids):
        codes = np.ascontiguousarray(codes, np.uint8)
        rc = self.ref.lib.ref_ivf_add(self.h, codes, np.ascontiguousarray(ids, np.uint64),
                                      codes.shape[0])
        self.ref._check(rc, "ivf_add")

    def merge(self, other):
        st = C.c_int()
        h = self.ref.lib.ref_ivf_merge(self.h, other.h, C.byref(st))
        self.ref._check(st.value, "ivf_merge")
        return RefIndexHandle(self.ref, h, self.row_bytes, self.dims)

    def query_batch(self, queries, k, nprobe, max_sq_dist=None, threads=1):
        queries = np.ascontiguousarray(queries, np.float32).reshape(-1, self.dims)
        nq = queries.shape[0]
        ids = np.zeros((nq, k), np.uint64)
        dist = np.zeros((nq, k), np.float64)
        counts = np.zeros(nq, np.uint32)
        rc = self.ref.lib.ref_ivf_query_batch(
            self.h, queries, nq, k, nprobe, int(max_sq_dist is not None),
            0.0 if max_sq_dist is None else float(max_sq_dist), ids, dist, counts, threads)
        self.ref._check(rc, "ivf_query")
        return ids, dist, counts

    def query_subset(self, query, k, subset, nprobe, max_sq_dist=None):
        ids = np.zeros(k, np.uint64)
        dist = np.zeros(k, np.float64)
        cnt = np.zeros(1, np.uint32)
        subset = np.ascontiguousarray(subset, np.uint64)
        rc = self.ref.lib.ref_ivf_query_subset(
            self.h, np.ascontiguousarray(query, np.float32), k, subset, subset.size, nprobe,
            int(max_sq_dist is not None), 0.0 if max_sq_dist is None else float(max_sq_dist),
            ids, dist, cnt)
        self.ref._check(rc, "ivf_query_subset")
        return ids[: cnt[0]], dist[: cnt[0]]


_C = None
_R = None


def c_oracle() -> COracle:
    global _C
    if _C is None:
        if not os.path.exists(C_LIB_PATH):
            build()
        _C = COracle()
    return _C


def ref_available() -> bool:
    return os.path.exists(REF_LIB_PATH)


def ref_impl() -> RefImpl:
    global _R
    if _R is None:
        _R = RefImpl()
    return _R
