"""The reference's PQ / IVF API (namespace ``pqii``, proj/include/pqii/*.hpp)
re-exposed over the B200 path.

Names, argument meaning, defaults and errors follow the reference so tests
read like its own: ``kmeans_fit`` (kmeans.hpp:41-44), ``pq_fit`` /
``pq_encode`` / ``pq_decode`` / ``adc_table`` / ``adc_lookup`` / ``rmse`` /
``reconstruction_rmse`` (pq.hpp:66-88), ``ivf_build`` /
``ivf_build_with_centroids`` / ``ivf_add`` / ``ivf_merge`` / ``ivf_query`` /
``ivf_query_subset`` / ``flat_scan`` / ``default_nlist`` (ivf.hpp:46-86).
``std::invalid_argument`` maps to ``ValueError`` and ``std::out_of_range`` to
``IndexError`` with the reference's message substrings.

Arrays may be numpy (host) or torch CUDA tensors (device-resident); the C
ABI stages host buffers itself.  Every computation runs in libpqg.so on the
GPU; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import threading
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib

# ---------------------------------------------------------------------------
# context
# ---------------------------------------------------------------------------


_tls = threading.local()  # set by _ptr when a call receives a torch CUDA tensor


class _OrderedLib:
    """libpqg with torch stream ordering: a call that was handed a torch CUDA
    tensor first makes the context stream wait for torch's current stream
    (the kernels that produced the inputs), and afterwards makes torch's
    current stream wait for the context stream (device outputs are complete
    before torch reads them).  Both are event waits, no host sync."""

    def __init__(self, ctx: "Context", lib):
        self._ctx = ctx
        self._lib = lib

    def __getattr__(self, name):
        f = getattr(self._lib, name)
        if not name.startswith("pqg_"):
            return f

        def call(*args):
            torch_args = getattr(_tls, "torch_cuda", False)
            _tls.torch_cuda = False
            if torch_args:
                self._ctx._fence(into_ctx=True)
            try:
                return f(*args)
            finally:
                if torch_args:
                    self._ctx._fence(into_ctx=False)
        return call


class Context:
    """One GPU, one stream, one scratch arena (pqg_ctx)."""

    def __init__(self, device: int = 0):
        self._raw = _lib.load()
        h = C.c_void_p()
        _lib.check(self._raw.pqg_ctx_create(device, C.byref(h)), "ctx_create")
        self.h = h
        self.device = device
        self.lib = _OrderedLib(self, self._raw)
        self._ext = {}

    def _fence(self, into_ctx: bool):
        import torch
        cur = torch.cuda.current_stream(self.device)
        mine = self._raw.pqg_ctx_stream(self.h) or 0
        if mine == cur.cuda_stream:
            return
        ext = self._ext.get(mine)
        if ext is None:
            ext = self._ext[mine] = torch.cuda.ExternalStream(mine, device=self.device)
        if into_ctx:
            ext.wait_stream(cur)
        else:
            cur.wait_stream(ext)

    def close(self):
        if getattr(self, "h", None):
            self._raw.pqg_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: int | None):
        _lib.check(self.lib.pqg_ctx_set_stream(self.h, C.c_void_p(stream_ptr or 0)))

    def sync(self):
        _lib.check(self.lib.pqg_ctx_sync(self.h))

    @property
    def launches(self) -> int:
        return int(self.lib.pqg_ctx_launches(self.h))

    def profile(self, enable: bool):
        _lib.check(self.lib.pqg_profile_enable(self.h, int(enable)))

    def profile_read(self, cls: str):
        n = C.c_uint64()
        ms = C.c_double()
        _lib.check(self.lib.pqg_profile_read(self.h, cls.encode(), C.byref(n), C.byref(ms)))
        return int(n.value), float(ms.value)


_CTX: dict[int, Context] = {}


def get_context(device: int = 0) -> Context:
    if device not in _CTX:
        _CTX[device] = Context(device)
    return _CTX[device]


def _ptr(x):
    """(void* value, keep-alive) for a numpy array or a torch tensor."""
    if x is None:
        return None, None
    if hasattr(x, "data_ptr"):
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        if getattr(x, "is_cuda", False):
            _tls.torch_cuda = True
        return C.c_void_p(x.data_ptr()), x
    a = np.ascontiguousarray(x)
    return C.c_void_p(a.ctypes.data), a


def _f32(x):
    if hasattr(x, "data_ptr"):
        return x
    return np.ascontiguousarray(x, dtype=np.float32)


# ---------------------------------------------------------------------------
# data types (proj/include/pqii/*.hpp)
# ---------------------------------------------------------------------------


@dataclass
class KMeansResult:  # kmeans.hpp:14-20
    centroids: np.ndarray
    assignments: np.ndarray
    inertia: float
    iterations_run: int
    inertia_per_iter: np.ndarray


@dataclass
class Codebook:  # pq.hpp:15-31
    m_subspaces: int
    ks: int
    sub_dim: int
    tables: np.ndarray  # [M, ks, sub_dim] float32

    def dims(self) -> int:
        return self.m_subspaces * self.sub_dim

    def codeword(self, m: int, j: int) -> np.ndarray:
        return self.tables[m, j]

    def __eq__(self, o) -> bool:
        return (isinstance(o, Codebook) and self.m_subspaces == o.m_subspaces and self.ks == o.ks
                and self.sub_dim == o.sub_dim and np.array_equal(self.tables, o.tables))


def code_width(ks: int) -> int:
    return 1 if ks <= 256 else 2


@dataclass
class CodeMatrix:  # pq.hpp:36-55
    rows: int
    m_subspaces: int
    ks: int
    bytes: np.ndarray  # [rows, M * width] uint8

    @staticmethod
    def zeros(n: int, m: int, ks: int) -> "CodeMatrix":
        if m == 0:
            raise ValueError("codebook: M must be >= 1")
        if ks == 0 or ks > 65536:
            raise ValueError("codebook: Ks must be in [1, 65536]")
        return CodeMatrix(n, m, ks, np.zeros((n, m * code_width(ks)), np.uint8))

    def code_width(self) -> int:
        return code_width(self.ks)

    def row_bytes(self) -> int:
        return self.m_subspaces * self.code_width()

    def at(self, i: int, m: int) -> int:
        w = self.code_width()
        b = self.bytes[i, m * w: m * w + w]
        return int(b[0]) if w == 1 else int(b[0]) | (int(b[1]) << 8)

    def set(self, i: int, m: int, v: int) -> None:
        w = self.code_width()
        self.bytes[i, m * w] = v & 0xFF
        if w == 2:
            self.bytes[i, m * w + 1] = (v >> 8) & 0xFF

    def codes(self) -> np.ndarray:
        """[rows, M] integer view of the packed codes."""
        if self.code_width() == 1:
            return self.bytes.astype(np.uint32)
        return self.bytes.view("<u2").astype(np.uint32)

    def __eq__(self, o) -> bool:
        return (isinstance(o, CodeMatrix) and self.rows == o.rows
                and self.m_subspaces == o.m_subspaces and self.ks == o.ks
                and np.array_equal(self.bytes, o.bytes))


@dataclass
class DistanceTable:  # pq.hpp:58-64
    m_subspaces: int
    ks: int
    entries: np.ndarray  # [M, ks] float32

    def entry(self, m: int, j: int) -> float:
        return float(self.entries[m, j])


@dataclass
class Hit:  # ivf.hpp:33-38
    id: int
    sq_dist: float


@dataclass
class QueryResult:  # ivf.hpp:40-44
    hits: list = field(default_factory=list)
    k_requested: int = 0


# ---------------------------------------------------------------------------
# L1: kmeans.hpp
# ---------------------------------------------------------------------------


def nearest_batch(points, table, ctx: Context | None = None):
    """nearest_in_table (kmeans.cpp:20-31) for every row of ``points``."""
    ctx = ctx or get_context()
    points = _f32(points)
    table = _f32(table)
    n, d = points.shape
    k = table.shape[0]
    if table.shape[0] == 0:
        raise ValueError("nearest_centroid: empty centroid set")
    if table.shape[1] != d:
        raise ValueError("nearest_centroid: dimension mismatch")
    idx = np.empty(n, np.uint32)
    dist = np.empty(n, np.float64)
    pp, _a = _ptr(points)
    tp, _b = _ptr(table)
    _lib.check(ctx.lib.pqg_nearest_batch(ctx.h, pp, n, d, tp, k, idx.ctypes.data_as(C.c_void_p),
                                         dist.ctypes.data_as(C.c_void_p)), "nearest")
    return idx, dist


def nearest_centroid(point, centroids, ctx: Context | None = None):
    """(index, sq_dist) -- kmeans.cpp:33-40."""
    point = np.ascontiguousarray(point, np.float32).reshape(1, -1)
    centroids = np.ascontiguousarray(centroids, np.float32)
    if centroids.ndim != 2 or centroids.shape[0] == 0:
        raise ValueError("nearest_centroid: empty centroid set")
    if point.shape[1] != centroids.shape[1]:
        raise ValueError("nearest_centroid: dimension mismatch")
    i, d = nearest_batch(point, centroids, ctx)
    return int(i[0]), float(d[0])


def kmeans_fit(points, k: int, max_iters: int = 20, seed: int = 0, tol: float = 1e-4,
               ctx: Context | None = None) -> KMeansResult:
    """Lloyd k-means, bit-identical to kmeans.cpp:61-133."""
    ctx = ctx or get_context()
    points = _f32(points)
    n, d = points.shape
    if max_iters < 0:
        raise ValueError("kmeans_fit: max_iters must be >= 1")
    cent = np.empty((k, d), np.float32)
    assign = np.empty(n, np.uint32)
    inertia = C.c_double()
    iters = C.c_uint32()
    per = np.zeros(max(1, max_iters), np.float64)
    pp, _a = _ptr(points)
    _lib.check(ctx.lib.pqg_kmeans_fit(ctx.h, pp, n, d, k, max_iters, seed, tol,
                                      cent.ctypes.data_as(C.c_void_p),
                                      assign.ctypes.data_as(C.c_void_p), C.byref(inertia),
                                      C.byref(iters), per.ctypes.data_as(C.c_void_p)), "kmeans_fit")
    return KMeansResult(cent, assign, inertia.value, iters.value, per[: iters.value].copy())


# ---------------------------------------------------------------------------
# L1: pq.hpp
# ---------------------------------------------------------------------------


def pq_fit(data, m: int, ks: int, max_iters: int = 20, seed: int = 0,
           ctx: Context | None = None, stats: dict | None = None) -> Codebook:
    """pq.cpp:63-93 -- all M subspace fits batched on the device."""
    ctx = ctx or get_context()
    data = _f32(data)
    n, D = data.shape
    if m == 0:
        raise ValueError("pq_fit: M must be >= 1")
    if D % m:
        raise ValueError(f"pq_fit: D ({D}) is not divisible by M ({m})")
    ds = D // m
    tables = np.empty((m, max(ks, 0), ds), np.float32)
    iters = np.empty(m, np.uint32)
    inert = np.empty(m, np.float64)
    per = np.zeros((m, max(1, max_iters)), np.float64)
    dp, _a = _ptr(data)
    _lib.check(ctx.lib.pqg_pq_fit_ex(ctx.h, dp, n, D, m, ks, max_iters, seed,
                                     tables.ctypes.data_as(C.c_void_p),
                                     iters.ctypes.data_as(C.c_void_p),
                                     inert.ctypes.data_as(C.c_void_p),
                                     per.ctypes.data_as(C.c_void_p) if max_iters > 0 else None),
               "pq_fit")
    if stats is not None:
        stats["iterations_run"] = iters
        stats["inertia"] = inert
        for b in range(m):  # kmeans_fit's inertia_per_iter per subspace
            per[b, iters[b]:] = np.nan
        stats["inertia_per_iter"] = per
    return Codebook(m, ks, ds, tables)


def pq_encode(cb: Codebook, data, ctx: Context | None = None) -> CodeMatrix:
    """pq.cpp:95-111."""
    ctx = ctx or get_context()
    data = _f32(data)
    if data.shape[1] != cb.dims():
        raise ValueError(f"pq_encode: data dimension {data.shape[1]} does not match codebook "
                         f"dimension {cb.dims()}")
    n = data.shape[0]
    out = CodeMatrix.zeros(n, cb.m_subspaces, cb.ks)
    dp, _a = _ptr(data)
    tp, _b = _ptr(np.ascontiguousarray(cb.tables, np.float32))
    _lib.check(ctx.lib.pqg_pq_encode(ctx.h, dp, n, cb.m_subspaces, cb.ks, cb.sub_dim, tp,
                                     out.bytes.ctypes.data_as(C.c_void_p)), "pq_encode")
    return out


def _check_codes(cb: Codebook, codes: CodeMatrix, who: str):
    if codes.m_subspaces != cb.m_subspaces or codes.ks != cb.ks:
        raise ValueError(f"{who}: codes do not match the codebook")


def pq_decode(cb: Codebook, codes: CodeMatrix, ctx: Context | None = None) -> np.ndarray:
    """pq.cpp:125-130 (raises IndexError for a code >= Ks, :117-120)."""
    ctx = ctx or get_context()
    _check_codes(cb, codes, "pq_decode")
    out = np.empty((codes.rows, cb.dims()), np.float32)
    if codes.rows == 0:
        return out
    cp, _a = _ptr(codes.bytes)
    tp, _b = _ptr(np.ascontiguousarray(cb.tables, np.float32))
    _lib.check(ctx.lib.pqg_pq_decode(ctx.h, cp, codes.rows, cb.m_subspaces, cb.ks, cb.sub_dim, tp,
                                     out.ctypes.data_as(C.c_void_p)), "pq_decode")
    return out


def pq_decode_row(cb: Codebook, codes: CodeMatrix, i: int, ctx: Context | None = None):
    """pq.cpp:113-123."""
    sub = CodeMatrix(1, codes.m_subspaces, codes.ks, codes.bytes[i: i + 1].copy())
    return pq_decode(cb, sub, ctx)[0]


def rmse(a, b, ctx: Context | None = None) -> float:
    """pq.cpp:169-177."""
    ctx = ctx or get_context()
    a = _f32(a)
    b = _f32(b)
    if tuple(a.shape) != tuple(b.shape):
        raise ValueError("rmse: shape mismatch")
    count = int(np.prod(a.shape))
    sse = C.c_double()
    ap, _a = _ptr(a)
    bp, _b = _ptr(b)
    _lib.check(ctx.lib.pqg_sq_error(ctx.h, ap, bp, count, C.byref(sse)), "rmse")
    return math.sqrt(sse.value / count) if count else float("nan")


def reconstruction_rmse(cb: Codebook, data, ctx: Context | None = None) -> float:
    """pq.cpp:179-181: rmse(data, decode(encode(data))), fused on the device."""
    ctx = ctx or get_context()
    data = _f32(data)
    if data.shape[1] != cb.dims():
        raise ValueError(f"pq_encode: data dimension {data.shape[1]} does not match codebook "
                         f"dimension {cb.dims()}")
    n = data.shape[0]
    sse = C.c_double()
    dp, _a = _ptr(data)
    tp, _b = _ptr(np.ascontiguousarray(cb.tables, np.float32))
    _lib.check(ctx.lib.pqg_pq_encode_sse(ctx.h, dp, n, cb.m_subspaces, cb.ks, cb.sub_dim, tp,
                                         None, C.byref(sse)), "reconstruction_rmse")
    return math.sqrt(sse.value / (n * cb.dims())) if n else float("nan")


def adc_table(cb: Codebook, query, ctx: Context | None = None) -> DistanceTable:
    """pq.cpp:132-151."""
    ctx = ctx or get_context()
    q = np.ascontiguousarray(query, np.float32).reshape(-1)
    if q.size != cb.dims():
        raise ValueError(f"adc_table: query dimension {q.size} does not match codebook "
                         f"dimension {cb.dims()}")
    ent = np.empty((cb.m_subspaces, cb.ks), np.float32)
    tp, _b = _ptr(np.ascontiguousarray(cb.tables, np.float32))
    _lib.check(ctx.lib.pqg_adc_tables(ctx.h, tp, cb.m_subspaces, cb.ks, cb.sub_dim,
                                      q.ctypes.data_as(C.c_void_p), 1,
                                      ent.ctypes.data_as(C.c_void_p)), "adc_table")
    return DistanceTable(cb.m_subspaces, cb.ks, ent)


def adc_lookup_all(table: DistanceTable, codes: CodeMatrix, ctx: Context | None = None):
    """adc_lookup (pq.cpp:153-167) for every row of ``codes``."""
    ctx = ctx or get_context()
    if codes.m_subspaces != table.m_subspaces or codes.ks != table.ks:
        raise ValueError("adc_lookup: codes do not match the table")
    out = np.empty(codes.rows, np.float64)
    if codes.rows == 0:
        return out
    ep, _a = _ptr(np.ascontiguousarray(table.entries, np.float32))
    cp, _b = _ptr(codes.bytes)
    _lib.check(ctx.lib.pqg_adc_lookup(ctx.h, ep, table.m_subspaces, table.ks, cp, codes.rows,
                                      out.ctypes.data_as(C.c_void_p)), "adc_lookup")
    return out


def adc_lookup(table: DistanceTable, codes: CodeMatrix, row: int, ctx: Context | None = None):
    sub = CodeMatrix(1, codes.m_subspaces, codes.ks, codes.bytes[row: row + 1].copy())
    return float(adc_lookup_all(table, sub, ctx)[0])


# ---------------------------------------------------------------------------
# L2: ivf.hpp
# ---------------------------------------------------------------------------


class InvertedIndex:
    """Device-resident posting lists (CSR) -- ivf.hpp:14-31."""

    def __init__(self, handle, ctx: Context):
        self.h = handle
        self.ctx = ctx

    def __del__(self):
        if getattr(self, "h", None):
            try:
                self.ctx.lib.pqg_index_destroy(self.h)
            except Exception:
                pass
            self.h = None

    def _info(self):
        nl, n = C.c_uint64(), C.c_uint64()
        M, ks, ds = C.c_uint32(), C.c_uint32(), C.c_uint32()
        _lib.check(self.ctx.lib.pqg_index_info(self.h, C.byref(nl), C.byref(n), C.byref(M),
                                               C.byref(ks), C.byref(ds)))
        return nl.value, n.value, M.value, ks.value, ds.value

    def nlist(self) -> int:
        return self._info()[0]

    @property
    def n_items(self) -> int:
        return self._info()[1]

    def export(self):
        """(offsets[nlist+1], ids[n], codes[n, row_bytes], coarse, codebook)."""
        nl, n, M, ks, ds = self._info()
        off = np.empty(nl + 1, np.uint64)
        ids = np.empty(max(n, 1), np.uint64)
        codes = np.empty((max(n, 1), M * code_width(ks)), np.uint8)
        coarse = np.empty((nl, M * ds), np.float32)
        tables = np.empty((M, ks, ds), np.float32)
        v = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        _lib.check(self.ctx.lib.pqg_index_export(self.ctx.h, self.h, v(off), v(ids), v(codes),
                                                 v(coarse), v(tables)))
        return off, ids[:n], codes[:n], coarse, Codebook(M, ks, ds, tables)

    @property
    def codebook(self) -> Codebook:
        return self.export()[4]

    @property
    def coarse_centroids(self) -> np.ndarray:
        return self.export()[3]

    @property
    def lists(self):
        """[(ids, CodeMatrix)] per list, in list order."""
        off, ids, codes, _, cb = self.export()
        out = []
        for l in range(len(off) - 1):
            a, b = int(off[l]), int(off[l + 1])
            out.append((ids[a:b], CodeMatrix(b - a, cb.m_subspaces, cb.ks, codes[a:b])))
        return out


def default_nlist(n_items: int) -> int:
    """ivf.cpp:118-121: round(sqrt(n)) clamped to [1, n] (llround: half away)."""
    r = int(math.floor(math.sqrt(float(n_items)) + 0.5))
    return max(1, min(r, n_items if n_items else 1))


def ivf_build_with_centroids(cb: Codebook, codes: CodeMatrix, ids, coarse_centroids,
                             ctx: Context | None = None) -> InvertedIndex:
    """ivf.cpp:151-166."""
    ctx = ctx or get_context()
    ids = np.ascontiguousarray(ids, np.uint64)
    coarse = np.ascontiguousarray(coarse_centroids, np.float32)
    if ids.size == 0:
        raise ValueError("ivf_build: no items")
    if ids.size != codes.rows:
        raise ValueError("ivf_build: ids/codes length mismatch")
    if coarse.ndim != 2 or coarse.shape[0] == 0 or coarse.shape[1] != cb.dims():
        raise ValueError("ivf_build: coarse centroids do not match the codebook")
    h = C.c_void_p()
    tp, _a = _ptr(np.ascontiguousarray(cb.tables, np.float32))
    cp, _b = _ptr(codes.bytes)
    _lib.check(ctx.lib.pqg_ivf_build_with_centroids(
        ctx.h, tp, cb.m_subspaces, cb.ks, cb.sub_dim, cp, ids.ctypes.data_as(C.c_void_p),
        codes.rows, coarse.ctypes.data_as(C.c_void_p), coarse.shape[0], C.byref(h)), "ivf_build")
    return InvertedIndex(h, ctx)


def ivf_build(cb: Codebook, codes: CodeMatrix, ids, nlist: int, seed: int,
              kmeans_iters: int = 20, ctx: Context | None = None) -> InvertedIndex:
    """ivf.cpp:123-149."""
    ctx = ctx or get_context()
    ids = np.ascontiguousarray(ids, np.uint64)
    if ids.size == 0:
        raise ValueError("ivf_build: no items")
    if ids.size != codes.rows:
        raise ValueError("ivf_build: ids/codes length mismatch")
    h = C.c_void_p()
    tp, _a = _ptr(np.ascontiguousarray(cb.tables, np.float32))
    cp, _b = _ptr(codes.bytes)
    _lib.check(ctx.lib.pqg_ivf_build(ctx.h, tp, cb.m_subspaces, cb.ks, cb.sub_dim, cp,
                                     ids.ctypes.data_as(C.c_void_p), codes.rows, nlist, seed,
                                     kmeans_iters, C.byref(h)), "ivf_build")
    return InvertedIndex(h, ctx)


def ivf_add(index: InvertedIndex, codes: CodeMatrix, ids) -> None:
    """ivf.cpp:168-184."""
    ids = np.ascontiguousarray(ids, np.uint64)
    if ids.size != codes.rows:
        raise ValueError("ivf_add: ids/codes length mismatch")
    _, _, M, ks, _ = index._info()
    if codes.m_subspaces != M or codes.ks != ks:
        raise ValueError("ivf_add: codes do not match the index codebook")
    if ids.size == 0:
        return
    cp, _b = _ptr(codes.bytes)
    _lib.check(index.ctx.lib.pqg_index_add(index.ctx.h, index.h, cp,
                                           ids.ctypes.data_as(C.c_void_p), ids.size), "ivf_add")


def ivf_merge(a: InvertedIndex, b: InvertedIndex) -> InvertedIndex:
    """ivf.cpp:186-216."""
    h = C.c_void_p()
    _lib.check(a.ctx.lib.pqg_index_merge(a.ctx.h, a.h, b.h, C.byref(h)), "ivf_merge")
    return InvertedIndex(h, a.ctx)


# ---------------------------------------------------------------------------
# on-disk formats (pq.cpp:183-259, ivf.cpp:264-355): byte-identical files,
# posting lists packed / unpacked and validated on the device
# ---------------------------------------------------------------------------


def save_index(index: InvertedIndex, path: str) -> None:
    """save_index (ivf.cpp:264-293)."""
    _lib.check(index.ctx.lib.pqg_index_save(index.ctx.h, index.h, os.fsencode(path)), "save_index")


def load_index(path: str, ctx: Context | None = None) -> InvertedIndex:
    """load_index (ivf.cpp:295-355): device-resident index straight from the file."""
    ctx = ctx or get_context()
    h = C.c_void_p()
    _lib.check(ctx.lib.pqg_index_load(ctx.h, os.fsencode(path), C.byref(h)), "load_index")
    return InvertedIndex(h, ctx)


def serialize_index(index: InvertedIndex) -> bytes:
    """The PQII file image of ``index`` in memory."""
    n = C.c_uint64()
    _lib.check(index.ctx.lib.pqg_index_serialize(index.ctx.h, index.h, None, 0, C.byref(n)), "serialize")
    buf = np.empty(n.value, np.uint8)
    _lib.check(index.ctx.lib.pqg_index_serialize(index.ctx.h, index.h, buf.ctypes.data_as(C.c_void_p), n.value,
                                                 C.byref(n)), "serialize")
    return buf.tobytes()


def deserialize_index(image, name: str = "index image", ctx: Context | None = None) -> InvertedIndex:
    """load_index over an in-memory PQII image (bytes, numpy u8 or a CUDA tensor)."""
    ctx = ctx or get_context()
    if isinstance(image, (bytes, bytearray)):
        image = np.frombuffer(image, np.uint8)
    ip, _keep = _ptr(image)
    nbytes = int(image.nbytes) if hasattr(image, "nbytes") else int(image.numel() * image.element_size())
    h = C.c_void_p()
    _lib.check(ctx.lib.pqg_index_deserialize(ctx.h, ip, nbytes, name.encode(), C.byref(h)), "deserialize")
    return InvertedIndex(h, ctx)


def save_codes(codes: CodeMatrix, path: str, ctx: Context | None = None) -> None:
    """save_codes (pq.cpp:221-232)."""
    ctx = ctx or get_context()
    cp, _k = _ptr(codes.bytes)
    _lib.check(ctx.lib.pqg_codes_save(ctx.h, cp, codes.rows, codes.m_subspaces, codes.ks, os.fsencode(path)),
               "save_codes")


def load_codes(path: str, ctx: Context | None = None) -> CodeMatrix:
    """load_codes (pq.cpp:234-259): every code range-checked on the device."""
    ctx = ctx or get_context()
    n, M, ks = C.c_uint64(), C.c_uint32(), C.c_uint32()
    _lib.check(ctx.lib.pqg_codes_file_info(os.fsencode(path), C.byref(n), C.byref(M), C.byref(ks)), "load_codes")
    out = np.empty((n.value, M.value * code_width(ks.value)), np.uint8)
    _lib.check(ctx.lib.pqg_codes_load(ctx.h, os.fsencode(path), out.ctypes.data_as(C.c_void_p), out.nbytes),
               "load_codes")
    return CodeMatrix(n.value, M.value, ks.value, out)


def save_codebook(cb: Codebook, path: str, ctx: Context | None = None) -> None:
    """save_codebook (pq.cpp:183-194)."""
    ctx = ctx or get_context()
    tp, _k = _ptr(_f32(cb.tables))
    _lib.check(ctx.lib.pqg_codebook_save(ctx.h, tp, cb.m_subspaces, cb.ks, cb.sub_dim, os.fsencode(path)),
               "save_codebook")


def load_codebook(path: str, ctx: Context | None = None) -> Codebook:
    """load_codebook (pq.cpp:196-219): codewords checked finite on the device."""
    ctx = ctx or get_context()
    M, ks, ds = C.c_uint32(), C.c_uint32(), C.c_uint32()
    _lib.check(ctx.lib.pqg_codebook_file_info(os.fsencode(path), C.byref(M), C.byref(ks), C.byref(ds)),
               "load_codebook")
    t = np.empty((M.value, ks.value, ds.value), np.float32)
    _lib.check(ctx.lib.pqg_codebook_load(ctx.h, os.fsencode(path), t.ctypes.data_as(C.c_void_p), t.size),
               "load_codebook")
    return Codebook(M.value, ks.value, ds.value, t)


def ivf_query_batch(index: InvertedIndex, queries, k: int, nprobe: int, max_sq_dist=None,
                    out=None):
    """Batched ivf_query: (ids [nq,k] u64, dists [nq,k] f64, counts [nq] u32)."""
    ctx = index.ctx
    q = _f32(queries)
    nq = q.shape[0] if q.ndim == 2 else 1
    if out is None:
        ids = np.zeros((nq, max(k, 1)), np.uint64)
        dist = np.zeros((nq, max(k, 1)), np.float64)
        cnt = np.zeros(nq, np.uint32)
    else:
        ids, dist, cnt = out
    qp, _a = _ptr(q)
    ip, _b = _ptr(ids)
    dp, _c = _ptr(dist)
    cp, _d = _ptr(cnt)
    _lib.check(ctx.lib.pqg_index_search(ctx.h, index.h, qp, nq, k, nprobe,
                                        int(max_sq_dist is not None),
                                        0.0 if max_sq_dist is None else float(max_sq_dist),
                                        ip, dp, cp), "ivf_query")
    return ids, dist, cnt


def _to_result(ids, dist, cnt, k) -> QueryResult:
    c = int(cnt)
    return QueryResult([Hit(int(ids[j]), float(dist[j])) for j in range(c)], k)


def ivf_query(index: InvertedIndex, query, k: int, nprobe: int, max_sq_dist=None) -> QueryResult:
    """ivf.cpp:218-228."""
    q = np.ascontiguousarray(query, np.float32).reshape(1, -1)
    nl, _, M, _, ds = index._info()
    if k == 0:
        raise ValueError("query: k must be >= 1")
    if q.shape[1] != M * ds:
        raise ValueError("query: dimension mismatch")
    ids, dist, cnt = ivf_query_batch(index, q, k, nprobe, max_sq_dist)
    return _to_result(ids[0], dist[0], cnt[0], k)


def ivf_probe(index: InvertedIndex, queries, nprobe: int) -> np.ndarray:
    """probe_order (ivf.cpp:91-101) for a batch of queries."""
    ctx = index.ctx
    q = _f32(queries)
    nq = q.shape[0]
    out = np.empty((nq, nprobe), np.uint32)
    qp, _a = _ptr(q)
    _lib.check(ctx.lib.pqg_index_probe(ctx.h, index.h, qp, nq, nprobe,
                                       out.ctypes.data_as(C.c_void_p)), "ivf_probe")
    return out


def flat_scan_batch(cb: Codebook, codes: CodeMatrix, ids, queries, k: int, max_sq_dist=None,
                    ctx: Context | None = None):
    ctx = ctx or get_context()
    ids = np.ascontiguousarray(ids, np.uint64)
    if k == 0:
        raise ValueError("flat_scan: k must be >= 1")
    if ids.size != codes.rows:
        raise ValueError("flat_scan: ids/codes length mismatch")
    q = _f32(queries)
    if q.ndim == 1:
        q = q.reshape(1, -1)
    if q.shape[1] != cb.dims():
        raise ValueError("flat_scan: dimension mismatch")
    nq = q.shape[0]
    oi = np.zeros((nq, k), np.uint64)
    od = np.zeros((nq, k), np.float64)
    oc = np.zeros(nq, np.uint32)
    tp, _a = _ptr(np.ascontiguousarray(cb.tables, np.float32))
    cp, _b = _ptr(codes.bytes)
    qp, _c = _ptr(q)
    _lib.check(ctx.lib.pqg_flat_scan(ctx.h, tp, cb.m_subspaces, cb.ks, cb.sub_dim, cp,
                                     ids.ctypes.data_as(C.c_void_p), codes.rows, qp, nq, k,
                                     int(max_sq_dist is not None),
                                     0.0 if max_sq_dist is None else float(max_sq_dist),
                                     oi.ctypes.data_as(C.c_void_p), od.ctypes.data_as(C.c_void_p),
                                     oc.ctypes.data_as(C.c_void_p)), "flat_scan")
    return oi, od, oc


def flat_scan(cb: Codebook, codes: CodeMatrix, ids, query, k: int, max_sq_dist=None,
              ctx: Context | None = None) -> QueryResult:
    """ivf.cpp:247-262."""
    oi, od, oc = flat_scan_batch(cb, codes, ids, np.asarray(query).reshape(1, -1), k, max_sq_dist,
                                 ctx)
    return _to_result(oi[0], od[0], oc[0], k)


def ivf_query_subset(index: InvertedIndex, query, k: int, subset, nprobe: int,
                     max_sq_dist=None) -> QueryResult:
    """ivf.cpp:230-245: ivf_query restricted to ids in ``subset`` (sorted
    ascending, unique); the membership test runs inside the device scan."""
    subset = np.ascontiguousarray(subset, np.uint64)
    q = np.ascontiguousarray(query, np.float32).reshape(1, -1)
    _, _, M, _, ds = index._info()
    if k == 0:
        raise ValueError("query: k must be >= 1")
    if q.shape[1] != M * ds:
        raise ValueError("query: dimension mismatch")
    ctx = index.ctx
    ids = np.zeros((1, k), np.uint64)
    dist = np.zeros((1, k), np.float64)
    cnt = np.zeros(1, np.uint32)
    v = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    _lib.check(ctx.lib.pqg_index_search_subset(
        ctx.h, index.h, v(q), 1, k, v(subset) if subset.size else None, subset.size, nprobe,
        int(max_sq_dist is not None), 0.0 if max_sq_dist is None else float(max_sq_dist), v(ids),
        v(dist), v(cnt)), "ivf_query_subset")
    return _to_result(ids[0], dist[0], cnt[0], k)


# ---------------------------------------------------------------------------
# L3: pipeline.hpp -- the paper's chunked fit (proj/src/pipeline.cpp)
# ---------------------------------------------------------------------------
PIPELINE_MODES = ("single", "parallel_pq", "parallel_pq_index")
_PHASES = ("fit", "chunking", "local_fit", "global_fit", "coarse_fit", "encode", "index_build",
           "merge")


def parse_mode(name: str):
    """pipeline.cpp:78-83: the mode for a name, else None."""
    return name if name in PIPELINE_MODES else None


@dataclass
class PipelineConfig:  # pipeline.hpp:27-36
    n_chunks: int = 1
    m_subspaces: int = 8
    ks: int = 256
    nlist: int = 0
    kmeans_iters: int = 20
    seed: int = 0
    n_threads: int = 1
    mode: str = "single"


@dataclass
class ChunkOutput:  # pipeline.hpp:40-45
    chunk_id: int
    representatives: np.ndarray  # ks x D
    local_rmse: float
    wall_seconds: float = 0.0


@dataclass
class PipelineReport:  # pipeline.hpp:47-58
    config: PipelineConfig
    global_codebook: Codebook
    global_rmse: float
    single_rmse: float | None = None
    phase_seconds: dict = field(default_factory=dict)
    total_seconds: float = 0.0
    representatives: np.ndarray | None = None
    merged_index: InvertedIndex | None = None
    local_rmse: np.ndarray | None = None

    def summary(self) -> str:
        """PipelineReport::summary (pipeline.cpp:268-293)."""
        c = self.config
        out = [f"mode: {c.mode}",
               f"params: M={c.m_subspaces} Ks={c.ks} C={c.n_chunks} T={c.n_threads} "
               f"nlist={c.nlist} iters={c.kmeans_iters} seed={c.seed}",
               "phases:" + "".join(f" {k}={v:.3f}s" for k, v in sorted(self.phase_seconds.items())),
               f"total: {self.total_seconds:.3f}s",
               f"rmse: {self.global_rmse:.9g}"]
        if self.merged_index is not None:
            out.append(f"index: {self.merged_index.n_items} items across "
                       f"{self.merged_index.nlist()} lists")
        return "\n".join(out) + "\n"


def train_chunks(data, n_chunks: int, m: int, ks: int, max_iters: int = 20, seed: int = 0,
                 ctx: Context | None = None) -> list[ChunkOutput]:
    """train_chunk (pipeline.cpp:84-106) for every chunk of chunk_rows(n,
    n_chunks), chunk c with seed + c -- one batched k-means on the device."""
    ctx = ctx or get_context()
    data = _f32(data)
    n, D = data.shape
    reps = np.empty((max(n_chunks, 1) * max(ks, 1), D), np.float32)
    local = np.empty(max(n_chunks, 1), np.float64)
    dp, _a = _ptr(data)
    _lib.check(ctx.lib.pqg_train_chunks(ctx.h, dp, n, D, n_chunks, m, ks, max_iters, seed,
                                        reps.ctypes.data_as(C.c_void_p),
                                        local.ctypes.data_as(C.c_void_p), None), "train_chunk")
    return [ChunkOutput(c, reps[c * ks:(c + 1) * ks], float(local[c])) for c in range(n_chunks)]


def aggregate_representatives(outputs: list[ChunkOutput]) -> np.ndarray:
    """pipeline.cpp:108-135: row concatenation in ascending chunk_id order."""
    if not outputs:
        raise ValueError("aggregate_representatives: no outputs")
    d = outputs[0].representatives.shape[1]
    for o in outputs:
        if o.representatives.shape[1] != d:
            raise ValueError(f"aggregate_representatives: dimension mismatch at chunk {o.chunk_id}")
    return np.concatenate([o.representatives for o in sorted(outputs, key=lambda o: o.chunk_id)])


def fit_global(representatives, m: int, ks: int, iters: int, seed: int,
               ctx: Context | None = None) -> Codebook:
    """pipeline.cpp:137-140."""
    return pq_fit(representatives, m, ks, iters, seed, ctx=ctx)


def run_pipeline(data, config: PipelineConfig, ctx: Context | None = None) -> PipelineReport:
    """run_pipeline (pipeline.cpp:142-266) on the device: the chunks' local
    fits are one batched k-means, and the data stays resident between phases."""
    ctx = ctx or get_context()
    if config.n_threads == 0:
        raise ValueError("run_pipeline: n_threads must be >= 1")
    if config.mode not in PIPELINE_MODES:
        raise ValueError(f"run_pipeline: unknown mode {config.mode}")
    mode = PIPELINE_MODES.index(config.mode)
    data = _f32(data)
    n, D = data.shape
    t0 = time.perf_counter()
    M, ks = config.m_subspaces, config.ks
    ds = D // M if M and D % M == 0 else 1
    tables = np.empty((M, max(ks, 1), ds), np.float32)
    C_ = config.n_chunks
    reps = np.empty((max(C_, 1) * max(ks, 1), D), np.float32) if mode else None
    local = np.empty(max(C_, 1), np.float64) if mode else None
    rm = C.c_double()
    nl = C.c_uint64()
    h = C.c_void_p()
    ph = np.full(8, -1.0)
    dp, _a = _ptr(data)
    v = lambda a: None if a is None else a.ctypes.data_as(C.c_void_p)  # noqa: E731
    _lib.check(ctx.lib.pqg_pipeline_run(ctx.h, dp, n, D, C_, M, ks, config.nlist,
                                        config.kmeans_iters, config.seed, mode, v(tables),
                                        C.byref(rm), v(reps), v(local), C.byref(nl),
                                        C.byref(h) if mode == 2 else None, v(ph)),
               "run_pipeline")
    cfg = PipelineConfig(**{**config.__dict__, "nlist": nl.value})
    rep = PipelineReport(cfg, Codebook(M, ks, ds, tables), rm.value,
                         phase_seconds={k: float(t) for k, t in zip(_PHASES, ph) if t >= 0})
    if mode == 0:
        rep.single_rmse = rm.value
    else:
        rep.representatives = reps
        rep.local_rmse = local
    if h.value:
        rep.merged_index = InvertedIndex(h, ctx)
    rep.total_seconds = time.perf_counter() - t0
    return rep
