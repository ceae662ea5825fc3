"""The tensor-core screened search (adc_tc.cu) against the LUT scan and the
reference's golden fixtures: both are exact, so every id, fp64 distance and
count must be identical.  PQG_ADC=tc forces the tensor-core path at any batch
size, PQG_ADC=lut the LUT scan."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view({4: np.uint32, 8: np.uint64}[a.dtype.itemsize])


@pytest.fixture(scope="module")
def pq():
    from paper_2604_21645_b200 import pqii
    return pqii


class adc_mode:
    def __init__(self, mode):
        self.mode = mode

    def __enter__(self):
        self.old = os.environ.get("PQG_ADC")
        os.environ["PQG_ADC"] = self.mode

    def __exit__(self, *exc):
        if self.old is None:
            os.environ.pop("PQG_ADC", None)
        else:
            os.environ["PQG_ADC"] = self.old


def both(pq, index, q, k, nprobe, **kw):
    with adc_mode("lut"):
        a = pq.ivf_query_batch(index, q, k, nprobe, **kw)
    with adc_mode("tc"):
        b = pq.ivf_query_batch(index, q, k, nprobe, **kw)
    return a, b


def same(a, b):
    ai, ad, ac = a
    bi, bd, bc = b
    assert np.array_equal(ac, bc)
    for i in range(len(ac)):
        c = int(ac[i])
        assert np.array_equal(ai[i, :c], bi[i, :c]), i
        assert np.array_equal(bits(ad[i, :c]), bits(bd[i, :c])), i


@pytest.mark.parametrize("nprobe", [1, 4, 40])
def test_tc_search_golden(pq, golden, nprobe):
    tables = golden["pq/tables"]
    cb = pq.Codebook(*tables.shape, tables)
    codes = pq.CodeMatrix(golden["pq/codes"].shape[0], tables.shape[0], tables.shape[1],
                          golden["pq/codes"])
    index = pq.ivf_build_with_centroids(cb, codes, golden["ivf/ids"], golden["ivf/coarse"])
    with adc_mode("tc"):
        ids, dist, cnt = pq.ivf_query_batch(index, golden["ivf/queries"], 10, nprobe)
        mi, md, mc = pq.ivf_query_batch(index, golden["ivf/queries"], 10, 4, max_sq_dist=60.0)
    assert np.array_equal(cnt, golden[f"ivf/q_np{nprobe}_count"])
    for q in range(len(cnt)):
        c = int(cnt[q])
        assert np.array_equal(ids[q, :c], golden[f"ivf/q_np{nprobe}_ids"][q, :c])
        assert np.array_equal(bits(dist[q, :c]), bits(golden[f"ivf/q_np{nprobe}_dist"][q, :c]))
    assert np.array_equal(mc, golden["ivf/q_max_count"])
    for q in range(len(mc)):
        assert np.array_equal(mi[q, : mc[q]], golden["ivf/q_max_ids"][q, : mc[q]])


@pytest.mark.parametrize("M,ks,D", [(16, 256, 128), (8, 256, 64), (4, 16, 32), (12, 64, 96),
                                    (2, 300, 16)])
@pytest.mark.parametrize("k,nprobe", [(10, 16), (1, 3), (16, 64)])
def test_tc_vs_lut(pq, M, ks, D, k, nprobe):
    from paper_2604_21645_b200.datagen import gaussian_mixture
    n = 30_000
    x = gaussian_mixture(n, D, 40, 11)
    cb = pq.pq_fit(x[:5000], M, ks, 6, 3)
    codes = pq.pq_encode(cb, x)
    ids = (np.arange(n, dtype=np.uint64) * 3 + 7)
    coarse = pq.kmeans_fit(x[:5000], 64, 5, 2).centroids
    index = pq.ivf_build_with_centroids(cb, codes, ids, coarse)
    q = gaussian_mixture(700, D, 40, 11, stream=1)
    a, b = both(pq, index, q, k, min(nprobe, 64))
    same(a, b)


def test_tc_duplicate_codes_ties_and_max(pq, orc):
    # identical code rows -> exact distance ties broken by id, across lists
    rng = np.random.default_rng(4)
    tables = orc.random_matrix(8 * 16, 4, 9).reshape(8, 16, 4)
    base = rng.integers(0, 16, size=(50, 8), dtype=np.uint8)
    codes_b = base[rng.integers(0, 50, size=20000)]
    ids = rng.permutation(1000000)[:20000].astype(np.uint64)
    cb = pq.Codebook(8, 16, 4, np.ascontiguousarray(tables, np.float32))
    codes = pq.CodeMatrix(20000, 8, 16, np.ascontiguousarray(codes_b))
    coarse = pq.pq_decode(cb, pq.CodeMatrix(12, 8, 16, np.ascontiguousarray(base[:12])))
    index = pq.ivf_build_with_centroids(cb, codes, ids, coarse)
    q = orc.random_matrix(600, 32, 77)
    for k in (1, 10, 16):
        a, b = both(pq, index, q, k, 5)
        same(a, b)
    a, b = both(pq, index, q, 10, 12, max_sq_dist=9.0)
    same(a, b)


def test_tc_subset_and_add(pq):
    from paper_2604_21645_b200.datagen import gaussian_mixture
    x = gaussian_mixture(20_000, 32, 30, 5)
    cb = pq.pq_fit(x[:4000], 8, 64, 5, 1)
    codes = pq.pq_encode(cb, x)
    coarse = pq.kmeans_fit(x[:4000], 50, 5, 2).centroids
    index = pq.ivf_build_with_centroids(cb, pq.CodeMatrix(15000, 8, 64, codes.bytes[:15000]),
                                        np.arange(15000, dtype=np.uint64), coarse)
    q = gaussian_mixture(600, 32, 30, 5, stream=1)
    a, b = both(pq, index, q, 10, 8)  # builds the cached operand
    same(a, b)
    # ivf_add invalidates the cached decoded operand
    pq.ivf_add(index, pq.CodeMatrix(5000, 8, 64, codes.bytes[15000:]),
               np.arange(15000, 20000, dtype=np.uint64))
    a, b = both(pq, index, q, 10, 8)
    same(a, b)
    assert (a[0][a[2] > 0] >= 15000).any()
    sub = np.arange(0, 20000, 3, dtype=np.uint64)
    with adc_mode("lut"):
        la = [pq.ivf_query_subset(index, qq, 10, sub, 8) for qq in q[:40]]
    with adc_mode("tc"):
        lb = [pq.ivf_query_subset(index, qq, 10, sub, 8) for qq in q[:40]]
    for r1, r2 in zip(la, lb):
        assert r1.hits == r2.hits
