"""Writes tests/golden/formats/: PQII / PQCM / PQCB files written by the
REFERENCE's own save_index / save_codes / save_codebook (oracle/_ref, compiled
from /root/reference sources by `make -C oracle`), plus formats.npz with the
inputs and the CSR the reference's load_index reads back.

    python tests/golden/make_format_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2604_21645_b200.datagen import gaussian_mixture  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "formats")


def main() -> None:
    os.makedirs(OUT, exist_ok=True)
    R = oracle.ref_impl()
    g: dict[str, np.ndarray] = {}
    # byte codes (Ks <= 256): 150 rows, D=16, M=4, Ks=16, nlist 10 (test_ivf.cpp:357-384 shape)
    data = gaussian_mixture(150, 16, 8, 61)
    tables = R.pq_fit(data, 4, 16, 15, 3)
    codes = R.pq_encode(data, tables)
    ids = (np.arange(150, dtype=np.uint64) * 7 + 3)
    coarse = data[::15][:10].copy()
    h = R.ivf_build_with_centroids(codes, ids, tables, coarse)
    rc, msg = R.save_index(h, os.path.join(OUT, "byte.pqii"))
    assert rc == 0, msg
    off, lid, lcodes, co = h.export()
    g.update({"byte/tables": tables, "byte/codes": codes, "byte/ids": ids, "byte/coarse": coarse,
              "byte/offsets": off, "byte/list_ids": lid, "byte/list_codes": lcodes})
    assert R.save_codes(codes, 4, 16, os.path.join(OUT, "codes.pqcm"))[0] == 0
    assert R.save_codebook(tables, os.path.join(OUT, "codebook.pqcb"))[0] == 0
    # Ks = 200 < 256: byte codes whose range check is live (codes >= 200 are invalid)
    data2 = gaussian_mixture(400, 8, 16, 62)
    t2 = R.pq_fit(data2, 2, 200, 6, 4)
    c2 = R.pq_encode(data2, t2)
    ids2 = np.arange(400, dtype=np.uint64)
    h2 = R.ivf_build_with_centroids(c2, ids2, t2, data2[::50][:8].copy())
    assert R.save_index(h2, os.path.join(OUT, "ks200.pqii"))[0] == 0
    g.update({"ks200/tables": t2, "ks200/codes": c2})
    # wide codes (Ks > 256): test_ivf.cpp:385-404 shape (600 x 8, M=2, Ks=300)
    data3 = R.random_matrix(600, 8, 71, -10, 10)
    t3 = R.pq_fit(data3, 2, 300, 8, 3)
    c3 = R.pq_encode(data3, t3)
    ids3 = np.arange(600, dtype=np.uint64)
    h3 = R.ivf_build(c3, ids3, t3, 5, 7)
    assert R.save_index(h3, os.path.join(OUT, "wide.pqii"))[0] == 0
    off3, lid3, lcodes3, co3 = h3.export()
    g.update({"wide/tables": t3, "wide/codes": c3, "wide/offsets": off3, "wide/list_ids": lid3,
              "wide/list_codes": lcodes3, "wide/coarse": co3})
    np.savez_compressed(os.path.join(OUT, "formats.npz"), **g)
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
