"""On-disk formats: PQII / PQCM / PQCB.

Reference: proj/src/pq.cpp:183-259 (save/load_codebook, save/load_codes),
proj/src/ivf.cpp:264-355 (save/load_index), proj/src/io_util.hpp:45-87
(read_bytes / expect_magic messages); reference tests restated here:
proj/tests/test_ivf.cpp:357-407 ("index serialization round-trips
bit-exactly": byte codes, wide codes, bad magic) and
proj/tests/test_pq.cpp:302-329 ("codebook and code files round-trip").

Fixtures in tests/golden/formats/ were written by the reference's own savers
(tests/golden/make_format_golden.py).  CPU tests pin the fixtures' byte
layout with an independent struct reader; GPU tests load / save through the
C ABI (device pack / unpack / validation) and compare bytes, arrays and --
for every corruption -- the exception class and message with the compiled
reference (oracle/_ref) run on the same file.
"""
from __future__ import annotations

import os
import struct

import numpy as np
import pytest

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "formats")


def _npz():
    return np.load(os.path.join(GOLD, "formats.npz"))


def _read(name):
    with open(os.path.join(GOLD, name), "rb") as f:
        return f.read()


def parse_pqii(b: bytes):
    """Independent reader of the PQII layout (ivf.cpp:264-293), test-side."""
    assert b[:4] == b"PQII" and struct.unpack_from("<I", b, 4)[0] == 1
    assert b[8:12] == b"PQCB" and struct.unpack_from("<I", b, 12)[0] == 1
    M, ks, ds = struct.unpack_from("<III", b, 16)
    p = 28
    tables = np.frombuffer(b, np.float32, M * ks * ds, p).reshape(M, ks, ds)
    p += 4 * M * ks * ds
    nlist = struct.unpack_from("<I", b, p)[0]
    p += 4
    coarse = np.frombuffer(b, np.float32, nlist * M * ds, p).reshape(nlist, M * ds)
    p += 4 * nlist * M * ds
    rb = M * (1 if ks <= 256 else 2)
    off, ids, codes = [0], [], []
    for _ in range(nlist):
        n = struct.unpack_from("<Q", b, p)[0]
        p += 8
        for _ in range(n):
            ids.append(struct.unpack_from("<Q", b, p)[0])
            codes.append(np.frombuffer(b, np.uint8, rb, p + 8))
            p += 8 + rb
        off.append(off[-1] + n)
    assert p == len(b)
    return tables, coarse, np.array(off, np.uint64), np.array(ids, np.uint64), np.array(codes, np.uint8).reshape(-1, rb)


# ---------------------------------------------------------------------------
# CPU: the fixtures' byte layout
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("name", ["byte", "wide"])
def test_golden_pqii_layout(name):
    g = _npz()
    tables, coarse, off, ids, codes = parse_pqii(_read(f"{name}.pqii"))
    assert np.array_equal(tables, g[f"{name}/tables"])
    assert np.array_equal(off, g[f"{name}/offsets"])
    assert np.array_equal(ids, g[f"{name}/list_ids"])
    assert np.array_equal(codes, g[f"{name}/list_codes"])
    if name == "byte":
        assert np.array_equal(coarse, g["byte/coarse"])


def test_golden_pqcm_pqcb_layout():
    g = _npz()
    b = _read("codes.pqcm")
    assert b[:4] == b"PQCM" and struct.unpack_from("<IQII", b, 4) == (1, 150, 4, 16)
    assert np.array_equal(np.frombuffer(b, np.uint8, offset=24).reshape(150, 4), g["byte/codes"])
    b = _read("codebook.pqcb")
    assert b[:4] == b"PQCB" and struct.unpack_from("<IIII", b, 4) == (1, 4, 16, 4)
    assert np.array_equal(np.frombuffer(b, np.float32, offset=20).reshape(4, 16, 4), g["byte/tables"])


# ---------------------------------------------------------------------------
# GPU
# ---------------------------------------------------------------------------


def _gpu():
    from paper_2604_21645_b200 import _lib, pqii
    return pqii, _lib


def _ref():
    if not os.path.exists(oracle.REF_LIB_PATH):
        pytest.skip("oracle/_ref not built")
    return oracle.ref_impl()


def _outcome_ours(fn):
    pqii, _lib = _gpu()
    try:
        fn()
        return 0, ""
    except ValueError as e:
        return -1, str(e)
    except IndexError as e:
        return -2, str(e)
    except _lib.PQGError as e:
        return -4, str(e)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["byte", "ks200", "wide"])
def test_load_golden_index(name):
    pqii, _ = _gpu()
    ix = pqii.load_index(os.path.join(GOLD, f"{name}.pqii"))
    tables, coarse, off, ids, codes = parse_pqii(_read(f"{name}.pqii"))
    o, i, c, co, cb = ix.export()
    assert np.array_equal(o, off) and np.array_equal(i, ids) and np.array_equal(c, codes)
    assert np.array_equal(co, coarse) and np.array_equal(cb.tables, tables)
    assert ix.n_items == ids.size and ix.nlist() == off.size - 1


@pytest.mark.gpu
def test_save_matches_reference_bytes(tmp_path):
    """An index built on the GPU from the fixture inputs saves to the
    reference's own file byte for byte."""
    pqii, _ = _gpu()
    g = _npz()
    t = g["byte/tables"]
    cb = pqii.Codebook(*t.shape, t)
    codes = pqii.CodeMatrix(150, 4, 16, g["byte/codes"])
    ix = pqii.ivf_build_with_centroids(cb, codes, g["byte/ids"], g["byte/coarse"])
    p = str(tmp_path / "ours.pqii")
    pqii.save_index(ix, p)
    assert open(p, "rb").read() == _read("byte.pqii")
    assert pqii.serialize_index(ix) == _read("byte.pqii")


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["byte", "wide"])
def test_index_roundtrip_bit_exact(tmp_path, name):
    """test_ivf.cpp:357-404: save -> load -> save is byte-identical, the loaded
    index answers queries identically, wide codes survive."""
    pqii, _ = _gpu()
    a = pqii.load_index(os.path.join(GOLD, f"{name}.pqii"))
    p1, p2 = str(tmp_path / "a.pqii"), str(tmp_path / "b.pqii")
    pqii.save_index(a, p1)
    b = pqii.load_index(p1)
    pqii.save_index(b, p2)
    assert open(p1, "rb").read() == open(p2, "rb").read() == _read(f"{name}.pqii")
    D = a.codebook.dims()
    q = np.random.default_rng(9).standard_normal((8, D)).astype(np.float32)
    nprobe = min(5, a.nlist())
    ra = pqii.ivf_query_batch(a, q, 10, nprobe)
    rb = pqii.ivf_query_batch(b, q, 10, nprobe)
    for x, y in zip(ra, rb):
        assert np.array_equal(x, y)


@pytest.mark.gpu
def test_index_memory_images(tmp_path):
    """serialize / deserialize from host bytes and from a device buffer."""
    import torch
    pqii, _ = _gpu()
    img = _read("ks200.pqii")
    a = pqii.deserialize_index(img, "mem")
    assert pqii.serialize_index(a) == img
    dev = torch.from_numpy(np.frombuffer(img, np.uint8).copy()).cuda()
    b = pqii.deserialize_index(dev, "dev")
    assert pqii.serialize_index(b) == img


def _mutations(img: bytes, rb: int, hdr: int):
    """(label, bytes) corruptions of a PQII image covering every check of
    load_index in its order (ivf.cpp:295-355)."""
    out = []
    for n in sorted(set(list(range(0, min(len(img), 64))) + list(range(hdr - 6, hdr + 40)) +
                        list(range(len(img) - 30, len(img))) + list(range(64, len(img), 97)))):
        if 0 <= n < len(img):
            out.append((f"trunc{n}", img[:n]))
    out.append(("trailing", img + b"\x00"))
    b = bytearray(img); b[0] = ord("Z"); out.append(("bad_magic", bytes(b)))
    b = bytearray(img); b[9] = ord("x"); out.append(("bad_cb_magic", bytes(b)))
    b = bytearray(img); struct.pack_into("<I", b, 4, 2); out.append(("version", bytes(b)))
    b = bytearray(img); struct.pack_into("<I", b, 12, 3); out.append(("cb_version", bytes(b)))
    b = bytearray(img); struct.pack_into("<I", b, 16, 0); out.append(("M0", bytes(b)))
    b = bytearray(img); struct.pack_into("<I", b, 20, 70000); out.append(("ks_huge", bytes(b)))
    M, ks, ds = struct.unpack_from("<III", img, 16)
    p_nlist = 28 + 4 * M * ks * ds
    b = bytearray(img); struct.pack_into("<I", b, p_nlist, 0); out.append(("nlist0", bytes(b)))
    # entries: walk to find (list, entry) byte positions
    pos, ent = hdr, []
    nlist = struct.unpack_from("<I", img, p_nlist)[0]
    for l in range(nlist):
        n = struct.unpack_from("<Q", img, pos)[0]
        pos += 8
        for e in range(n):
            ent.append((l, e, pos))
            pos += 8 + rb
    if len(ent) > 10:
        first_id = struct.unpack_from("<Q", img, ent[0][2])[0]
        b = bytearray(img); struct.pack_into("<Q", b, ent[-1][2], first_id); out.append(("dup_last", bytes(b)))
        same = [e for e in ent if e[0] == ent[-1][0]]
        if len(same) >= 2:
            i0 = struct.unpack_from("<Q", img, same[0][2])[0]
            b = bytearray(img); struct.pack_into("<Q", b, same[1][2], i0); out.append(("dup_same_list", bytes(b)))
        if ks < 256 and rb == M:
            mid = ent[len(ent) // 2]
            b = bytearray(img); b[mid[2] + 8] = 255; out.append(("code_range", bytes(b)))
            # a range error in an early list beats a duplicate in a later one, not vice versa
            b2 = bytearray(b); struct.pack_into("<Q", b2, ent[-1][2], first_id); out.append(("range_then_dup", bytes(b2)))
            b3 = bytearray(img); b3[ent[-1][2] + 8] = 254
            struct.pack_into("<Q", b3, ent[1][2], first_id); out.append(("dup_then_range", bytes(b3)))
            b4 = bytearray(img); b4[ent[0][2] + 8] = 253; out.append(("range_then_trunc", bytes(b4[:-5])))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["byte", "ks200", "wide"])
def test_index_load_errors_match_reference(tmp_path, name):
    pqii, _ = _gpu()
    R = _ref()
    img = _read(f"{name}.pqii")
    M, ks, ds = struct.unpack_from("<III", img, 16)
    rb = M * (1 if ks <= 256 else 2)
    nlist = struct.unpack_from("<I", img, 28 + 4 * M * ks * ds)[0]
    hdr = 28 + 4 * M * ks * ds + 4 + 4 * nlist * M * ds
    cases = _mutations(img, rb, hdr)
    assert len(cases) > 80
    for label, data in cases:
        p = str(tmp_path / f"{label}.pqii")
        with open(p, "wb") as f:
            f.write(data)
        rs, rm, rh = R.load_index(p, rb, M * ds)
        os_, om = _outcome_ours(lambda: pqii.load_index(p))
        assert (os_, om) == (rs, rm), (label, (os_, om), (rs, rm))
        if rs == 0:  # loadable: same lists
            ours = pqii.load_index(p).export()
            ref = rh.export()
            for x, y in zip(ours[:3], ref[:3]):
                assert np.array_equal(x, y), label


@pytest.mark.gpu
def test_codebook_and_code_files_roundtrip(tmp_path):
    """test_pq.cpp:302-329 (plus byte equality with the reference's files)."""
    pqii, _ = _gpu()
    R = _ref()
    g = _npz()
    cb = pqii.Codebook(4, 16, 4, g["byte/tables"])
    codes = pqii.CodeMatrix(150, 4, 16, g["byte/codes"])
    pc, pk = str(tmp_path / "cb.pqcb"), str(tmp_path / "codes.pqcm")
    pqii.save_codebook(cb, pc)
    assert pqii.load_codebook(pc) == cb
    pqii.save_codes(codes, pk)
    assert pqii.load_codes(pk) == codes
    assert open(pc, "rb").read() == _read("codebook.pqcb")
    assert open(pk, "rb").read() == _read("codes.pqcm")
    pc2 = str(tmp_path / "cb2.pqcb")
    pqii.save_codebook(pqii.load_codebook(pc), pc2)
    assert open(pc2, "rb").read() == open(pc, "rb").read()
    # wide codes
    w = pqii.CodeMatrix(600, 2, 300, g["wide/codes"])
    pw = str(tmp_path / "w.pqcm")
    pqii.save_codes(w, pw)
    assert pqii.load_codes(pw) == w
    rc, msg, val = R.load_codes(pw)
    assert rc == 0 and np.array_equal(val[0], w.bytes)


@pytest.mark.gpu
def test_codebook_and_code_errors_match_reference(tmp_path):
    pqii, _ = _gpu()
    R = _ref()
    cases = []
    cbb, cmb = _read("codebook.pqcb"), _read("codes.pqcm")
    for n in list(range(0, 24)) + [len(cbb) - 1]:
        cases.append(("cb", f"cbtrunc{n}", cbb[:n]))
    for n in list(range(0, 28)) + [len(cmb) - 1]:
        cases.append(("cm", f"cmtrunc{n}", cmb[:n]))
    b = bytearray(cbb); b[1] = ord("x"); cases.append(("cb", "cb_magic", bytes(b)))  # test_pq.cpp:317-327
    b = bytearray(cbb); struct.pack_into("<I", b, 4, 9); cases.append(("cb", "cb_version", bytes(b)))
    b = bytearray(cbb); struct.pack_into("<f", b, 20 + 4 * 37, float("nan")); cases.append(("cb", "cb_nan", bytes(b)))
    b = bytearray(cbb); struct.pack_into("<f", b, 20 + 4 * 5, float("inf")); cases.append(("cb", "cb_inf", bytes(b)))
    b = bytearray(cbb); struct.pack_into("<I", b, 8, 0); cases.append(("cb", "cb_M0", bytes(b)))
    b = bytearray(cbb); struct.pack_into("<I", b, 16, 0); cases.append(("cb", "cb_ds0", bytes(b)))
    b = bytearray(cmb); b[0] = ord("Q"); cases.append(("cm", "cm_magic", bytes(b)))
    b = bytearray(cmb); struct.pack_into("<I", b, 4, 5); cases.append(("cm", "cm_version", bytes(b)))
    b = bytearray(cmb); b[24 + 4 * 7 + 2] = 20; cases.append(("cm", "cm_range_row7", bytes(b)))
    b = bytearray(cmb); b[24 + 4 * 149] = 16; b[24 + 4 * 3] = 99; cases.append(("cm", "cm_range_row3", bytes(b)))
    b = bytearray(cmb); struct.pack_into("<I", b, 20, 70000); cases.append(("cm", "cm_ks_huge", bytes(b)))
    cases.append(("cm", "cm_trailing_ok", cmb + b"\x01\x02"))  # load_codes has no trailing check
    for kind, label, data in cases:
        p = str(tmp_path / label)
        with open(p, "wb") as f:
            f.write(data)
        if kind == "cb":
            rs, rm, rv = R.load_codebook(p)
            os_, om = _outcome_ours(lambda: pqii.load_codebook(p))
            if rs == 0:
                assert np.array_equal(pqii.load_codebook(p).tables, rv), label
        else:
            rs, rm, rv = R.load_codes(p)
            os_, om = _outcome_ours(lambda: pqii.load_codes(p))
            if rs == 0:
                assert np.array_equal(pqii.load_codes(p).bytes, rv[0]), label
        assert (os_, om) == (rs, rm), (label, (os_, om), (rs, rm))


@pytest.mark.gpu
def test_index_save_load_large_device_roundtrip(tmp_path):
    """A 200k-item device index (M=16) through the file and back: the device
    pack / unpack at a size where every list and entry layout varies."""
    pqii, _ = _gpu()
    from paper_2604_21645_b200.datagen import gaussian_mixture
    x = gaussian_mixture(200_000, 64, 32, 5)
    cb = pqii.pq_fit(x[:20_000], 16, 256, max_iters=3, seed=1)
    codes = pqii.pq_encode(cb, x)
    ids = np.arange(200_000, dtype=np.uint64)[::-1].copy()
    ix = pqii.ivf_build_with_centroids(cb, codes, ids, x[::400][:300].copy())
    p = str(tmp_path / "big.pqii")
    pqii.save_index(ix, p)
    b = pqii.load_index(p)
    for u, v in zip(ix.export()[:4], b.export()[:4]):
        assert np.array_equal(u, v)
    tables, coarse, off, lid, lcodes = parse_pqii(open(p, "rb").read())
    e = ix.export()
    assert np.array_equal(off, e[0]) and np.array_equal(lid, e[1]) and np.array_equal(lcodes, e[2])
