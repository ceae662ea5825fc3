"""CPU checks of the drop-in boundary: libpqg.so loads without a GPU and exports
every entry point include/pqg.h declares; the Python binding covers them all;
the product path refuses to run without a GPU instead of falling back."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pqg.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(pqg_\w+)\s*\(", src, re.M)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ["pqg_kmeans_fit", "pqg_pq_fit", "pqg_pq_encode", "pqg_pq_decode",
                 "pqg_pq_recon_sse", "pqg_adc_tables", "pqg_ivf_build_with_centroids",
                 "pqg_index_search", "pqg_flat_scan", "pqg_topk_merge", "pqg_last_error"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2604_21645_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libpqg.so not built")
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\b(pqg_\w+)\b", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing
    lib = _lib.load()
    assert lib.pqg_version().startswith(b"pqg")
    assert set(declared()) == set(_lib.EXPORTED)


def test_no_cpu_fallback():
    """Without a GPU the product path raises; it never computes on the host."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2604_21645_b200 import _lib, pqii
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libpqg.so not built")
    with pytest.raises(_lib.PQGError):
        pqii.Context(0)


def test_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2604_21645_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "liboracle" not in src and "libpqii_ref" not in src, f
