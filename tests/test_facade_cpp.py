"""The reference's unit-test cases restated in C++ against the drop-in
libpqg_pqii.so (tests/cpp/facade_test.cpp), compiled with g++ and run on a GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2604_21645_b200")


def build_binary(out):
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "facade_test.cpp"), "-L", PKG,
                    "-lpqg_pqii", "-lpqg", f"-Wl,-rpath,{PKG}", "-o", out], check=True)


def test_facade_compiles(tmp_path):
    if not os.path.exists(os.path.join(PKG, "libpqg_pqii.so")):
        pytest.skip("libpqg_pqii.so not built")
    build_binary(str(tmp_path / "facade_test"))


@pytest.mark.gpu
def test_facade_reference_cases(tmp_path):
    out = str(tmp_path / "facade_test")
    build_binary(out)
    p = subprocess.run([out], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr
