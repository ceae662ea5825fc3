"""Drop-in proof: the reference's own acceptance harness
(proj/tests/acceptance_main.cpp) and its callers (pipeline, bench,
dataset_io), compiled from the reference's sources and headers, linked
against libpqg_pqii.so (the namespace-pqii facade over the C ABI) instead of
the reference's kmeans/pq/ivf.  Built by `make -C oracle` where the reference
is present; the binaries travel in oracle/_ref."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PQG_BIN = os.path.join(ROOT, "oracle", "_ref", "pqii_acceptance_pqg")
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "pqii_acceptance_ref")


def run(binary, criteria, timeout=900):
    args = [binary]
    for c in criteria:
        args += ["--only", str(c)]
    p = subprocess.run(args, capture_output=True, text=True, timeout=timeout)
    lines = [l for l in p.stdout.splitlines() if l.startswith("criterion ")]
    out = {}
    for l in lines:
        m = re.match(r"criterion (\d+) (PASS|FAIL) \[[^\]]*\] ([^:]*): (.*)", l)
        if m:
            # wall-clock fields differ by construction; every other value must match
            detail = re.sub(r"elapsed [0-9.eE+-]+s", "elapsed <t>", m.group(4))
            out[int(m.group(1))] = (m.group(2), detail)
    return out, p


@pytest.mark.gpu
def test_reference_acceptance_on_pqg():
    if not os.path.exists(PQG_BIN):
        pytest.skip("drop-in acceptance binary not built (needs the reference sources)")
    crit = [1, 2, 3, 5, 6, 7, 9, 10]
    res, p = run(PQG_BIN, crit)
    assert set(res) == set(crit), p.stdout + p.stderr
    failed = {c: v for c, v in res.items() if v[0] != "PASS"}
    assert not failed, failed


@pytest.mark.gpu
def test_acceptance_details_match_reference():
    """Deterministic criteria print result values; the drop-in must print the
    same values as the reference's own hot path on the same seeds."""
    if not (os.path.exists(PQG_BIN) and os.path.exists(REF_BIN)):
        pytest.skip("acceptance binaries not built")
    crit = [1, 3, 5, 6, 9]
    ours, _ = run(PQG_BIN, crit)
    ref, _ = run(REF_BIN, crit)
    for c in crit:
        assert ours[c][0] == ref[c][0] == "PASS", (c, ours.get(c), ref.get(c))
        assert ours[c][1] == ref[c][1], (c, ours[c][1], ref[c][1])
