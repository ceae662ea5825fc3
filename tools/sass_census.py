"""SASS instruction census of the built library objects: per kernel, the
counts of the instructions that prove the Blackwell paths (tensor-core MMA
UTC*MMA, TMEM loads LDTM, TMA / bulk copies UTMALDG / UBLKCP, packed FP32
FFMA2 / FADD2, fp64 DFMA/DADD/DMUL, shared-memory LDS) -- static counts from
cuobjdump -sass (run here; no GPU needed).

  python tools/sass_census.py [out.md]
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "paper_2604_21645_b200", "csrc", "build")
KEYS = ["UTCHMMA", "UTCQMMA", "UTCIMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UBLKCP", "SYNCS", "FFMA2", "FADD2",
        "FFMA", "DFMA", "DADD", "DMUL", "LDS", "LDG", "VIMNMX", "VIMNMX3"]


def demangle(name):
    try:
        return subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    except Exception:
        return name


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r2_sass_census.md")
    rows = []
    for f in sorted(os.listdir(OBJ)):
        if not f.endswith(".o"):
            continue
        sass = subprocess.run(["cuobjdump", "-sass", os.path.join(OBJ, f)], capture_output=True, text=True).stdout
        cur, cnt = None, None
        for line in sass.splitlines():
            m = re.search(r"Function : (\S+)", line)
            if m:
                if cur:
                    rows.append((f, cur, cnt))
                cur, cnt = m.group(1), collections.Counter()
                continue
            m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
            if m and cur:
                op = m.group(1)
                cnt[op] += 1
        if cur:
            rows.append((f, cur, cnt))
    keep = [r for r in rows if any(r[2][k] for k in ("UTCHMMA", "UTCQMMA", "LDTM", "UTMALDG", "UBLKCP", "FFMA2"))]
    with open(out, "w") as fo:
        fo.write("# SASS census (static instruction counts, cuobjdump -sass of the sm_100a objects)\n\n")
        fo.write("Kernels that use tcgen05 (UTCHMMA = tcgen05.mma kind::tf32, LDTM = tcgen05.ld), TMA / bulk "
                 "copies (UTMALDG = cp.async.bulk.tensor, UBLKCP = cp.async.bulk) or packed FP32 (FFMA2/FADD2).\n\n")
        fo.write("| object | kernel | " + " | ".join(KEYS) + " |\n|" + "---|" * (len(KEYS) + 2) + "\n")
        for f, k, c in keep:
            name = demangle(k)
            name = re.sub(r"pqg::\(anonymous namespace\)::", "", name)
            name = name.split("(")[0][:80]
            fo.write(f"| {f} | `{name}` | " + " | ".join(str(c[x]) for x in KEYS) + " |\n")
    print(f"wrote {out}: {len(keep)} kernels")


if __name__ == "__main__":
    main()
