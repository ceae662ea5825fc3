"""Summarise ncu captures into profiles/ (run here, on the CPU box).

  python tools/ncu_summarize.py <tag> gpurun_out/prof_x.ncu-rep [...] [--launches gpurun_out/launches.csv]

Writes profiles/<tag>_ncu.md (key metrics per captured kernel, launch-list
shares) and merges dram bytes per launch into profiles/ncu_summary.json.
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    ("GPU Speed Of Light Throughput", "Duration"),
    ("GPU Speed Of Light Throughput", "SM Frequency"),
    ("GPU Speed Of Light Throughput", "Compute (SM) Throughput"),
    ("GPU Speed Of Light Throughput", "Memory Throughput"),
    ("GPU Speed Of Light Throughput", "DRAM Throughput"),
    ("GPU Speed Of Light Throughput", "L1/TEX Cache Throughput"),
    ("GPU Speed Of Light Throughput", "L2 Cache Throughput"),
    ("Compute Workload Analysis", "Issue Slots Busy"),
    ("Compute Workload Analysis", "Executed Ipc Active"),
    ("Occupancy", "Achieved Occupancy"),
    ("Occupancy", "Theoretical Occupancy"),
    ("Launch Statistics", "Registers Per Thread"),
    ("Launch Statistics", "Grid Size"),
    ("Launch Statistics", "Block Size"),
    ("Warp State Statistics", "Warp Cycles Per Issued Instruction"),
    ("Instruction Statistics", "Executed Instructions"),
    ("Memory Workload Analysis", "L2 Hit Rate"),
]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fma.sum",
       "sm__inst_executed_pipe_alu.sum", "sm__inst_executed_pipe_lsu.sum",
       "smsp__inst_executed.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio"]


def ncu_csv(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True,
                         text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def summarize(rep):
    rows = ncu_csv(rep, "details")
    h = rows[0]
    per = collections.OrderedDict()
    for r in rows[1:]:
        kid = r[h.index("ID")]
        d = per.setdefault(kid, {"kernel": r[h.index("Kernel Name")]})
        key = (r[h.index("Section Name")], r[h.index("Metric Name")])
        if key in KEYS:
            d[key[1]] = f"{r[h.index('Metric Value')]} {r[h.index('Metric Unit')]}".strip()
    raw = ncu_csv(rep, "raw")
    hdr, units = raw[0], raw[1]
    for r in raw[2:]:
        d = per.setdefault(r[hdr.index("ID")], {})
        for m in RAW:
            if m in hdr:
                d[m] = f"{r[hdr.index(m)]} {units[hdr.index(m)]}".strip()
    return per


def to_bytes(s):
    v, _, u = s.partition(" ")
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def main():
    tag = sys.argv[1]
    reps = [a for a in sys.argv[2:] if a.endswith(".ncu-rep")]
    launches = sys.argv[sys.argv.index("--launches") + 1] if "--launches" in sys.argv else None
    md = [f"# ncu summary -- {tag}", ""]
    js_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    js = json.load(open(js_path)) if os.path.exists(js_path) else {}
    for rep in reps:
        per = summarize(rep)
        md.append(f"## {os.path.basename(rep)}")
        for kid, d in per.items():
            md.append(f"### launch {kid}: `{d.get('kernel', '?')[:140]}`")
            md += [f"- {k}: {v}" for k, v in d.items() if k != "kernel"]
            md.append("")
        vals = [d for d in per.values() if "dram__bytes_read.sum" in d]
        if vals:
            rb = [to_bytes(d["dram__bytes_read.sum"]) + to_bytes(d["dram__bytes_write.sum"]) for d in vals]
            js[os.path.basename(rep).replace(".ncu-rep", "")] = {
                "kernel": vals[0].get("kernel", "")[:200],
                "dram_bytes_per_launch": sum(rb) / len(rb), "tag": tag}
    if launches:
        rows = list(csv.reader(open(launches)))
        hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
        h = rows[hi]
        agg = collections.OrderedDict()
        for r in rows[hi + 1:]:
            if len(r) <= h.index("Metric Value"):
                continue
            a = agg.setdefault(r[h.index("Kernel Name")].split("(")[0], [0, 0.0])
            a[0] += 1
            a[1] += float(r[h.index("Metric Value")].replace(",", ""))
        tot = sum(v[1] for v in agg.values())
        md += ["## launch list (gpu__time_duration.sum in ns; cold-cache, serialised: compare shares)",
               "| kernel | launches | total ms | avg us | share |", "|---|---|---|---|---|"]
        for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
            md.append(f"| `{k[:70]}` | {v[0]} | {v[1] / 1e6:.3f} | {v[1] / v[0] / 1e3:.2f} | "
                      f"{v[1] / tot * 100:.1f}% |")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    with open(js_path, "w") as f:
        json.dump(js, f, indent=1)
    print("wrote", f"profiles/{tag}_ncu.md")


if __name__ == "__main__":
    main()
