"""Print the key ncu metrics of every kernel in a report (run here, no GPU).
  python tools/ncu_brief.py gpurun_out/x.ncu-rep [kernel-regex]"""
import csv
import io
import re
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Compute (SM) Throughput", "Issue Slots Busy", "Executed Ipc Active",
        "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread", "Grid Size", "Block Size",
        "L2 Hit Rate", "No Eligible", "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction"]
RAW = ["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__pipe_tensor_op_tmem_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
       "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__inst_executed.sum",
       "dram__bytes_read.sum", "dram__bytes_write.sum"]
STALL = "smsp__average_warps_issue_stalled_"


def main():
    rep = sys.argv[1]
    pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(det)))
    h = rows[0]
    ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    cur = None
    for r in rows[1:]:
        if pat and not pat.search(r[ki]):
            continue
        if r[ii] != cur:
            cur = r[ii]
            print(f"== [{cur}] {r[ki][:110]}")
        if r[mi] in WANT:
            print(f"   {r[mi]}: {r[vi]} {r[ui]}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h = rr[0]
    kn = h.index("Kernel Name")
    for r in rr[2:]:
        if pat and not pat.search(r[kn]):
            continue
        print(f"-- raw {r[kn][:90]}")
        for i, name in enumerate(h):
            if name in RAW or ("pipe_t" in name and "pct_of_peak_sustained_active" in name and ".avg." in name):
                print(f"   {name}: {r[i]}")
        st = [(float(r[i].replace(',', '') or 0), name[len(STALL):]) for i, name in enumerate(h)
              if name.startswith(STALL) and name.endswith("per_issue_active.ratio")]
        st.sort(reverse=True)
        print("   stalls/issue:", ", ".join(f"{n.replace('_per_issue_active.ratio','')}={v:.2f}" for v, n in st[:8]))


if __name__ == "__main__":
    main()
