"""Brief per-kernel view of an ncu --set full report: time, occupancy, issue,
L1/L2/DRAM load, instruction count and the top stall reasons (pc samples).
usage: python tools/ncu_brief.py REPORT.ncu-rep"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[0], rows[2:]
want = ["gpu__time_duration.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"]
stall = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")]
for d in data:
    print("==", d[hdr.index("Kernel Name")][:90])
    for w in want:
        if w in hdr:
            print(f"   {w:62s} {d[hdr.index(w)]}")
    st = sorted([(float(d[hdr.index(h)] or 0), h) for h in stall], reverse=True)[:5]
    tot = sum(float(d[hdr.index(h)] or 0) for h in stall) or 1.0
    print("   stalls: " + ", ".join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_', '')} {v / tot:.0%}" for v, h in st))
