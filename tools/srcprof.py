"""Top CUDA source lines of one kernel in an ncu report (needs -lineinfo)."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kern}", "--launch-skip", sys.argv[4] if len(sys.argv) > 4 else "0", "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
si = hdr.index("Warp Stall Sampling (All Samples)")
ii = hdr.index("Instructions Executed")
data = [r for r in rows if len(r) == len(hdr) and r[0].isdigit()]
f = lambda v: float(v) if v not in ("", "-") else 0.0
tot = sum(f(r[si]) for r in data) or 1
for r in sorted(data, key=lambda r: -f(r[si]))[:top]:
    print(f"{f(r[si]) / tot * 100:5.1f}% L{r[0]:>4} inst={f(r[ii]):9.0f}  {r[1].strip()[:95]}")
