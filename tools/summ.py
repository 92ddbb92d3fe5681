"""Print the key fields of bench JSON lines (tools/gpu logs)."""
import json
import sys

for path in sys.argv[1:]:
    for line in open(path):
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        print(path, d.get("config", {}).get("workload", "")[:40])
        print("  value %.4g  ms/step %.4f  e2e %.4g" % (d["value"], d["ms_per_step"] * 1e3 / 1e3,
                                                      (d.get("e2e") or {}).get("value", 0)))
        if "phases_ms" in d:
            print("  phases(us):", {k: round(v * 1e3, 1) for k, v in d["phases_ms"].items()})
        if "clocks" in d:
            print("  clocks:", d["clocks"])
