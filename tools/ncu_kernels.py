"""Fold an ncu --metrics CSV launch list (one bench.py run) into per-kernel means.

usage: python tools/ncu_kernels.py LAUNCHES.csv CONFIG [profiles/ncu_kernels.json]
Kernel names are mapped to the phase names bench.py's event profile uses, so the
bench line can quote the ncu dram traffic of its dominant kernel ("traffic")."""
import collections
import csv
import json
import re
import sys

PHASE = {"f3_hist": "hist", "f3_scan": "scan", "f3_scatter": "scatter", "f3_fwd": "f3_fwd",
         "f3_bwd1": "f3_bwd1", "f3_bwd2": "f3_bwd2", "f3_combine": "f3_combine"}
SCALE = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3, "ms": 1e3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main():
    path, config = sys.argv[1], sys.argv[2]
    out = sys.argv[3] if len(sys.argv) > 3 else None
    rows = list(csv.reader(open(path)))
    hdr, per = None, collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        m = re.search(r"(f3_\w+|k_\w+|\w+_kernel)", d["Kernel Name"])
        name = m.group(1) if m else d["Kernel Name"][:40]
        name = PHASE.get(name, name)
        v = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1.0)
        per[(name, d["ID"])][d["Metric Name"]] = v
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    for (name, _), ms in per.items():
        for k, v in ms.items():
            agg[name][k].append(v)
    res = {}
    for name, ms in agg.items():
        e = {"launches": len(next(iter(ms.values())))}
        mean = {k: sum(v) / len(v) for k, v in ms.items()}
        if "gpu__time_duration.sum" in mean:
            e["us"] = mean["gpu__time_duration.sum"]
        if "dram__bytes_read.sum" in mean:
            e["dram_bytes"] = mean["dram__bytes_read.sum"] + mean.get("dram__bytes_write.sum", 0.0)
        if "lts__t_bytes.sum" in mean:
            e["l2_bytes"] = mean["lts__t_bytes.sum"]
        if "sm__sass_thread_inst_executed_op_ffma_pred_on.sum" in mean:
            e["ffma_thread_inst"] = mean["sm__sass_thread_inst_executed_op_ffma_pred_on.sum"]
            # FFMA2 (fma.rn.f32x2) is counted separately: 2 lanes x 2 flops
            e["ffma2_thread_inst"] = mean.get("sm__sass_thread_inst_executed_op_ffma2_pred_on.sum", 0.0)
            if "us" in e:
                fl = 2 * e["ffma_thread_inst"] + 4 * e["ffma2_thread_inst"]
                e["executed_ffma_tflops"] = fl / (e["us"] * 1e-6) / 1e12
        res[name] = e
    for n, e in sorted(res.items(), key=lambda x: -x[1].get("us", 0)):
        print(f"{n:16s} " + " ".join(f"{k}={v:.4g}" for k, v in e.items()))
    if out:
        try:
            allc = json.load(open(out))
        except Exception:  # noqa: BLE001
            allc = {}
        allc[config] = res
        json.dump(allc, open(out, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
