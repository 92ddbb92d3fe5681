"""Summarise an `ncu --set full` report (one row per captured kernel) into the
figures the DESIGN/bench rooflines quote.

usage: python tools/ncu_full_summary.py REPORT.ncu-rep > profiles/ncu_full_<tag>.txt"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem %"),
    ("dram__bytes_read.sum", "dram rd"),
    ("dram__bytes_write.sum", "dram wr"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__shared_mem_per_block_static", "smem static"),
    ("launch__shared_mem_per_block_dynamic", "smem dyn"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA cyc %"),
    ("sm__sass_thread_inst_executed_op_ffma_pred_on.sum", "FFMA thr-inst"),
    ("sm__sass_thread_inst_executed_op_fmul_pred_on.sum", "FMUL thr-inst"),
    ("sm__sass_thread_inst_executed_op_fadd_pred_on.sum", "FADD thr-inst"),
    ("smsp__average_warp_latency_issue_stalled_long_scoreboard", "stall long_sb"),
    ("smsp__average_warp_latency_issue_stalled_barrier", "stall barrier"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def main():
    raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    for r in data:
        name = r[col["Kernel Name"]].split("(")[0]
        print(f"== {name}  (ID {r[col['ID']]}, grid {r[col['Grid Size']]}, block {r[col['Block Size']]})")
        for key, label in KEYS:
            if key in col:
                print(f"   {label:16s} {r[col[key]]:>14s} {units[col[key]]}  [{key}]")


if __name__ == "__main__":
    main()
