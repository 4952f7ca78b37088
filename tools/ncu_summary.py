"""Summarise an ncu report (one launch per kernel) into the per-kernel metrics quoted in
DESIGN.md / profiles/.  Usage: python tools/ncu_summary.py rep.ncu-rep out.json"""
import csv
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "sm__cycles_active.sum", "sm__warps_active.avg.per_cycle_active", "smsp__cycles_elapsed.avg",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed",
]


def _num(v):
    return float(v.split()[0].replace(",", ""))


def main(rep, out, note=None):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = f"{r[i]} {units[i]}".strip()
        try:   # fp64 FLOPs of the launch: (2 dfma + dadd + dmul) thread instructions
            cyc = _num(d["smsp__cycles_elapsed.avg"])
            d["fp64_flop"] = cyc * (2 * _num(d["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed"])
                                    + _num(d["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed"])
                                    + _num(d["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed"]))
        except (KeyError, ValueError):
            pass
        res.append(d)
    with open(out, "w") as f:
        json.dump({"meta": {"note": note or "", "units_per_round": None}, "rows": res} if note else res, f, indent=1)
    for d in res:
        print(d["kernel"], d.get("gpu__time_duration.sum"), "issue", d.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
              "dram", d.get("dram__bytes_read.sum"), d.get("dram__bytes_write.sum"), "fp64 GFLOP",
              round(d.get("fp64_flop", 0) / 1e9, 3))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
