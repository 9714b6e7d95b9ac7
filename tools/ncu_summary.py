"""Summarise ncu --set full captures (.ncu-rep) into a JSON for profiles/.

usage: python tools/ncu_summary.py OUT.json REP [REP ...]
"""
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "smsp__warps_active.avg.per_cycle_active", "smsp__warps_eligible.avg.per_cycle_active"] + [
        f"smsp__average_warps_issue_stalled_{r}_per_issue_active.ratio"
        for r in ("wait", "not_selected", "math_pipe_throttle", "long_scoreboard",
                  "short_scoreboard", "barrier", "mio_throttle", "lg_throttle")]


def summarise(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    if len(rows) < 3:
        return []
    h, u = rows[0], rows[1]
    out = []
    for row in rows[2:]:
        d = {"kernel": row[h.index("Kernel Name")][:90]}
        for k in KEYS:
            if k in h:
                d[k] = f"{row[h.index(k)]} {u[h.index(k)]}".strip()
        out.append(d)
    return out


if __name__ == "__main__":
    if len(sys.argv) < 3 or sys.argv[1].startswith("-"):
        sys.exit(__doc__)
    res = {r.split("/")[-1]: summarise(r) for r in sys.argv[2:]}
    json.dump(res, open(sys.argv[1], "w"), indent=1)
    print(json.dumps(res, indent=1))
