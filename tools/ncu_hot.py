"""Summarise an ncu --set full report (.ncu-rep) per launch: time, DRAM bytes, instructions,
pipe utilisation, occupancy, cache hit rates and the top stall reasons per issue.

python tools/ncu_hot.py gpurun_out/prof.ncu-rep "command line used" > profiles/<name>.json
"""
import csv
import io
import json
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
           "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]


def main():
    rep = sys.argv[1]
    cmd = sys.argv[2] if len(sys.argv) > 2 else ""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    ki = h.index("Kernel Name")
    out = {}
    for n, r in enumerate(rows[2:]):
        name = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        d = {m: r[h.index(m)] for m in METRICS if m in h}
        stall = [c for c in h if c.startswith("smsp__average_warps_issue_stalled_") and
                 c.endswith("_per_issue_active.ratio")]
        top = sorted(((float(r[h.index(c)] or 0), c) for c in stall), reverse=True)[:8]
        d["stall_per_issue_top"] = {c.replace("smsp__average_warps_issue_stalled_", "").replace(
            "_per_issue_active.ratio", ""): round(v, 2) for v, c in top}
        out[f"{n}:{name}"] = d
    out["_units"] = {m: units[h.index(m)] for m in METRICS if m in h}
    out["_command"] = cmd
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
