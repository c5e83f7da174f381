"""Summarise `ncu --set full` reports into profiles/<tag>_ncu_summary.json.

    python tools/ncu_summary.py <tag> <report.ncu-rep>:<params>:<algorithmic bytes/param> ...

Reads the raw page of each report (one kernel per report) and records
duration, DRAM bytes (-> DRAM bytes per param, the roofline `traffic`),
throughputs, occupancy and the top warp-stall reasons.
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "sm__cycles_elapsed.avg.per_second",
        "dram__cycles_elapsed.avg.per_second"]
UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
TUNIT = {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return {h: (u, v) for h, u, v in zip(rows[0], rows[1], rows[2])}


def summarise(rep, n, bpp):
    r = raw(rep)
    d = {k: f"{r[k][1]} {r[k][0]}".strip() for k in KEYS if k in r}
    stalls = []
    for k, (u, v) in r.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
            try:
                stalls.append((float(v), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(x for x, _ in stalls) or 1.0
    d["top_stalls_pct"] = {k: round(100 * x / tot, 1) for x, k in sorted(stalls, reverse=True)[:6]}
    rb = float(r["dram__bytes_read.sum"][1]) * UNIT[r["dram__bytes_read.sum"][0]]
    wb = float(r["dram__bytes_write.sum"][1]) * UNIT[r["dram__bytes_write.sum"][0]]
    t = float(r["gpu__time_duration.sum"][1]) * TUNIT[r["gpu__time_duration.sum"][0]]
    d.update(params=n, algorithmic_bytes=n * bpp, dram_bytes=rb + wb,
             dram_bytes_per_param=round((rb + wb) / n, 4),
             algorithmic_gbs_cold_serialised=round(n * bpp / t / 1e9, 1))
    return d


def main():
    tag = sys.argv[1]
    out = {}
    for spec in sys.argv[2:]:
        rep, n, bpp = spec.split(":")
        out[os.path.basename(rep)] = summarise(rep, int(n), float(bpp))
    path = os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(path)


if __name__ == "__main__":
    main()
