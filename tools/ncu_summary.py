#!/usr/bin/env python3
"""Summaries of ncu captures for profiles/:

  python tools/ncu_summary.py full  <report.ncu-rep> <out.json> [algorithmic_bytes_per_launch]
  python tools/ncu_summary.py launches <launches.csv> <out.json>

`full` reads `ncu -i --page raw --csv` of a `--set full` capture (one kernel launch) and keeps the
numbers DESIGN.md / bench.py cite: time, DRAM bytes, IPC, pipe utilisation, warps, stalls per issue.
`launches` sums the `gpu__time_duration.sum` launch list per kernel (share of the GPU time)."""
import csv
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__inst_executed.avg.per_cycle_active", "sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.sum.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.sum.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "sm__warps_active.avg.per_cycle_active", "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
]
UNIT = {"G": 1e9, "M": 1e6, "K": 1e3, "": 1.0}


def full(rep, out, alg=None):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, units, v = rows[0], rows[1], rows[2]
    d = dict(zip(h, v))
    u = dict(zip(h, units))
    s = {k: d.get(k) for k in KEYS}
    s["units"] = {k: u.get(k) for k in KEYS}
    st = {}
    for k in d:
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            name = k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]
            try:
                if float(d[k]) > 0.01:
                    st[name] = round(float(d[k]), 3)
            except ValueError:
                pass
    s["stalls_per_issue"] = st

    def nbytes(key):
        unit = (u.get(key) or "byte").strip()
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
        return float(d[key].replace(",", "")) * scale

    dram = nbytes("dram__bytes_read.sum") + nbytes("dram__bytes_write.sum")
    s["dram_bytes_per_launch"] = dram
    if alg:
        s["algorithmic_bytes_per_launch"] = int(alg)
        s["traffic_over_algorithmic"] = dram / float(alg)
    s["source"] = rep
    json.dump(s, open(out, "w"), indent=1)
    print(json.dumps(s, indent=1))


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    tot, cnt = {}, {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0]
        tot[k] = tot.get(k, 0.0) + float(d["Metric Value"].replace(",", ""))
        cnt[k] = cnt.get(k, 0) + 1
    T = sum(tot.values())
    s = {k: {"launches": cnt[k], "total_ns": tot[k], "avg_ns": tot[k] / cnt[k], "share": tot[k] / T} for k in tot}
    s["source"] = path
    json.dump(s, open(out, "w"), indent=1)
    print(json.dumps(s, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
    else:
        launches(sys.argv[2], sys.argv[3])
