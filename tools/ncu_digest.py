#!/usr/bin/env python3
"""Digest of one ncu --set full capture (first kernel in the report) into a small JSON for
profiles/: time, DRAM bytes, pipe utilisation, warps, issue, stall reasons per issue, the executed
SASS opcode histogram and the 20 most-stalled instructions.  Runs on the GPU box so the (large)
.ncu-rep need not travel back:  python tools/ncu_digest.py report.ncu-rep out.json [--rm]"""
import csv
import json
import os
import subprocess
import sys
from collections import Counter

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.avg.per_cycle_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "lts__t_sector_hit_rate.pct", "sm__cycles_active.avg",
        "smsp__warps_eligible.avg.per_cycle_active"]


def ncu_csv(rep, *args):
    r = subprocess.run(["ncu", "-i", rep] + list(args) + ["--csv"], capture_output=True, text=True)
    return list(csv.reader(r.stdout.splitlines()))


def main():
    rep, out = sys.argv[1], sys.argv[2]
    rows = ncu_csv(rep, "--page", "raw")
    h, units, v = rows[0], rows[1], rows[2]
    d = dict(zip(h, v))
    u = dict(zip(h, units))
    res = {"report": os.path.basename(rep), "kernel": d.get("Kernel Name", "")[:120],
           "metrics": {k: d.get(k) for k in KEYS}, "units": {k: u.get(k) for k in KEYS}, "stalls_per_issue": {}}
    for k in d:
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                x = float(d[k])
            except ValueError:
                continue
            if x > 0.01:
                res["stalls_per_issue"][k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = x
    src = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    if len(src) > 2:
        hh = src[1]
        ia, isrc = hh.index("Instructions Executed"), hh.index("Source")
        iss = hh.index("Warp Stall Sampling (All Samples)")
        ops, stall_ops = Counter(), Counter()
        lines = []
        for r in src[2:]:
            if len(r) <= max(ia, isrc, iss) or not r[ia].isdigit():
                continue
            t = r[isrc].split()
            if not t:
                continue
            op = (t[1] if t[0].startswith("@") and len(t) > 1 else t[0]).split(".")[0]
            ops[op] += int(r[ia])
            st = int(r[iss]) if r[iss].isdigit() else 0
            stall_ops[op] += st
            lines.append((st, int(r[ia]), r[isrc].strip()[:100]))
        tot = sum(ops.values()) or 1
        res["sass_static_instructions"] = len(lines)
        res["sass_opcode_executed"] = {k: [n, round(100.0 * n / tot, 2), stall_ops[k]] for k, n in ops.most_common(30)}
        res["top_stalled_instructions"] = [list(x) for x in sorted(lines, reverse=True)[:20]]
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    if "--rm" in sys.argv:
        os.remove(rep)


if __name__ == "__main__":
    main()
