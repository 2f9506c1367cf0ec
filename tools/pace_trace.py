"""Per-group timing of the group-specialised encode kernel (run with PMRC_GEN=trace=1[,pace_lag=N]):
CTA start/end (globaltimer), time spent pacing and pacing timeouts, per group, from the last launch."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import inputs
import paper_1412_3022_b200 as pm

k, d, n, S = 8, 14, 16, 1 << 20
code = pm.pmrc_create(0, k, d, n)
info = pm.pmrc_info(code)
B, P = info["B"], info["parity_rows"]
stripes = -(-(1 << 30) // (B * S))
data = torch.empty((stripes, B, S), dtype=torch.uint8, device="cuda")
par = torch.empty((stripes, P, S), dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
inputs.fill_device(data.data_ptr(), data.numel(), 1, stream=st)
for _ in range(4):
    pm.pmrc_encode(code, data.data_ptr(), par.data_ptr(), S, stripes, st)
torch.cuda.synchronize()
c = pm.pmrc_debug_counters(code)
E = len(c) // 6
G = 7
t0 = [x for x in c[E:2 * E] if x]
base = min(t0)
teams = None
rows = []
for i in range(E):
    if not c[E + i]:
        continue
    rows.append((i, (c[E + i] - base) / 1e3, (c[2 * E + i] - base) / 1e3, c[3 * E + i] / 1e3, c[4 * E + i]))
# infer teams per CTA from the used entries: grid = G * spg
used = len(rows)
print(json.dumps({"entries": E, "used": used}))
import collections
per = collections.defaultdict(list)
grid_teams = max(r[0] for r in rows) + 1
print("grid x teams", grid_teams)
for T in range(1, 17):
    if grid_teams % T == 0 and (grid_teams // T) % G == 0:
        teams = T
for i, s0, e0, w, f in rows:
    blk = i // teams
    spg = (grid_teams // teams) // G
    g = blk // spg
    per[g].append((s0, e0, w, f))
for g in sorted(per):
    v = per[g]
    ends = [x[1] for x in v]
    waits = [x[2] for x in v]
    print("group %d: n=%d start max %.1f us, end min/mean/max %.1f/%.1f/%.1f us, wait mean %.1f us, timeouts %d" % (
        g, len(v), max(x[0] for x in v), min(ends), sum(ends) / len(ends), max(ends), sum(waits) / len(waits),
        sum(x[3] for x in v)))

pre = c[5 * E: 5 * E + 2048]
post = c[5 * E + 2048: 5 * E + 4096]
for g in range(G):
    its = [(pre[g * 256 + i], post[g * 256 + i]) for i in range(256) if pre[g * 256 + i]]
    print("g%d iters=%d" % (g, len(its)), " ".join("%.1f+%.1f" % ((a - base) / 1e3, (b - a) / 1e3 if b else -1) for a, b in its[:40]))
