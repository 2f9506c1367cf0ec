"""Per-group timing of a group-specialised encode kernel (layouts 1/2), run with PMRC_GEN=trace=1:
CTA start/end (globaltimer), time spent pacing and pacing timeouts per group, from the last launch.
  PMRC_GEN=trace=1 python tools/pace_trace.py [kind k n S]"""
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import inputs
import paper_1412_3022_b200 as pm

a = [int(x) for x in sys.argv[1:]]
kind, k, n, S = (a + [0, 8, 16, 1 << 20][len(a):])[:4] if a else (0, 8, 16, 1 << 20)
d = k if kind == 3 else 2 * k - 2
code = pm.pmrc_create(kind, k, d, n)
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
base = min(x for x in c[E:2 * E] if x)
per = collections.defaultdict(list)
for i in range(E):
    if not c[E + i]:
        continue
    g = (c[4 * E + i] >> 32) & 0xFFFF
    per[g].append(((c[E + i] - base) / 1e3, (c[2 * E + i] - base) / 1e3, c[3 * E + i] / 1e3, c[4 * E + i] & 0xFFFFFFFF))
print(json.dumps({"kind": kind, "k": k, "S": S, "groups": len(per)}))
for g in sorted(per):
    v = per[g]
    ends = [x[1] for x in v]
    print("group %d: teams=%d end min/mean/max %.1f/%.1f/%.1f us, wait mean %.1f us, timeouts %d" % (
        g, len(v), min(ends), sum(ends) / len(ends), max(ends), sum(x[2] for x in v) / len(v), sum(x[3] for x in v)))
