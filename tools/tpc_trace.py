"""Which SMs finish late, and do the two SMs of a TPC run the same group?  Encode (or decode with
--decode) kernel with PMRC_GEN=trace=1: per-(CTA, team) end time, %smid and group, aggregated per
TPC (smid // 2).
  PMRC_GEN=trace=1 python tools/tpc_trace.py [--decode]"""
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from sweep import Job, MSR  # noqa: E402
import paper_1412_3022_b200 as pm  # noqa: E402

gen = os.environ.get("PMRC_GEN", "")
j = Job(MSR, 8, 16, 1 << 20)
if "--decode" in sys.argv:
    ids = [0, 1, 4, 5, 9, 12, 14, 15]
    out = torch.zeros_like(j.data)
    f = lambda: pm.pmrc_decode(j.code, ids, [j.piece(i) for i in ids], out.data_ptr(), j.S, j.stripes, j.st)
else:
    f = j.encode
for _ in range(4):
    f()
torch.cuda.synchronize()
c = pm.pmrc_debug_counters(j.code)
E = len(c) // 6
base = min(x for x in c[E:2 * E] if x)
sm = collections.defaultdict(list)
for i in range(E):
    if c[E + i]:
        sm[c[4 * E + i] >> 48].append(((c[2 * E + i] - base) / 1e3, (c[4 * E + i] >> 32) & 0xFFFF))
tpc = collections.defaultdict(dict)
for s, v in sm.items():
    tpc[s // 2][s] = (max(x[0] for x in v), sorted(set(x[1] for x in v)))
rows = []
for t in sorted(tpc):
    d = tpc[t]
    groups = [tuple(d[s][1]) for s in sorted(d)]
    rows.append((max(d[s][0] for s in d), t, len(set(groups)) > 1, groups))
rows.sort(reverse=True)
mixed = [r for r in rows if r[2]]
print(json.dumps({"gen": gen, "tpcs": len(rows), "mixed_tpcs": len(mixed),
                  "end_us_mixed_mean": sum(r[0] for r in mixed) / max(1, len(mixed)),
                  "end_us_same_mean": sum(r[0] for r in rows if not r[2]) / max(1, len(rows) - len(mixed))}))
for r in rows[:16]:
    print("tpc %3d end %.1f us mixed=%s groups=%s" % (r[1], r[0], r[2], r[3]))
j.close()
