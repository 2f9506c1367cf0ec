"""Per-CTA timing of the config-4 decode kernel (group-specialised layouts), run with PMRC_GEN=trace=1:
start / end of every (CTA, team) from the globaltimer, per group, and the spread of CTA end times.
  PMRC_GEN=trace=1 python tools/dec_trace.py [survivor ids]"""
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from sweep import Job, MSR  # noqa: E402
import paper_1412_3022_b200 as pm  # noqa: E402

ids = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "0,1,4,5,9,12,14,15").split(",")]
gen = os.environ.pop("PMRC_GEN", "")
j = Job(MSR, 8, 16, 1 << 20)  # encode without the trace (its counters would be reported first)
j.encode()
torch.cuda.synchronize()
os.environ["PMRC_GEN"] = gen
pm.pmrc_destroy(j.code)
j.code = pm.pmrc_create(MSR, 8, 14, 16)
out = torch.zeros_like(j.data)
for _ in range(4):
    pm.pmrc_decode(j.code, ids, [j.piece(i) for i in ids], out.data_ptr(), j.S, j.stripes, j.st)
torch.cuda.synchronize()
c = pm.pmrc_debug_counters(j.code)
E = len(c) // 6
base = min(x for x in c[E:2 * E] if x)
per = collections.defaultdict(list)
for i in range(E):
    if c[E + i]:
        per[(c[4 * E + i] >> 32) & 0xFFFF].append(((c[E + i] - base) / 1e3, (c[2 * E + i] - base) / 1e3, i,
                                                   c[4 * E + i] >> 48))
print(json.dumps({"ids": ids, "groups": len(per), "gen": gen}))
for g in sorted(per):
    v = per[g]
    st = sorted(x[0] for x in v)
    en = sorted(x[1] for x in v)
    q = lambda a, f: a[min(len(a) - 1, int(f * len(a)))]
    print("group %d: teams=%d start max %.1f us; end min/p10/p50/p90/max %.1f/%.1f/%.1f/%.1f/%.1f us" % (
        g, len(v), st[-1], en[0], q(en, .1), q(en, .5), q(en, .9), en[-1]))
teams = max(len(v) for v in per.values()) and None
for g in sorted(per):
    slow = sorted(per[g], key=lambda x: -x[1])[:24]
    print("group %d slowest (end us, slot, smid):" % g, " ".join("%.0f/%d/%d" % (x[1], x[2], x[3]) for x in slow))
j.close()
