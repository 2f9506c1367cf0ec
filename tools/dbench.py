"""Kernel-only timing of one decode or repair plan of config 4 (MSR k=8 n=16, 1 GiB, 1 MiB
sub-blocks) through the C ABI, for generator experiments and ncu:
  python tools/dbench.py decode 0,1,4,5,9,12,14,15
  python tools/dbench.py repair 15 0,1,2,3,4,5,6,7,8,9,11,12,13,14"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from sweep import Job, timed, MSR  # noqa: E402
import paper_1412_3022_b200 as pm  # noqa: E402


def main():
    op = sys.argv[1]
    kind = int(os.environ.get("KIND", MSR))
    j = Job(kind, 8, 16, int(os.environ.get("S", 1 << 20)))
    # the generated (JIT) kernels unless PMRC_POLICY=runtime
    pm.pmrc_set_plan_policy(j.code, pm.PMRC_PLAN_RUNTIME if os.environ.get("PMRC_POLICY") == "runtime"
                            else pm.PMRC_PLAN_JIT)
    j.encode()
    torch.cuda.synchronize()
    if op == "decode":
        ids = [int(x) for x in sys.argv[2].split(",")]
        out = torch.zeros_like(j.data)
        f = lambda: pm.pmrc_decode(j.code, ids, [j.piece(i) for i in ids], out.data_ptr(), j.S, j.stripes, j.st)
        f()
        ms = timed(f, 10)
        print(json.dumps({"op": op, "ids": ids, "ms": ms, "GBps": j.stripes * j.B * j.S / ms / 1e6,
                          "gen": os.environ.get("PMRC_GEN", "")}))
    else:
        lost = int(sys.argv[2])
        H = [int(x) for x in sys.argv[3].split(",")]
        out = torch.empty((j.stripes, j.alpha, j.S), dtype=torch.uint8, device="cuda")
        f = lambda: pm.pmrc_repair(j.code, lost, H, [j.piece(i) for i in H], (out.data_ptr(), j.alpha * j.S), j.S,
                                   j.stripes, j.st)
        f()
        ms = timed(f, 10)
        print(json.dumps({"op": op, "lost": lost, "ms": ms, "GBps_repaired": j.stripes * j.alpha * j.S / ms / 1e6,
                          "gen": os.environ.get("PMRC_GEN", "")}))
    j.close()


if __name__ == "__main__":
    main()
