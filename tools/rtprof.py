#!/usr/bin/env python3
"""One launch each of the runtime-coefficient kernel on the config-4 decode / repair plans and the
config-2 encode (1 GiB jobs), for ncu (kernel filter: rlc_kernel).  usage: rtprof.py [decode|repair|encode|all]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import inputs
import paper_1412_3022_b200 as pm


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    k, n, d, S = 8, 16, 14, 1 << 20
    code = pm.pmrc_create(0, k, d, n)
    info = pm.pmrc_info(code)
    a, B, P = info["alpha"], info["B"], info["parity_rows"]
    stripes = 19
    data = torch.empty((stripes, B, S), dtype=torch.uint8, device="cuda")
    par = torch.empty((stripes, P, S), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    inputs.fill_device(data.data_ptr(), data.numel(), 3, stream=st)
    pm.pmrc_encode(code, data.data_ptr(), par.data_ptr(), S, stripes, st)
    pm.pmrc_set_plan_policy(code, pm.PMRC_PLAN_RUNTIME)

    def piece(i):
        return (par.data_ptr() + (i - k) * a * S, P * S) if i >= k else (data.data_ptr() + i * a * S, B * S)
    if what in ("all", "decode"):
        ids = [0, 1, 4, 5, 9, 12, 14, 15]
        dec = torch.zeros_like(data)
        pm.pmrc_decode(code, ids, [piece(i) for i in ids], dec.data_ptr(), S, stripes, st)
    if what in ("all", "repair"):
        H = [i for i in range(n) if i not in (15, 9)]
        out = torch.empty((stripes, a, S), dtype=torch.uint8, device="cuda")
        pm.pmrc_repair(code, 15, H, [piece(i) for i in H], (out.data_ptr(), a * S), S, stripes, st)
    if what in ("all", "encode"):
        par2 = torch.empty_like(par)
        pm.pmrc_encode(code, data.data_ptr(), par2.data_ptr(), S, stripes, st)
    torch.cuda.synchronize()
    pm.pmrc_destroy(code)


if __name__ == "__main__":
    main()
