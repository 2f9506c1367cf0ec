#!/usr/bin/env python3
"""One launch each of the runtime-coefficient kernel (1 GiB jobs), for ncu (kernel filter:
rlc_kernel):  rtprof.py decode|repair|encode|rs_encode [...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import inputs
import paper_1412_3022_b200 as pm


def job(kind, k, S):
    d = k if kind == pm.PMRC_RS_VANDERMONDE else 2 * k - 2
    code = pm.pmrc_create(kind, k, d, 2 * k)
    info = pm.pmrc_info(code)
    a, B, P = info["alpha"], info["B"], info["parity_rows"]
    stripes = -(-(1 << 30) // (B * S))
    data = torch.empty((stripes, B, S), dtype=torch.uint8, device="cuda")
    par = torch.empty((stripes, P, S), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    inputs.fill_device(data.data_ptr(), data.numel(), 3, stream=st)
    pm.pmrc_encode(code, data.data_ptr(), par.data_ptr(), S, stripes, st)
    pm.pmrc_set_plan_policy(code, pm.PMRC_PLAN_RUNTIME)
    return code, data, par, a, B, P, stripes, st


def main():
    whats = sys.argv[1:] or ["decode", "repair", "encode"]
    k, S = 8, 1 << 20
    code, data, par, a, B, P, stripes, st = job(pm.PMRC_MSR_SPARSE, k, S)

    def piece(i):
        return (par.data_ptr() + (i - k) * a * S, P * S) if i >= k else (data.data_ptr() + i * a * S, B * S)
    for what in whats:
        if what == "decode":
            ids = [0, 1, 4, 5, 9, 12, 14, 15]
            dec = torch.zeros_like(data)
            pm.pmrc_decode(code, ids, [piece(i) for i in ids], dec.data_ptr(), S, stripes, st)
        elif what == "repair":
            H = [i for i in range(16) if i not in (15, 9)]
            out = torch.empty((stripes, a, S), dtype=torch.uint8, device="cuda")
            pm.pmrc_repair(code, 15, H, [piece(i) for i in H], (out.data_ptr(), a * S), S, stripes, st)
        elif what == "encode":
            par2 = torch.empty_like(par)
            pm.pmrc_encode(code, data.data_ptr(), par2.data_ptr(), S, stripes, st)
        elif what in ("batch_repair", "batch_decode"):
            r = inputs.rng(2026)
            reps, decs = [], []
            for t in range(stripes):
                while True:
                    f = int(r.integers(16))
                    H = sorted(r.choice([i for i in range(16) if i != f], 14, replace=False).tolist())
                    om = [i for i in range(16) if i != f and i not in H]
                    if not (f < a and len(om) == 1 and om[0] < a):
                        break
                reps.append((f, H))
                decs.append(sorted(r.choice(16, 8, replace=False).tolist()))
            nodes = [piece(i) for i in range(16)]
            if what == "batch_repair":
                out = torch.empty((stripes, a, S), dtype=torch.uint8, device="cuda")
                pm.pmrc_repair_batch(code, [f for f, _ in reps], [H for _, H in reps], nodes, (out.data_ptr(), a * S),
                                     S, stripes, st)
            else:
                dec = torch.zeros_like(data)
                pm.pmrc_decode_batch(code, decs, nodes, dec.data_ptr(), S, stripes, st)
        elif what == "rs_encode":
            c2, d2, p2, _, _, _, s2, _ = job(pm.PMRC_RS_VANDERMONDE, 8, S)
            pm.pmrc_encode(c2, d2.data_ptr(), p2.data_ptr(), S, s2, st)
            torch.cuda.synchronize()
            pm.pmrc_destroy(c2)
    torch.cuda.synchronize()
    pm.pmrc_destroy(code)


if __name__ == "__main__":
    main()
