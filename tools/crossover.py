#!/usr/bin/env python3
"""The paper's linear-vs-specific decode axis (the linearised decode is faster than the
specific PM decoder "for k < 12 (non-systematic) and k < 21 (systematic)"; P:398 for MBR, k < 7) on
one B200: for k in {4, 8, 16} (d = 2k-2, n = 2k) and f = 1..k lost systematic nodes (the k
survivors are the k - f remaining systematic nodes and f parity nodes), time pmrc_decode (one
launch of G'^-1's missing rows) against pmrc_decode_specific (the symmetric-matrix method, one
launch per step, P:55 / S:406-423), both on the same engine, kernel-only (CUDA events, inputs
resident, ~1 GiB of source data per job), and check both outputs against the data.  One JSON line
per point.  usage: crossover.py [--engine runtime|jit] [--ks 4,8,16] [--kinds msr,mbr]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import inputs
import paper_1412_3022_b200 as pm


def timed(fn, steps=5, warmup=2):
    st = torch.cuda.current_stream()
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--engine", default="runtime", choices=["runtime", "jit"])
    ap.add_argument("--ks", default="4,8,16")
    ap.add_argument("--kinds", default="msr,mbr")
    ap.add_argument("--gib", type=float, default=1.0)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    pol = pm.PMRC_PLAN_RUNTIME if args.engine == "runtime" else pm.PMRC_PLAN_JIT
    for kname in args.kinds.split(","):
        kind = pm.PMRC_MSR_SPARSE if kname == "msr" else pm.PMRC_MBR
        for k in [int(x) for x in args.ks.split(",")]:
            n, d = 2 * k, 2 * k - 2
            code = pm.pmrc_create(kind, k, d, n)
            pm.pmrc_set_plan_policy(code, pol)
            info = pm.pmrc_info(code)
            a, B, P = info["alpha"], info["B"], info["parity_rows"]
            S = 256 << 10
            stripes = max(1, int(args.gib * (1 << 30)) // (B * S))
            data = torch.empty((stripes, B, S), dtype=torch.uint8, device="cuda")
            par = torch.empty((stripes, P, S), dtype=torch.uint8, device="cuda")
            st = torch.cuda.current_stream().cuda_stream
            inputs.fill_device(data.data_ptr(), data.numel(), 77, stream=st)
            pm.pmrc_encode(code, data.data_ptr(), par.data_ptr(), S, stripes, st)
            L = pm.pmrc_layout(code)
            mbr_rows = {}

            def piece(i):
                if i >= k:
                    return (par.data_ptr() + (i - k) * a * S, P * S)
                if kind != pm.PMRC_MBR:
                    return (data.data_ptr() + i * a * S, B * S)
                if i not in mbr_rows:
                    mbr_rows[i] = data.index_select(1, torch.tensor([int(v) - 1 for v in L[i]], device="cuda"))
                return (mbr_rows[i].data_ptr(), a * S)
            nbytes = pm.pmrc_decode_specific_scratch(code, S, stripes)
            scratch = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
            for f in range(1, k + 1):
                ids = list(range(f, k)) + list(range(k, k + f))
                held = set()
                for i in ids:
                    if i < k:
                        held |= ({i * a + j for j in range(a)} if kind != pm.PMRC_MBR else {int(v) - 1 for v in L[i]})
                miss = sorted(set(range(B)) - held)
                out_l = torch.zeros_like(data)
                out_s = torch.zeros_like(data)
                pcs = [piece(i) for i in ids]
                lin = lambda: pm.pmrc_decode(code, ids, pcs, out_l.data_ptr(), S, stripes, st)
                spe = lambda: pm.pmrc_decode_specific(code, ids, pcs, out_s.data_ptr(), scratch.data_ptr(), nbytes,
                                                      S, stripes, st)
                lin()
                spe()
                torch.cuda.synchronize()
                ok = bool(torch.equal(out_l[:, miss], data[:, miss])) and bool(torch.equal(out_s[:, miss], data[:, miss]))
                ms_l = timed(lin)
                ms_s = timed(spe)
                src = stripes * B * S
                print(json.dumps({"op": "decode_crossover", "kind": kname, "engine": args.engine, "k": k, "n": n,
                                  "lost_systematic": f, "survivors": ids, "S": S, "stripes": stripes,
                                  "missing_blocks": len(miss), "bit_exact": ok, "linear_ms": round(ms_l, 4),
                                  "specific_ms": round(ms_s, 4), "linear_GBps": round(src / ms_l / 1e6, 1),
                                  "specific_GBps": round(src / ms_s / 1e6, 1),
                                  "faster": "linear" if ms_l < ms_s else "specific"}), flush=True)
            pm.pmrc_destroy(code)
            del data, par, scratch, mbr_rows


if __name__ == "__main__":
    main()
