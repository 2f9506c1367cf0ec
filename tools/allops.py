#!/usr/bin/env python3
"""One small run of every product call on the GPU (python tools/allops.py):

Each op runs once on a few stripes with ragged block sizes (every kernel family: the generated
bitsliced encode / decode / fused repair / split repair / apply, the runtime-coefficient kernel's
single and batch calls, the specific decoders, the host-staged encode), and its result is checked
against the oracle / the unique answer.  Prints one line per op."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np
import torch

import oracle as O
import paper_1412_3022_b200 as pm
from gpu_util import DEV, Stripes, oracle_kind


def check(name, ok):
    print("%-48s %s" % (name, "ok" if ok else "MISMATCH"), flush=True)
    if not ok:
        raise SystemExit(1)


def missing(st, ids):
    held = set()
    for i in ids:
        if i < st.k:
            held |= ({i * st.alpha + j for j in range(st.alpha)} if st.kind != pm.PMRC_MBR
                     else {int(v) - 1 for v in st.L[i]})
    return sorted(set(range(st.B)) - held)


def run(kind, k, n, S, stripes, policy):
    tag = "%s k=%d S=%d %s" % ({0: "msr", 2: "mbr", 3: "rs"}[kind], k, S, {1: "jit", 2: "rt"}[policy])
    st = Stripes(kind, k, n, S, stripes, seed=11 + k, policy=policy)
    try:
        st.encode()
        check("encode " + tag, np.array_equal(st.parity.cpu().numpy(),
                                              O.encode(oracle_kind(kind), n, k, st.d, st.host_data())))
        # decode from the last k nodes (every systematic block of the first nodes missing)
        surv = list(range(n - k, n))
        out = torch.full_like(st.data, 0x5A)
        pm.pmrc_decode(st.code, surv, [st.piece(i) for i in surv], out.data_ptr(), S, stripes, st.stream)
        torch.cuda.synchronize()
        miss = missing(st, surv)
        check("decode " + tag, torch.equal(out[:, miss], st.data[:, miss]))
        # fused repair of a systematic and a parity node
        need = k if kind == pm.PMRC_RS_VANDERMONDE else st.d
        for f in (1, n - 1):
            H = [i for i in range(n) if i != f][:need]
            piece = torch.full((stripes, st.alpha, S), 0x3C, dtype=torch.uint8, device=DEV)
            pm.pmrc_repair(st.code, f, H, [st.piece(i) for i in H], (piece.data_ptr(), st.alpha * S), S, stripes,
                           st.stream)
            torch.cuda.synchronize()
            check("repair f=%d %s" % (f, tag), torch.equal(piece, st.piece_tensor(f)))
        # batch calls: a pattern per stripe, one launch
        reps = [((t * 3) % n, None) for t in range(stripes)]
        reps = [(f, [i for i in range(n) if i != f][:need]) for f, _ in reps]
        out = torch.full((stripes * st.alpha * S,), 0x3C, dtype=torch.uint8, device=DEV)
        pm.pmrc_repair_batch(st.code, [f for f, _ in reps], [H for _, H in reps], st.nodes(),
                             (out.data_ptr(), st.alpha * S), S, stripes, st.stream)
        torch.cuda.synchronize()
        got = out.view(stripes, st.alpha, S)
        check("repair_batch " + tag, all(torch.equal(got[t], st.piece_tensor(f)[t]) for t, (f, _) in enumerate(reps)))
        decs = [[(t + j) % n for j in range(k)] for t in range(stripes)]
        dec = torch.full_like(st.data, 0xA5)
        pm.pmrc_decode_batch(st.code, decs, st.nodes(), dec.data_ptr(), S, stripes, st.stream)
        torch.cuda.synchronize()
        check("decode_batch " + tag, all(torch.equal(dec[t, missing(st, decs[t])], st.data[t, missing(st, decs[t])])
                                         for t in range(stripes)))
        if kind != pm.PMRC_RS_VANDERMONDE:
            surv = list(range(n - k, n))
            scratch_bytes = pm.pmrc_decode_specific_scratch(st.code, S, stripes)
            scratch = torch.empty((max(1, scratch_bytes),), dtype=torch.uint8, device=DEV)
            out = torch.full_like(st.data, 0x5A)
            pm.pmrc_decode_specific(st.code, surv, [st.piece(i) for i in surv], out.data_ptr(), scratch.data_ptr(),
                                    scratch_bytes, S, stripes, st.stream)
            torch.cuda.synchronize()
            miss = missing(st, surv)
            check("decode_specific " + tag, torch.equal(out[:, miss], st.data[:, miss]))
        if kind == pm.PMRC_MSR_SPARSE and policy == pm.PMRC_PLAN_JIT:
            f, H = n - 1, list(range(need))
            betas = torch.empty((need, stripes, S), dtype=torch.uint8, device=DEV)
            for j, h in enumerate(H):
                pm.pmrc_repair_project(st.code, f, st.piece(h), (betas[j].data_ptr(), S), S, stripes, st.stream)
            piece = torch.empty((stripes, st.alpha, S), dtype=torch.uint8, device=DEV)
            pm.pmrc_repair_combine(st.code, f, H, [(betas[j].data_ptr(), S) for j in range(need)],
                                   (piece.data_ptr(), st.alpha * S), S, stripes, st.stream)
            torch.cuda.synchronize()
            check("repair_project/combine " + tag, torch.equal(piece, st.piece_tensor(f)))
            hd = st.data.cpu().pin_memory()
            hp = torch.empty((stripes, st.P, S), dtype=torch.uint8).pin_memory()
            pm.pmrc_encode_host(st.code, hd.data_ptr(), hp.data_ptr(), S, stripes, st.stream)
            torch.cuda.synchronize()
            check("encode_host " + tag, torch.equal(hp, st.parity.cpu()))
    finally:
        st.close()


def main():
    torch.cuda.set_device(0)
    for policy in (pm.PMRC_PLAN_JIT, pm.PMRC_PLAN_RUNTIME):
        run(pm.PMRC_MSR_SPARSE, 8, 16, 2048 + 16, 3, policy)
        run(pm.PMRC_MSR_SPARSE, 3, 6, 1024 + 48, 4, policy)
        run(pm.PMRC_MBR, 8, 16, 1024 + 16, 2, policy)
        run(pm.PMRC_RS_VANDERMONDE, 8, 16, 4096, 2, policy)
    print("sanitize: all ops ok")


if __name__ == "__main__":
    main()
