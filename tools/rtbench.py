#!/usr/bin/env python3
"""Runtime-coefficient kernel (csrc/rt/rlc.cu) vs the generated bitsliced kernels (JIT), kernel-only
(CUDA events, inputs resident, 1 GiB jobs > L2), one JSON line per measurement:

  config 4 as BASELINE.json writes it: per-stripe (lost, helpers) and survivor sets, ONE launch
           each (pmrc_repair_batch / pmrc_decode_batch), bit-exact against the data / the pieces
  single-pattern repair (systematic / parity lost node) and decode: runtime vs JIT policy
  encode (config 2 and config 3 codes) on the runtime kernel vs the JIT kernel (the north star's
           formulation choice: PRMT tables vs bitsliced XOR networks)

Roofline per measurement: algorithmic HBM bytes (distinct blocks read + written) at the measured
HBM peak; the PRMT formulation's own ALU-pipe work (rt_alu_per_word, counted from the plan blob)
at 148 x 64 lanes/clk x 1.965 GHz ("rt_formulation_alu_frac" / "rt_alu_frac"); and the SURVEY §8(d)
naive-W issue term of the same plan ("naive_W_alu_frac").
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import inputs
import paper_1412_3022_b200 as pm

ALU = 148 * 64 * 1965e6


def hbm_peak():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] * 1e9
    except Exception:
        return 6545.3e9


def timed(fn, steps=10, warmup=3):
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


def emit(d):
    print(json.dumps(d), flush=True)


def singular(k, n, f, H):
    alpha = k - 1
    om = [i for i in range(n) if i != f and i not in H]
    return n >= 2 * k and f < alpha and len(om) == 1 and om[0] < alpha


class Job:
    def __init__(self, kind, k, n, S, seed=5):
        self.kind, self.k, self.n, self.S = kind, k, n, S
        self.d = k if kind == 3 else 2 * k - 2
        self.code = pm.pmrc_create(kind, k, self.d, n)
        info = pm.pmrc_info(self.code)
        self.a, self.B, self.P = info["alpha"], info["B"], info["parity_rows"]
        self.stripes = -(-(1 << 30) // (self.B * S))
        self.data = torch.empty((self.stripes, self.B, S), dtype=torch.uint8, device="cuda")
        self.par = torch.empty((self.stripes, self.P, S), dtype=torch.uint8, device="cuda")
        self.st = torch.cuda.current_stream().cuda_stream
        inputs.fill_device(self.data.data_ptr(), self.data.numel(), seed, stream=self.st)
        pm.pmrc_encode(self.code, self.data.data_ptr(), self.par.data_ptr(), S, self.stripes, self.st)
        torch.cuda.synchronize()

    def piece(self, i):
        if i >= self.k:
            return (self.par.data_ptr() + (i - self.k) * self.a * self.S, self.P * self.S)
        return (self.data.data_ptr() + i * self.a * self.S, self.B * self.S)

    def piece_t(self, i):
        a = self.a
        return self.par[:, (i - self.k) * a:(i - self.k + 1) * a] if i >= self.k else self.data[:, i * a:(i + 1) * a]


HDR = ["magic", "words", "n_in", "n_out", "n_terms", "R", "n_rb", "flags", "off_tabA", "off_tabB", "off_ttabA",
       "off_ttabB", "off_terms", "off_outs", "off_masks", "smem_words", "G", "n_pass", "off_pstart", "off_seq",
       "seq_len"]


def rt_alu_per_word(blob):
    """ALU-pipe lane-ops per 32-bit word position of the runtime kernel's formulation for a plan blob
    (rlc.cu): every streamed coefficient term 3 LOP3 + 3 LEA.HI (selectors) + 3 PRMT + 1.5 LOP3,
    every completed input 3 + 3 (selectors) + 1 (unpermute), every nonzero coefficient of a row block
    3 PRMT + 2 LOP3, each counted once per row group that streams it."""
    h = dict(zip(HDR, [int(v) for v in blob[:len(HDR)]]))
    ops = 0.0
    for ps in range(h["n_pass"]):
        e0, e1 = int(blob[h["off_pstart"] + ps]), int(blob[h["off_pstart"] + ps + 1])
        for g in range(h["G"]):
            rb = ps * h["G"] + g
            if rb >= h["n_rb"]:
                continue
            for e in range(e0, e1):
                j = int(blob[h["off_seq"] + e])
                w0, w1 = int(blob[h["off_terms"] + 2 * j]), int(blob[h["off_terms"] + 2 * j + 1])
                if not w0 & 0x80000000:
                    ops += 10.5
                if w0 & 0x40000000:
                    mask = int(blob[h["off_masks"] + (w1 >> 16) * h["n_rb"] + rb])
                    ops += 7 + 5 * bin(mask).count("1")
    return ops


def config4_batch(steps):
    j = Job(0, 8, 16, 1 << 20)
    S, a, k, n = j.S, j.a, j.k, j.n
    r = inputs.rng(2026)
    reps, decs, rej = [], [], 0
    for t in range(j.stripes):
        while True:
            f = int(r.integers(n))
            H = sorted(r.choice([i for i in range(n) if i != f], j.d, replace=False).tolist())
            if not singular(k, n, f, H):
                break
            rej += 1
        reps.append((f, H))
        decs.append(sorted(r.choice(n, k, replace=False).tolist()))
    nodes = [j.piece(i) for i in range(n)]
    out = torch.zeros((j.stripes, a, S), dtype=torch.uint8, device="cuda")
    dec = torch.zeros_like(j.data)
    t0 = time.perf_counter()
    pm.pmrc_repair_batch(j.code, [f for f, _ in reps], [H for _, H in reps], nodes, (out.data_ptr(), a * S), S,
                         j.stripes, j.st)
    init_r = time.perf_counter() - t0
    t0 = time.perf_counter()
    pm.pmrc_decode_batch(j.code, decs, nodes, dec.data_ptr(), S, j.stripes, j.st)
    init_d = time.perf_counter() - t0
    torch.cuda.synchronize()
    ok_r = all(bool(torch.equal(out[t], j.piece_t(f)[t])) for t, (f, _) in enumerate(reps))
    ok_d = True
    for t, ids in enumerate(decs):
        miss = [i * a + x for i in range(k) if i not in ids for x in range(a)]
        if miss:
            ok_d &= bool(torch.equal(dec[t, miss], j.data[t, miss]))
    ms_r = timed(lambda: pm.pmrc_repair_batch(j.code, [f for f, _ in reps], [H for _, H in reps], nodes,
                                              (out.data_ptr(), a * S), S, j.stripes, j.st), steps)
    ms_d = timed(lambda: pm.pmrc_decode_batch(j.code, decs, nodes, dec.data_ptr(), S, j.stripes, j.st), steps)
    # algorithmic bytes: repair reads nnz(mu) blocks per helper, writes alpha; decode reads the used
    # survivor blocks, writes the missing data blocks (pmrc_plan_stats per pattern)
    rb = db = 0
    r_ops = d_ops = 0.0
    for f, H in reps:
        s = pm.pmrc_plan_stats(j.code, 1, f, H)
        rb += (s["in_blocks"] + s["out_blocks"]) * S
        r_ops += rt_alu_per_word(pm.pmrc_rt_plan_blob(j.code, 1, f, H)) * (S // 4)
    for ids in decs:
        try:
            s = pm.pmrc_plan_stats(j.code, 0, 0, ids)
        except pm.PmrcError:
            continue
        db += (s["in_blocks"] + s["out_blocks"]) * S
        d_ops += rt_alu_per_word(pm.pmrc_rt_plan_blob(j.code, 0, 0, ids)) * (S // 4)
    hb = hbm_peak()
    emit({"op": "repair_batch", "config": "config4", "stripes": j.stripes, "launches": 1, "bit_exact": ok_r,
          "singular_rejected": rej, "ms": round(ms_r, 4), "GBps_repaired": round(j.stripes * a * S / ms_r / 1e6, 1),
          "host_init_ms": round(init_r * 1e3, 2), "hbm_bytes": rb, "hbm_frac": round(rb / hb / (ms_r * 1e-3), 3),
          "rt_alu_frac": round(r_ops / ALU / (ms_r * 1e-3), 3)})
    emit({"op": "decode_batch", "config": "config4", "stripes": j.stripes, "launches": 1, "bit_exact": ok_d,
          "ms": round(ms_d, 4), "GBps": round(j.stripes * j.B * S / ms_d / 1e6, 1),
          "host_init_ms": round(init_d * 1e3, 2), "hbm_bytes": db, "hbm_frac": round(db / hb / (ms_d * 1e-3), 3),
          "rt_alu_frac": round(d_ops / ALU / (ms_d * 1e-3), 3)})
    if os.environ.get("RTB_PROMOTED", "1") == "1":
        promoted(j, reps, decs, nodes, out, dec, rb, db, hb, steps)
    return j


def promoted(j, reps, decs, nodes, out, dec, rb, db, hb, steps):
    """The same batch calls after every pattern was promoted to its generated kernel (AUTO policy:
    one JIT launch per stripe, no runtime launch), without and with independent (PDL) launches."""
    S, a, k = j.S, j.a, j.k
    pats = [("repair", f, H) for f, H in reps] + [("decode", ids) for ids in decs]
    for indep in (0, 1):
        t0 = time.perf_counter()
        res = pm.prepare_plans(0, k, j.d, j.n, pats, independent=bool(indep))   # NVRTC, parallel
        prep = time.perf_counter() - t0
        pm.pmrc_set_independent_launches(j.code, indep)
        t0 = time.perf_counter()
        for (pt, rc) in res:
            if rc == pm.PMRC_OK:
                if pt[0] == "repair":
                    pm.pmrc_plan_prepare(j.code, 1, pt[1], pt[2])
                else:
                    pm.pmrc_plan_prepare(j.code, 0, 0, pt[1])
        load = time.perf_counter() - t0
        out.zero_()
        dec.zero_()
        l0 = pm.pmrc_launch_count()
        pm.pmrc_repair_batch(j.code, [f for f, _ in reps], [H for _, H in reps], nodes, (out.data_ptr(), a * S), S,
                             j.stripes, j.st)
        lr = pm.pmrc_launch_count() - l0
        l0 = pm.pmrc_launch_count()
        pm.pmrc_decode_batch(j.code, decs, nodes, dec.data_ptr(), S, j.stripes, j.st)
        ld = pm.pmrc_launch_count() - l0
        torch.cuda.synchronize()
        ok_r = all(bool(torch.equal(out[t], j.piece_t(f)[t])) for t, (f, _) in enumerate(reps))
        ok_d = True
        for t, ids in enumerate(decs):
            miss = [i * a + x for i in range(k) if i not in ids for x in range(a)]
            if miss:
                ok_d &= bool(torch.equal(dec[t, miss], j.data[t, miss]))
        ms_r = timed(lambda: pm.pmrc_repair_batch(j.code, [f for f, _ in reps], [H for _, H in reps], nodes,
                                                  (out.data_ptr(), a * S), S, j.stripes, j.st), steps)
        ms_d = timed(lambda: pm.pmrc_decode_batch(j.code, decs, nodes, dec.data_ptr(), S, j.stripes, j.st), steps)
        tag = "promoted_pdl" if indep else "promoted"
        emit({"op": "repair_batch", "config": "config4", "plans": tag, "stripes": j.stripes, "launches": lr,
              "bit_exact": ok_r, "ms": round(ms_r, 4), "GBps_repaired": round(j.stripes * a * S / ms_r / 1e6, 1),
              "nvrtc_s": round(prep, 2), "load_s": round(load, 2), "hbm_frac": round(rb / hb / (ms_r * 1e-3), 3)})
        emit({"op": "decode_batch", "config": "config4", "plans": tag, "stripes": j.stripes, "launches": ld,
              "bit_exact": ok_d, "ms": round(ms_d, 4), "GBps": round(j.stripes * j.B * S / ms_d / 1e6, 1),
              "hbm_frac": round(db / hb / (ms_d * 1e-3), 3)})
    pm.pmrc_set_independent_launches(j.code, 0)


def single(j, steps):
    S, a = j.S, j.a
    H6 = [i for i in range(16) if i not in (6, 12)]
    H15 = [i for i in range(16) if i not in (15, 9)]
    ids = [0, 1, 4, 5, 9, 12, 14, 15]
    for pol, name in ((pm.PMRC_PLAN_RUNTIME, "runtime"), (pm.PMRC_PLAN_JIT, "jit")):
        pm.pmrc_set_plan_policy(j.code, pol)
        for f, H in ((6, H6), (15, H15)):
            out = torch.empty((j.stripes, a, S), dtype=torch.uint8, device="cuda")
            fn = lambda: pm.pmrc_repair(j.code, f, H, [j.piece(i) for i in H], (out.data_ptr(), a * S), S,
                                        j.stripes, j.st)
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            init = time.perf_counter() - t0
            ok = bool(torch.equal(out, j.piece_t(f)))
            ms = timed(fn, steps)
            s = pm.pmrc_plan_stats(j.code, 1, f, H)
            byts = (s["in_blocks"] + s["out_blocks"]) * S * j.stripes
            rt = rt_alu_per_word(pm.pmrc_rt_plan_blob(j.code, 1, f, H)) * (S // 4) * j.stripes
            emit({"op": "repair", "engine": name, "lost": f, "bit_exact": ok, "ms": round(ms, 4),
                  "GBps_repaired": round(j.stripes * a * S / ms / 1e6, 1), "first_call_s": round(init, 3),
                  "hbm_frac": round(byts / hbm_peak() / (ms * 1e-3), 3),
                  "rt_formulation_alu_frac": round(rt / ALU / (ms * 1e-3), 3)})
        dec = torch.zeros_like(j.data)
        fn = lambda: pm.pmrc_decode(j.code, ids, [j.piece(i) for i in ids], dec.data_ptr(), S, j.stripes, j.st)
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        init = time.perf_counter() - t0
        miss = [i * a + x for i in range(8) if i not in ids for x in range(a)]
        ok = bool(torch.equal(dec[:, miss], j.data[:, miss]))
        ms = timed(fn, steps)
        s = pm.pmrc_plan_stats(j.code, 0, 0, ids)
        byts = (s["in_blocks"] + s["out_blocks"]) * S * j.stripes
        naive = s["naive_lop3"] * (S // 32) * j.stripes
        rt = rt_alu_per_word(pm.pmrc_rt_plan_blob(j.code, 0, 0, ids)) * (S // 4) * j.stripes
        emit({"op": "decode", "engine": name, "survivors": ids, "bit_exact": ok, "ms": round(ms, 4),
              "GBps": round(j.stripes * j.B * S / ms / 1e6, 1), "first_call_s": round(init, 3),
              "hbm_frac": round(byts / hbm_peak() / (ms * 1e-3), 3),
              "naive_W_alu_frac": round(naive / ALU / (ms * 1e-3), 3),
              "rt_formulation_alu_frac": round(rt / ALU / (ms * 1e-3), 3)})
    pm.pmrc_set_plan_policy(j.code, pm.PMRC_PLAN_AUTO)


def encode_cmp(steps):
    for kind, k, S in ((0, 8, 1 << 20), (2, 8, 256 << 10), (3, 8, 1 << 20)):
        j = Job(kind, k, 2 * k, S)
        ref = j.par.clone()
        for pol, name in ((pm.PMRC_PLAN_JIT, "jit_bitsliced"), (pm.PMRC_PLAN_RUNTIME, "runtime_prmt")):
            pm.pmrc_set_plan_policy(j.code, pol)
            j.par.zero_()
            fn = lambda: pm.pmrc_encode(j.code, j.data.data_ptr(), j.par.data_ptr(), S, j.stripes, j.st)
            fn()
            torch.cuda.synchronize()
            ok = bool(torch.equal(j.par, ref))
            ms = timed(fn, steps)
            info = pm.pmrc_info(j.code)
            naive = info["xor_ops_naive"] * (S // 32) * j.stripes
            byts = (j.B + j.P) * S * j.stripes
            rt = rt_alu_per_word(pm.pmrc_rt_plan_blob(j.code, 2)) * (S // 4) * j.stripes
            emit({"op": "encode", "engine": name, "kind": kind, "k": k, "S": S, "same_as_jit": ok, "ms": round(ms, 4),
                  "GBps": round(j.stripes * j.B * S / ms / 1e6, 1),
                  "naive_W_alu_frac": round(naive / ALU / (ms * 1e-3), 3),
                  "rt_alu_frac": round(rt / ALU / (ms * 1e-3), 3),
                  "hbm_frac": round(byts / hbm_peak() / (ms * 1e-3), 3)})
        pm.pmrc_destroy(j.code)
        del j


def main():
    torch.cuda.set_device(0)
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    steps = 10
    if what in ("all", "config4"):
        j = config4_batch(steps)
        if what == "all":
            single(j, steps)
        pm.pmrc_destroy(j.code)
    if what in ("all", "encode"):
        encode_cmp(steps)


if __name__ == "__main__":
    main()
