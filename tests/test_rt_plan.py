"""CPU tier: the runtime-coefficient kernel's plan blobs (built by the product's host code, no GPU),
executed by a plain numpy emulation of the kernel's semantics (pass sequences, derived-input terms,
row masks, 3-3-2 table lookups from the blob's PRMT tables, output wiring), against the oracle:
encode equals O.encode, decode returns the data, repair returns the encoded piece.  This pins the
blob builder (tables, masks, row clustering, pass sequences, term flags) independently of the GPU;
the PRMT selector arithmetic itself is pinned in test_rt_formulation.py."""
import numpy as np
import pytest

import inputs
import oracle as O
import paper_1412_3022_b200 as pm

HDR = ["magic", "words", "n_in", "n_out", "n_terms", "R", "n_rb", "flags", "off_tabA", "off_tabB", "off_ttabA",
       "off_ttabB", "off_terms", "off_outs", "off_masks", "smem_words", "G", "n_pass", "off_pstart", "off_seq",
       "seq_len"]


def _bytes(w):
    return [(int(w) >> (8 * i)) & 0xFF for i in range(4)]


def _mul(tA, tB, x):
    """c * x through the blob's tables: T0 = bytes of (tA[0], tA[1]), T1 = (tA[2], tA[3]), T2 = tB."""
    T0 = np.array(_bytes(tA[0]) + _bytes(tA[1]), np.uint8)
    T1 = np.array(_bytes(tA[2]) + _bytes(tA[3]), np.uint8)
    T2 = np.array(_bytes(tB), np.uint8)
    return T0[x & 7] ^ T1[(x >> 3) & 7] ^ T2[x >> 6]


def emulate(blob, slots, out_slot_arrays):
    """slots[s] = uint8 [blocks][S] (one stripe); out_slot_arrays[s] written in place."""
    h = dict(zip(HDR, [int(v) for v in blob[:len(HDR)]]))
    assert h["magic"] == 0x524C4331 and h["words"] == len(blob)
    R, G, n_rb, n_out = h["R"], h["G"], h["n_rb"], h["n_out"]
    S = next(iter(slots.values())).shape[1]
    for ps in range(h["n_pass"]):
        e0, e1 = blob[h["off_pstart"] + ps], blob[h["off_pstart"] + ps + 1]
        for g in range(G):
            rb = ps * G + g
            if rb >= n_rb:
                continue
            acc = np.zeros((R, S), np.uint8)
            w = np.zeros(S, np.uint8)
            for e in range(e0, e1):
                j = int(blob[h["off_seq"] + e])
                w0, w1 = int(blob[h["off_terms"] + 2 * j]), int(blob[h["off_terms"] + 2 * j + 1])
                x = slots[w0 & 0xFFFF][w1 & 0xFFFF]
                if w0 & 0x80000000:
                    w = w ^ x
                else:
                    w = w ^ _mul(blob[h["off_ttabA"] + 4 * j: h["off_ttabA"] + 4 * j + 4], blob[h["off_ttabB"] + j], x)
                if not w0 & 0x40000000:
                    continue
                i = w1 >> 16
                mask = int(blob[h["off_masks"] + i * n_rb + rb])
                for r in range(R):
                    if mask >> r & 1:
                        t = i * n_out + rb * R + r
                        acc[r] ^= _mul(blob[h["off_tabA"] + 4 * t: h["off_tabA"] + 4 * t + 4], blob[h["off_tabB"] + t], w)
                w = np.zeros(S, np.uint8)
            for r in range(R):
                row = rb * R + r
                if row < n_out:
                    s_, b_ = int(blob[h["off_outs"] + 2 * row]), int(blob[h["off_outs"] + 2 * row + 1])
                    out_slot_arrays[s_][b_] = acc[r]
    return h


@pytest.mark.parametrize("kind,k,n", [(0, 3, 6), (0, 8, 16), (2, 4, 8), (3, 8, 16), (1, 4, 8)])
def test_rt_encode_blob_emulated_equals_oracle(kind, k, n):
    d = k if kind == 3 else 2 * k - 2
    code = pm.pmrc_create(kind, k, d, n)
    try:
        info = pm.pmrc_info(code)
        B, P = info["B"], info["parity_rows"]
        blob = pm.pmrc_rt_plan_blob(code, 2)
        x = inputs.stripe_data(1, B, 64, seed=3 + k)[0]
        par = np.zeros((P, 64), np.uint8)
        h = emulate(blob, {0: x}, {1: par})
        okind = {0: O.MSR_SPARSE, 1: O.MSR_VANILLA, 2: O.MBR, 3: O.RS}[kind]
        assert np.array_equal(par, O.encode(okind, n, k, d, x[None])[0])
        # every pass streams only the inputs its rows read; when a symbol group's n - k rows fill
        # whole row blocks (k = 8: 8 rows, R = 8) the sparse MSR rows cluster so that every
        # (input, row block) mask is all or nothing
        assert h["seq_len"] <= h["n_pass"] * h["n_terms"]
        if kind == 0 and (n - k) % h["R"] == 0:
            masks = blob[h["off_masks"]: h["off_masks"] + h["n_in"] * h["n_rb"]]
            full = [(1 << min(h["R"], h["n_out"] - b * h["R"])) - 1 for b in range(h["n_rb"])]
            for i in range(h["n_in"]):
                for b in range(h["n_rb"]):
                    assert int(masks[i * h["n_rb"] + b]) in (0, full[b])
    finally:
        pm.pmrc_destroy(code)


@pytest.mark.parametrize("kind,k,n", [(0, 3, 6), (0, 8, 16), (2, 3, 6), (3, 8, 16)])
def test_rt_decode_and_repair_blobs_emulated(kind, k, n):
    d = k if kind == 3 else 2 * k - 2
    code = pm.pmrc_create(kind, k, d, n)
    try:
        info = pm.pmrc_info(code)
        B, P, a = info["B"], info["parity_rows"], info["alpha"]
        S = 48
        x = inputs.stripe_data(1, B, S, seed=9 + k)[0]
        okind = {0: O.MSR_SPARSE, 2: O.MBR, 3: O.RS}[kind]
        par = O.encode(okind, n, k, d, x[None])[0]
        L = pm.pmrc_layout(code)

        def piece(i):
            if i >= k:
                return par[(i - k) * a:(i - k + 1) * a]
            if kind == 2:
                return x[[int(v) - 1 for v in L[i]]]
            return x[i * a:(i + 1) * a]
        r = inputs.rng(5 + k)
        for _ in range(4):
            ids = sorted(r.choice(n, k, replace=False).tolist())
            held = set()
            for i in ids:
                if i < k:
                    held |= {int(v) - 1 for v in L[i]} if kind == 2 else {i * a + j for j in range(a)}
            miss = sorted(set(range(B)) - held)
            if not miss:
                continue
            blob = pm.pmrc_rt_plan_blob(code, 0, 0, ids)
            out = np.zeros((B, S), np.uint8)
            emulate(blob, {q: piece(i) for q, i in enumerate(ids)}, {len(ids): out})
            assert np.array_equal(out[miss], x[miss]), ids
        need = k if kind == 3 else d
        for _ in range(4):
            f = int(r.integers(n))
            H = sorted(r.choice([i for i in range(n) if i != f], need, replace=False).tolist())
            try:
                blob = pm.pmrc_rt_plan_blob(code, 1, f, H)
            except pm.PmrcError as e:
                assert e.rc == pm.PMRC_ESINGULAR
                continue
            out = np.zeros((a, S), np.uint8)
            emulate(blob, {q: piece(i) for q, i in enumerate(H)}, {len(H): out})
            assert np.array_equal(out, piece(f)), (f, H)
    finally:
        pm.pmrc_destroy(code)


def test_rt_decode_blob_k16_tables_in_device_memory():
    # k = 16 decode from 16 parity nodes: 240 x 240 coefficients (1.15 MB of tables) exceed the
    # shared-memory budget, so the blob flags its tables to be read from device memory; the
    # emulation of that blob still returns the data
    kind, k, n, d = 0, 16, 32, 30
    code = pm.pmrc_create(kind, k, d, n)
    try:
        info = pm.pmrc_info(code)
        B, a = info["B"], info["alpha"]
        S = 16
        x = inputs.stripe_data(1, B, S, seed=161)[0]
        par = O.encode(O.MSR_SPARSE, n, k, d, x[None])[0]
        ids = list(range(16, 32))
        blob = pm.pmrc_rt_plan_blob(code, 0, 0, ids)
        h = dict(zip(HDR, [int(v) for v in blob[:len(HDR)]]))
        assert h["flags"] & 1 and h["smem_words"] == h["off_tabA"] < h["words"]
        out = np.zeros((B, S), np.uint8)
        emulate(blob, {q: par[(i - k) * a:(i - k + 1) * a] for q, i in enumerate(ids)}, {len(ids): out})
        assert np.array_equal(out, x)
    finally:
        pm.pmrc_destroy(code)


def test_rt_rows_per_thread_follow_the_plan_size():
    # rows per thread: 7 or 8, the one with fewer passes and then fewer row slots (rtplan.cpp
    # rt_shape): MSR k = 8 repairs (7 rows) and 4-missing-node decodes (28 rows) take 7, the
    # 56-row encode (8-row symbol groups) and a 15-row MBR decode keep 8
    code = pm.pmrc_create(0, 8, 14, 16)
    mbr = pm.pmrc_create(2, 8, 14, 16)
    try:
        def shape(c, op, lost=0, ids=()):
            h = dict(zip(HDR, [int(v) for v in pm.pmrc_rt_plan_blob(c, op, lost, ids)[:len(HDR)]]))
            return h["n_out"], h["R"], h["G"], h["n_pass"]
        assert shape(code, 1, 15, list(range(14))) == (7, 7, 1, 1)
        assert shape(code, 1, 3, [i for i in range(15) if i != 3]) == (7, 7, 1, 1)
        assert shape(code, 0, 0, [0, 1, 4, 5, 9, 12, 14, 15]) == (28, 7, 2, 2)
        assert shape(code, 2) == (56, 8, 2, 4)
        assert shape(mbr, 0, 0, [0, 1, 4, 5, 6, 7, 11, 14]) == (15, 8, 2, 1)
    finally:
        pm.pmrc_destroy(code)
        pm.pmrc_destroy(mbr)
