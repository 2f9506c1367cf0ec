"""GPU parity (-m gpu), randomised: seeded random codes (from the pre-compiled encode set), block
sizes (16 B up to several tiles, ragged), stripe counts and failure patterns; encode on both engines
against the oracle, decode and repair on the runtime engine (no NVRTC per pattern) against the
unique answers, per-stripe batches against the same.  A property sweep on top of the targeted
tests: any wrong offset, tail mask, table or wiring shows up on some draw."""
import numpy as np
import pytest
import torch

import inputs
import oracle as O
import paper_1412_3022_b200 as pm
from gpu_util import DEV, Stripes, oracle_kind

pytestmark = pytest.mark.gpu

# (kind, k, n): codes whose encode kernels build() pre-compiles (no NVRTC at create)
CODES = [(0, 8, 16), (0, 3, 6), (2, 8, 16), (3, 8, 16), (0, 8, 15), (1, 8, 16), (0, 4, 8), (2, 4, 8), (1, 3, 6),
         (2, 3, 6), (3, 3, 6)]
SIZES = [16, 48, 1008, 1024, 4096 + 16, 8192 + 1024 + 32, 65536 + 48]


def _singular(kind, k, n, f, H):
    alpha = k - 1
    om = [i for i in range(n) if i != f and i not in H]
    return kind == 0 and n >= 2 * k and f < alpha and len(om) == 1 and om[0] < alpha


@pytest.mark.parametrize("case", range(32))
def test_fuzz_encode_decode_repair(case):
    r = inputs.rng(1000 + case)
    kind, k, n = CODES[int(r.integers(len(CODES)))]
    S = SIZES[int(r.integers(len(SIZES)))]
    stripes = int(r.integers(1, 6))
    st = Stripes(kind, k, n, S, stripes, seed=2000 + case, policy=pm.PMRC_PLAN_RUNTIME)
    try:
        # encode, runtime engine and the generated kernel, both against the oracle
        st.encode()
        want = O.encode(oracle_kind(kind), n, k, st.d, st.host_data())
        assert np.array_equal(st.parity.cpu().numpy(), want), (kind, k, n, S, stripes)
        pm.pmrc_set_plan_policy(st.code, pm.PMRC_PLAN_JIT)
        st.parity.fill_(0)
        st.encode()
        assert np.array_equal(st.parity.cpu().numpy(), want)
        pm.pmrc_set_plan_policy(st.code, pm.PMRC_PLAN_AUTO)
        need = k if kind == 3 else st.d
        # single-pattern decode and repair (AUTO: runtime kernel, no NVRTC)
        ids = sorted(r.choice(n, k + int(r.integers(0, n - k + 1)), replace=False).tolist())
        dec = torch.full_like(st.data, 0x5A)
        nw = pm.pmrc_decode(st.code, ids, [st.piece(i) for i in ids], dec.data_ptr(), S, stripes, st.stream)
        torch.cuda.synchronize()
        held = set()
        for i in ids:
            if i < k:
                held |= {int(v) - 1 for v in st.L[i]} if kind == 2 else {i * st.alpha + j for j in range(st.alpha)}
        miss = sorted(set(range(st.B)) - held)
        assert nw == len(miss)
        if miss:
            assert torch.equal(dec[:, miss], st.data[:, miss]), ids
        while True:
            f = int(r.integers(n))
            H = sorted(r.choice([i for i in range(n) if i != f], need, replace=False).tolist())
            if not _singular(kind, k, n, f, H):
                break
        out = torch.zeros((stripes, st.alpha, S), dtype=torch.uint8, device=DEV)
        pm.pmrc_repair(st.code, f, H, [st.piece(i) for i in H], (out.data_ptr(), st.alpha * S), S, stripes, st.stream)
        torch.cuda.synchronize()
        assert torch.equal(out, st.piece_tensor(f)), (f, H)
        # per-stripe batch of random patterns
        reps, decs = [], []
        for _ in range(stripes):
            while True:
                f = int(r.integers(n))
                H = [int(x) for x in r.permutation(r.choice([i for i in range(n) if i != f], need, replace=False))]
                if not _singular(kind, k, n, f, H):
                    break
            reps.append((f, H))
            decs.append([int(x) for x in r.choice(n, k, replace=False)])
        out.zero_()
        pm.pmrc_repair_batch(st.code, [f for f, _ in reps], [H for _, H in reps], st.nodes(),
                             (out.data_ptr(), st.alpha * S), S, stripes, st.stream)
        dec.zero_()
        pm.pmrc_decode_batch(st.code, decs, st.nodes(), dec.data_ptr(), S, stripes, st.stream)
        torch.cuda.synchronize()
        for t, (f, _) in enumerate(reps):
            assert torch.equal(out[t], st.piece_tensor(f)[t]), (t, f)
        for t, ids in enumerate(decs):
            held = set()
            for i in ids:
                if i < k:
                    held |= {int(v) - 1 for v in st.L[i]} if kind == 2 else {i * st.alpha + j for j in range(st.alpha)}
            miss = sorted(set(range(st.B)) - held)
            if miss:
                assert torch.equal(dec[t, miss], st.data[t, miss]), (t, ids)
    finally:
        st.close()
