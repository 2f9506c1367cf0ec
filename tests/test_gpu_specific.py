"""GPU parity (-m gpu) of the paper's specific product-matrix decoders (NEXT-2; P:336, P:398;
S:406-423) run as region linear combinations on both engines: the MSR message Z the GPU computes
(stage 4, in scratch) equals the oracle's specific decoder's Z (O.decode_msr_specific_Z), and the
decoded data blocks equal the data (the decoded data is unique: "decoding method is independent of
the encoding method") and pmrc_decode's output."""
import itertools

import numpy as np
import pytest
import torch

import inputs
import oracle as O
import paper_1412_3022_b200 as pm
from gpu_util import DEV, POLICIES, Stripes, oracle_kind

pytestmark = pytest.mark.gpu


def _missing(st, ids):
    held = set()
    for i in ids:
        if i < st.k:
            held |= ({i * st.alpha + j for j in range(st.alpha)} if st.kind != pm.PMRC_MBR
                     else {int(v) - 1 for v in st.L[i]})
    return sorted(set(range(st.B)) - held)


def _check(st, ids, policy):
    S, stripes = st.S, st.stripes
    nbytes = pm.pmrc_decode_specific_scratch(st.code, S, stripes)
    scratch = torch.zeros(nbytes, dtype=torch.uint8, device=DEV)
    out = torch.full_like(st.data, 0xA5)
    nw = pm.pmrc_decode_specific(st.code, list(ids), [st.piece(i) for i in ids], out.data_ptr(), scratch.data_ptr(),
                                 nbytes, S, stripes, st.stream)
    torch.cuda.synchronize()
    miss = _missing(st, ids)
    assert nw == len(miss)
    keep = [b for b in range(st.B) if b not in miss]
    if miss:
        assert torch.equal(out[:, miss], st.data[:, miss]), ids
    assert bool((out[:, keep] == 0xA5).all()), ids
    if st.kind != pm.PMRC_MBR:
        # stage 4's message Z (scratch buffers: A k^2, P/Q 2k^2, U 2k alpha, then Z B blocks per stripe)
        k, a = st.k, st.alpha
        off = (k * k + 2 * k * k + 2 * k * a) * S * stripes
        Z = scratch[off:off + st.B * S * stripes].view(stripes, st.B, S).cpu().numpy()
        sids = sorted(ids)
        for t in range(stripes):
            pieces = np.stack([st.piece_tensor(i)[t].cpu().numpy() for i in sids])
            want = O.decode_msr_specific_Z(oracle_kind(st.kind), st.n, st.k, st.d, sids, pieces)
            assert np.array_equal(Z[t], want), (ids, t)
    else:
        sids = sorted(ids)
        for t in range(stripes):
            pieces = np.stack([st.piece_tensor(i)[t].cpu().numpy() for i in sids])
            want = O.decode_mbr_specific(st.n, st.k, st.d, sids, pieces)
            assert np.array_equal(want, st.host_data()[t]), (ids, t)     # the oracle's own cross-check


@pytest.mark.parametrize("policy", POLICIES)
@pytest.mark.parametrize("kind", [pm.PMRC_MSR_SPARSE, pm.PMRC_MSR_VANILLA, pm.PMRC_MBR])
def test_specific_decode_k3_every_subset(kind, policy):
    st = Stripes(kind, 3, 6, 2048 + 16, 3, seed=5, policy=policy)
    try:
        st.encode()
        subsets = list(itertools.combinations(range(6), 3))
        if policy == pm.PMRC_PLAN_JIT and kind != pm.PMRC_MSR_SPARSE:
            subsets = subsets[::3]   # exhaustive on the runtime engine and for the sparse code
        for ids in subsets:
            _check(st, ids, policy)
    finally:
        st.close()


@pytest.mark.parametrize("policy", POLICIES)
@pytest.mark.parametrize("kind,k,n", [(pm.PMRC_MSR_SPARSE, 8, 16), (pm.PMRC_MBR, 8, 16), (pm.PMRC_MSR_SPARSE, 4, 8),
                                      (pm.PMRC_MSR_SPARSE_N2K, 8, 16)])
def test_specific_decode_random_subsets(kind, k, n, policy):
    st = Stripes(kind, k, n, 4096 + 32, 2, seed=6 + k, policy=policy)
    try:
        st.encode()
        r = inputs.rng(31 + k)
        sets = [list(range(n - k, n)), list(range(k))] + [r.choice(n, k, replace=False).tolist() for _ in range(3)]
        if policy == pm.PMRC_PLAN_JIT:
            sets = sets[::2]   # every set costs 5 NVRTC compiles on the JIT engine
        for ids in sets:
            _check(st, [int(x) for x in r.permutation(ids)], policy)
    finally:
        st.close()


def test_specific_equals_linear_decode_k16():
    # k = 16 (the paper's crossover region): specific and linear decode write the same bytes
    st = Stripes(pm.PMRC_MSR_SPARSE, 16, 32, 1024, 1, seed=16, policy=pm.PMRC_PLAN_RUNTIME)
    try:
        st.encode()
        ids = list(range(20, 32)) + [0, 5, 9, 13]
        nbytes = pm.pmrc_decode_specific_scratch(st.code, st.S, st.stripes)
        scratch = torch.empty(nbytes, dtype=torch.uint8, device=DEV)
        a = torch.zeros_like(st.data)
        b = torch.zeros_like(st.data)
        pm.pmrc_decode_specific(st.code, ids, [st.piece(i) for i in ids], a.data_ptr(), scratch.data_ptr(), nbytes,
                                st.S, st.stripes, st.stream)
        pm.pmrc_decode(st.code, ids, [st.piece(i) for i in ids], b.data_ptr(), st.S, st.stripes, st.stream)
        torch.cuda.synchronize()
        assert torch.equal(a, b)
        miss = _missing(st, ids)
        assert torch.equal(a[:, miss], st.data[:, miss])
    finally:
        st.close()


def test_specific_decode_errors():
    st = Stripes(pm.PMRC_MSR_SPARSE, 3, 6, 1024, 1, seed=2)
    try:
        st.encode()
        with pytest.raises(pm.PmrcError) as e:      # exactly k survivors
            pm.pmrc_decode_specific(st.code, [0, 1, 2, 3], [st.piece(i) for i in range(4)], st.data.data_ptr(),
                                    st.data.data_ptr(), 1 << 20, st.S, 1, st.stream)
        assert e.value.rc == pm.PMRC_EINVAL
        rs = pm.pmrc_create(pm.PMRC_RS_VANDERMONDE, 8, 8, 16)
        try:
            with pytest.raises(pm.PmrcError) as e:
                pm.pmrc_decode_specific_scratch(rs, 1024, 1)
            assert e.value.rc == pm.PMRC_EUNSUPPORTED
        finally:
            pm.pmrc_destroy(rs)
    finally:
        st.close()
