"""GPU parity (-m gpu): the CUDA path through the C ABI vs the oracle, element by element, on the
same seeded inputs; sizes span several 1 KiB chunks and ragged tails.  Plus full-size config 2
(1 GiB, the bench's launch configuration) on sampled stripes/windows."""
import itertools

import numpy as np
import pytest
import torch

import inputs
import oracle as O
import paper_1412_3022_b200 as pm
from gpu_util import DEV, POLICIES, Stripes, oracle_kind

pytestmark = pytest.mark.gpu

ENC_CASES = [
    (pm.PMRC_MSR_SPARSE, 3, 6, 2048, 16),     # config 1 shape
    (pm.PMRC_MSR_SPARSE, 8, 16, 4096 + 1024 + 16, 3),   # config 2 code, ragged chunk tail
    (pm.PMRC_MSR_SPARSE, 8, 15, 1040, 2),
    (pm.PMRC_MSR_VANILLA, 8, 16, 2064, 2),
    (pm.PMRC_MBR, 8, 16, 3072 + 48, 2),       # config 3 code
    (pm.PMRC_RS_VANDERMONDE, 8, 16, 4096, 3),
    (pm.PMRC_MSR_SPARSE, 4, 8, 1024, 5),
    (pm.PMRC_MBR, 4, 8, 1008, 4),
    (pm.PMRC_MSR_SPARSE, 16, 32, 1024 + 32, 1),
    (pm.PMRC_MSR_SPARSE, 2, 3, 16, 7),        # smallest code, one vector per block
    (pm.PMRC_MSR_SPARSE_N2K, 8, 16, 2048 + 32, 2),   # R15 extension
    (pm.PMRC_MBR, 16, 32, 1024 + 16, 1),      # config 5's MBR k=16 plan (30 groups, 16-row groups, layout 0)
    (pm.PMRC_MSR_SPARSE, 8, 16, (4 << 20) + 16, 1),   # config 5's largest sub-block (4 MiB), ragged
    (pm.PMRC_MSR_VANILLA, 3, 6, 2048, 16),    # the k=3 codes the decode / repair tests start from
    (pm.PMRC_MBR, 3, 6, 2048, 16),
    (pm.PMRC_RS_VANDERMONDE, 3, 6, 2048, 16),
]


@pytest.mark.parametrize("policy", POLICIES)
@pytest.mark.parametrize("kind,k,n,S,stripes", ENC_CASES)
def test_encode_bit_exact(kind, k, n, S, stripes, policy):
    st = Stripes(kind, k, n, S, stripes, seed=11 + k, policy=policy)
    try:
        st.encode()
        want = O.encode(oracle_kind(kind), n, k, st.d, st.host_data())
        got = st.parity.cpu().numpy()
        assert np.array_equal(got, want)
    finally:
        st.close()


def test_encode_empty_and_alignment():
    st = Stripes(pm.PMRC_MSR_SPARSE, 3, 6, 32, 2, seed=3)
    try:
        before = st.parity.clone()
        pm.pmrc_encode(st.code, st.data.data_ptr(), st.parity.data_ptr(), 0, 2, st.stream)
        pm.pmrc_encode(st.code, st.data.data_ptr(), st.parity.data_ptr(), 32, 0, st.stream)
        torch.cuda.synchronize()
        assert torch.equal(before, st.parity)
        with pytest.raises(pm.PmrcError) as e:
            pm.pmrc_encode(st.code, st.data.data_ptr() + 8, st.parity.data_ptr(), 32, 1, st.stream)
        assert e.value.rc == pm.PMRC_EALIGN
    finally:
        st.close()


def test_encode_does_not_touch_beyond_parity():
    # the kernel writes exactly stripes x P x S bytes: guard bytes after the buffer stay intact
    k, n, S, stripes = 8, 16, 1024 + 16, 2
    st = Stripes(pm.PMRC_MSR_SPARSE, k, n, S, stripes, seed=5)
    try:
        big = torch.full((stripes * st.P * S + 4096,), 0x5A, dtype=torch.uint8, device=DEV)
        pm.pmrc_encode(st.code, st.data.data_ptr(), big.data_ptr(), S, stripes, st.stream)
        torch.cuda.synchronize()
        assert bool((big[stripes * st.P * S:] == 0x5A).all())
        want = O.encode(O.MSR_SPARSE, n, k, st.d, st.host_data())
        assert np.array_equal(big[: stripes * st.P * S].cpu().numpy().reshape(stripes, st.P, S), want)
    finally:
        st.close()


@pytest.mark.parametrize("policy", POLICIES)
@pytest.mark.parametrize("kind", [pm.PMRC_MSR_SPARSE, pm.PMRC_MSR_VANILLA, pm.PMRC_MBR, pm.PMRC_RS_VANDERMONDE])
def test_decode_config1_every_subset(kind, policy):
    # config 1: k=3, n=6 (RS uses the same k, n): decode from every 3-subset
    k, n, S, stripes = 3, 6, 2048, 16
    st = Stripes(kind, k, n, S, stripes, seed=1, policy=policy)
    try:
        st.encode()
        # the parity every decode starts from is itself the oracle's (not only self-consistent)
        assert np.array_equal(st.parity.cpu().numpy(), O.encode(oracle_kind(kind), n, k, st.d, st.host_data()))
        for ids in itertools.combinations(range(n), k):
            out = torch.zeros_like(st.data)
            nw = pm.pmrc_decode(st.code, list(ids), [st.piece(i) for i in ids], out.data_ptr(), S, stripes, st.stream)
            torch.cuda.synchronize()
            held = set()
            for i in ids:
                if i < k:
                    held |= ({i * st.alpha + j for j in range(st.alpha)} if kind != pm.PMRC_MBR
                             else {int(v) - 1 for v in st.L[i]})
            missing = sorted(set(range(st.B)) - held)
            assert nw == len(missing)
            assert torch.equal(out[:, missing], st.data[:, missing]), ids
            untouched = sorted(held)
            assert not out[:, untouched].any()   # only missing blocks are written
    finally:
        st.close()


@pytest.mark.parametrize("policy", POLICIES)
@pytest.mark.parametrize("kind", [pm.PMRC_MSR_SPARSE, pm.PMRC_MBR])
def test_decode_k8_random_subsets(kind, policy):
    k, n, S, stripes = 8, 16, 2048 + 16, 2
    st = Stripes(kind, k, n, S, stripes, seed=9, policy=policy)
    try:
        st.encode()
        r = inputs.rng(4)
        for trial in range(6):
            ids = sorted(r.choice(n, k, replace=False).tolist())
            if policy == pm.PMRC_PLAN_JIT and trial % 2:
                continue   # half the sets on the JIT engine (an NVRTC compile each)
            out = st.data.clone()
            lost = [i for i in range(k) if i not in ids]
            # poison the lost systematic blocks, decode in place
            for i in lost:
                if kind != pm.PMRC_MBR:
                    out[:, i * st.alpha:(i + 1) * st.alpha] = 0xCC
            pm.pmrc_decode(st.code, ids, [st.piece(i) for i in ids], out.data_ptr(), S, stripes, st.stream)
            torch.cuda.synchronize()
            if kind != pm.PMRC_MBR:
                assert torch.equal(out, st.data), ids
            else:
                # oracle cross-check of the decoded blocks
                got = out.cpu().numpy()
                want = st.host_data()
                assert np.array_equal(got, want), ids
    finally:
        st.close()


def test_decode_more_than_k_survivors_and_errors():
    k, n, S = 3, 6, 1024
    st = Stripes(pm.PMRC_MSR_SPARSE, k, n, S, 4, seed=2)
    try:
        st.encode()
        ids = [5, 1, 4, 3]   # unsorted, one systematic
        out = torch.zeros_like(st.data)
        pm.pmrc_decode(st.code, ids, [st.piece(i) for i in ids], out.data_ptr(), S, 4, st.stream)
        torch.cuda.synchronize()
        miss = [0, 1, 4, 5]
        assert torch.equal(out[:, miss], st.data[:, miss])
        with pytest.raises(pm.PmrcError) as e:
            pm.pmrc_decode(st.code, [3, 4], [st.piece(3), st.piece(4)], out.data_ptr(), S, 4, st.stream)
        assert e.value.rc == pm.PMRC_ESINGULAR
    finally:
        st.close()


def _predicted_singular(kind, k, n, f, H):
    alpha = k - 1
    if kind != pm.PMRC_MSR_SPARSE or n < 2 * k:
        return False
    omitted = [i for i in range(n) if i != f and i not in H]
    return f < alpha and len(omitted) == 1 and omitted[0] < alpha


@pytest.mark.parametrize("policy", POLICIES)
@pytest.mark.parametrize("kind", [pm.PMRC_MSR_SPARSE, pm.PMRC_MSR_VANILLA, pm.PMRC_MBR, pm.PMRC_MSR_SPARSE_N2K])
def test_repair_config1_every_node_every_helper_set(kind, policy):
    k, n, S, stripes = 3, 6, 2048, 16
    st = Stripes(kind, k, n, S, stripes, seed=1, policy=policy)
    try:
        st.encode()
        assert np.array_equal(st.parity.cpu().numpy(), O.encode(oracle_kind(kind), n, k, st.d, st.host_data()))
        d = st.d
        n_sing = 0
        for f in range(n):
            for H in itertools.combinations([i for i in range(n) if i != f], d):
                H = list(H)
                out = torch.empty((stripes, st.alpha, S), dtype=torch.uint8, device=DEV)
                try:
                    pm.pmrc_repair(st.code, f, H, [st.piece(i) for i in H], (out.data_ptr(), st.alpha * S), S,
                                   stripes, st.stream)
                except pm.PmrcError as e:
                    assert e.rc == pm.PMRC_ESINGULAR and _predicted_singular(kind, k, n, f, H), (f, H)
                    n_sing += 1
                    continue
                torch.cuda.synchronize()
                assert not _predicted_singular(kind, k, n, f, H)
                assert torch.equal(out, st.piece_tensor(f)), (f, H)
        assert n_sing == (2 if kind == pm.PMRC_MSR_SPARSE else 0)
    finally:
        st.close()


@pytest.mark.parametrize("policy", POLICIES)
@pytest.mark.parametrize("kind", [pm.PMRC_MSR_SPARSE, pm.PMRC_MBR, pm.PMRC_RS_VANDERMONDE])
def test_repair_k8_random(kind, policy):
    k, n, S, stripes = 8, 16, 4096 + 16, 2
    st = Stripes(kind, k, n, S, stripes, seed=21, policy=policy)
    try:
        st.encode()
        r = inputs.rng(8)
        need = k if kind == pm.PMRC_RS_VANDERMONDE else st.d
        done = 0
        while done < 5:
            f = int(r.integers(n))
            H = sorted(r.choice([i for i in range(n) if i != f], need, replace=False).tolist())
            if _predicted_singular(kind, k, n, f, H):
                continue
            out = torch.empty((stripes, st.alpha, S), dtype=torch.uint8, device=DEV)
            pm.pmrc_repair(st.code, f, H, [st.piece(i) for i in H], (out.data_ptr(), st.alpha * S), S, stripes,
                           st.stream)
            torch.cuda.synchronize()
            assert torch.equal(out, st.piece_tensor(f)), (f, H)
            done += 1
    finally:
        st.close()


@pytest.mark.parametrize("policy", POLICIES)
def test_repair_project_combine_split_equals_oracle(policy):
    # helper side (projection) and newcomer side (combine) as separate calls, vs the oracle
    k, n, S, stripes = 8, 16, 2048, 2
    st = Stripes(pm.PMRC_MSR_SPARSE, k, n, S, stripes, seed=33, policy=policy)
    try:
        st.encode()
        for f in (2, 11):
            H = [i for i in range(n) if i not in (f, 15)]   # omit a Cauchy node: never singular (R10)
            betas = torch.empty((len(H), stripes, S), dtype=torch.uint8, device=DEV)
            for j, h in enumerate(H):
                pm.pmrc_repair_project(st.code, f, st.piece(h), (betas[j].data_ptr(), S), S, stripes, st.stream)
            torch.cuda.synchronize()
            for j, h in enumerate(H):
                piece = st.piece_tensor(h).cpu().numpy()
                for t in range(stripes):
                    want = O.repair_project(O.MSR_SPARSE, n, k, st.d, f, piece[t])
                    assert np.array_equal(betas[j, t].cpu().numpy(), want)
            out = torch.empty((stripes, st.alpha, S), dtype=torch.uint8, device=DEV)
            pm.pmrc_repair_combine(st.code, f, H, [(betas[j].data_ptr(), S) for j in range(len(H))],
                                   (out.data_ptr(), st.alpha * S), S, stripes, st.stream)
            torch.cuda.synchronize()
            assert torch.equal(out, st.piece_tensor(f))
    finally:
        st.close()


def test_encode_host_path_equals_device_path():
    k, n, S, stripes = 8, 16, 8192, 9
    st = Stripes(pm.PMRC_MSR_SPARSE, k, n, S, stripes, seed=44)
    try:
        st.encode()
        hd = torch.from_numpy(st.host_data()).pin_memory()
        hp = torch.zeros((stripes, st.P, S), dtype=torch.uint8).pin_memory()
        pm.pmrc_encode_host(st.code, hd.data_ptr(), hp.data_ptr(), S, stripes, st.stream)
        assert torch.equal(hp, st.parity.cpu())
    finally:
        st.close()


def test_encode_host_block_size_grows_between_calls():
    # the host path's staging ring must follow the block size, not only the stripe
    # count: a small S then a larger S on one handle (same stripes) must stay bit-exact
    k, n = 8, 16
    code = pm.pmrc_create(pm.PMRC_MSR_SPARSE, k, 14, n)
    try:
        # stripes of > 16 MiB go through the host path in column ranges (2-D copies), ragged last one
        for S, stripes in ((64 * 1024, 1), (1 << 20, 1), (16 * 1024, 3), (2 << 20, 2), ((1 << 20) + 48, 3)):
            x = inputs.stripe_data(stripes, 56, S, seed=S)
            hd = torch.from_numpy(x).pin_memory()
            hp = torch.zeros((stripes, 56, S), dtype=torch.uint8).pin_memory()
            pm.pmrc_encode_host(code, hd.data_ptr(), hp.data_ptr(), S, stripes, torch.cuda.current_stream().cuda_stream)
            d = torch.from_numpy(x).to(DEV)
            par = torch.empty((stripes, 56, S), dtype=torch.uint8, device=DEV)
            pm.pmrc_encode(code, d.data_ptr(), par.data_ptr(), S, stripes, torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            assert torch.equal(hp, par.cpu()), S
            w = min(S, 4096)
            assert np.array_equal(hp[:, :, :w].numpy(), O.encode(O.MSR_SPARSE, n, k, 14, x[:, :, :w]))
            assert np.array_equal(hp[:, :, S - w:].numpy(), O.encode(O.MSR_SPARSE, n, k, 14, x[:, :, S - w:]))
    finally:
        pm.pmrc_destroy(code)


def test_full_size_config2_sampled():
    # config 2 in the bench's launch configuration: 1 GiB real data (R11: 19 stripes of 56 x 1 MiB,
    # last one zero padded), generated on the device; sampled stripes and byte windows vs oracle
    k, n, S = 8, 16, 1 << 20
    B = 56
    real = 1 << 30
    stripes = -(-real // (B * S))
    code = pm.pmrc_create(pm.PMRC_MSR_SPARSE, k, 14, n)
    try:
        data = torch.empty((stripes, B, S), dtype=torch.uint8, device=DEV)
        par = torch.empty((stripes, B, S), dtype=torch.uint8, device=DEV)
        stream = torch.cuda.current_stream().cuda_stream
        inputs.fill_device(data.data_ptr(), data.numel(), 1234, real_len=real, stream=stream)
        pm.pmrc_encode(code, data.data_ptr(), par.data_ptr(), S, stripes, stream)
        torch.cuda.synchronize()
        r = inputs.rng(77)
        for t in (0, stripes - 1, int(r.integers(1, stripes - 1))):
            for p0 in (0, S - 4096, int(r.integers(0, S // 16 - 256)) * 16):
                W = 4096
                x = np.stack([inputs.host_bytes(W, 1234, t * B * S + c * S + p0, real) for c in range(B)])
                want = O.encode(O.MSR_SPARSE, n, k, 14, x[None])[0]
                assert np.array_equal(par[t, :, p0:p0 + W].cpu().numpy(), want), (t, p0)
        # R11: the last stripe holds the remaining 16 MiB of real data in its first 16 blocks and
        # zero padding after them (its parity, which mixes both, is in the sampled windows above)
        last_real = real - (stripes - 1) * B * S
        full_blocks = last_real // S
        assert full_blocks == 16 and last_real % S == 0
        assert data[stripes - 1, :full_blocks].any() and not data[stripes - 1, full_blocks:].any()
    finally:
        pm.pmrc_destroy(code)


def _full_job(kind, k, S, seed):
    n, d = 2 * k, 2 * k - 2
    code = pm.pmrc_create(kind, k, d, n)
    info = pm.pmrc_info(code)
    B, P, a = info["B"], info["parity_rows"], info["alpha"]
    real = 1 << 30
    stripes = -(-real // (B * S))
    data = torch.empty((stripes, B, S), dtype=torch.uint8, device=DEV)
    par = torch.empty((stripes, P, S), dtype=torch.uint8, device=DEV)
    stream = torch.cuda.current_stream().cuda_stream
    inputs.fill_device(data.data_ptr(), data.numel(), seed, real_len=real, stream=stream)
    pm.pmrc_encode(code, data.data_ptr(), par.data_ptr(), S, stripes, stream)
    torch.cuda.synchronize()
    return code, data, par, (n, d, B, P, a, stripes, real, stream)


@pytest.mark.parametrize("policy", POLICIES)
def test_full_size_config4_repair_and_decode(policy):
    # config 4 at full size (1 GiB, 1 MiB sub-blocks, 19 stripes) in the sweep's launch
    # configuration: a repair of a parity node (alpha blocks per helper) and of a systematic node
    # (1 block per helper) regenerate the encoded pieces exactly; decode from a random
    # 8-subset returns the data; a sampled window of the parity is checked against the oracle
    k, S = 8, 1 << 20
    code, data, par, (n, d, B, P, a, stripes, real, stream) = _full_job(pm.PMRC_MSR_SPARSE, k, S, 99)
    pm.pmrc_set_plan_policy(code, policy)
    try:
        def piece(i):
            return (par.data_ptr() + (i - k) * a * S, P * S) if i >= k else (data.data_ptr() + i * a * S, B * S)

        def piece_t(i):
            return par[:, (i - k) * a:(i - k + 1) * a] if i >= k else data[:, i * a:(i + 1) * a]
        x = np.stack([inputs.host_bytes(2048, 99, 5 * B * S + c * S + 4096, real) for c in range(B)])
        assert np.array_equal(par[5, :, 4096:4096 + 2048].cpu().numpy(), O.encode(O.MSR_SPARSE, n, k, d, x[None])[0])
        out = torch.empty((stripes, a, S), dtype=torch.uint8, device=DEV)
        for f, H in ((13, [i for i in range(n) if i not in (13, 9)]), (3, [i for i in range(n) if i not in (3, 11)])):
            out.fill_(0)
            pm.pmrc_repair(code, f, H, [piece(i) for i in H], (out.data_ptr(), a * S), S, stripes, stream)
            torch.cuda.synchronize()
            assert torch.equal(out, piece_t(f)), f
        ids = sorted(inputs.rng(4).choice(n, k, replace=False).tolist())
        dec = torch.zeros_like(data)
        nw = pm.pmrc_decode(code, ids, [piece(i) for i in ids], dec.data_ptr(), S, stripes, stream)
        torch.cuda.synchronize()
        miss = [i * a + x for i in range(k) if i not in ids for x in range(a)]
        assert nw == len(miss)
        assert torch.equal(dec[:, miss], data[:, miss])
    finally:
        pm.pmrc_destroy(code)


@pytest.mark.parametrize("policy", POLICIES)
def test_full_size_config3_mbr_encode_decode(policy):
    # config 3 at full size (MBR k=8, 1 GiB, 256 KiB sub-blocks, 49 stripes): sampled parity windows
    # vs the oracle, then decode from a random 8-subset of nodes returns every missing data block
    k, S = 8, 256 << 10
    code, data, par, (n, d, B, P, a, stripes, real, stream) = _full_job(pm.PMRC_MBR, k, S, 7)
    pm.pmrc_set_plan_policy(code, policy)
    try:
        for t, p0 in ((0, 0), (stripes - 2, S - 1024), (17, 77 * 16)):
            x = np.stack([inputs.host_bytes(1024, 7, t * B * S + c * S + p0, real) for c in range(B)])
            assert np.array_equal(par[t, :, p0:p0 + 1024].cpu().numpy(), O.encode(O.MBR, n, k, d, x[None])[0])
        L = pm.pmrc_layout(code)
        ids = sorted(inputs.rng(3).choice(n, k, replace=False).tolist())
        sysp = {}
        pieces = []
        for i in ids:
            if i >= k:
                pieces.append((par.data_ptr() + (i - k) * a * S, P * S))
            else:                      # MBR systematic node i = row i of M(X) (R6), materialised
                sysp[i] = data.index_select(1, torch.tensor([int(v) - 1 for v in L[i]], device=DEV)).contiguous()
                pieces.append((sysp[i].data_ptr(), a * S))
        dec = torch.zeros_like(data)
        pm.pmrc_decode(code, ids, pieces, dec.data_ptr(), S, stripes, stream)
        torch.cuda.synchronize()
        held = set()
        for i in ids:
            if i < k:
                held |= {int(v) - 1 for v in L[i]}
        miss = sorted(set(range(B)) - held)
        assert miss and torch.equal(dec[:, miss], data[:, miss])
    finally:
        pm.pmrc_destroy(code)


def test_per_stripe_patterns_one_launch_each():
    # config 4's per-stripe failure patterns: each stripe repaired / decoded with its own plan by
    # offsetting the piece pointers to that stripe (stripes = 1 per launch)
    k, n, S, stripes = 8, 16, 4096 + 512, 4
    st = Stripes(pm.PMRC_MSR_SPARSE, k, n, S, stripes, seed=61)
    try:
        st.encode()
        r = inputs.rng(12)
        out = torch.zeros((stripes, st.alpha, S), dtype=torch.uint8, device=DEV)
        want = []
        for t in range(stripes):
            while True:
                f = int(r.integers(n))
                H = sorted(r.choice([i for i in range(n) if i != f], st.d, replace=False).tolist())
                if not _predicted_singular(pm.PMRC_MSR_SPARSE, k, n, f, H):
                    break
            pieces = [(st.piece(i)[0] + t * st.piece(i)[1], st.piece(i)[1]) for i in H]
            pm.pmrc_repair(st.code, f, H, pieces, (out[t].data_ptr(), st.alpha * S), S, 1, st.stream)
            want.append(st.piece_tensor(f)[t])
        torch.cuda.synchronize()
        for t in range(stripes):
            assert torch.equal(out[t], want[t]), t
    finally:
        st.close()


def test_n2k_extension_repairs_paper_singular_sets_k8():
    # R15: the (lost, helpers) pairs for which the paper's construction returns PMRC_ESINGULAR at
    # k = 8, n = 16 (f < alpha, H omits another identity node) repair exactly with kind 4
    k, n, S, stripes = 8, 16, 4096 + 16, 2
    paper = Stripes(pm.PMRC_MSR_SPARSE, k, n, S, stripes, seed=71)
    ext = Stripes(pm.PMRC_MSR_SPARSE_N2K, k, n, S, stripes, seed=71)
    try:
        ext.encode()
        paper.encode()
        for f, omit in ((0, 1), (3, 6), (6, 2)):
            H = [i for i in range(n) if i not in (f, omit)]
            out = torch.empty((stripes, ext.alpha, S), dtype=torch.uint8, device=DEV)
            with pytest.raises(pm.PmrcError) as e:
                pm.pmrc_repair(paper.code, f, H, [paper.piece(i) for i in H], (out.data_ptr(), paper.alpha * S), S,
                               stripes, paper.stream)
            assert e.value.rc == pm.PMRC_ESINGULAR
            pm.pmrc_repair(ext.code, f, H, [ext.piece(i) for i in H], (out.data_ptr(), ext.alpha * S), S, stripes,
                           ext.stream)
            torch.cuda.synchronize()
            assert torch.equal(out, ext.piece_tensor(f)), (f, H)
    finally:
        paper.close()
        ext.close()


@pytest.mark.parametrize("policy", POLICIES)
def test_apply_matches_encode_specific_and_precode_paths(policy):
    # pmrc_apply (general region linear combination) on the paper's comparison paths:
    #  * non-systematic encode Y = G Z equals the oracle's specific PM encode C = Psi M(Z)
    #  * precode Z = Gtilde^{-1} X, then parity = G_parity Z, equals the linearised systematic
    #    encode G'' X (the two systematic encoders give identical codewords)
    k, n, S, stripes = 8, 16, 2048 + 48, 2
    st = Stripes(pm.PMRC_MSR_SPARSE, k, n, S, stripes, seed=81, policy=policy)
    try:
        st.encode()
        G = pm.pmrc_matrix(st.code, pm.MATRIX_G)
        Gti = pm.pmrc_matrix(st.code, pm.MATRIX_GTINV)
        B, a = st.B, st.alpha
        Y = torch.empty((stripes, n * a, S), dtype=torch.uint8, device=DEV)
        pm.pmrc_apply(st.code, G, st.data.data_ptr(), B * S, Y.data_ptr(), n * a * S, S, stripes, st.stream)
        torch.cuda.synchronize()
        Z = st.host_data()
        want = np.stack([O.encode_specific(O.MSR_SPARSE, n, k, st.d, Z[t]).reshape(n * a, S) for t in range(stripes)])
        assert np.array_equal(Y.cpu().numpy(), want)
        Zd = torch.empty_like(st.data)
        pm.pmrc_apply(st.code, Gti, st.data.data_ptr(), B * S, Zd.data_ptr(), B * S, S, stripes, st.stream)
        par = torch.empty_like(st.parity)
        pm.pmrc_apply(st.code, G[k * a:], Zd.data_ptr(), B * S, par.data_ptr(), st.P * S, S, stripes, st.stream)
        torch.cuda.synchronize()
        assert torch.equal(par, st.parity)
        Gpp = pm.pmrc_matrix(st.code, pm.MATRIX_GPP)
        pm.pmrc_apply(st.code, Gpp, st.data.data_ptr(), B * S, par.data_ptr(), st.P * S, S, stripes, st.stream)
        torch.cuda.synchronize()
        assert torch.equal(par, st.parity)
    finally:
        st.close()


@pytest.mark.parametrize("policy", POLICIES)
def test_decode_and_repair_write_only_their_outputs(policy):
    # no compute-sanitizer on this pool: bounds by sentinels instead.  Decode writes exactly the
    # missing data blocks (every other byte of data_out keeps its sentinel); repair writes exactly
    # stripes x alpha x S bytes (guard bytes after the piece stay intact); ragged S
    k, n, S, stripes = 8, 16, 3072 + 16, 3
    st = Stripes(pm.PMRC_MSR_SPARSE, k, n, S, stripes, seed=91, policy=policy)
    try:
        st.encode()
        ids = [1, 2, 5, 6, 9, 10, 13, 15]
        out = torch.full_like(st.data, 0xA5)
        nw = pm.pmrc_decode(st.code, ids, [st.piece(i) for i in ids], out.data_ptr(), S, stripes, st.stream)
        torch.cuda.synchronize()
        miss = [i * st.alpha + a for i in range(k) if i not in ids for a in range(st.alpha)]
        keep = [b for b in range(st.B) if b not in miss]
        assert nw == len(miss)
        assert torch.equal(out[:, miss], st.data[:, miss])
        assert bool((out[:, keep] == 0xA5).all())
        f, H = 12, [i for i in range(n) if i not in (12, 4)]
        big = torch.full((stripes * st.alpha * S + 8192,), 0x3C, dtype=torch.uint8, device=DEV)
        pm.pmrc_repair(st.code, f, H, [st.piece(i) for i in H], (big.data_ptr(), st.alpha * S), S, stripes,
                       st.stream)
        torch.cuda.synchronize()
        assert bool((big[stripes * st.alpha * S:] == 0x3C).all())
        assert torch.equal(big[: stripes * st.alpha * S].view(stripes, st.alpha, S), st.piece_tensor(f))
    finally:
        st.close()


def test_distributed_repair_single_rank_with_product_kernels():
    # NEXT-3's orchestration (paper_1412_3022_b200/dist.py) with the product's projection and
    # combine kernels; all helpers on this rank (the gloo test covers the cross-rank transfers)
    from paper_1412_3022_b200 import dist as pdist
    k, n, S, stripes = 8, 16, 2048 + 16, 2
    st = Stripes(pm.PMRC_MSR_SPARSE, k, n, S, stripes, seed=95)
    try:
        st.encode()
        f, H = 11, [i for i in range(n) if i not in (11, 14)]
        owner = {i: 0 for i in range(n)}

        def project(h, piece):
            b = torch.empty((stripes, S), dtype=torch.uint8, device=DEV)
            pm.pmrc_repair_project(st.code, f, piece, (b.data_ptr(), S), S, stripes, st.stream)
            return b

        def combine(ids, betas, dst):
            pm.pmrc_repair_combine(st.code, f, ids, [(b.data_ptr(), S) for b in betas],
                                   (dst.data_ptr(), st.alpha * S), S, stripes, st.stream)
        out = torch.empty((stripes, st.alpha, S), dtype=torch.uint8, device=DEV)
        sent = pdist.distributed_repair(f, H, owner, {h: st.piece(h) for h in H}, out, project, combine,
                                        torch.empty((stripes, S), dtype=torch.uint8, device=DEV), None, 0)
        torch.cuda.synchronize()
        assert sent == 0
        assert torch.equal(out, st.piece_tensor(f))
    finally:
        st.close()


@pytest.mark.parametrize("k,n,S,stripes", [(8, 16, 2048 + 48, 2), (4, 8, 4096, 3), (8, 15, 64, 5)])
def test_encode_gf16_bit_exact(k, n, S, stripes):
    # w = 16 extension: the GPU encode of the sparse MSR code over GF(2^16)
    # (little-endian byte pairs) equals the GF(2^16) oracle (oracle/gf16.py); ragged chunk tails
    import oracle.gf16 as G16
    code = pm.pmrc_create(pm.PMRC_MSR_SPARSE, k, 2 * k - 2, n, w=16)
    try:
        info = pm.pmrc_info(code)
        B, P = info["B"], info["parity_rows"]
        x = inputs.stripe_data(stripes, B, S, seed=40 + k)
        data = torch.from_numpy(x).to(DEV)
        par = torch.full((stripes, P, S), 0xEE, dtype=torch.uint8, device=DEV)
        pm.pmrc_encode(code, data.data_ptr(), par.data_ptr(), S, stripes, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        assert np.array_equal(par.cpu().numpy(), G16.encode(n, k, x))
    finally:
        pm.pmrc_destroy(code)


@pytest.mark.parametrize("ids", [[0, 1, 4, 5, 9, 12, 14, 15], list(range(8, 16))])
def test_decode_gf16(ids):
    # w = 16: decode from a survivor set returns the data (unique result) -- the GF(2^16)
    # oracle's decode round trip pins the same algebra on the CPU (tests/test_oracle_gf16.py)
    k, n, S, stripes = 8, 16, 2048 + 48, 2
    code = pm.pmrc_create(pm.PMRC_MSR_SPARSE, k, 14, n, w=16)
    try:
        info = pm.pmrc_info(code)
        B, P, a = info["B"], info["parity_rows"], info["alpha"]
        data = torch.from_numpy(inputs.stripe_data(stripes, B, S, seed=71)).to(DEV)
        par = torch.empty((stripes, P, S), dtype=torch.uint8, device=DEV)
        st = torch.cuda.current_stream().cuda_stream
        pm.pmrc_encode(code, data.data_ptr(), par.data_ptr(), S, stripes, st)
        pieces = [(par.data_ptr() + (i - k) * a * S, P * S) if i >= k else (data.data_ptr() + i * a * S, B * S)
                  for i in ids]
        out = torch.zeros_like(data)
        nw = pm.pmrc_decode(code, ids, pieces, out.data_ptr(), S, stripes, st)
        torch.cuda.synchronize()
        miss = [i * a + x for i in range(k) if i not in ids for x in range(a)]
        assert nw == len(miss)
        assert torch.equal(out[:, miss], data[:, miss])
    finally:
        pm.pmrc_destroy(code)


def test_repair_gf16():
    # w = 16: exact repair (P:53 footnote) of a parity node (alpha blocks per helper) and a
    # systematic node (1 block per helper); the R10 singular set is singular over GF(2^16) too
    k, n, S, stripes = 8, 16, 2048 + 48, 2
    code = pm.pmrc_create(pm.PMRC_MSR_SPARSE, k, 14, n, w=16)
    try:
        info = pm.pmrc_info(code)
        B, P, a = info["B"], info["parity_rows"], info["alpha"]
        data = torch.from_numpy(inputs.stripe_data(stripes, B, S, seed=72)).to(DEV)
        par = torch.empty((stripes, P, S), dtype=torch.uint8, device=DEV)
        st = torch.cuda.current_stream().cuda_stream
        pm.pmrc_encode(code, data.data_ptr(), par.data_ptr(), S, stripes, st)

        def piece(i):
            return (par.data_ptr() + (i - k) * a * S, P * S) if i >= k else (data.data_ptr() + i * a * S, B * S)

        def piece_t(i):
            return par[:, (i - k) * a:(i - k + 1) * a] if i >= k else data[:, i * a:(i + 1) * a]
        for f, omit in ((15, 10), (3, 11)):
            H = [i for i in range(n) if i not in (f, omit)]
            out = torch.zeros((stripes, a, S), dtype=torch.uint8, device=DEV)
            pm.pmrc_repair(code, f, H, [piece(i) for i in H], (out.data_ptr(), a * S), S, stripes, st)
            torch.cuda.synchronize()
            assert torch.equal(out, piece_t(f)), f
        H = [i for i in range(n) if i not in (0, 1)]
        with pytest.raises(pm.PmrcError) as e:
            pm.pmrc_repair(code, 0, H, [piece(i) for i in H], (16 * 1024, a * S), S, stripes, st)
        assert e.value.rc == pm.PMRC_ESINGULAR
    finally:
        pm.pmrc_destroy(code)


def test_decode_dynamic_schedule_concurrent_streams_and_tiny():
    # decode plans take chunks from per-group counters (a ring of counter slots, one per launch):
    # the same plan launched back to back on two streams, more launches than a slot ring's worth of
    # in-flight work, and launches with fewer chunks than teams must all stay bit-exact
    k, n = 8, 16
    ids = [0, 1, 4, 5, 9, 12, 14, 15]
    for S, stripes in ((64 * 1024, 6), (16, 1), (1024 + 16, 3)):
        st = Stripes(pm.PMRC_MSR_SPARSE, k, n, S, stripes, seed=21, policy=pm.PMRC_PLAN_JIT)
        try:
            st.encode()
            assert "atomicAdd(dctr" in pm.pmrc_plan_source(st.code, 0, 0, ids)
            streams = [torch.cuda.Stream(), torch.cuda.Stream()]
            outs = [st.data.clone() for _ in range(4)]
            for o in outs:
                for i in (2, 3, 6, 7):
                    o[:, i * st.alpha:(i + 1) * st.alpha] = 0xCC
            torch.cuda.synchronize()
            for rep in range(80):       # > 64 launches of one plan, alternating streams
                o = outs[rep % 4]
                s = streams[rep % 2]
                pm.pmrc_decode(st.code, ids, [st.piece(i) for i in ids], o.data_ptr(), S, stripes, s.cuda_stream)
            torch.cuda.synchronize()
            for o in outs:
                assert torch.equal(o, st.data), (S, stripes)
        finally:
            st.close()


def test_independent_launches_per_stripe_repair_and_decode():
    # config 4's per-stripe patterns with consecutive launches declared independent (programmatic
    # dependent launch: a launch's CTAs start while the previous launch's CTAs retire)
    k, n, S, stripes = 8, 16, 64 * 1024, 6
    st = Stripes(pm.PMRC_MSR_SPARSE, k, n, S, stripes, seed=31, policy=pm.PMRC_PLAN_JIT)
    try:
        st.encode()
        pm.pmrc_set_independent_launches(st.code, 1)
        rep = [(0, 6, [0, 1, 2, 3, 4, 5, 7, 8, 9, 10, 11, 13, 14, 15]),
               (1, 15, [0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 11, 12, 13, 14]),
               (2, 8, [0, 1, 2, 3, 4, 5, 6, 9, 10, 11, 12, 13, 14, 15]),
               (3, 3, [0, 1, 2, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14]),
               (4, 12, [0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 13, 14]),
               (5, 0, [1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 15])]
        dec = [(t, ids) for t, ids in enumerate(([0, 1, 4, 5, 9, 12, 14, 15], list(range(8, 16)),
                                                 [2, 3, 6, 7, 8, 10, 11, 13], [0, 1, 2, 3, 4, 5, 6, 15],
                                                 [1, 3, 5, 7, 9, 11, 13, 15], [0, 2, 4, 6, 8, 10, 12, 14]))]
        a = st.alpha
        out = torch.full((stripes, a, S), 0xAB, dtype=torch.uint8, device=DEV)
        dout = st.data.clone()
        for t, ids in dec:
            for i in range(k):
                if i not in ids:
                    dout[t, i * a:(i + 1) * a] = 0xCC
        for rnd in range(3):
            for t, f, H in rep:
                pcs = [(p + t * s_, s_) for p, s_ in (st.piece(i) for i in H)]
                pm.pmrc_repair(st.code, f, H, pcs, (out[t].data_ptr(), a * S), S, 1, st.stream)
            for t, ids in dec:
                pcs = [(p + t * s_, s_) for p, s_ in (st.piece(i) for i in ids)]
                pm.pmrc_decode(st.code, ids, pcs, dout[t].data_ptr(), S, 1, st.stream)
        torch.cuda.synchronize()
        for t, f, _ in rep:
            assert torch.equal(out[t], st.piece_tensor(f)[t]), (t, f)
        assert torch.equal(dout, st.data)
        pm.pmrc_set_independent_launches(st.code, 0)
    finally:
        st.close()
