"""GPU parity (-m gpu) of the runtime-coefficient kernel's batch calls: per-stripe failure patterns
in ONE launch (config 4 as BASELINE.json states it), against the unique answers (the data, the
encoded pieces) of parity that is itself checked against the oracle; a new pattern costs no NVRTC."""
import time

import numpy as np
import pytest
import torch

import inputs
import oracle as O
import paper_1412_3022_b200 as pm
from gpu_util import DEV, Stripes, oracle_kind

pytestmark = pytest.mark.gpu


def _predicted_singular(kind, k, n, f, H):
    alpha = k - 1
    if kind != pm.PMRC_MSR_SPARSE or n < 2 * k:
        return False
    omitted = [i for i in range(n) if i != f and i not in H]
    return f < alpha and len(omitted) == 1 and omitted[0] < alpha


def _patterns(kind, k, n, need, stripes, seed):
    r = inputs.rng(seed)
    reps, decs = [], []
    for t in range(stripes):
        while True:
            f = int(r.integers(n))
            H = sorted(r.choice([i for i in range(n) if i != f], need, replace=False).tolist())
            if not _predicted_singular(kind, k, n, f, H):
                break
        reps.append((f, [int(x) for x in r.permutation(H)]))     # any helper order
        decs.append([int(x) for x in r.permutation(r.choice(n, k, replace=False))])
    return reps, decs


def _missing(st, ids):
    held = set()
    for i in ids:
        if i < st.k:
            held |= ({i * st.alpha + j for j in range(st.alpha)} if st.kind != pm.PMRC_MBR
                     else {int(v) - 1 for v in st.L[i]})
    return sorted(set(range(st.B)) - held)


@pytest.mark.parametrize("kind,k,n,S,stripes", [
    (pm.PMRC_MSR_SPARSE, 8, 16, 4096 + 512, 7),     # config 4's code, ragged tile tail
    (pm.PMRC_MSR_SPARSE, 3, 6, 2048, 16),            # config 1's code
    (pm.PMRC_MBR, 8, 16, 2048 + 16, 5),
    (pm.PMRC_RS_VANDERMONDE, 8, 16, 1024, 6),
    (pm.PMRC_MSR_SPARSE_N2K, 8, 16, 16, 9),          # one 16-B vector per block
    (pm.PMRC_MSR_SPARSE, 16, 32, 1024 + 32, 3),
])
def test_batch_repair_and_decode_per_stripe_patterns(kind, k, n, S, stripes):
    st = Stripes(kind, k, n, S, stripes, seed=100 + k)
    try:
        st.encode()
        assert np.array_equal(st.parity.cpu().numpy(), O.encode(oracle_kind(kind), n, k, st.d, st.host_data()))
        need = k if kind == pm.PMRC_RS_VANDERMONDE else st.d
        reps, decs = _patterns(kind, k, n, need, stripes, seed=7 + k)
        decs[0] = list(range(k))                     # a stripe whose data all survives: nothing written
        nodes = st.nodes()
        # repair: stripe t regenerates node reps[t][0] from its own helpers; one launch
        out = torch.full((stripes * st.alpha * S + 4096,), 0x3C, dtype=torch.uint8, device=DEV)
        l0 = pm.pmrc_launch_count()
        pm.pmrc_repair_batch(st.code, [f for f, _ in reps], [H for _, H in reps], nodes,
                             (out.data_ptr(), st.alpha * S), S, stripes, st.stream)
        torch.cuda.synchronize()
        assert pm.pmrc_launch_count() - l0 == 1
        got = out[: stripes * st.alpha * S].view(stripes, st.alpha, S)
        for t, (f, _) in enumerate(reps):
            assert torch.equal(got[t], st.piece_tensor(f)[t]), (t, f)
        assert bool((out[stripes * st.alpha * S:] == 0x3C).all())          # nothing beyond the pieces
        # decode: stripe t from its own survivors; missing blocks only, others keep the sentinel
        dec = torch.full_like(st.data, 0xA5)
        nw = pm.pmrc_decode_batch(st.code, decs, nodes, dec.data_ptr(), S, stripes, st.stream)
        torch.cuda.synchronize()
        for t, ids in enumerate(decs):
            miss = _missing(st, ids)
            assert nw[t] == len(miss)
            keep = [b for b in range(st.B) if b not in miss]
            if miss:
                assert torch.equal(dec[t, miss], st.data[t, miss]), (t, ids)
            assert bool((dec[t, keep] == 0xA5).all()), (t, ids)
    finally:
        st.close()


def test_batch_singular_and_errors():
    k, n, S, stripes = 8, 16, 1024, 3
    st = Stripes(pm.PMRC_MSR_SPARSE, k, n, S, stripes, seed=5)
    try:
        st.encode()
        good = (11, [i for i in range(n) if i not in (11, 15)])
        bad = (0, [i for i in range(n) if i not in (0, 1)])          # R10: predicted singular pair
        out = torch.empty((stripes, st.alpha, S), dtype=torch.uint8, device=DEV)
        with pytest.raises(pm.PmrcError) as e:
            pm.pmrc_repair_batch(st.code, [good[0], bad[0], good[0]], [good[1], bad[1], good[1]], st.nodes(),
                                 (out.data_ptr(), st.alpha * S), S, stripes, st.stream)
        assert e.value.rc == pm.PMRC_ESINGULAR and "stripe 1" in str(e.value)
        with pytest.raises(pm.PmrcError) as e:   # lost node among its helpers
            pm.pmrc_repair_batch(st.code, [3] * stripes, [list(range(14))] * stripes, st.nodes(),
                                 (out.data_ptr(), st.alpha * S), S, stripes, st.stream)
        assert e.value.rc == pm.PMRC_EINVAL
        dec = torch.empty_like(st.data)
        with pytest.raises(pm.PmrcError) as e:   # fewer than k survivors cannot span the data
            pm.pmrc_decode_batch(st.code, [[8, 9, 10]] * stripes, st.nodes(), dec.data_ptr(), S, stripes, st.stream)
        assert e.value.rc == pm.PMRC_ESINGULAR
        with pytest.raises(pm.PmrcError) as e:
            pm.pmrc_decode_batch(st.code, [list(range(8))] * stripes, st.nodes(), dec.data_ptr() + 8, S, stripes,
                                 st.stream)
        assert e.value.rc == pm.PMRC_EALIGN
    finally:
        st.close()


def test_new_pattern_costs_no_jit():
    # the per-pattern initialisation is the host inversion; under the default policy a new
    # (lost, helpers) pair / survivor set launches the runtime-coefficient kernel at once (no
    # kernel generation, no NVRTC), and gives the same bytes as the generated kernel of the pattern
    k, n, S, stripes = 8, 16, 64 * 1024, 2
    st = Stripes(pm.PMRC_MSR_SPARSE, k, n, S, stripes, seed=17)
    try:
        st.encode()
        assert pm.pmrc_get_plan_policy(st.code) == pm.PMRC_PLAN_AUTO
        r = inputs.rng(99)
        for trial in range(6):
            f = int(r.integers(n))
            while True:
                H = sorted(r.choice([i for i in range(n) if i != f], st.d, replace=False).tolist())
                if not _predicted_singular(pm.PMRC_MSR_SPARSE, k, n, f, H):
                    break
            out = torch.empty((stripes, st.alpha, S), dtype=torch.uint8, device=DEV)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            pm.pmrc_repair(st.code, f, H, [st.piece(i) for i in H], (out.data_ptr(), st.alpha * S), S, stripes,
                           st.stream)
            host_ms = (time.perf_counter() - t0) * 1e3
            torch.cuda.synchronize()
            assert torch.equal(out, st.piece_tensor(f))
            if trial:                      # (the first call also creates the stream-ordered pool)
                assert host_ms < 50, host_ms
            if trial:
                continue
            # promote the pattern to its generated kernel (hot-pattern cache, NVRTC): same bytes
            pm.pmrc_plan_prepare(st.code, 1, f, H)
            out2 = torch.empty_like(out)
            pm.pmrc_repair(st.code, f, H, [st.piece(i) for i in H], (out2.data_ptr(), st.alpha * S), S, stripes,
                           st.stream)
            torch.cuda.synchronize()
            assert torch.equal(out2, out)
    finally:
        st.close()


def test_full_size_config4_batch():
    # config 4 exactly as BASELINE.json writes it, at full size: 1 GiB encoded as config 2 (19 stripes
    # of 1 MiB sub-blocks); every stripe repairs its own uniformly chosen lost node from its own
    # random non-singular 14-helper set, and decodes from its own random 8-node set -- one launch each
    k, n, d, S = 8, 16, 14, 1 << 20
    B, real = 56, 1 << 30
    stripes = -(-real // (B * S))
    code = pm.pmrc_create(pm.PMRC_MSR_SPARSE, k, d, n)
    try:
        info = pm.pmrc_info(code)
        a, P = info["alpha"], info["parity_rows"]
        data = torch.empty((stripes, B, S), dtype=torch.uint8, device=DEV)
        par = torch.empty((stripes, P, S), dtype=torch.uint8, device=DEV)
        stream = torch.cuda.current_stream().cuda_stream
        inputs.fill_device(data.data_ptr(), data.numel(), 4321, real_len=real, stream=stream)
        pm.pmrc_encode(code, data.data_ptr(), par.data_ptr(), S, stripes, stream)
        torch.cuda.synchronize()
        x = np.stack([inputs.host_bytes(1024, 4321, 7 * B * S + c * S + 5 * 4096, real) for c in range(B)])
        assert np.array_equal(par[7, :, 5 * 4096:5 * 4096 + 1024].cpu().numpy(),
                              O.encode(O.MSR_SPARSE, n, k, d, x[None])[0])
        nodes = [(data.data_ptr() + i * a * S, B * S) for i in range(k)] + \
                [(par.data_ptr() + (i - k) * a * S, P * S) for i in range(k, n)]
        reps, decs = _patterns(pm.PMRC_MSR_SPARSE, k, n, d, stripes, seed=2026)
        out = torch.zeros((stripes, a, S), dtype=torch.uint8, device=DEV)
        pm.pmrc_repair_batch(code, [f for f, _ in reps], [H for _, H in reps], nodes, (out.data_ptr(), a * S), S,
                             stripes, stream)
        dec = torch.zeros_like(data)
        pm.pmrc_decode_batch(code, decs, nodes, dec.data_ptr(), S, stripes, stream)
        torch.cuda.synchronize()
        for t, (f, _) in enumerate(reps):
            want = data[t, f * a:(f + 1) * a] if f < k else par[t, (f - k) * a:(f - k + 1) * a]
            assert torch.equal(out[t], want), (t, f)
        for t, ids in enumerate(decs):
            miss = [i * a + x for i in range(k) if i not in ids for x in range(a)]
            if miss:
                assert torch.equal(dec[t, miss], data[t, miss]), (t, ids)
    finally:
        pm.pmrc_destroy(code)


def test_batch_many_small_stripes_and_empty_calls():
    # thousands of stripes of one 1 KiB tile each (the CTA item ranges are balanced by each stripe's
    # plan cost across many plan switches), and the empty calls (no stripes / S = 0) do nothing
    k, n, S, stripes = 8, 16, 1024, 3000
    st = Stripes(pm.PMRC_MSR_SPARSE, k, n, S, stripes, seed=123)
    try:
        st.encode()
        reps, decs = _patterns(pm.PMRC_MSR_SPARSE, k, n, st.d, 40, seed=77)
        reps = [reps[t % 40] for t in range(stripes)]
        decs = [decs[t % 40] for t in range(stripes)]
        out = torch.zeros((stripes, st.alpha, S), dtype=torch.uint8, device=DEV)
        pm.pmrc_repair_batch(st.code, [f for f, _ in reps], [H for _, H in reps], st.nodes(),
                             (out.data_ptr(), st.alpha * S), S, stripes, st.stream)
        dec = torch.zeros_like(st.data)
        pm.pmrc_decode_batch(st.code, decs, st.nodes(), dec.data_ptr(), S, stripes, st.stream)
        torch.cuda.synchronize()
        for t in range(stripes):
            f = reps[t][0]
            assert torch.equal(out[t], st.piece_tensor(f)[t]), t
            miss = _missing(st, decs[t])
            if miss:
                assert torch.equal(dec[t, miss], st.data[t, miss]), t
        before = out.clone()
        pm.pmrc_repair_batch(st.code, [], [], st.nodes(), (out.data_ptr(), st.alpha * S), S, 0, st.stream)
        pm.pmrc_repair_batch(st.code, [f for f, _ in reps], [H for _, H in reps], st.nodes(),
                             (out.data_ptr(), st.alpha * S), 0, stripes, st.stream)
        torch.cuda.synchronize()
        assert torch.equal(before, out)
    finally:
        st.close()


def test_new_plan_used_on_another_stream_right_away():
    # a runtime plan uploaded on stream A (its first call) and used by a launch on stream B issued
    # immediately after: the launch waits for the upload (event), so the result is exact
    k, n, S, stripes = 8, 16, 256 * 1024, 3
    st = Stripes(pm.PMRC_MSR_SPARSE, k, n, S, stripes, seed=321, policy=pm.PMRC_PLAN_RUNTIME)
    try:
        st.encode()
        a_, b_ = torch.cuda.Stream(), torch.cuda.Stream()
        ids = [2, 3, 6, 7, 8, 10, 11, 13]
        outs = [torch.zeros_like(st.data) for _ in range(2)]
        torch.cuda.synchronize()
        pm.pmrc_decode(st.code, ids, [st.piece(i) for i in ids], outs[0].data_ptr(), S, stripes, a_.cuda_stream)
        pm.pmrc_decode(st.code, ids, [st.piece(i) for i in ids], outs[1].data_ptr(), S, stripes, b_.cuda_stream)
        torch.cuda.synchronize()
        miss = _missing(st, ids)
        for o in outs:
            assert torch.equal(o[:, miss], st.data[:, miss])
    finally:
        st.close()


def test_batch_runs_promoted_patterns_on_their_generated_kernels():
    # "the JIT kernels stay as a cache for hot patterns": under AUTO, stripes whose pattern was
    # promoted (pmrc_plan_prepare) run its generated kernel, one launch per run of consecutive
    # stripes with that pattern; the other stripes share one runtime launch; same bytes either way
    k, n, S, stripes = 8, 16, 4096 + 512, 7
    st = Stripes(pm.PMRC_MSR_SPARSE, k, n, S, stripes, seed=71)
    try:
        st.encode()
        A = (15, [i for i in range(15) if i != 9])           # parity node, helpers without node 9
        B = (6, [i for i in range(n) if i not in (6, 15)])   # systematic node
        C = (11, [i for i in range(n) if i not in (11, 2)])
        reps = [A, A, A, B, A, A, C]
        da, db, dc = [0, 1, 4, 5, 9, 12, 14, 15], [2, 3, 8, 9, 10, 11, 12, 13], list(range(8, 16))
        decs = [da, da, db, dc, dc, da, db]
        pm.pmrc_plan_prepare(st.code, 1, A[0], A[1])
        pm.pmrc_plan_prepare(st.code, 1, C[0], C[1])
        pm.pmrc_plan_prepare(st.code, 0, 0, da)
        pm.pmrc_plan_prepare(st.code, 0, 0, dc)
        nodes = st.nodes()
        for policy, launches in ((pm.PMRC_PLAN_AUTO, (4, 4)), (pm.PMRC_PLAN_RUNTIME, (1, 1))):
            pm.pmrc_set_plan_policy(st.code, policy)
            out = torch.full((stripes, st.alpha, S), 0x3C, dtype=torch.uint8, device=DEV)
            l0 = pm.pmrc_launch_count()
            pm.pmrc_repair_batch(st.code, [f for f, _ in reps], [list(reversed(H)) for _, H in reps], nodes,
                                 (out.data_ptr(), st.alpha * S), S, stripes, st.stream)
            torch.cuda.synchronize()
            assert pm.pmrc_launch_count() - l0 == launches[0], policy   # A x2 runs + C, then B
            for t, (f, _) in enumerate(reps):
                assert torch.equal(out[t], st.piece_tensor(f)[t]), (policy, t, f)
            dec = torch.full_like(st.data, 0xA5)
            l0 = pm.pmrc_launch_count()
            nw = pm.pmrc_decode_batch(st.code, decs, nodes, dec.data_ptr(), S, stripes, st.stream)
            torch.cuda.synchronize()
            assert pm.pmrc_launch_count() - l0 == launches[1], policy   # da x2 runs + dc, then db
            for t, ids in enumerate(decs):
                miss = _missing(st, ids)
                keep = [b for b in range(st.B) if b not in miss]
                assert nw[t] == len(miss)
                assert torch.equal(dec[t, miss], st.data[t, miss]), (policy, t)
                assert bool((dec[t, keep] == 0xA5).all()), (policy, t)
    finally:
        st.close()


def test_auto_promotion_of_a_hot_pattern(tmp_path, monkeypatch):
    # AUTO: a pattern past the promotion threshold is compiled in a host thread while its calls keep
    # running on the runtime kernel; a later call loads the generated kernel (bit-exact either way)
    monkeypatch.setenv("PMRC_KCACHE", str(tmp_path))        # empty cache: the promotion compiles
    k, n, S, stripes = 4, 8, 64 * 1024, 2
    st = Stripes(pm.PMRC_MSR_SPARSE, k, n, S, stripes, seed=23)
    try:
        st.encode()
        assert np.array_equal(st.parity.cpu().numpy(), O.encode(O.MSR_SPARSE, n, k, st.d, st.host_data()))
        pm.pmrc_set_auto_promotion(st.code, 1 << 20)       # 1 MiB of plan traffic
        f, H = 7, [0, 1, 2, 3, 4, 5]
        cold = (5, [0, 1, 2, 3, 4, 6])
        assert pm.pmrc_plan_state(st.code, 1, f, H) == pm.PLAN_RUNTIME_ONLY
        out = torch.zeros((stripes, st.alpha, S), dtype=torch.uint8, device=DEV)
        states = []
        t0 = time.time()
        while True:
            out.zero_()
            pm.pmrc_repair(st.code, f, list(reversed(H)), [st.piece(i) for i in reversed(H)],
                           (out.data_ptr(), st.alpha * S), S, stripes, st.stream)
            torch.cuda.synchronize()
            assert torch.equal(out, st.piece_tensor(f)), states
            states.append(pm.pmrc_plan_state(st.code, 1, f, H))
            if states[-1] == pm.PLAN_LOADED or time.time() - t0 > 300:
                break
            time.sleep(0.05)
        assert states[0] in (pm.PLAN_COMPILING, pm.PLAN_COMPILED), states   # promoted after the first call
        assert states[-1] == pm.PLAN_LOADED, states
        # a pattern below the threshold stays on the runtime kernel
        pm.pmrc_set_auto_promotion(st.code, 1 << 40)
        pm.pmrc_repair(st.code, cold[0], cold[1], [st.piece(i) for i in cold[1]], (out.data_ptr(), st.alpha * S), S,
                       stripes, st.stream)
        torch.cuda.synchronize()
        assert torch.equal(out, st.piece_tensor(cold[0]))
        assert pm.pmrc_plan_state(st.code, 1, cold[0], cold[1]) == pm.PLAN_RUNTIME_ONLY
    finally:
        st.close()
