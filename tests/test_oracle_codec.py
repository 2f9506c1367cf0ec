"""Pins of the oracle's data path (oracle/pmrc_oracle.c: or_encode, or_encode_specific,
or_decode_linear, or_decode_*_specific, or_repair*) by cross-paths the paper states are
equivalent, round trips, the exact-repair property, closed-form
singular sets, the read accounting of P:209 and brute force at k = 2."""
import itertools
import os

import numpy as np
import pytest

import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
rng = np.random.default_rng(2024)


def _rand(*shape):
    return rng.integers(0, 256, shape, dtype=np.uint8)


def _d(kind, k):
    return k if kind == O.RS else 2 * k - 2


@pytest.mark.parametrize("kind,k,n", [(O.MSR_SPARSE, 3, 6), (O.MSR_VANILLA, 3, 6), (O.MSR_SPARSE, 4, 8),
                                      (O.MSR_SPARSE, 8, 16), (O.MSR_VANILLA, 8, 16), (O.MBR, 3, 6),
                                      (O.MBR, 8, 16), (O.RS, 8, 16)])
def test_linear_equals_specific_nonsystematic(kind, k, n):
    # the linearised generator G reproduces C = Psi M, for every construction
    d = _d(kind, k)
    alpha, B = O.params(kind, n, k, d)
    X = _rand(B, 40)
    assert (O.apply(O.generator(kind, n, k, d), X) == O.encode_specific(kind, n, k, d, X)).all()


@pytest.mark.parametrize("kind,k,n", [(O.MSR_SPARSE, 3, 6), (O.MSR_VANILLA, 3, 6), (O.MSR_SPARSE, 4, 8),
                                      (O.MSR_SPARSE, 8, 16), (O.MSR_VANILLA, 8, 16), (O.MSR_SPARSE, 8, 15)])
def test_systematic_linear_equals_precode_then_encode(kind, k, n):
    # systematic = decode X with the specific MSR decoder applied to the first k
    # nodes, then encode Z with C = Psi M(Z).  Must equal the linearised G'' X bit-exactly,
    # and the first k nodes of Psi M(Z) must give back X (systematic prefix).
    d = 2 * k - 2
    alpha, B = O.params(kind, n, k, d)
    S = 33
    X = _rand(B, S)
    Z = O.decode_msr_specific_Z(kind, n, k, d, list(range(k)), X.reshape(k, alpha, S))
    C = O.encode_specific(kind, n, k, d, Z)
    assert (C[:B] == X).all()
    assert (C[B:] == O.encode(kind, n, k, d, X[None])[0]).all()
    # and Z is Gtilde^{-1} X (the linear-algebra form of the same precoding)
    G = O.generator(kind, n, k, d)
    assert (O.apply(O.mat_inv(G[:B]), X) == Z).all()


@pytest.mark.parametrize("kind,k,n", [(O.MSR_SPARSE, 8, 16), (O.MBR, 8, 16), (O.RS, 8, 16), (O.MSR_VANILLA, 4, 8)])
def test_sparse_skipping_equals_dense(kind, k, n):
    # north star: the sparsified (zero-skipping) and dense products give identical codewords
    d = _d(kind, k)
    alpha, B = O.params(kind, n, k, d)
    X = _rand(B, 64)
    G2 = O.parity_matrix(kind, n, k, d)
    assert (O.apply(G2, X, skip_zeros=True) == O.apply(G2, X, skip_zeros=False)).all()


def test_encode_gf_linearity():
    k, n, d = 8, 16, 14
    alpha, B = O.params(O.MSR_SPARSE, n, k, d)
    X, Y = _rand(3, B, 20), _rand(3, B, 20)
    a = 0x53
    aX = np.vectorize(lambda v: O.gf_mul(a, int(v)), otypes=[np.uint8])(X)
    lhs = O.encode(O.MSR_SPARSE, n, k, d, aX ^ Y)
    EX = O.encode(O.MSR_SPARSE, n, k, d, X)
    rhs = np.vectorize(lambda v: O.gf_mul(a, int(v)), otypes=[np.uint8])(EX) ^ O.encode(O.MSR_SPARSE, n, k, d, Y)
    assert (lhs == rhs).all()
    assert not O.encode(O.MSR_SPARSE, n, k, d, np.zeros((1, B, 8), np.uint8)).any()


@pytest.mark.parametrize("kind,k,n", [(O.MSR_SPARSE, 3, 6), (O.MSR_VANILLA, 3, 6), (O.MBR, 3, 6),
                                      (O.MSR_SPARSE, 4, 8), (O.MBR, 4, 8), (O.RS, 4, 8), (O.MSR_N2K, 4, 8)])
def test_decode_every_k_subset(kind, k, n):
    # any k nodes recover the data; exhaustive over all k-subsets (and all larger sets at k=3)
    d = _d(kind, k)
    alpha, B = O.params(kind, n, k, d)
    X = _rand(B, 24)
    code = O.full_code(kind, n, k, d, X)
    for r in range(k, n + 1 if k == 3 else k + 1):
        for ids in itertools.combinations(range(n), r):
            got = O.decode_linear(kind, n, k, d, list(ids), code[list(ids)])
            assert (got == X).all(), ids


def test_decode_k8_sampled_and_underdetermined():
    for kind in (O.MSR_SPARSE, O.MBR):
        k, n = 8, 16
        d = 14
        alpha, B = O.params(kind, n, k, d)
        X = _rand(B, 16)
        code = O.full_code(kind, n, k, d, X)
        r = np.random.default_rng(7)
        for _ in range(40):
            ids = sorted(r.choice(n, k, replace=False).tolist())
            assert (O.decode_linear(kind, n, k, d, ids, code[ids]) == X).all()
        with pytest.raises(O.OracleError) as e:
            O.decode_linear(kind, n, k, d, list(range(k - 1)), code[: k - 1])
        assert e.value.rc == O.ESING


@pytest.mark.parametrize("kind,k,n,trials", [(O.MSR_SPARSE, 3, 6, None), (O.MSR_VANILLA, 3, 6, None),
                                             (O.MSR_SPARSE, 4, 8, None), (O.MSR_SPARSE, 8, 16, 60),
                                             (O.MSR_VANILLA, 8, 16, 30)])
def test_specific_msr_decode_equals_linear(kind, k, n, trials):
    # "decoding method is independent of the encoding method" -- the specific MSR decoder
    # on linear-encoded stripes returns Z; the data is the first k nodes of Psi M(Z)
    d = 2 * k - 2
    alpha, B = O.params(kind, n, k, d)
    X = _rand(B, 12)
    code = O.full_code(kind, n, k, d, X)
    subsets = list(itertools.combinations(range(n), k))
    if trials:
        idx = np.random.default_rng(3).choice(len(subsets), trials, replace=False)
        subsets = [subsets[i] for i in idx]
    for ids in subsets:
        Z = O.decode_msr_specific_Z(kind, n, k, d, list(ids), code[list(ids)])
        assert (O.encode_specific(kind, n, k, d, Z)[:B] == X).all(), ids


@pytest.mark.parametrize("k,d,n,trials", [(3, 4, 6, None), (4, 6, 8, None), (8, 14, 16, 60)])
def test_specific_mbr_decode_equals_data(k, d, n, trials):
    alpha, B = O.params(O.MBR, n, k, d)
    X = _rand(B, 12)
    code = O.full_code(O.MBR, n, k, d, X)
    subsets = list(itertools.combinations(range(n), k))
    if trials:
        idx = np.random.default_rng(4).choice(len(subsets), trials, replace=False)
        subsets = [subsets[i] for i in idx]
    for ids in subsets:
        assert (O.decode_mbr_specific(n, k, d, list(ids), code[list(ids)]) == X).all(), ids


def _sparse_n2k_singular(k, f, H, n):
    # R10 closed form (SURVEY §8c-A7 proof): at n = 2k, Psi_H is singular iff the lost node is an
    # identity node (f < alpha) and the helper set omits another identity node (so it holds all
    # n - alpha Cauchy nodes)
    alpha = k - 1
    omitted = [i for i in range(n) if i != f and i not in H]
    return f < alpha and len(omitted) == 1 and omitted[0] < alpha


@pytest.mark.parametrize("kind,k,n", [(O.MSR_SPARSE, 3, 6), (O.MSR_VANILLA, 3, 6), (O.MSR_SPARSE, 4, 8),
                                      (O.MSR_SPARSE, 3, 5), (O.MBR, 3, 6), (O.MBR, 4, 8),
                                      (O.MSR_N2K, 3, 6), (O.MSR_N2K, 4, 8)])
def test_repair_every_node_every_helper_set(kind, k, n):
    # exact repair (P:53 fn): every lost node from every d-helper subset regenerates the
    # lost piece bit-exactly, except the predicted singular sets of the sparse code at n = 2k (R10)
    d = 2 * k - 2
    alpha, B = O.params(kind, n, k, d)
    X = _rand(B, 20)
    code = O.full_code(kind, n, k, d, X)
    n_sing = 0
    for f in range(n):
        others = [i for i in range(n) if i != f]
        for H in itertools.combinations(others, d):
            H = list(H)
            predicted = kind == O.MSR_SPARSE and n == 2 * k and _sparse_n2k_singular(k, f, H, n)
            try:
                got = O.repair(kind, n, k, d, f, H, code[H])
            except O.OracleError as e:
                assert e.rc == O.ESING and predicted, (f, H)
                n_sing += 1
                continue
            assert not predicted, (f, H)
            assert (got == code[f]).all(), (f, H)
    if kind == O.MSR_SPARSE and n == 2 * k:
        assert n_sing == (k - 1) * (k - 2)   # alpha (alpha-1): 2/30 at k=3, 6/56 at k=4
    else:
        assert n_sing == 0


def test_repair_k8_sampled_and_singular_fraction():
    k, n, d = 8, 16, 14
    alpha, B = O.params(O.MSR_SPARSE, n, k, d)
    X = _rand(B, 8)
    code = O.full_code(O.MSR_SPARSE, n, k, d, X)
    n_sing = 0
    for f in range(n):
        others = [i for i in range(n) if i != f]
        for omit in others:
            H = [i for i in others if i != omit]
            pred = _sparse_n2k_singular(k, f, H, n)
            try:
                got = O.repair(O.MSR_SPARSE, n, k, d, f, H, code[H])
                assert not pred and (got == code[f]).all()
            except O.OracleError as e:
                assert pred and e.rc == O.ESING
                n_sing += 1
    assert n_sing == 42   # 42 / 240 = 17.5 % of (f, H) pairs at k = 8, n = 16


def test_repair_rs_and_mbr_k8():
    X = _rand(84, 8)
    code = O.full_code(O.MBR, 16, 8, 14, X)
    r = np.random.default_rng(11)
    for _ in range(20):
        f = int(r.integers(16))
        others = [i for i in range(16) if i != f]
        H = sorted(r.choice(others, 14, replace=False).tolist())
        assert (O.repair(O.MBR, 16, 8, 14, f, H, code[H]) == code[f]).all()
    Xr = _rand(8, 8)
    coder = O.full_code(O.RS, 16, 8, 8, Xr)
    for f in range(16):
        H = [i for i in range(16) if i != f][:8]
        assert (O.repair(O.RS, 16, 8, 8, f, H, coder[H]) == coder[f]).all()


def test_read_accounting_paper():
    # helpers read 1 block for a failure of the alpha first nodes and alpha blocks otherwise;
    # the average reduction (k-2)/(2k-2) gives 43% at k=8 and 33% at k=4 (n = 2k-1)
    claims = {}
    for line in open(os.path.join(HERE, "golden", "claims.txt")):
        if not line.startswith("#") and line.strip():
            a, b = line.split()
            claims[a] = int(b)
    for k, key in ((8, "read_reduction_k8_percent"), (4, "read_reduction_k4_percent")):
        d, n, alpha = 2 * k - 2, 2 * k - 1, k - 1
        reads = [O.repair_reads(O.MSR_SPARSE, n, k, d, f) for f in range(n)]
        assert reads == [1] * alpha + [alpha] * (n - alpha)
        saved = sum(alpha - r for r in reads)
        # the paper's average: per-node saving averaged over d = 2k-2 nodes (R10b)
        assert round(100 * saved / (alpha * d)) == claims[key]
        assert [O.repair_reads(O.MSR_VANILLA, n, k, d, f) for f in range(n)] == [alpha] * n


def test_repair_projection_reads_only_nonzero_blocks():
    # the helper's beta depends only on the blocks with nonzero phi_f: poison the others
    k, n, d = 8, 16, 14
    alpha = 7
    piece = _rand(alpha, 32)
    for f in range(n):
        mu = O.repair_mu(O.MSR_SPARSE, n, k, d, f)
        p2 = piece.copy()
        p2[mu == 0] ^= 0xA5
        assert (O.repair_project(O.MSR_SPARSE, n, k, d, f, piece) ==
                O.repair_project(O.MSR_SPARSE, n, k, d, f, p2)).all()


@pytest.mark.parametrize("kind,n", [(O.MSR_SPARSE, 3), (O.MSR_SPARSE, 4), (O.MSR_VANILLA, 3), (O.MSR_VANILLA, 4)])
def test_bruteforce_k2(kind, n):
    # k = 2: alpha = 1, d = 2, B = 2.  Blocks of 65,536 bytes hold every (x1, x2) pair once, so one
    # call enumerates the whole message space: every 2-node projection must be injective and decode
    # must invert it; every repair must regenerate the lost byte.
    k, d = 2, 2
    a = np.arange(65536, dtype=np.uint32)
    X = np.stack([(a & 0xFF).astype(np.uint8), (a >> 8).astype(np.uint8)])
    code = O.full_code(kind, n, k, d, X)
    for ids in itertools.combinations(range(n), 2):
        pair = code[list(ids), 0].astype(np.uint32)
        assert len(np.unique(pair[0] | (pair[1] << 8))) == 65536
        assert (O.decode_linear(kind, n, k, d, list(ids), code[list(ids)]) == X).all()
    for f in range(n):
        for H in itertools.combinations([i for i in range(n) if i != f], d):
            assert (O.repair(kind, n, k, d, f, list(H), code[list(H)]) == code[f]).all()


def test_n2k_extension_repairs_the_paper_singular_sets_at_k8():
    # R15 (extension): with the greedy Lambda every (f, H) pair repairs exactly at k = 8, n = 16,
    # including the 42 pairs that are singular for the paper's construction (R10)
    k, n, d = 8, 16, 14
    alpha, B = O.params(O.MSR_N2K, n, k, d)
    X = _rand(B, 8)
    code = O.full_code(O.MSR_N2K, n, k, d, X)
    was_singular = 0
    for f in range(n):
        others = [i for i in range(n) if i != f]
        for omit in others:
            H = [i for i in others if i != omit]
            was_singular += _sparse_n2k_singular(k, f, H, n)
            got = O.repair(O.MSR_N2K, n, k, d, f, H, code[H])
            assert (got == code[f]).all(), (f, H)
    assert was_singular == 42
