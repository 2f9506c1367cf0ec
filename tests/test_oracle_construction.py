"""Pins of the oracle's code construction (oracle/pmrc_oracle.c: or_index_matrix, or_psi,
or_generator, or_systematic, or_validate) against PAPER.md's printed examples, Table 1, the
validity range of P:189 and closed forms derived from the constructions."""
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
import gfref

HERE = os.path.dirname(os.path.abspath(__file__))


def _golden_rows(name):
    rows = []
    for line in open(os.path.join(HERE, "golden", name)):
        if line.startswith("#") or not line.strip():
            continue
        rows.append(line.split())
    return rows


def test_index_matrix_msr_k3_paper():
    # P:77-83
    want = np.array(_golden_rows("index_matrix_msr_k3.txt"), np.int32)
    assert (O.index_matrix(O.MSR_SPARSE, 3, 4) == want).all()


def test_index_matrix_mbr_k3_spec():
    want = np.array(_golden_rows("index_matrix_mbr_k3_d4.txt"), np.int32)
    assert (O.index_matrix(O.MBR, 3, 4) == want).all()


@pytest.mark.parametrize("k", [2, 3, 4, 5, 8, 16])
def test_index_matrix_msr_invariants(k):
    d = 2 * k - 2
    alpha, B = O.params(O.MSR_SPARSE, d + 1, k, d)
    L = O.index_matrix(O.MSR_SPARSE, k, d)
    S1, S2 = L[:alpha], L[alpha:]
    assert (S1 == S1.T).all() and (S2 == S2.T).all()          # north star: [S1;S2] symmetric
    assert sorted(set(L.flatten())) == list(range(1, B + 1))  # every data symbol once per S
    for j in range(alpha):                                     # no duplicate in a column
        assert len(set(L[:, j])) == d
    for i in range(d):                                         # ... nor in a row
        assert len(set(L[i])) == alpha


@pytest.mark.parametrize("k,d", [(2, 2), (3, 4), (4, 6), (8, 14), (5, 9)])
def test_index_matrix_mbr_invariants(k, d):
    alpha, B = O.params(O.MBR, d + 1, k, d)
    assert B == k * (2 * d - k + 1) // 2
    L = O.index_matrix(O.MBR, k, d)
    assert (L == L.T).all()                                    # north star: [[S,T],[T^t,0]]
    assert (L[k:, k:] == 0).all()
    assert sorted(set(L.flatten()) - {0}) == list(range(1, B + 1))
    for j in range(d):
        col = [v for v in L[:, j] if v]
        assert len(col) == len(set(col))


def test_params_paper():
    # (5,3,4,MSR) -> alpha 2, B 6; (5,3,4,MBR) -> alpha 4, B 9
    assert O.params(O.MSR_SPARSE, 5, 3, 4) == (2, 6)
    assert O.params(O.MBR, 5, 3, 4) == (4, 9)
    assert O.params(O.MSR_SPARSE, 16, 8, 14) == (7, 56)
    assert O.params(O.MBR, 16, 8, 14) == (14, 84)
    with pytest.raises(O.OracleError):
        O.params(O.MSR_SPARSE, 6, 3, 3)  # MSR needs d = 2k-2


def test_vanilla_psi_paper_display():
    # P:135-157, n=5 k=3 d=4 alpha=2: Psi_{i,j} = g^{(i-1)(j-1)}, Lambda = diag(1, g^2, g^4, g^6, g^8)
    P, lam = O.psi(O.MSR_VANILLA, 5, 3, 4)
    for i in range(5):
        for j in range(4):
            assert P[i, j] == gfref.gexp(i * j)
    assert [int(x) for x in lam] == [gfref.gexp(e) for e in (0, 2, 4, 6, 8)]


def test_sparse_psi_paper_display():
    # P:168-186, n=5 k=3 d=4 alpha=2 (1-based i, R2):
    #   Phi rows 1,2 = I;  Phi_{i,j} = 1/(g^{2 alpha + (i-2)} - g^{j-1}) for rows i = 3..5 as displayed
    #   Lambda_ii = (g^{i+alpha} - g^0)/(g^{i+alpha} - g^alpha);  Psi = [Phi  Lambda Phi]
    a = 2
    P, lam = O.psi(O.MSR_SPARSE, 5, 3, 4)
    g = gfref
    assert list(P[0, :2]) == [1, 0] and list(P[1, :2]) == [0, 1]
    for row, e in ((2, 2 * a + 1), (3, 2 * a + 2), (4, 2 * a + 3)):
        for j in range(2):
            assert P[row, j] == g.inv(g.gexp(e) ^ g.gexp(j))
    exps = [a + 1, a + 2, 2 * a + 1, 2 * a + 2, 2 * a + 3]   # the displayed Lambda numerators
    for i, e in enumerate(exps):
        want = g.mul(g.gexp(e) ^ 1, g.inv(g.gexp(e) ^ g.gexp(a)))
        assert lam[i] == want
        for j in range(2):
            assert P[i, a + j] == g.mul(want, int(P[i, j]))


def _sparsity(M):
    return Fraction(int((M == 0).sum()), M.size)


def test_table1_sparsity():
    # PAPER.md Table 1, n = 2k-1, d = 2k-2
    rows = {r[0]: [int(x) for x in r[1:]] for r in _golden_rows("table1_sparsity.txt")}
    for col, k in enumerate((4, 8, 16)):
        n, d = 2 * k - 1, 2 * k - 2
        got = {
            "vanilla_nonsys": _sparsity(O.generator(O.MSR_VANILLA, n, k, d)),
            "sparse_nonsys": _sparsity(O.generator(O.MSR_SPARSE, n, k, d)),
            "vanilla_sys": _sparsity(O.parity_matrix(O.MSR_VANILLA, n, k, d)),
            "sparse_sys": _sparsity(O.parity_matrix(O.MSR_SPARSE, n, k, d)),
        }
        for name, frac in got.items():
            assert abs(float(frac) * 100 - rows[name][col]) <= 0.5, (name, k, float(frac) * 100)
        alpha = k - 1
        # closed forms (derived from the constructions):
        assert got["vanilla_nonsys"] == 1 - Fraction(d, k * alpha)         # d nonzeros per row
        nnz_sparse = 2 * alpha * alpha + (n - alpha) * alpha * d              # identity rows: 2 each
        assert got["sparse_nonsys"] == 1 - Fraction(nnz_sparse, n * alpha * k * alpha)
        assert got["sparse_sys"] == Fraction(k - 2, k)                     # exactly d nonzeros per row


@pytest.mark.parametrize("k,n", [(3, 5), (3, 6), (4, 8), (8, 15), (8, 16), (16, 32)])
def test_sparse_sys_rows_have_d_nonzeros_and_group_support(k, n):
    # every row of the sparse systematic G'' has exactly d nonzeros, and the parity rows of PM symbol
    # j all read the same d inputs: data column j across the systematic nodes plus the other symbols
    # of identity node j (the group structure the kernel exploits)
    d = 2 * k - 2
    alpha = k - 1
    G2 = O.parity_matrix(O.MSR_SPARSE, n, k, d)
    for r in range(G2.shape[0]):
        assert (G2[r] != 0).sum() == d
    for j in range(alpha):
        want = {s * alpha + j for s in range(k)} | {j * alpha + t for t in range(alpha)}
        for p in range(n - k):
            assert set(np.nonzero(G2[p * alpha + j])[0]) == want


def test_mbr_parity_nnz_closed_form():
    # MBR G'' = parity rows of G (R6); Cauchy rows are dense, so row (i,j) has as many nonzeros as
    # column j of L has nonzero entries: d for j <= k, k for j > k.
    for k, d, n in ((3, 4, 6), (4, 6, 8), (8, 14, 16)):
        G2 = O.parity_matrix(O.MBR, n, k, d)
        assert int((G2 != 0).sum()) == (n - k) * (k * d + (d - k) * k)
    assert int((O.parity_matrix(O.MBR, 16, 8, 14) != 0).sum()) == 1280


@pytest.mark.parametrize("kind", [O.MSR_SPARSE, O.MSR_VANILLA, O.RS])
def test_systematic_prefix(kind):
    # G' = G Gtilde^{-1} has the identity on top
    for k, n in ((3, 6), (4, 8), (8, 16)):
        d = k if kind == O.RS else 2 * k - 2
        alpha, B = O.params(kind, n, k, d)
        Gp = O.systematic(kind, n, k, d)
        assert (Gp[:B] == np.eye(B, dtype=np.uint8)).all()


def test_mbr_systematic_rows_are_unit():
    # R5/R6: Psi = [I_k 0; Psi''] makes the systematic rows of G unit rows e_{L_{i,j}}
    k, d, n = 8, 14, 16
    G = O.generator(O.MBR, n, k, d)
    L = O.index_matrix(O.MBR, k, d)
    alpha = d
    for i in range(k):
        for j in range(alpha):
            row = G[i * alpha + j]
            assert (row != 0).sum() == 1 and row[L[i, j] - 1] == 1


def test_validity_range_paper():
    # valid for k in {2..39} in GF(2^8) (Lambda distinct and all n d x d submatrices of Psi
    # invertible, n = d+1), and the construction is claimed only up to 39: k = 40 fails.
    claims = {r[0]: int(r[1]) for r in _golden_rows("claims.txt")}
    for k in range(claims["valid_k_min"], claims["valid_k_max"] + 1):
        d = 2 * k - 2
        flags, _ = O.validate(O.MSR_SPARSE, d + 1, k, d, check_phi=False)
        assert flags == 0, k
    flags, _ = O.validate(O.MSR_SPARSE, 79, 40, 78, check_phi=False)
    assert flags & 2


@pytest.mark.parametrize("k", [3, 4, 5])
def test_full_validation_small(k):
    # exhaustive version of the P:121-127 constraints at n = d+1 (both constructions) and MBR
    d = 2 * k - 2
    for kind in (O.MSR_SPARSE, O.MSR_VANILLA):
        flags, _ = O.validate(kind, d + 1, k, d)
        assert flags == 0
    flags, _ = O.validate(O.MBR, 2 * k, k, d)
    assert flags == 0


@pytest.mark.parametrize("k", [3, 4, 8])
def test_sparse_n2k_singular_d_subsets(k):
    # DESIGN.md R10: at n = 2k the Cauchy rows of Psi lie in an (alpha+1)-dim space,
    # so a d-subset with >= alpha+2 Cauchy rows is singular; with <= alpha+1 it is not.
    import itertools
    d, alpha, n = 2 * k - 2, k - 1, 2 * k
    P, _ = O.psi(O.MSR_SPARSE, n, k, d)
    cauchy = P[alpha:]
    assert O.mat_rank(cauchy) == alpha + 1
    for sub in itertools.combinations(range(n), d):
        nc = sum(1 for i in sub if i >= alpha)
        full = O.mat_rank(P[list(sub)]) == d
        assert full == (nc <= alpha + 1), sub


def test_vanilla_lambda_collision():
    # R8: vanilla lambda_i = g^{(i-1)alpha} collide iff n > 255/gcd(alpha,255): k=16 (alpha=15,
    # gcd 15) collides from n = 18 on, so Table 1's vanilla k=16 column is not a valid MSR code in
    # GF(2^8) even though its generator (and sparsity) is well defined.
    flags, _ = O.validate(O.MSR_VANILLA, 31, 16, 30, check_phi=False, max_subsets=100)
    assert flags & 1
    for k in (3, 4, 8, 15):
        d = 2 * k - 2
        flags, _ = O.validate(O.MSR_VANILLA, 2 * k, k, d, check_phi=False, max_subsets=10 ** 5)
        assert not flags & 1, k


@pytest.mark.parametrize("k", [3, 4, 8, 16])
def test_n2k_extension_valid_and_sparse(k):
    # R15 (extension, not the paper's): the sparse Phi = [I; Cauchy] with the greedy Lambda
    # passes the P:121-127 constraints at n = 2k by brute force over every d-row subset (the
    # paper's Lambda does not, R10), and keeps the systematic sparsity (k-2)/k of Table 1
    d, n = 2 * k - 2, 2 * k
    flags, _ = O.validate(O.MSR_N2K, n, k, d, check_phi=(k <= 8))
    assert flags == 0
    assert O.validate(O.MSR_SPARSE, n, k, d, check_phi=False)[0] & 2
    G2 = O.parity_matrix(O.MSR_N2K, n, k, d)
    assert (G2 == 0).mean() >= (k - 2) / k
    P, lam = O.psi(O.MSR_N2K, n, k, d)
    Ps, _ = O.psi(O.MSR_SPARSE, n, k, d)
    alpha = k - 1
    assert (P[:, :alpha] == Ps[:, :alpha]).all()        # same Phi as the paper's sparse code
    for i in range(n):                                     # Psi = [Phi  Lambda Phi]
        assert all(P[i, alpha + j] == O.gf_mul(lam[i], P[i, j]) for j in range(alpha))


def test_validity_range_gf16_paper():
    # "valid ... k in {2...64} in GF(2^16)" (GF-Complete's default field, R1 extended to
    # w = 16: polynomial 0x1100B, g = 2): Lambda distinct and all n d x d submatrices of the sparse
    # Psi invertible at n = d+1, for every k the paper checked
    for k in range(2, 65):
        assert O.validate16_sparse(k) == 0, k


@pytest.mark.parametrize("k", [2, 3, 4, 5, 8, 12])
def test_validity_gf16_negative_at_n2k(k):
    # negative pin of the GF(2^16) validity check (a check that always answered "valid" would pass
    # the test above): at n = 2k the sparse Psi's n - alpha = alpha + 2 Cauchy rows span only
    # alpha + 1 dimensions (SURVEY §8(c) A7 -- a field-independent rank argument), so exactly the
    # d-subsets that omit two identity rows (C(alpha, 2) of them, none for k = 2) are singular;
    # at n = 2k - 1 (the paper's n = d + 1) none is.
    from math import comb
    alpha = k - 1
    flags, sing = O.validate16_sparse_n(k, 2 * k)
    assert sing == comb(alpha, 2)
    assert bool(flags & 2) == (k >= 3)
    flags1, sing1 = O.validate16_sparse_n(k, 2 * k - 1)
    assert (flags1, sing1) == (0, 0) and O.validate16_sparse(k) == 0


def test_gf16_field_vs_carryless():
    # the w = 16 field the check above uses: products equal carry-less multiplication reduced by
    # 0x1100B (independent reference), and g = 2 generates all 65,535 nonzero elements
    import random

    def clmul16(a, b):
        r = 0
        for i in range(16):
            if (b >> i) & 1:
                r ^= a << i
        for bit in range(30, 15, -1):
            if (r >> bit) & 1:
                r ^= 0x1100B << (bit - 16)
        return r
    rnd = random.Random(16)
    for _ in range(5000):
        a, b = rnd.randrange(65536), rnd.randrange(65536)
        assert O.gf16_mul(a, b) == clmul16(a, b)
    x, seen = 1, set()
    for _ in range(65535):
        seen.add(x)
        x = clmul16(x, 2)
    assert len(seen) == 65535 and x == 1
