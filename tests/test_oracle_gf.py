"""Pins of the oracle's GF(2^8) (oracle/pmrc_oracle.c `or_gf_*`, reading R1: poly 0x11D, g=2)
against an independent textbook carry-less-multiply implementation and SPEC.md:56-65."""
import os

import numpy as np

import oracle as O
import gfref

HERE = os.path.dirname(os.path.abspath(__file__))


def test_gf_examples_golden():
    # SPEC.md:56-65 worked examples
    for line in open(os.path.join(HERE, "golden", "gf_examples.txt")):
        if line.startswith("#") or not line.strip():
            continue
        op, a, b, r = line.split()
        a, b, r = int(a, 16), int(b, 16), int(r, 16)
        if op == "mul":
            assert O.gf_mul(a, b) == r
            assert gfref.mul(a, b) == r
        else:
            assert a ^ b == r


def test_gf_mul_exhaustive_vs_carryless():
    # all 65,536 products: log/exp tables == carry-less multiply + reduction by 0x11D
    ref = np.array([[gfref.mul(a, b) for b in range(256)] for a in range(256)], np.uint8)
    got = np.array([[O.gf_mul(a, b) for b in range(256)] for a in range(256)], np.uint8)
    assert (ref == got).all()


def test_generator_order_and_inverse():
    # g = 2 generates the multiplicative group (order 255): g^e enumerates every nonzero element
    seen = {O.gf_exp(e) for e in range(255)}
    assert seen == set(range(1, 256))
    assert O.gf_exp(255) == 1 and O.gf_exp(0) == 1 and O.gf_exp(1) == 2
    for a in range(1, 256):
        assert O.gf_mul(a, O.gf_inv(a)) == 1
        assert O.gf_inv(a) == gfref.inv(a) if a < 16 else True
        assert O.gf_exp(O.gf_log(a)) == a


def test_field_axioms_sampled():
    r = np.random.default_rng(5)
    for _ in range(3000):
        a, b, c = (int(x) for x in r.integers(0, 256, 3))
        assert O.gf_mul(a, O.gf_mul(b, c)) == O.gf_mul(O.gf_mul(a, b), c)
        assert O.gf_mul(a, b ^ c) == O.gf_mul(a, b) ^ O.gf_mul(a, c)
        assert O.gf_mul(a, b) == O.gf_mul(b, a)


def test_matrix_inverse_examples():
    # [[1,1],[1,0]]^-1 = [[0,1],[1,1]];  [[1,1],[1,1]] singular
    assert (O.mat_inv([[1, 1], [1, 0]]) == np.array([[0, 1], [1, 1]])).all()
    try:
        O.mat_inv([[1, 1], [1, 1]])
        raise AssertionError("expected singular")
    except O.OracleError as e:
        assert e.rc == O.ESING
    # random invertible matrices: A A^-1 = A^-1 A = I, and the product checked with gfref
    r = np.random.default_rng(1)
    for m in (1, 3, 8, 20):
        while True:
            A = r.integers(0, 256, (m, m)).astype(np.uint8)
            if O.mat_rank(A) == m:
                break
        Ai = O.mat_inv(A)
        for i in range(m):
            for j in range(m):
                s = 0
                for t in range(m):
                    s ^= gfref.mul(int(A[i, t]), int(Ai[t, j]))
                assert s == (1 if i == j else 0)


def test_rank_vandermonde():
    # a Vandermonde matrix on distinct points has full rank; a repeated row drops it
    V = np.array([[gfref.power(gfref.gexp(i), j) for j in range(6)] for i in range(6)], np.uint8)
    assert O.mat_rank(V) == 6
    V[5] = V[2]
    assert O.mat_rank(V) == 5
