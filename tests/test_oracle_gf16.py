"""CPU tier: pins of the GF(2^16) oracle (oracle/gf16.py, the w = 16 extension)."""
import itertools
import random

import numpy as np
import pytest

import inputs
import oracle.gf16 as G16


def _clmul16(a, b):
    r = 0
    for i in range(16):
        if (b >> i) & 1:
            r ^= a << i
    for bit in range(30, 15, -1):
        if (r >> bit) & 1:
            r ^= 0x1100B << (bit - 16)
    return r


def test_field_vs_carryless():
    rnd = random.Random(3)
    for _ in range(3000):
        a, b = rnd.randrange(65536), rnd.randrange(65536)
        assert int(G16.mul(a, b)) == _clmul16(a, b)


@pytest.mark.parametrize("k,n", [(3, 5), (4, 7), (4, 8), (8, 16)])
def test_systematic_prefix_and_sparsity(k, n):
    # G' = G Gtilde^-1 starts with I_B; the sparse construction keeps (k-2)/k zeros in
    # the systematic parity part (Table 1's "sparse sys" column) in GF(2^16) too
    a, B = k - 1, k * (k - 1)
    Gs = G16.systematic(n, k)
    assert (Gs[:B] == np.eye(B, dtype=np.int64)).all()
    Gpp = Gs[k * a:]
    assert (Gpp == 0).mean() == pytest.approx((k - 2) / k)
    assert all((row != 0).sum() == 2 * k - 2 for row in Gpp)     # d nonzeros per row


@pytest.mark.parametrize("k,n", [(3, 6), (4, 8)])
def test_linear_equals_specific_and_precode(k, n):
    # the linearised G Z equals the specific PM encode Psi M(Z) (different algorithm);
    # the systematic encode G'' X equals the specific encode of the precoded Z = Gtilde^-1 X
    a, B = k - 1, k * (k - 1)
    rng = np.random.default_rng(k)
    Z = rng.integers(0, 65536, (B, 12))
    G = G16.generator(n, k)
    assert (G16.mat_mul(G, Z) == G16.encode_specific(n, k, Z)).all()
    X = rng.integers(0, 65536, (B, 12))
    Zp = G16.mat_mul(G16.mat_inv(G[:B]), X)
    par = G16.symbols(G16.encode(n, k, G16.to_bytes(X)[None]))[0]
    assert (par == G16.encode_specific(n, k, Zp)[k * a:]).all()
    assert (G16.encode_specific(n, k, Zp)[:k * a] == X).all()   # systematic nodes hold X


def test_decode_every_k_subset_k3():
    # any k nodes recover the data (k = 3, n = 6, every 3-subset of nodes)
    k, n = 3, 6
    a, B = 2, 6
    Gs = G16.systematic(n, k)
    X = np.random.default_rng(1).integers(0, 65536, (B, 5))
    Y = G16.mat_mul(Gs, X)
    for ids in itertools.combinations(range(n), k):
        rows = [i * a + j for i in ids for j in range(a)]
        assert (G16.mat_mul(G16.mat_inv(Gs[rows]), Y[rows]) == X).all(), ids


def test_bytes_roundtrip_little_endian():
    x = inputs.stripe_data(1, 3, 64, seed=2)
    assert (G16.to_bytes(G16.symbols(x)) == x).all()
    assert G16.symbols(np.array([[0x34, 0x12]], np.uint8))[0, 0] == 0x1234
