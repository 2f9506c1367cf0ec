"""The runtime-coefficient kernel's GF(2^8) multiply formulation (csrc/rt/rlc.cu), emulated on the
CPU and pinned to the oracle's field (log/exp tables, 0x11D): for every coefficient c and byte x,
  c*x = T0[x & 7] ^ T1[(x >> 3) & 7] ^ T2[x >> 6]      (T0[j] = c*j, T1[j] = c*(j<<3), T2[j] = c*(j<<6))
with each lookup done by a byte permute (PRMT) whose selector nibbles come from u + (u >> 12),
u = the masked bit field of each byte, which leaves the 4 products in byte order (0, 2, 1, 3);
PRMT(acc, 0, 0x3120) restores the order.  A wrong shift, mask, table index or permutation fails
here for some (c, x)."""
import numpy as np

import oracle as O


def prmt(a, b, s):
    """PTX prmt.b32 (default mode) on numpy uint32 arrays: byte i of the result is byte
    ((s >> 4i) & 7) of the 8-byte value b:a (bit 3 of a selector nibble = sign mode, never set)."""
    a, b, s = (np.asarray(v, dtype=np.uint64) for v in (a, b, s))
    src = a | (b << np.uint64(32))
    out = np.zeros(np.broadcast(a, b, s).shape, dtype=np.uint64)
    for i in range(4):
        nib = (s >> np.uint64(4 * i)) & np.uint64(0xF)
        assert not np.any(nib & np.uint64(8)), "sign-mode bit set in a selector"
        byte = (src >> (np.uint64(8) * (nib & np.uint64(7)))) & np.uint64(0xFF)
        out |= byte << np.uint64(8 * i)
    return out.astype(np.uint32)


def madhi(a, b, c):
    """mad.hi.u32: ((a * b) >> 32) + c (mod 2^32)."""
    a, b, c = (np.asarray(v, dtype=np.uint64) for v in (a, b, c))
    return ((((a * b) >> np.uint64(32)) + c) & np.uint64(0xFFFFFFFF)).astype(np.uint32)


def selectors(w):
    u0 = w & np.uint32(0x07070707)
    s0 = madhi(u0, 1 << 20, u0)
    u1 = madhi(w, 1 << 29, 0) & np.uint32(0x07070707)
    s1 = madhi(u1, 1 << 20, u1)
    u2 = madhi(w, 1 << 26, 0) & np.uint32(0x03030303)
    s2 = madhi(u2, 1 << 20, u2)
    return s0, s1, s2


def pack(bs):
    return int(bs[0]) | (int(bs[1]) << 8) | (int(bs[2]) << 16) | (int(bs[3]) << 24)


def tables(c):
    t0 = [O.gf_mul(c, j) for j in range(8)]
    t1 = [O.gf_mul(c, j << 3) for j in range(8)]
    t2 = [O.gf_mul(c, j << 6) for j in range(4)]
    return pack(t0), pack(t0[4:]), pack(t1), pack(t1[4:]), pack(t2)


def test_prmt_formulation_every_coefficient_and_byte():
    # words holding every byte value at every byte position (64 words x 4 positions x 4 rotations)
    xs = np.arange(256, dtype=np.uint32)
    words = []
    for rot in range(4):
        b = [np.roll(xs, 64 * ((rot + i) % 4)) for i in range(4)]
        words.append(b[0] | (b[1] << 8) | (b[2] << 16) | (b[3] << 24))
    w = np.concatenate(words).astype(np.uint32)
    s0, s1, s2 = selectors(w)
    mul = np.array([[O.gf_mul(c, x) for x in range(256)] for c in range(256)], dtype=np.uint8)
    for c in range(256):
        t0a, t0b, t1a, t1b, t2 = tables(c)
        acc = prmt(t0a, t0b, s0) ^ prmt(t1a, t1b, s1) ^ prmt(t2, t2, s2)
        got = prmt(acc, 0, 0x3120)
        want = np.zeros_like(w)
        for i in range(4):
            want |= mul[c][(w >> np.uint32(8 * i)) & np.uint32(0xFF)].astype(np.uint32) << np.uint32(8 * i)
        assert np.array_equal(got, want), c


def test_selector_permutation_is_fixed():
    # the products come out in byte order (0, 2, 1, 3) whatever the word: with the identity table
    # c = 1 the permuted word is the input with bytes 1 and 2 swapped, and 0x3120 is an involution
    rnd = np.random.default_rng(3).integers(0, 2 ** 32, size=4096, dtype=np.uint64).astype(np.uint32)
    s0, s1, s2 = selectors(rnd)
    t0a, t0b, t1a, t1b, t2 = tables(1)
    acc = prmt(t0a, t0b, s0) ^ prmt(t1a, t1b, s1) ^ prmt(t2, t2, s2)
    assert np.array_equal(acc, prmt(rnd, 0, 0x3120))
    assert np.array_equal(prmt(prmt(rnd, 0, 0x3120), 0, 0x3120), rnd)
