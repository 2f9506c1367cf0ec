"""Independent textbook GF(2^8) for the oracle pins: carry-less multiply then reduction by the
primitive polynomial x^8+x^4+x^3+x^2+1 (0x11D), inverse by exhaustive search.  Shares nothing
with oracle/ (which uses log/antilog tables) nor with the product."""

POLY = 0x11D


def clmul(a, b):
    r = 0
    for i in range(8):
        if (b >> i) & 1:
            r ^= a << i
    return r


def reduce(r):
    for bit in range(14, 7, -1):
        if (r >> bit) & 1:
            r ^= POLY << (bit - 8)
    return r


def mul(a, b):
    return reduce(clmul(a, b))


def power(a, e):
    r = 1
    for _ in range(e % 255):
        r = mul(r, a)
    return r


def inv(a):
    assert a != 0
    for x in range(1, 256):
        if mul(a, x) == 1:
            return x
    raise AssertionError


def gexp(e):
    """g^e with g = 2."""
    return power(2, e)
