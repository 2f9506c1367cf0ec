"""GF(2^16) oracle for the w = 16 extension (reading R1b: polynomial 0x1100B, g = 2).

TEST INFRASTRUCTURE ONLY (like the rest of oracle/): only tests/ may import it; the product never
calls it.  Plain numpy / Python, following the paper's formulas in its notation (1-based i, j):
the sparse PM-MSR Psi, the index matrix L (R4), the linearised generator G
(P:95-104), the systematic G' = G Gtilde^{-1} and its parity part G'', the encode
parity = G'' X on little-endian 16-bit symbols, and the specific encode
C = Psi M as an independent cross-path."""
import numpy as np

POLY = 0x1100B
_EXP = np.zeros(2 * 65535, np.int64)
_LOG = np.full(65536, -1, np.int64)
_x = 1
for _e in range(65535):
    _EXP[_e] = _x
    _LOG[_x] = _e
    _x <<= 1
    if _x & 0x10000:
        _x ^= POLY
_EXP[65535:] = _EXP[:65535]


def mul(a, b):
    """Elementwise GF(2^16) product of integer arrays / scalars."""
    a = np.asarray(a, np.int64)
    b = np.asarray(b, np.int64)
    out = _EXP[(_LOG[np.where(a == 0, 1, a)] + _LOG[np.where(b == 0, 1, b)]) % 65535]
    return np.where((a == 0) | (b == 0), 0, out)


def inv(a):
    return int(_EXP[(65535 - _LOG[a]) % 65535])


def gexp(e):
    return int(_EXP[e % 65535])


def psi_sparse(n, k):
    """x_i = g^{i+alpha}, y_j = g^{j-1}, Phi = [I; 1/(x_i - y_j)],
    Lambda_ii = (x_i - 1)/(x_i - g^alpha), Psi = [Phi  Lambda Phi] (n x d)."""
    a, d = k - 1, 2 * k - 2
    P = np.zeros((n, d), np.int64)
    lam = np.zeros(n, np.int64)
    for i in range(1, n + 1):
        x = gexp(i + a)
        lam[i - 1] = mul(x ^ 1, inv(x ^ gexp(a)))
        for j in range(1, a + 1):
            phi = int(i == j) if i <= a else inv(x ^ gexp(j - 1))
            P[i - 1, j - 1] = phi
            P[i - 1, a + j - 1] = mul(lam[i - 1], phi)
    return P, lam


def index_matrix(k):
    """P:75-83 / R4: M = [S1; S2] (d x alpha), symmetric blocks numbered row-major over the upper
    triangle, 1-based data indices."""
    a = k - 1
    L = np.zeros((2 * a, a), np.int64)
    v = 1
    for blk in range(2):
        for r in range(a):
            for c in range(r, a):
                L[blk * a + r, c] = L[blk * a + c, r] = v
                v += 1
    return L


def generator(n, k):
    """G_{alpha(i-1)+j, L_{l,j}} = Psi_{i,l}  ((n alpha) x B)."""
    a, d, B = k - 1, 2 * k - 2, k * (k - 1)
    P, _ = psi_sparse(n, k)
    L = index_matrix(k)
    G = np.zeros((n * a, B), np.int64)
    for i in range(n):
        for j in range(a):
            for l in range(d):
                G[i * a + j, L[l, j] - 1] = P[i, l]
    return G


def mat_inv(A):
    A = [list(map(int, r)) for r in A]
    m = len(A)
    Iv = [[int(i == j) for j in range(m)] for i in range(m)]
    for c in range(m):
        p = next(r for r in range(c, m) if A[r][c])
        A[c], A[p] = A[p], A[c]
        Iv[c], Iv[p] = Iv[p], Iv[c]
        s = inv(A[c][c])
        A[c] = [int(mul(v, s)) for v in A[c]]
        Iv[c] = [int(mul(v, s)) for v in Iv[c]]
        for r in range(m):
            if r != c and A[r][c]:
                f = A[r][c]
                A[r] = [x ^ int(mul(f, y)) for x, y in zip(A[r], A[c])]
                Iv[r] = [x ^ int(mul(f, y)) for x, y in zip(Iv[r], Iv[c])]
    return np.array(Iv, np.int64)


def mat_mul(A, B):
    C = np.zeros((A.shape[0], B.shape[1]), np.int64)
    for t in range(A.shape[1]):
        C ^= mul(A[:, t:t + 1], B[t:t + 1, :])
    return C


def systematic(n, k):
    """G' = G Gtilde^{-1} (Gtilde = the first B rows)."""
    G = generator(n, k)
    B = k * (k - 1)
    return mat_mul(G, mat_inv(G[:B]))


def parity_matrix(n, k):
    a = k - 1
    return systematic(n, k)[k * a:]


def symbols(data):
    """bytes (..., S) -> little-endian 16-bit symbols (..., S/2)."""
    d = np.asarray(data, np.uint8)
    return d[..., 0::2].astype(np.int64) | (d[..., 1::2].astype(np.int64) << 8)


def to_bytes(sym):
    sym = np.asarray(sym, np.int64)
    out = np.zeros(sym.shape[:-1] + (2 * sym.shape[-1],), np.uint8)
    out[..., 0::2] = sym & 0xFF
    out[..., 1::2] = sym >> 8
    return out


def encode(n, k, data, Gpp=None):
    """parity = G'' X, zero coefficients skipped: data (stripes, B, S) bytes ->
    parity (stripes, (n-k) alpha, S) bytes."""
    Gpp = parity_matrix(n, k) if Gpp is None else Gpp
    X = symbols(data)
    out = np.zeros((X.shape[0], Gpp.shape[0], X.shape[2]), np.int64)
    for r in range(Gpp.shape[0]):
        for c in np.nonzero(Gpp[r])[0]:
            out[:, r] ^= mul(Gpp[r, c], X[:, c])
    return to_bytes(out)


def encode_specific(n, k, Z):
    """C = Psi M(Z) for message symbols Z (B, S/2): node i's piece c_i = psi_i^T M."""
    a, d = k - 1, 2 * k - 2
    P, _ = psi_sparse(n, k)
    L = index_matrix(k)
    M = Z[L - 1]                       # (d, alpha, S/2)
    C = np.zeros((n, a, Z.shape[1]), np.int64)
    for i in range(n):
        for l in range(d):
            if P[i, l]:
                C[i] ^= mul(P[i, l], M[l])
    return C.reshape(n * a, Z.shape[1])
