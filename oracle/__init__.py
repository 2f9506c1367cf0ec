"""CPU oracle for the product-matrix regenerating-code hot path (arxiv 1412.3022).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()``, ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs and the measurement tools' sampled correctness
checks (``tools/sweep.py``) may import this package.  The product path
(``paper_1412_3022_b200``) shares no code with it and never calls it.

Thin ctypes/numpy wrapper over ``pmrc_oracle.c`` (plain scalar log/exp GF(2^8) arithmetic,
primitive polynomial 0x11D, g = 2).  Every function cites the passage it follows in the C file.
"""
import ctypes
import os
import subprocess

import numpy as np

MSR_SPARSE, MSR_VANILLA, MBR, RS = 0, 1, 2, 3
MSR_N2K = 4   # extension (R15): sparse Phi, greedy Lambda valid at n = 2k; not the paper's
OK, EINVAL, EUNSUP, ESING = 0, -1, -2, -3

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "pmrc_oracle.c")
_L = None


def build():
    """Compile the oracle (plain gcc, -O2, no SIMD intrinsics)."""
    if (not os.path.exists(_SO)) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-o", _SO, _SRC])


def _lib():
    global _L
    if _L is None:
        build()
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        I = ctypes.c_int
        Z = ctypes.c_size_t
        sig = {
            "or_init": ([], None),
            "or_gf_mul": ([ctypes.c_uint8, ctypes.c_uint8], ctypes.c_uint8),
            "or_gf_inv": ([ctypes.c_uint8], ctypes.c_uint8),
            "or_gf_div": ([ctypes.c_uint8, ctypes.c_uint8], ctypes.c_uint8),
            "or_gf_exp": ([ctypes.c_long], ctypes.c_uint8),
            "or_gf_log": ([ctypes.c_uint8], I),
            "or_mat_mul": ([P, P, P, I, I, I], None),
            "or_mat_inv": ([P, P, I], I),
            "or_mat_rank": ([P, I, I], I),
            "or_params": ([I, I, I, I, P, P], I),
            "or_index_matrix": ([I, I, I, P], I),
            "or_psi": ([I, I, I, I, P, P], I),
            "or_generator": ([I, I, I, I, P], I),
            "or_systematic": ([I, I, I, I, P], I),
            "or_parity_matrix": ([I, I, I, I, P], I),
            "or_apply_flat": ([P, I, I, P, P, Z, I], None),
            "or_encode": ([I, I, I, I, P, P, Z, Z], I),
            "or_encode_specific": ([I, I, I, I, P, P, Z], I),
            "or_decode_linear": ([I, I, I, I, P, I, P, P, Z], I),
            "or_decode_msr_specific_Z": ([I, I, I, I, P, P, P, Z], I),
            "or_decode_mbr_specific": ([I, I, I, P, P, P, Z], I),
            "or_repair_mu": ([I, I, I, I, I, P, P], I),
            "or_repair_reads": ([I, I, I, I, I], I),
            "or_repair_project": ([I, I, I, I, I, P, P, Z], I),
            "or_validate16_sparse": ([I, ctypes.POINTER(ctypes.c_int)], I),
            "or_validate16_sparse_n": ([I, I, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)], I),
            "or_gf16_mul": ([ctypes.c_uint16, ctypes.c_uint16], ctypes.c_uint16),
            "or_repair_combine": ([I, I, I, I, I, P, P, P, Z], I),
            "or_repair": ([I, I, I, I, I, P, P, P, Z], I),
            "or_validate": ([I, I, I, I, ctypes.c_long, I, P], I),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        L.or_init()
        _L = L
    return _L


def _p(a):
    return a.ctypes.data if a is not None else None


def _u8(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


class OracleError(RuntimeError):
    def __init__(self, rc, what):
        super().__init__("%s failed: rc=%d" % (what, rc))
        self.rc = rc


def _chk(rc, what):
    if rc != 0:
        raise OracleError(rc, what)


# ---------------------------------------------------------------- GF(2^8)
def gf_mul(a, b):
    return int(_lib().or_gf_mul(a, b))


def gf_inv(a):
    return int(_lib().or_gf_inv(a))


def gf_div(a, b):
    return int(_lib().or_gf_div(a, b))


def gf_exp(e):
    return int(_lib().or_gf_exp(e))


def gf_log(a):
    return int(_lib().or_gf_log(a))


def mat_mul(A, B):
    A, B = _u8(A), _u8(B)
    C = np.zeros((A.shape[0], B.shape[1]), np.uint8)
    _lib().or_mat_mul(_p(A), _p(B), _p(C), A.shape[0], A.shape[1], B.shape[1])
    return C


def mat_inv(A):
    A = _u8(A)
    R = np.zeros_like(A)
    _chk(_lib().or_mat_inv(_p(A), _p(R), A.shape[0]), "mat_inv")
    return R


def mat_rank(A):
    A = _u8(A)
    return int(_lib().or_mat_rank(_p(A), A.shape[0], A.shape[1]))


# ---------------------------------------------------------------- construction
def params(kind, n, k, d):
    a = ctypes.c_int()
    b = ctypes.c_int()
    _chk(_lib().or_params(kind, n, k, d, ctypes.byref(a), ctypes.byref(b)), "params")
    return a.value, b.value


def index_matrix(kind, k, d):
    alpha, _ = params(kind, d + 1, k, d)
    cols = d if kind == MBR else alpha
    L = np.zeros((d, cols), np.int32)
    _chk(_lib().or_index_matrix(kind, k, d, _p(L)), "index_matrix")
    return L


def psi(kind, n, k, d):
    cols = k if kind == RS else d
    P = np.zeros((n, cols), np.uint8)
    lam = np.zeros(n, np.uint8)
    _chk(_lib().or_psi(kind, n, k, d, _p(P), _p(lam)), "psi")
    return P, lam


def generator(kind, n, k, d):
    alpha, B = params(kind, n, k, d)
    G = np.zeros((n * alpha, B), np.uint8)
    _chk(_lib().or_generator(kind, n, k, d, _p(G)), "generator")
    return G


def systematic(kind, n, k, d):
    alpha, B = params(kind, n, k, d)
    G = np.zeros((n * alpha, B), np.uint8)
    _chk(_lib().or_systematic(kind, n, k, d, _p(G)), "systematic")
    return G


def parity_matrix(kind, n, k, d):
    alpha, B = params(kind, n, k, d)
    G = np.zeros(((n - k) * alpha, B), np.uint8)
    _chk(_lib().or_parity_matrix(kind, n, k, d, _p(G)), "parity_matrix")
    return G


def validate(kind, n, k, d, max_subsets=10 ** 6, check_phi=True):
    w = np.zeros(256, np.int32)
    rc = _lib().or_validate(kind, n, k, d, max_subsets, int(check_phi), _p(w))
    if rc < 0:
        raise OracleError(rc, "validate")
    return rc, w


# ---------------------------------------------------------------- data path
def apply(A, X, skip_zeros=True):
    """Y = A X over GF(2^8); X: (C, S) uint8 blocks."""
    A, X = _u8(A), _u8(X)
    R, C = A.shape
    S = X.shape[1]
    Y = np.zeros((R, S), np.uint8)
    _lib().or_apply_flat(_p(A), R, C, _p(X), _p(Y), S, int(skip_zeros))
    return Y


def encode(kind, n, k, d, data):
    """data: (stripes, B, S) -> parity (stripes, (n-k) alpha, S)."""
    data = _u8(data)
    alpha, B = params(kind, n, k, d)
    st, b, S = data.shape
    assert b == B
    par = np.zeros((st, (n - k) * alpha, S), np.uint8)
    _chk(_lib().or_encode(kind, n, k, d, _p(data), _p(par), S, st), "encode")
    return par


def encode_specific(kind, n, k, d, Z):
    """C = Psi M(Z): Z (B, S) -> code (n*alpha, S), node-major."""
    Z = _u8(Z)
    alpha, B = params(kind, n, k, d)
    C = np.zeros((n * alpha, Z.shape[1]), np.uint8)
    _chk(_lib().or_encode_specific(kind, n, k, d, _p(Z), _p(C), Z.shape[1]), "encode_specific")
    return C


def decode_linear(kind, n, k, d, ids, pieces):
    """ids: node ids; pieces: (len(ids), alpha, S) -> X (B, S)."""
    ids = _i32(ids)
    pieces = _u8(pieces)
    alpha, B = params(kind, n, k, d)
    S = pieces.shape[2]
    X = np.zeros((B, S), np.uint8)
    _chk(_lib().or_decode_linear(kind, n, k, d, _p(ids), len(ids), _p(pieces), _p(X), S), "decode_linear")
    return X


def decode_msr_specific_Z(kind, n, k, d, ids, pieces):
    ids = _i32(ids)
    pieces = _u8(pieces)
    alpha, B = params(kind, n, k, d)
    S = pieces.shape[2]
    Z = np.zeros((B, S), np.uint8)
    _chk(_lib().or_decode_msr_specific_Z(kind, n, k, d, _p(ids), _p(pieces), _p(Z), S), "decode_msr_specific")
    return Z


def decode_mbr_specific(n, k, d, ids, pieces):
    ids = _i32(ids)
    pieces = _u8(pieces)
    alpha, B = params(MBR, n, k, d)
    S = pieces.shape[2]
    X = np.zeros((B, S), np.uint8)
    _chk(_lib().or_decode_mbr_specific(n, k, d, _p(ids), _p(pieces), _p(X), S), "decode_mbr_specific")
    return X


def repair_mu(kind, n, k, d, f):
    mu = np.zeros(256, np.uint8)
    ln = ctypes.c_int()
    _chk(_lib().or_repair_mu(kind, n, k, d, f, _p(mu), ctypes.byref(ln)), "repair_mu")
    return mu[: ln.value].copy()


def repair_reads(kind, n, k, d, f):
    return int(_lib().or_repair_reads(kind, n, k, d, f))


def repair_project(kind, n, k, d, f, piece):
    piece = _u8(piece)
    S = piece.shape[1]
    beta = np.zeros(S, np.uint8)
    _chk(_lib().or_repair_project(kind, n, k, d, f, _p(piece), _p(beta), S), "repair_project")
    return beta


def gf16_mul(a, b):
    """GF(2^16) product, polynomial 0x1100B (R1 extended to w = 16)."""
    return int(_lib().or_gf16_mul(a, b))


def validate16_sparse(k):
    """P:189 in GF(2^16): flags of the sparse construction at n = d+1 (1 lambda collision,
    2 a singular d x d submatrix of Psi)."""
    f = ctypes.c_int(0)
    _chk(_lib().or_validate16_sparse(k, ctypes.byref(f)), "validate16_sparse")
    return f.value


def validate16_sparse_n(k, n):
    """The same check over EVERY d-row subset at n = d+1 or n = d+2 (= 2k): (flags, number of
    singular d-subsets)."""
    f, ns = ctypes.c_int(0), ctypes.c_int(0)
    _chk(_lib().or_validate16_sparse_n(k, n, ctypes.byref(f), ctypes.byref(ns)), "validate16_sparse_n")
    return f.value, ns.value


def repair_combine(kind, n, k, d, f, H, betas):
    """Newcomer side: betas (len(H), S) of helpers H -> lost piece (alpha, S)."""
    H = _i32(H)
    betas = _u8(betas)
    alpha, B = params(kind, n, k, d)
    S = betas.shape[1]
    out = np.zeros((alpha, S), np.uint8)
    _chk(_lib().or_repair_combine(kind, n, k, d, f, _p(H), _p(betas), _p(out), S), "repair_combine")
    return out


def repair(kind, n, k, d, f, H, pieces):
    """H: helper ids (d of them; RS: k); pieces (len(H), alpha, S) -> lost piece (alpha, S).
    Raises OracleError(rc=ESING) if Psi_H is singular."""
    H = _i32(H)
    pieces = _u8(pieces)
    alpha, B = params(kind, n, k, d)
    S = pieces.shape[2]
    out = np.zeros((alpha, S), np.uint8)
    _chk(_lib().or_repair(kind, n, k, d, f, _p(H), _p(pieces), _p(out), S), "repair")
    return out


def full_code(kind, n, k, d, data):
    """All n nodes' pieces of one stripe of systematic code: (n, alpha, S).  Systematic nodes hold
    the data (MSR/RS: blocks i*alpha..; MBR: row i of M(X), R6); parity nodes from encode()."""
    data = _u8(data)
    alpha, B = params(kind, n, k, d)
    S = data.shape[1]
    par = encode(kind, n, k, d, data[None])[0]
    out = np.zeros((n, alpha, S), np.uint8)
    if kind == MBR:
        L = index_matrix(MBR, k, d)
        for i in range(k):
            for j in range(alpha):
                out[i, j] = data[L[i, j] - 1]
    else:
        out[:k] = data.reshape(k, alpha, S)
    out[k:] = par.reshape(n - k, alpha, S)
    return out
