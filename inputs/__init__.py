"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

Holds none of the method's arithmetic: only the counter-based byte stream defined in
``pmrc_inputs.h`` (splitmix64 of the global source offset) and the host PCG64 draws of
failure patterns.  Both sides call the same functions with the same seed, so neither
ever needs the other's output to build its inputs.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libpmrc_inputs.so")
        if not os.path.exists(path):
            raise RuntimeError("inputs/libpmrc_inputs.so not built: run __graft_entry__.build()")
        L = ctypes.CDLL(path)
        L.pmrc_inputs_fill_host.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint64,
                                            ctypes.c_uint64, ctypes.c_uint64]
        L.pmrc_inputs_fill_host.restype = None
        L.pmrc_inputs_fill_device.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint64,
                                              ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p]
        L.pmrc_inputs_fill_device.restype = ctypes.c_int
        _LIB = L
    return _LIB


NO_PAD = (1 << 64) - 1


def host_bytes(n, seed, offset=0, real_len=NO_PAD):
    """numpy uint8[n] of the stream at global offsets [offset, offset+n)."""
    out = np.empty(int(n), dtype=np.uint8)
    if n:
        lib().pmrc_inputs_fill_host(out.ctypes.data, int(n), seed, offset, real_len)
    return out


def stripe_data(stripes, blocks, S, seed, t0=0, real_len=NO_PAD):
    """uint8[stripes, blocks, S]: the source data of stripes t0..t0+stripes-1 (global offsets
    t*blocks*S + c*S + p)."""
    flat = host_bytes(stripes * blocks * S, seed, t0 * blocks * S, real_len)
    return flat.reshape(stripes, blocks, S)


def fill_device(ptr, n, seed, offset=0, real_len=NO_PAD, stream=0):
    """Fill device memory at ``ptr`` (int address) with the stream; async on ``stream``."""
    rc = lib().pmrc_inputs_fill_device(ctypes.c_void_p(ptr), int(n), seed, offset, real_len,
                                       ctypes.c_void_p(stream))
    if rc != 0:
        raise RuntimeError("pmrc_inputs_fill_device: CUDA error %d" % rc)


def rng(seed):
    """Host PCG64 stream for pattern draws (lost node, helpers, survivors)."""
    return np.random.Generator(np.random.PCG64(seed))
