"""In-tree build of libpmrc.so (host C++ + NVRTC JIT of the generated bitsliced kernels, and the
nvcc-compiled runtime-coefficient kernels of csrc/rt/) and the shared input generator.

The bitsliced kernels are generated per plan and compiled by NVRTC for sm_100a at
``pmrc_create`` / first use (``-arch=sm_100a``); ``build()`` pre-compiles the encode kernels of the
benchmark configurations and the decode / repair plans the GPU tests use into the in-tree kernel
cache (``kcache/``), so the GPU box loads cubins instead of running NVRTC.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
HOST_SRC = ["gf256.cpp", "construct.cpp", "xorprog.cpp", "codegen.cpp", "plan.cpp", "cudrv.cpp", "rtplan.cpp",
            "capi.cpp"]
RT_SRC = ["rlc.cu"]   # hand-written sm_100a kernels compiled by nvcc into libpmrc.so
LIB = os.path.join(HERE, "libpmrc.so")
INPUTS_LIB = os.path.join(ROOT, "inputs", "libpmrc_inputs.so")
NVCC_ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError("build failed: %s" % cmd[0])
    return r


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build_lib(force=False):
    srcs = [os.path.join(HERE, "csrc", "host", s) for s in HOST_SRC]
    rt = [os.path.join(HERE, "csrc", "rt", s) for s in RT_SRC]
    hdrs = [os.path.join(HERE, "csrc", d, h) for d in ("host", "rt") for h in os.listdir(os.path.join(HERE, "csrc", d))
            if h.endswith(".hpp")]
    deps = srcs + rt + hdrs + [os.path.join(ROOT, "include", "pmrc.h")]
    if force or _stale(LIB, deps):
        objs = []
        for cu in rt:
            obj = os.path.join(HERE, "csrc", "rt", os.path.basename(cu)[:-3] + ".o")
            _run([os.path.join(CUDA, "bin", "nvcc")] + NVCC_ARCH +
                 ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-warn-spills",
                  "-c", "-o", obj, cu])
            objs.append(obj)
        _run(["g++", "-O2", "-g", "-std=c++17", "-fPIC", "-shared", "-Wall", "-Wno-unused-function",
              "-I" + os.path.join(CUDA, "include"), "-o", LIB] + srcs + objs +
             ["-L" + os.path.join(CUDA, "lib64"), "-lnvrtc", "-lcudart", "-ldl", "-lpthread",
              "-Wl,-rpath," + os.path.join(CUDA, "lib64")])
    return LIB


def build_inputs(force=False):
    src = os.path.join(ROOT, "inputs", "pmrc_inputs.cu")
    hdr = os.path.join(ROOT, "inputs", "pmrc_inputs.h")
    if force or _stale(INPUTS_LIB, [src, hdr]):
        _run([os.path.join(CUDA, "bin", "nvcc")] + NVCC_ARCH +
             ["-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-shared", "-o", INPUTS_LIB, src])
    return INPUTS_LIB


# encode plans pre-compiled (NVRTC, sm_100a) into the in-tree kernel cache by build(): the bench
# configuration and the GPU-test shapes.  (kind, k, d, n)
PRECOMPILE = [(0, 8, 14, 16), (0, 3, 4, 6), (2, 8, 14, 16), (3, 8, 8, 16), (0, 8, 14, 15), (1, 8, 14, 16),
              (0, 4, 6, 8), (2, 4, 6, 8), (0, 2, 2, 3), (1, 3, 4, 6), (2, 3, 4, 6), (3, 3, 3, 6), (0, 16, 30, 32), (2, 16, 30, 32),
              (0, 8, 14, 16, 16), (0, 4, 6, 8, 16), (0, 8, 14, 15, 16)]   # + GF(2^16) encodes (w = 16)


def _precompile_one(args):
    import ctypes
    L = ctypes.CDLL(LIB)
    h = ctypes.c_void_p()
    kind, k, d, n = args[:4]
    w = args[4] if len(args) > 4 else 8
    rc = L.pmrc_create(ctypes.byref(h), kind, k, d, n, w)
    if rc == 0:
        rc = L.pmrc_precompile(h)
        L.pmrc_destroy(h)
    return args, rc


# decode (op 0) / repair (op 1) plans of fixed failure patterns the GPU tests use (GF(2^16): NVRTC
# takes 20-80 s each).  (kind, k, d, n, w, op, lost id, node ids)
PRECOMPILE_DECODE = [(0, 8, 14, 16, 16, 0, 0, (0, 1, 4, 5, 9, 12, 14, 15)),
                     (0, 8, 14, 16, 16, 0, 0, tuple(range(8, 16))),
                     (0, 8, 14, 16, 16, 1, 15, (0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 11, 12, 13, 14)),
                     (0, 8, 14, 16, 16, 1, 3, (0, 1, 2, 4, 5, 6, 7, 8, 9, 10, 12, 13, 14, 15))]
# + the independent-launch (programmatic dependent launch) plans of
# test_independent_launches_per_stripe_repair_and_decode: (..., independent=1)
_IND_REP = [(6, (0, 1, 2, 3, 4, 5, 7, 8, 9, 10, 11, 13, 14, 15)), (15, (0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 11, 12, 13, 14)),
            (8, (0, 1, 2, 3, 4, 5, 6, 9, 10, 11, 12, 13, 14, 15)), (3, (0, 1, 2, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14)),
            (12, (0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 13, 14)), (0, (1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 15))]
_IND_DEC = [(0, 1, 4, 5, 9, 12, 14, 15), tuple(range(8, 16)), (2, 3, 6, 7, 8, 10, 11, 13), (0, 1, 2, 3, 4, 5, 6, 15),
            (1, 3, 5, 7, 9, 11, 13, 15), (0, 2, 4, 6, 8, 10, 12, 14)]
PRECOMPILE_DECODE += [(0, 8, 14, 16, 8, 1, f, H, 1) for f, H in _IND_REP] + [(0, 8, 14, 16, 8, 0, 0, ids, 1) for ids in _IND_DEC]


def _precompile_decode(args):
    import ctypes
    L = ctypes.CDLL(LIB)
    h = ctypes.c_void_p()
    kind, k, d, n, w, op, lost, ids = args[:8]
    rc = L.pmrc_create(ctypes.byref(h), kind, k, d, n, w)
    if rc == 0 and len(args) > 8 and args[8]:
        rc = L.pmrc_set_independent_launches(h, 1)
    if rc == 0:
        arr = (ctypes.c_int * len(ids))(*ids)
        n_ = ctypes.c_size_t(0)
        rc = L.pmrc_plan_source(h, op, lost, arr, len(ids), 1, None, ctypes.c_size_t(0), ctypes.byref(n_))
        L.pmrc_destroy(h)
    return args, rc


def precompile(configs=PRECOMPILE, clean=True):
    """NVRTC-compile the encode kernels of `configs` into paper_1412_3022_b200/kcache (no GPU).
    clean=True first drops cubins of earlier generator versions (the cache is keyed by source) and the
    plan index of earlier library builds (its key includes the build)."""
    from multiprocessing import get_context
    kdir = os.path.join(HERE, "kcache")
    if clean and os.path.isdir(kdir):
        for f in os.listdir(kdir):
            if f.endswith(".cubin") or f.endswith(".meta"):
                os.remove(os.path.join(kdir, f))
    with get_context("spawn").Pool(min(len(configs), os.cpu_count() or 4)) as pool:
        res = pool.map(_precompile_one, configs)
        res += pool.map(_precompile_decode, PRECOMPILE_DECODE)
    bad = [r for r in res if r[1] != 0]
    if bad:
        raise RuntimeError("precompile failed: %s" % bad)
    return res


def build_all(force=False, kernels=True):
    build_inputs(force)
    build_lib(force)
    if kernels:
        precompile()


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
    print("built", LIB, INPUTS_LIB)
