"""Python binding of libpmrc (include/pmrc.h) — argument marshalling only.

Every function below has the name of the C-ABI entry point it calls; buffers are passed as
integer device addresses (e.g. ``tensor.data_ptr()``) and streams as ``cudaStream_t`` handles
(e.g. ``torch.cuda.current_stream().cuda_stream``).  There is no CPU fallback: every data-path
call runs the library's CUDA kernels and raises ``PmrcError`` on any error, including a missing
GPU or a missing ``libpmrc.so``.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpmrc.so")

PMRC_MSR_SPARSE, PMRC_MSR_VANILLA, PMRC_MBR, PMRC_RS_VANDERMONDE, PMRC_MSR_SPARSE_N2K = 0, 1, 2, 3, 4
PMRC_OK, PMRC_EINVAL, PMRC_EUNSUPPORTED, PMRC_ESINGULAR = 0, -1, -2, -3
PMRC_EALIGN, PMRC_ENOMEM, PMRC_ECUDA, PMRC_EJIT = -4, -5, -6, -7

PMRC_PLAN_AUTO, PMRC_PLAN_JIT, PMRC_PLAN_RUNTIME = 0, 1, 2

MATRIX_PSI, MATRIX_G, MATRIX_GSYS, MATRIX_GPP, MATRIX_LAMBDA, MATRIX_GTINV = 0, 1, 2, 3, 4, 5

EXPORTS = ["pmrc_create", "pmrc_destroy", "pmrc_info", "pmrc_matrix", "pmrc_layout", "pmrc_encode",
           "pmrc_encode_host", "pmrc_decode", "pmrc_repair", "pmrc_repair_project", "pmrc_repair_combine",
           "pmrc_read_cost", "pmrc_launch_count", "pmrc_strerror", "pmrc_last_error", "pmrc_precompile",
           "pmrc_encode_source", "pmrc_debug_counters", "pmrc_plan_source", "pmrc_plan_stats", "pmrc_apply", "pmrc_apply_stats", "pmrc_set_max_ctas",
           "pmrc_set_independent_launches", "pmrc_set_plan_policy", "pmrc_get_plan_policy", "pmrc_plan_prepare",
           "pmrc_decode_batch", "pmrc_repair_batch", "pmrc_decode_specific", "pmrc_decode_specific_scratch",
           "pmrc_rt_plan_blob", "pmrc_set_auto_promotion", "pmrc_plan_state"]


class PmrcError(RuntimeError):
    def __init__(self, rc, where, detail=""):
        self.rc = rc
        super().__init__("%s: %s (%d)%s" % (where, _strerror(rc), rc, (": " + detail) if detail else ""))


class pmrc_cregion(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("stripe_stride", ctypes.c_size_t)]


class pmrc_region(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("stripe_stride", ctypes.c_size_t)]


class pmrc_info_t(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("n", ctypes.c_int), ("k", ctypes.c_int), ("d", ctypes.c_int),
                ("w", ctypes.c_int), ("alpha", ctypes.c_int), ("B", ctypes.c_int), ("parity_rows", ctypes.c_int),
                ("nnz", ctypes.c_int), ("zero_pct", ctypes.c_double), ("repair_complete", ctypes.c_int),
                ("xor_ops", ctypes.c_long), ("xor_ops_naive", ctypes.c_long)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class pmrc_plan_stats_t(ctypes.Structure):
    _fields_ = [("groups", ctypes.c_int), ("in_blocks", ctypes.c_int), ("out_blocks", ctypes.c_int),
                ("naive_lop3", ctypes.c_longlong), ("xor2", ctypes.c_longlong), ("transposes", ctypes.c_int)]


_L = None


def lib():
    """Load libpmrc.so (raises if it was not built: no fallback)."""
    global _L
    if _L is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError("libpmrc.so not built (run __graft_entry__.build()); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        P, I, Z = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
        IP = ctypes.POINTER(ctypes.c_int)
        sig = {
            "pmrc_create": ([ctypes.POINTER(ctypes.c_void_p), I, I, I, I, I], I),
            "pmrc_destroy": ([P], None),
            "pmrc_info": ([P, ctypes.POINTER(pmrc_info_t)], I),
            "pmrc_matrix": ([P, I, P, IP, IP], I),
            "pmrc_layout": ([P, P, IP, IP], I),
            "pmrc_encode": ([P, P, P, Z, Z, P], I),
            "pmrc_encode_host": ([P, P, P, Z, Z, P], I),
            "pmrc_decode": ([P, IP, I, ctypes.POINTER(pmrc_cregion), P, Z, Z, IP, P], I),
            "pmrc_repair": ([P, I, IP, I, ctypes.POINTER(pmrc_cregion), pmrc_region, Z, Z, P], I),
            "pmrc_repair_project": ([P, I, pmrc_cregion, pmrc_region, Z, Z, P], I),
            "pmrc_repair_combine": ([P, I, IP, I, ctypes.POINTER(pmrc_cregion), pmrc_region, Z, Z, P], I),
            "pmrc_read_cost": ([P, I, IP], I),
            "pmrc_launch_count": ([], ctypes.c_ulonglong),
            "pmrc_precompile": ([P], I),
            "pmrc_encode_source": ([P, P, Z, ctypes.POINTER(ctypes.c_size_t)], I),
            "pmrc_debug_counters": ([P, P, Z, ctypes.POINTER(ctypes.c_size_t)], I),
            "pmrc_plan_source": ([P, I, I, IP, I, I, P, Z, ctypes.POINTER(ctypes.c_size_t)], I),
            "pmrc_plan_stats": ([P, I, I, IP, I, ctypes.POINTER(pmrc_plan_stats_t)], I),
            "pmrc_apply": ([P, P, I, I, P, Z, P, Z, Z, Z, P], I),
            "pmrc_apply_stats": ([P, P, I, I, ctypes.POINTER(pmrc_plan_stats_t)], I),
            "pmrc_set_max_ctas": ([P, I], I),
            "pmrc_set_independent_launches": ([P, I], I),
            "pmrc_set_plan_policy": ([P, I], I),
            "pmrc_get_plan_policy": ([P], I),
            "pmrc_plan_prepare": ([P, I, I, IP, I], I),
            "pmrc_set_auto_promotion": ([P, ctypes.c_ulonglong], I),
            "pmrc_plan_state": ([P, I, I, IP, I], I),
            "pmrc_decode_batch": ([P, IP, I, ctypes.POINTER(pmrc_cregion), P, Z, Z, IP, P], I),
            "pmrc_repair_batch": ([P, IP, IP, I, ctypes.POINTER(pmrc_cregion), pmrc_region, Z, Z, P], I),
            "pmrc_decode_specific_scratch": ([P, Z, Z, ctypes.POINTER(ctypes.c_size_t)], I),
            "pmrc_decode_specific": ([P, IP, I, ctypes.POINTER(pmrc_cregion), P, P, Z, Z, Z, IP, P], I),
            "pmrc_rt_plan_blob": ([P, I, I, IP, I, P, Z, ctypes.POINTER(ctypes.c_size_t)], I),
            "pmrc_strerror": ([I], ctypes.c_char_p),
            "pmrc_last_error": ([], ctypes.c_char_p),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _L = L
    return _L


def _strerror(rc):
    try:
        return lib().pmrc_strerror(rc).decode()
    except Exception:
        return "error"


def _check(rc, where):
    if rc != PMRC_OK:
        raise PmrcError(rc, where, lib().pmrc_last_error().decode())


def _ints(seq):
    seq = [int(x) for x in seq]
    return (ctypes.c_int * max(1, len(seq)))(*seq), len(seq)


# ------------------------------------------------------------------ C-ABI mirrors
def pmrc_create(kind, k, d, n, w=8):
    h = ctypes.c_void_p()
    _check(lib().pmrc_create(ctypes.byref(h), kind, k, d, n, w), "pmrc_create")
    return h


def pmrc_destroy(code):
    lib().pmrc_destroy(code)


def pmrc_info(code):
    info = pmrc_info_t()
    _check(lib().pmrc_info(code, ctypes.byref(info)), "pmrc_info")
    return info.as_dict()


def pmrc_matrix(code, which):
    import numpy as np
    r, c = ctypes.c_int(), ctypes.c_int()
    _check(lib().pmrc_matrix(code, which, None, ctypes.byref(r), ctypes.byref(c)), "pmrc_matrix")
    out = np.zeros((r.value, c.value), np.uint8)
    _check(lib().pmrc_matrix(code, which, out.ctypes.data, ctypes.byref(r), ctypes.byref(c)), "pmrc_matrix")
    return out


def pmrc_layout(code):
    import numpy as np
    r, c = ctypes.c_int(), ctypes.c_int()
    _check(lib().pmrc_layout(code, None, ctypes.byref(r), ctypes.byref(c)), "pmrc_layout")
    out = np.zeros((r.value, c.value), np.int32)
    _check(lib().pmrc_layout(code, out.ctypes.data, ctypes.byref(r), ctypes.byref(c)), "pmrc_layout")
    return out


def pmrc_encode(code, data_ptr, parity_ptr, S, stripes, stream=0):
    _check(lib().pmrc_encode(code, data_ptr, parity_ptr, S, stripes, stream), "pmrc_encode")


def pmrc_encode_host(code, data_host_ptr, parity_host_ptr, S, stripes, stream=0):
    _check(lib().pmrc_encode_host(code, data_host_ptr, parity_host_ptr, S, stripes, stream), "pmrc_encode_host")


def pmrc_decode(code, surv_ids, pieces, data_out_ptr, S, stripes, stream=0):
    """pieces: list of (ptr, stripe_stride) per survivor.  Returns blocks written per stripe."""
    ids, n = _ints(surv_ids)
    regs = (pmrc_cregion * max(1, n))(*[pmrc_cregion(p, s) for p, s in pieces])
    nw = ctypes.c_int()
    _check(lib().pmrc_decode(code, ids, n, regs, data_out_ptr, S, stripes, ctypes.byref(nw), stream), "pmrc_decode")
    return nw.value


def pmrc_repair(code, lost_id, helper_ids, helper_pieces, out_piece, S, stripes, stream=0):
    ids, n = _ints(helper_ids)
    regs = (pmrc_cregion * max(1, n))(*[pmrc_cregion(p, s) for p, s in helper_pieces])
    _check(lib().pmrc_repair(code, lost_id, ids, n, regs, pmrc_region(*out_piece), S, stripes, stream), "pmrc_repair")


def pmrc_repair_project(code, lost_id, piece, beta, S, stripes, stream=0):
    _check(lib().pmrc_repair_project(code, lost_id, pmrc_cregion(*piece), pmrc_region(*beta), S, stripes, stream),
           "pmrc_repair_project")


def pmrc_repair_combine(code, lost_id, helper_ids, betas, out_piece, S, stripes, stream=0):
    ids, n = _ints(helper_ids)
    regs = (pmrc_cregion * max(1, n))(*[pmrc_cregion(p, s) for p, s in betas])
    _check(lib().pmrc_repair_combine(code, lost_id, ids, n, regs, pmrc_region(*out_piece), S, stripes, stream),
           "pmrc_repair_combine")


def pmrc_read_cost(code, lost_id):
    b = ctypes.c_int()
    _check(lib().pmrc_read_cost(code, lost_id, ctypes.byref(b)), "pmrc_read_cost")
    return b.value


def pmrc_precompile(code):
    _check(lib().pmrc_precompile(code), "pmrc_precompile")


def pmrc_encode_source(code):
    n = ctypes.c_size_t()
    _check(lib().pmrc_encode_source(code, None, 0, ctypes.byref(n)), "pmrc_encode_source")
    buf = ctypes.create_string_buffer(n.value + 1)
    _check(lib().pmrc_encode_source(code, buf, n.value + 1, ctypes.byref(n)), "pmrc_encode_source")
    return buf.value.decode()


def pmrc_plan_source(code, op, lost_id, ids, compile=False):
    """Generated source of a decode (op 0, ids = survivors) or repair (op 1) plan; no GPU needed."""
    n = ctypes.c_size_t(0)
    arr, _ = _ints(ids)
    _check(lib().pmrc_plan_source(code, op, lost_id, arr, len(ids), int(compile), None, 0, ctypes.byref(n)),
           "pmrc_plan_source")
    buf = ctypes.create_string_buffer(n.value + 1)
    _check(lib().pmrc_plan_source(code, op, lost_id, arr, len(ids), 0, buf, n.value + 1, ctypes.byref(n)),
           "pmrc_plan_source")
    return buf.value.decode()


def pmrc_apply(code, A, in_ptr, in_stride, out_ptr, out_stride, S, stripes, stream=0):
    """out block r = XOR_c A[r][c] * in block c for every stripe (A: host uint8 rows x cols)."""
    import numpy as np
    A = np.ascontiguousarray(A, dtype=np.uint8)
    rows, cols = A.shape
    _check(lib().pmrc_apply(code, A.ctypes.data, rows, cols, in_ptr, in_stride, out_ptr, out_stride, S, stripes,
                            stream), "pmrc_apply")


def pmrc_set_max_ctas(code, max_ctas):
    """Grid cap for every launch on this handle (0 = one full wave)."""
    _check(lib().pmrc_set_max_ctas(code, max_ctas), "pmrc_set_max_ctas")


def pmrc_set_independent_launches(code, on):
    """Declare consecutive launches of this handle independent (programmatic dependent launch)."""
    _check(lib().pmrc_set_independent_launches(code, int(on)), "pmrc_set_independent_launches")


def pmrc_set_plan_policy(code, policy):
    """PMRC_PLAN_AUTO (default), PMRC_PLAN_JIT or PMRC_PLAN_RUNTIME (include/pmrc.h)."""
    _check(lib().pmrc_set_plan_policy(code, int(policy)), "pmrc_set_plan_policy")


def pmrc_get_plan_policy(code):
    return int(lib().pmrc_get_plan_policy(code))


def pmrc_plan_prepare(code, op, lost_id, ids):
    """JIT-compile and keep the generated kernel of a decode (op 0) / repair (op 1) pattern."""
    arr, n = _ints(ids)
    _check(lib().pmrc_plan_prepare(code, op, lost_id, arr, n), "pmrc_plan_prepare")


def pmrc_set_auto_promotion(code, nbytes):
    """AUTO policy: compile a pattern's generated kernel in a host thread once it moved nbytes of
    plan traffic on the runtime kernel (0 = off; default 1 GiB)."""
    _check(lib().pmrc_set_auto_promotion(code, nbytes), "pmrc_set_auto_promotion")


PLAN_RUNTIME_ONLY, PLAN_COMPILING, PLAN_COMPILED, PLAN_LOADED = 0, 1, 2, 3


def pmrc_plan_state(code, op, lost_id, ids):
    """0 runtime kernel only, 1 promotion compiling, 2 compiled (loads at the next call), 3 loaded."""
    arr, n = _ints(ids)
    rc = lib().pmrc_plan_state(code, op, lost_id, arr, n)
    if rc < 0:
        _check(rc, "pmrc_plan_state")
    return rc


def pmrc_decode_batch(code, surv_ids, nodes, data_out_ptr, S, stripes, stream=0):
    """surv_ids: stripes x n_surv survivor ids (per stripe); nodes: n (ptr, stripe_stride) piece
    regions, one per node.  Returns the list of blocks written per stripe."""
    rows = [list(r) for r in surv_ids]
    n_surv = len(rows[0]) if rows else 0
    assert len(rows) == stripes and all(len(r) == n_surv for r in rows)
    ids, _ = _ints([x for r in rows for x in r])
    regs = (pmrc_cregion * max(1, len(nodes)))(*[pmrc_cregion(p, s) for p, s in nodes])
    nw = (ctypes.c_int * max(1, stripes))()
    _check(lib().pmrc_decode_batch(code, ids, n_surv, regs, data_out_ptr, S, stripes, nw, stream), "pmrc_decode_batch")
    return list(nw[:stripes])


def pmrc_repair_batch(code, lost_ids, helper_ids, nodes, out_piece, S, stripes, stream=0):
    """lost_ids: per stripe; helper_ids: stripes x d; nodes: n (ptr, stripe_stride) piece regions;
    out_piece: (ptr, stripe_stride) of the repaired pieces."""
    rows = [list(r) for r in helper_ids]
    nh = len(rows[0]) if rows else 0
    assert len(rows) == stripes == len(lost_ids) and all(len(r) == nh for r in rows)
    lost, _ = _ints(lost_ids)
    ids, _ = _ints([x for r in rows for x in r])
    regs = (pmrc_cregion * max(1, len(nodes)))(*[pmrc_cregion(p, s) for p, s in nodes])
    _check(lib().pmrc_repair_batch(code, lost, ids, nh, regs, pmrc_region(*out_piece), S, stripes, stream),
           "pmrc_repair_batch")


def pmrc_decode_specific_scratch(code, S, stripes):
    """Bytes of device scratch pmrc_decode_specific needs for (S, stripes)."""
    n = ctypes.c_size_t()
    _check(lib().pmrc_decode_specific_scratch(code, S, stripes, ctypes.byref(n)), "pmrc_decode_specific_scratch")
    return n.value


def pmrc_decode_specific(code, surv_ids, pieces, data_out_ptr, scratch_ptr, scratch_bytes, S, stripes, stream=0):
    """The paper's specific MSR / MBR decoder from exactly k survivors (pieces: (ptr, stride) each).
    Returns blocks written per stripe."""
    ids, n = _ints(surv_ids)
    regs = (pmrc_cregion * max(1, n))(*[pmrc_cregion(p, s) for p, s in pieces])
    nw = ctypes.c_int()
    _check(lib().pmrc_decode_specific(code, ids, n, regs, data_out_ptr, scratch_ptr, scratch_bytes, S, stripes,
                                      ctypes.byref(nw), stream), "pmrc_decode_specific")
    return nw.value


def pmrc_rt_plan_blob(code, op, lost_id=0, ids=()):
    """The runtime-coefficient plan blob (numpy uint32) of a decode (0) / repair (1) / encode (2) plan."""
    import numpy as np
    arr, n = _ints(ids)
    nw = ctypes.c_size_t()
    _check(lib().pmrc_rt_plan_blob(code, op, lost_id, arr, n, None, 0, ctypes.byref(nw)), "pmrc_rt_plan_blob")
    out = np.zeros(nw.value, np.uint32)
    _check(lib().pmrc_rt_plan_blob(code, op, lost_id, arr, n, out.ctypes.data, nw.value, ctypes.byref(nw)),
           "pmrc_rt_plan_blob")
    return out


def pmrc_apply_stats(code, A):
    """Per-stripe work of the pmrc_apply plan for matrix A."""
    import numpy as np
    A = np.ascontiguousarray(A, dtype=np.uint8)
    st = pmrc_plan_stats_t()
    _check(lib().pmrc_apply_stats(code, A.ctypes.data, A.shape[0], A.shape[1], ctypes.byref(st)), "pmrc_apply_stats")
    return {f: getattr(st, f) for f, _ in pmrc_plan_stats_t._fields_}


def pmrc_plan_stats(code, op, lost_id=0, ids=()):
    """Per-stripe work of a decode (op 0) / repair (op 1) / encode (op 2) plan (roofline accounting)."""
    st = pmrc_plan_stats_t()
    arr, n = _ints(ids)
    _check(lib().pmrc_plan_stats(code, op, lost_id, arr, n, ctypes.byref(st)), "pmrc_plan_stats")
    return {f: getattr(st, f) for f, _ in pmrc_plan_stats_t._fields_}


def prepare_plans(kind, k, d, n, patterns, threads=None, independent=False):
    """Pre-compile the decode / repair plans of many failure patterns in parallel (NVRTC runs
    outside the GIL; each worker thread uses its own handle, and the cubins land in the shared
    in-tree kernel cache, keyed by source), so that the first pmrc_decode / pmrc_repair of each
    pattern only loads a cubin.  patterns: iterable of ("decode", survivor_ids) or
    ("repair", lost_id, helper_ids).  Returns the list of (pattern, rc) (rc = PMRC_ESINGULAR for
    singular helper sets).  independent=True prepares the kernels a handle uses after
    pmrc_set_independent_launches(code, 1)."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    pats = list(patterns)
    threads = threads or min(len(pats), os.cpu_count() or 4) or 1
    handles = [pmrc_create(kind, k, d, n) for _ in range(threads)]
    try:
        if independent:
            for h in handles:
                pmrc_set_independent_launches(h, 1)
        def work(i):
            h = handles[i % threads]
            out = []
            for pt in pats[i::threads]:
                try:
                    if pt[0] == "decode":
                        pmrc_plan_source(h, 0, 0, pt[1], compile=True)
                    else:
                        pmrc_plan_source(h, 1, pt[1], pt[2], compile=True)
                    out.append((pt, PMRC_OK))
                except PmrcError as e:
                    out.append((pt, e.rc))
            return out
        with ThreadPoolExecutor(threads) as ex:
            res = [r for part in ex.map(work, range(threads)) for r in part]
    finally:
        for h in handles:
            pmrc_destroy(h)
    return res


def pmrc_debug_counters(code):
    """Pacing counters / trace of the encode kernel as a list of ints (diagnostics)."""
    n = ctypes.c_size_t(0)
    _check(lib().pmrc_debug_counters(code, None, 0, ctypes.byref(n)), "pmrc_debug_counters")
    buf = (ctypes.c_ulonglong * max(1, n.value))()
    _check(lib().pmrc_debug_counters(code, buf, n.value, ctypes.byref(n)), "pmrc_debug_counters")
    return list(buf[: n.value])


def pmrc_launch_count():
    return int(lib().pmrc_launch_count())


def pmrc_strerror(rc):
    return _strerror(rc)


def pmrc_last_error():
    return lib().pmrc_last_error().decode()
