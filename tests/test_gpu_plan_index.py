"""GPU (-m gpu): a plan built on one handle is loaded by another handle from the kernel cache's
plan index (no source generation, no NVRTC) and computes the same bytes."""
import time

import numpy as np
import pytest
import torch

import oracle as O
import paper_1412_3022_b200 as pm
from gpu_util import DEV, Stripes

pytestmark = pytest.mark.gpu


def test_second_handle_loads_plans_from_the_index(tmp_path, monkeypatch):
    monkeypatch.setenv("PMRC_KCACHE", str(tmp_path))       # empty cache: the first builds compile
    k, n, S, stripes = 4, 8, 4096 + 32, 2
    ids = [1, 4, 6, 7]
    t0 = time.perf_counter()
    a = Stripes(pm.PMRC_MSR_SPARSE, k, n, S, stripes, seed=8, policy=pm.PMRC_PLAN_JIT)
    t_create_a = time.perf_counter() - t0
    b = None
    try:
        a.encode()
        assert np.array_equal(a.parity.cpu().numpy(), O.encode(O.MSR_SPARSE, n, k, a.d, a.host_data()))
        out_a = torch.zeros_like(a.data)
        t0 = time.perf_counter()
        pm.pmrc_decode(a.code, ids, [a.piece(i) for i in ids], out_a.data_ptr(), S, stripes, a.stream)
        torch.cuda.synchronize()
        t_a = time.perf_counter() - t0
        t0 = time.perf_counter()
        b = pm.pmrc_create(pm.PMRC_MSR_SPARSE, k, a.d, n)
        t_create_b = time.perf_counter() - t0
        pm.pmrc_set_plan_policy(b, pm.PMRC_PLAN_JIT)
        out_b = torch.zeros_like(a.data)
        t0 = time.perf_counter()
        pm.pmrc_decode(b, ids, [a.piece(i) for i in ids], out_b.data_ptr(), S, stripes, a.stream)
        torch.cuda.synchronize()
        t_b = time.perf_counter() - t0
        assert torch.equal(out_a, out_b)
        miss = [x for x in range(a.B) if x // a.alpha not in ids]
        assert torch.equal(out_b[:, miss], a.data[:, miss])
        par_b = torch.zeros_like(a.parity)
        pm.pmrc_encode(b, a.data.data_ptr(), par_b.data_ptr(), S, stripes, a.stream)
        torch.cuda.synchronize()
        assert torch.equal(par_b, a.parity)
        # generation + NVRTC on the first handle, an index lookup + cubin load on the second
        assert t_b < 0.5 * t_a, (t_a, t_b)
        assert t_create_b < 0.5 * t_create_a, (t_create_a, t_create_b)
    finally:
        a.close()
        if b is not None:
            pm.pmrc_destroy(b)
