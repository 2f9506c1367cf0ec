"""CPU tier: libpmrc.so loads without a GPU, exports every symbol include/pmrc.h declares, and its
host logic (construction, info, error paths) behaves; the data path fails loudly without a GPU."""
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_1412_3022_b200 as pm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_symbols_exported():
    hdr = open(os.path.join(ROOT, "include", "pmrc.h")).read()
    declared = set(re.findall(r"\b(pmrc_[a-z_]+)\s*\(", hdr))
    assert declared == set(pm.EXPORTS)
    L = pm.lib()
    for name in declared:
        assert hasattr(L, name), name


@pytest.mark.parametrize("kind,k,n", [(0, 3, 6), (0, 8, 16), (1, 8, 16), (2, 8, 16), (3, 8, 16), (0, 4, 8), (2, 3, 6),
                                      (0, 16, 32), (4, 3, 6), (4, 8, 16)])
def test_host_matrices_equal_oracle(kind, k, n):
    # the product's host construction (independent code) reproduces the oracle's matrices
    d = k if kind == 3 else 2 * k - 2
    c = pm.pmrc_create(kind, k, d, n)
    try:
        assert np.array_equal(pm.pmrc_matrix(c, pm.MATRIX_GPP), O.parity_matrix(kind, n, k, d))
        assert np.array_equal(pm.pmrc_matrix(c, pm.MATRIX_G), O.generator(kind, n, k, d))
        assert np.array_equal(pm.pmrc_matrix(c, pm.MATRIX_GSYS), O.systematic(kind, n, k, d))
        psi, lam = O.psi(kind, n, k, d)
        assert np.array_equal(pm.pmrc_matrix(c, pm.MATRIX_PSI), psi)
        if kind != 3:
            assert np.array_equal(pm.pmrc_layout(c), O.index_matrix(kind, k, d))
        info = pm.pmrc_info(c)
        G2 = O.parity_matrix(kind, n, k, d)
        assert info["nnz"] == int((G2 != 0).sum())
        for f in range(n):
            want = 1 if kind == 3 else O.repair_reads(kind, n, k, d, f)
            assert pm.pmrc_read_cost(c, f) == want
    finally:
        pm.pmrc_destroy(c)


def test_info_config2():
    c = pm.pmrc_create(pm.PMRC_MSR_SPARSE, 8, 14, 16)
    info = pm.pmrc_info(c)
    pm.pmrc_destroy(c)
    assert (info["alpha"], info["B"], info["parity_rows"], info["nnz"]) == (7, 56, 56, 784)
    assert info["zero_pct"] == 75.0
    assert info["repair_complete"] == 0          # R10: n = 2k
    assert info["xor_ops_naive"] == 12584        # SURVEY §8(d) W for config 2
    assert 0 < info["xor_ops"] < 2 * info["xor_ops_naive"]


def test_create_errors():
    with pytest.raises(pm.PmrcError) as e:
        pm.pmrc_create(pm.PMRC_MSR_SPARSE, 3, 3, 6)   # MSR needs d = 2k-2
    assert e.value.rc == pm.PMRC_EUNSUPPORTED
    with pytest.raises(pm.PmrcError) as e:
        pm.pmrc_create(pm.PMRC_MSR_SPARSE, 8, 14, 16, w=12)        # only w = 8 and (encode) w = 16
    assert e.value.rc == pm.PMRC_EUNSUPPORTED
    with pytest.raises(pm.PmrcError) as e:
        pm.pmrc_create(pm.PMRC_MSR_VANILLA, 16, 30, 32)  # R8 lambda collision
    assert e.value.rc == pm.PMRC_EUNSUPPORTED
    with pytest.raises(pm.PmrcError):
        pm.pmrc_create(pm.PMRC_MBR, 8, 14, 14)           # n must exceed d


def test_argument_errors_without_gpu_work():
    c = pm.pmrc_create(pm.PMRC_MSR_SPARSE, 3, 4, 6)
    try:
        with pytest.raises(pm.PmrcError) as e:
            pm.pmrc_encode(c, 16, 16, 24, 1)              # S % 16 != 0
        assert e.value.rc == pm.PMRC_EALIGN
        with pytest.raises(pm.PmrcError) as e:
            pm.pmrc_encode(c, 8, 16, 32, 1)               # misaligned pointer
        assert e.value.rc == pm.PMRC_EALIGN
        pm.pmrc_encode(c, 16, 16, 0, 5)                   # empty: no work, no error
        pm.pmrc_encode(c, 16, 16, 32, 0)
        with pytest.raises(pm.PmrcError) as e:
            pm.pmrc_repair(c, 0, [0, 1, 2, 3], [(16, 0)] * 4, (16, 0), 32, 1)   # lost among helpers
        assert e.value.rc == pm.PMRC_EINVAL
        with pytest.raises(pm.PmrcError) as e:
            pm.pmrc_repair(c, 0, [1, 2, 3], [(16, 0)] * 3, (16, 0), 32, 1)      # needs d helpers
        assert e.value.rc == pm.PMRC_EINVAL
        with pytest.raises(pm.PmrcError) as e:
            pm.pmrc_decode(c, [0, 0, 1], [(16, 0)] * 3, 16, 32, 1)            # duplicate ids
        assert e.value.rc == pm.PMRC_EINVAL
    finally:
        pm.pmrc_destroy(c)


def test_no_silent_cpu_fallback():
    # without a GPU the data path must fail loudly (PMRC_ECUDA), never compute on the CPU
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    c = pm.pmrc_create(pm.PMRC_MSR_SPARSE, 3, 4, 6)
    try:
        with pytest.raises(pm.PmrcError) as e:
            pm.pmrc_encode(c, 16, 16, 32, 1)
        assert e.value.rc == pm.PMRC_ECUDA
    finally:
        pm.pmrc_destroy(c)


def test_plan_stats_and_source_without_gpu():
    # plan generation is host-only: the per-stripe work of the config-2 plans
    c = pm.pmrc_create(pm.PMRC_MSR_SPARSE, 8, 14, 16)
    try:
        enc = pm.pmrc_plan_stats(c, 2)
        assert (enc["groups"], enc["in_blocks"], enc["out_blocks"], enc["naive_lop3"]) == (7, 56, 56, 12584)
        assert enc["transposes"] == 7 * (14 + 8)          # every group: its 14 inputs + 8 outputs
        dec = pm.pmrc_plan_stats(c, 0, 0, list(range(4, 12)))
        assert dec["out_blocks"] == 4 * 7 and dec["in_blocks"] == 56   # nodes 0..3 lost
        rep_par = pm.pmrc_plan_stats(c, 1, 15, [i for i in range(16) if i not in (15, 10)])
        assert (rep_par["in_blocks"], rep_par["out_blocks"]) == (14 * 7, 7)     # f >= alpha: alpha blocks each
        rep_sys = pm.pmrc_plan_stats(c, 1, 2, [i for i in range(16) if i not in (2, 12)])
        assert (rep_sys["in_blocks"], rep_sys["out_blocks"]) == (14, 7)          # f < alpha: 1 block each
        with pytest.raises(pm.PmrcError) as e:                                    # R10 singular set
            pm.pmrc_plan_stats(c, 1, 0, [i for i in range(16) if i not in (0, 1)])
        assert e.value.rc == pm.PMRC_ESINGULAR
        with pytest.raises(pm.PmrcError) as e:                                    # all data survives
            pm.pmrc_plan_stats(c, 0, 0, list(range(8)))
        assert e.value.rc == pm.PMRC_EINVAL
        src = pm.pmrc_plan_source(c, 1, 15, [i for i in range(16) if i not in (15, 10)])
        assert "pmrc_kernel" in src and "lop3" in src
        # schedules: the config-4 decode takes chunks from per-group counters (and helps the other
        # group when its own run out); the encode keeps static, aligned chunk ranges
        dsrc = pm.pmrc_plan_source(c, 0, 0, [0, 1, 4, 5, 9, 12, 14, 15])
        assert "atomicAdd(dctr, 1u)" in dsrc and "for (u32 hop = 0; hop < 2u; hop++)" in dsrc
        esrc = pm.pmrc_encode_source(c)
        assert "atomicAdd" not in esrc and "c1 = (u32)((u64)total * (r + 1u) / spg)" in esrc
    finally:
        pm.pmrc_destroy(c)


def test_tuned_plan_shapes_without_gpu():
    # the measured defaults: 16 warps per CTA, static ranges for the sparse encode,
    # group-specialised 8-row groups with the stealing counters for k = 16, and the stealing
    # counters for GF(2^16) k = 8 (14 groups)
    c = pm.pmrc_create(pm.PMRC_MSR_SPARSE, 8, 14, 16)
    try:
        src = pm.pmrc_encode_source(c)
        assert "__launch_bounds__(512, 1)" in src and "atomicAdd" not in src
        assert pm.pmrc_plan_stats(c, 2)["xor2"] <= 12305          # best of 4 CSE runs
    finally:
        pm.pmrc_destroy(c)
    c = pm.pmrc_create(pm.PMRC_MSR_SPARSE, 16, 30, 32)
    try:
        st = pm.pmrc_plan_stats(c, 2)
        assert st["groups"] == 30                                  # 8-row groups (auto_wide16)
        assert "for (u32 hop = 0; hop < 30u; hop++)" in pm.pmrc_encode_source(c)   # layout 1, dyn 2
    finally:
        pm.pmrc_destroy(c)
    c = pm.pmrc_create(pm.PMRC_MSR_SPARSE, 8, 14, 16, 16)
    try:
        assert "for (u32 hop = 0; hop < 14u; hop++)" in pm.pmrc_encode_source(c)
    finally:
        pm.pmrc_destroy(c)
    # one group of 9-16 rows: decodes (clustered rows) on 12 warps with 8-input sub-networks, the
    # MBR fused repair (parity node: 14 stages; systematic node: ALU-heavy) on 12 warps too
    c = pm.pmrc_create(pm.PMRC_MBR, 8, 14, 16)
    try:
        assert pm.pmrc_plan_stats(c, 2)["xor2"] <= 19700          # + the input / row partition search
        dec = pm.pmrc_plan_source(c, 0, 0, [0, 1, 4, 5, 6, 7, 11, 14])
        assert "__launch_bounds__(384, 1)" in dec
        assert pm.pmrc_plan_stats(c, 0, 0, [0, 1, 4, 5, 6, 7, 11, 14])["xor2"] <= 6927
        rep = pm.pmrc_plan_source(c, 1, 15, list(range(14)))
        assert "__launch_bounds__(384, 1)" in rep
        rep = pm.pmrc_plan_source(c, 1, 3, [i for i in range(15) if i != 3])
        assert "__launch_bounds__(384, 1)" in rep                  # systematic node: ALU-heavy class
    finally:
        pm.pmrc_destroy(c)


def test_partition_search_is_deterministic_and_optional(monkeypatch):
    # encode plans of unequal groups search the input / row partition of their CSE
    # sub-networks (parallel host threads, fixed seeds): the same source every time, fewer XORs than
    # the unsearched plan, the same naive count (the matrix is untouched); part_search < 0 searches
    # every plan, enc_part_search=0 none
    def stats_and_source(kind, k, d, n):
        c = pm.pmrc_create(kind, k, d, n)
        try:
            return pm.pmrc_plan_stats(c, 2), pm.pmrc_encode_source(c)
        finally:
            pm.pmrc_destroy(c)
    st1, src1 = stats_and_source(pm.PMRC_MBR, 8, 14, 16)
    st2, src2 = stats_and_source(pm.PMRC_MBR, 8, 14, 16)
    assert src1 == src2 and st1 == st2
    monkeypatch.setenv("PMRC_GEN", "enc_part_search=0")
    st0, src0 = stats_and_source(pm.PMRC_MBR, 8, 14, 16)
    assert st0["naive_lop3"] == st1["naive_lop3"] and st1["xor2"] < st0["xor2"] and src0 != src1
    msr0, _ = stats_and_source(pm.PMRC_MSR_SPARSE, 4, 6, 8)
    monkeypatch.setenv("PMRC_GEN", "part_search=-60")
    msr1, _ = stats_and_source(pm.PMRC_MSR_SPARSE, 4, 6, 8)      # equal groups: searched only on request
    assert msr1["xor2"] <= msr0["xor2"] and msr1["naive_lop3"] == msr0["naive_lop3"]
    monkeypatch.delenv("PMRC_GEN")
    msr2, _ = stats_and_source(pm.PMRC_MSR_SPARSE, 4, 6, 8)
    assert msr2 == msr0


def test_independent_launches_flag_without_gpu():
    c = pm.pmrc_create(pm.PMRC_MSR_SPARSE, 8, 14, 16)
    try:
        pm.pmrc_set_independent_launches(c, 1)     # nothing built yet: no device work
        assert "griddepcontrol.launch_dependents" in pm.pmrc_encode_source(c)
        assert "griddepcontrol.wait" not in pm.pmrc_encode_source(c)
        pm.pmrc_set_independent_launches(c, 0)
        assert "griddepcontrol" not in pm.pmrc_encode_source(c)
        with pytest.raises(pm.PmrcError) as e:
            pm.pmrc_set_independent_launches(c, 2)
        assert e.value.rc == pm.PMRC_EINVAL
    finally:
        pm.pmrc_destroy(c)


def test_prepare_plans_parallel_without_gpu():
    # config-4-style patterns compiled in parallel host threads (no GPU): singular helper sets (R10)
    # and all-systematic survivor sets are reported, the rest compile
    pats = [("repair", 15, [i for i in range(16) if i not in (15, 3)]),
            ("repair", 0, [i for i in range(16) if i not in (0, 1)]),        # R10 singular
            ("decode", [0, 1, 2, 3, 12, 13, 14, 15]),
            ("decode", list(range(8)))]                                      # nothing to decode
    res = dict((str(p), rc) for p, rc in pm.prepare_plans(pm.PMRC_MSR_SPARSE, 3, 4, 6, []))
    assert res == {}
    out = pm.prepare_plans(pm.PMRC_MSR_SPARSE, 8, 14, 16, pats, threads=2)
    rcs = {str(p): rc for p, rc in out}
    assert rcs[str(pats[0])] == pm.PMRC_OK and rcs[str(pats[2])] == pm.PMRC_OK
    assert rcs[str(pats[1])] == pm.PMRC_ESINGULAR
    assert rcs[str(pats[3])] == pm.PMRC_EINVAL


def test_gf16_code_host_side():
    # w = 16: the sparse MSR code builds, keeps Table 1's sparsity; encode, decode
    # and fused repair run, the other operations are refused loudly
    c = pm.pmrc_create(pm.PMRC_MSR_SPARSE, 8, 14, 16, w=16)
    try:
        info = pm.pmrc_info(c)
        assert (info["w"], info["B"], info["parity_rows"], info["nnz"], info["zero_pct"]) == (16, 56, 56, 784, 75.0)
        with pytest.raises(pm.PmrcError) as e:
            pm.pmrc_repair_project(c, 15, (16, 0), (16, 0), 32, 1)
        assert e.value.rc == pm.PMRC_EUNSUPPORTED
        with pytest.raises(pm.PmrcError) as e:
            pm.pmrc_matrix(c, pm.MATRIX_GPP)
        assert e.value.rc == pm.PMRC_EUNSUPPORTED
        assert "pm_tr16" in pm.pmrc_encode_source(c)
    finally:
        pm.pmrc_destroy(c)
    for kind in (pm.PMRC_MSR_VANILLA, pm.PMRC_MBR, pm.PMRC_RS_VANDERMONDE):
        with pytest.raises(pm.PmrcError) as e:
            pm.pmrc_create(kind, 8, 8 if kind == pm.PMRC_RS_VANDERMONDE else 14, 16, w=16)
        assert e.value.rc == pm.PMRC_EUNSUPPORTED
