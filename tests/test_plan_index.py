"""CPU tier: the kernel cache's plan index (csrc/host/plan.cpp).  Compiling a plan (NVRTC, no GPU
needed) stores its cubin under the source key and a <plan key>.meta index entry that names that
cubin, so a later build of the same plan (same spec, generator options and library build) loads the
cubin without generating the source again; other options index separately."""
import os

import paper_1412_3022_b200 as pm


def _entries(d):
    return sorted(f for f in os.listdir(d) if f.endswith(".meta")), sorted(f for f in os.listdir(d) if f.endswith(".cubin"))


def test_plan_index_names_the_compiled_cubin(tmp_path, monkeypatch):
    monkeypatch.setenv("PMRC_KCACHE", str(tmp_path))
    code = pm.pmrc_create(pm.PMRC_MSR_SPARSE, 3, 4, 6)
    try:
        src = pm.pmrc_plan_source(code, 1, 5, [0, 1, 2, 3], compile=True)
        metas, cubins = _entries(tmp_path)
        assert len(metas) == 1 and len(cubins) == 1
        lines = (tmp_path / metas[0]).read_text().split("\n")
        assert lines[0] == "pmrc-plan-meta 1"
        assert lines[1] + ".cubin" == cubins[0]
        # the cubin key is the generated source's (FNV-1a 64 + length)
        h = 1469598103934665603
        for b in src.encode():
            h = ((h ^ b) * 1099511628211) & (2 ** 64 - 1)
        assert lines[1] == "%016x_%d" % (h, len(src.encode()))
        stats = lines[2].split()
        assert int(stats[0]) >= 1                     # groups
        opts = [int(v) for v in lines[3].split()]
        assert opts[0] % 32 == 0 and opts[0] == 32 * opts[4]   # tpb = 32 x warps
        # compiling again finds the index (no new entries); another plan adds one of each
        pm.pmrc_plan_source(code, 1, 5, [0, 1, 2, 3], compile=True)
        assert _entries(tmp_path) == (metas, cubins)
        pm.pmrc_plan_source(code, 0, 0, [3, 4, 5], compile=True)
        m2, c2 = _entries(tmp_path)
        assert len(m2) == 2 and len(c2) == 2
    finally:
        pm.pmrc_destroy(code)


def test_plan_index_key_follows_generator_options(tmp_path, monkeypatch):
    monkeypatch.setenv("PMRC_KCACHE", str(tmp_path))
    code = pm.pmrc_create(pm.PMRC_MSR_SPARSE, 3, 4, 6)
    monkeypatch.setenv("PMRC_GEN", "net_in=3")
    code2 = pm.pmrc_create(pm.PMRC_MSR_SPARSE, 3, 4, 6)
    try:
        pm.pmrc_plan_source(code, 1, 5, [0, 1, 2, 3], compile=True)
        pm.pmrc_plan_source(code2, 1, 5, [0, 1, 2, 3], compile=True)
        metas, _ = _entries(tmp_path)
        assert len(metas) == 2                         # same plan, other options: its own entry
    finally:
        pm.pmrc_destroy(code)
        pm.pmrc_destroy(code2)


def test_promotion_controls_without_a_gpu():
    # the AUTO promotion knobs are host state: a pattern never run is on the runtime kernel (0),
    # bad ops are EINVAL, and the threshold accepts any 64-bit value (0 = off)
    code = pm.pmrc_create(pm.PMRC_MSR_SPARSE, 3, 4, 6)
    try:
        assert pm.pmrc_plan_state(code, 0, 0, [0, 1, 5]) == pm.PLAN_RUNTIME_ONLY
        assert pm.pmrc_plan_state(code, 1, 5, [0, 1, 2, 3]) == pm.PLAN_RUNTIME_ONLY
        for v in (0, 1, 1 << 30, 2 ** 64 - 1):
            pm.pmrc_set_auto_promotion(code, v)
        try:
            pm.pmrc_plan_state(code, 2, 0, [0, 1, 2])
            raise AssertionError("op 2 accepted")
        except pm.PmrcError as e:
            assert e.rc == pm.PMRC_EINVAL
    finally:
        pm.pmrc_destroy(code)
