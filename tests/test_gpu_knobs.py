"""GPU parity (-m gpu) of non-default generator / runtime-kernel shapes that PMRC_GEN accepts (only
result-preserving options are accepted, include/pmrc.h): a 3-deep stage ring under the dynamic
chunk schedule (the decode and the parity-node repair plans), and 8-row runtime thread blocks for
plans that default to 7.  Each is checked against the unique answer (the data, the encoded piece)
of parity that is itself checked against the oracle."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_1412_3022_b200 as pm
from gpu_util import DEV, Stripes, oracle_kind

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("gen,policy", [("nbuf=3", pm.PMRC_PLAN_JIT), ("nbuf=4,in_block=8", pm.PMRC_PLAN_JIT),
                                        ("rt_rows=8", pm.PMRC_PLAN_RUNTIME)])
def test_decode_and_repair_with_non_default_shapes(monkeypatch, gen, policy):
    monkeypatch.setenv("PMRC_GEN", gen)
    k, n, S, stripes = 8, 16, 8192 + 1024 + 16, 5    # several chunks per stripe and a ragged tail
    st = Stripes(pm.PMRC_MSR_SPARSE, k, n, S, stripes, seed=41, policy=policy)
    try:
        st.encode()
        assert np.array_equal(st.parity.cpu().numpy(),
                              O.encode(oracle_kind(st.kind), n, k, st.d, st.host_data()))
        ids = [0, 1, 4, 5, 9, 12, 14, 15]                 # 4 missing nodes: 28 rows, multi-stage plan
        out = torch.full_like(st.data, 0x5A)
        nw = pm.pmrc_decode(st.code, ids, [st.piece(i) for i in ids], out.data_ptr(), S, stripes, st.stream)
        torch.cuda.synchronize()
        assert nw == 28
        miss = [b for b in range(st.B) if b // st.alpha not in ids]
        assert torch.equal(out[:, miss], st.data[:, miss])
        for f in (15, 6):                                  # parity node (98 blocks, 7 stages), systematic
            H = [i for i in range(n) if i != f][:st.d]
            piece = torch.full((stripes, st.alpha, S), 0x3C, dtype=torch.uint8, device=DEV)
            pm.pmrc_repair(st.code, f, H, [st.piece(i) for i in H], (piece.data_ptr(), st.alpha * S), S, stripes,
                           st.stream)
            torch.cuda.synchronize()
            assert torch.equal(piece, st.piece_tensor(f)), f
    finally:
        st.close()


@pytest.mark.parametrize("kind,k,n", [(pm.PMRC_MSR_SPARSE, 8, 16), (pm.PMRC_MSR_SPARSE, 16, 32), (pm.PMRC_MBR, 4, 8)])
def test_encode_with_the_partition_search_on_every_plan(monkeypatch, kind, k, n):
    # part_search < 0: equal groups and multi-stage groups (k = 16) are searched too; the reordered
    # inputs / rows must not change a byte
    monkeypatch.setenv("PMRC_GEN", "part_search=-40")
    S, stripes = 2048 + 1024 + 16, 2
    st = Stripes(kind, k, n, S, stripes, seed=43)
    try:
        st.encode()
        assert np.array_equal(st.parity.cpu().numpy(),
                              O.encode(oracle_kind(st.kind), n, k, st.d, st.host_data()))
    finally:
        st.close()
