"""NEXT-3 over a real interconnect (-m gpu): distributed repair with the helpers on two GPUs and
the newcomer on one of them, NCCL point-to-point over NVLink, the product's projection / combine
kernels on each rank.  Needs >= 2 visible GPUs; skipped otherwise (one GPU per gpurun box), so the
path runs the moment a multi-GPU box is available.  The CPU tier covers the same orchestration with
gloo (tests/test_dist.py)."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import inputs
    import paper_1412_3022_b200 as pm
    from paper_1412_3022_b200 import dist as pdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        k, n, d, S, stripes = 8, 16, 14, 64 * 1024, 3
        code = pm.pmrc_create(pm.PMRC_MSR_SPARSE, k, d, n)
        info = pm.pmrc_info(code)
        a, B, P = info["alpha"], info["B"], info["parity_rows"]
        # every rank holds the whole (seeded, identical) codeword; node i is "owned" by rank i % world
        data = torch.from_numpy(inputs.stripe_data(stripes, B, S, 123)).to(dev)
        par = torch.empty((stripes, P, S), dtype=torch.uint8, device=dev)
        st = torch.cuda.current_stream().cuda_stream
        pm.pmrc_encode(code, data.data_ptr(), par.data_ptr(), S, stripes, st)

        def piece(i):
            return (par.data_ptr() + (i - k) * a * S, P * S) if i >= k else (data.data_ptr() + i * a * S, B * S)
        f = 12
        H = [i for i in range(n) if i not in (f, 3)]
        owner = {i: i % world for i in range(n)}

        def project(h, pc):
            b = torch.empty((stripes, S), dtype=torch.uint8, device=dev)
            pm.pmrc_repair_project(code, f, pc, (b.data_ptr(), S), S, stripes, st)
            return b

        def combine(ids, betas, dst):
            pm.pmrc_repair_combine(code, f, ids, [(b.data_ptr(), S) for b in betas], (dst.data_ptr(), a * S), S,
                                   stripes, st)
        out = torch.zeros((stripes, a, S), dtype=torch.uint8, device=dev)
        sent = pdist.distributed_repair(f, H, owner, {h: piece(h) for h in H if owner[h] == rank}, out, project,
                                        combine, torch.empty((stripes, S), dtype=torch.uint8, device=dev), dist, rank)
        torch.cuda.synchronize()
        ok = True
        if rank == owner[f]:
            ok = bool(torch.equal(out, par[:, (f - k) * a:(f - k + 1) * a]))
        q.put((rank, ok, sent))
        pm.pmrc_destroy(code)
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_distributed_repair_nccl_two_gpus():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(60)
    assert all(ok for _, ok, _ in res)
    # the newcomer's rank receives d/2 betas of one block per stripe from the other rank
    sent = {r: s for r, _, s in res}
    assert sent[1 - (12 % world)] == 7 * 3 * 64 * 1024
