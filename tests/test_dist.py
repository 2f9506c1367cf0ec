"""CPU tier: the multi-GPU host logic (sharding, max-over-ranks timing, aggregate throughput) on
a world_size-2 gloo process group; plus per-rank encodes through the oracle covering exactly the
job's stripes (no data-path collective)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1412_3022_b200 import dist as pdist


def test_shard_covers_exactly():
    for total in (0, 1, 7, 19, 64):
        for world in (1, 2, 3, 8):
            spans = [pdist.shard(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        pdist.shard(10, 2, 2)


def test_aggregate():
    assert pdist.aggregate_gbps(1e9, 8, 0.5) == 16.0
    assert pdist.global_offset(3, 19, 56, 1 << 20) == 3 * 19 * 56 * (1 << 20)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import inputs
    import oracle as O
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # strong scaling: 5 stripes of k=3 MSR split over 2 ranks; each rank encodes its own stripes
    k, n, d, S, total = 3, 6, 4, 64, 5
    lo, hi = pdist.shard(total, world, rank)
    B = 6
    x = inputs.stripe_data(hi - lo, B, S, seed=9, t0=lo)
    par = O.encode(O.MSR_SPARSE, n, k, d, x)
    elapsed = 0.25 + rank   # a fake per-rank time: the max rule must pick the slowest
    m = pdist.max_over_ranks(elapsed, dist)
    q.put((rank, lo, hi, par.tobytes(), m))
    dist.destroy_process_group()


def test_two_rank_gloo_sharded_encode_and_max_time():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    import inputs
    import oracle as O
    full = O.encode(O.MSR_SPARSE, 6, 3, 4, inputs.stripe_data(5, 6, 64, seed=9))
    got = np.concatenate([np.frombuffer(r[3], np.uint8).reshape(r[2] - r[1], 6, 64) for r in res])
    assert np.array_equal(got, full)          # the ranks' stripes tile the job exactly
    assert all(r[4] == 1.25 for r in res)     # max over ranks, seen by every rank


def _repair_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import inputs
    import oracle as O
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # MSR k=4 n=8 (d=6): nodes spread over the ranks, the lost node's newcomer on owner[f]
    kind, k, n, d, S = O.MSR_SPARSE, 4, 8, 6, 96
    alpha, B = O.params(kind, n, k, d)
    code = O.full_code(kind, n, k, d, inputs.stripe_data(1, B, S, seed=13)[0])   # (n, alpha, S)
    owner = {i: i % world for i in range(n)}
    res = []
    for f, H in ((5, [0, 1, 2, 3, 4, 6]), (1, [0, 2, 3, 5, 6, 7])):
        pieces = {h: torch.from_numpy(code[h].copy()) for h in H if owner[h] == rank}
        out = torch.zeros((alpha, S), dtype=torch.uint8)

        def project(h, piece):
            return torch.from_numpy(O.repair_project(kind, n, k, d, f, piece.numpy()))

        def combine(ids, betas, dst):
            dst.copy_(torch.from_numpy(O.repair_combine(kind, n, k, d, f, ids, torch.stack(betas).numpy())))
        sent = pdist.distributed_repair(f, H, owner, pieces, out, project, combine,
                                        torch.empty(S, dtype=torch.uint8), dist, rank)
        res.append((f, sent, out.numpy().tobytes() if owner[f] == rank else None,
                    code[f].tobytes()))
    q.put((rank, res))
    dist.destroy_process_group()


def test_two_rank_gloo_distributed_repair():
    # NEXT-3: helpers project locally, ship one block each to the newcomer's rank, which combines;
    # the regenerated piece is exact and each rank sends exactly its remote helpers' betas
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_repair_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    S = 96
    for idx, (f, H) in enumerate(((5, [0, 1, 2, 3, 4, 6]), (1, [0, 2, 3, 5, 6, 7]))):
        new_rank = f % world
        got = res[new_rank][idx][2]
        assert got == res[new_rank][idx][3]                      # exact regeneration
        for r in range(world):
            remote = sum(1 for h in H if h % world == r and r != new_rank)
            assert res[r][idx][1] == remote * S                   # d blocks in total, one per helper
