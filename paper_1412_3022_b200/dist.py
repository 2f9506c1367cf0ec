"""Multi-GPU plumbing for the encode path: stripes are independent, so ranks never
exchange data; torch.distributed (NCCL on GPUs, gloo in the CPU tests) is used only for the
barrier before/after the timed region and the max-over-ranks reduction of the elapsed time.

Weak scaling: every rank encodes its own `stripes_per_rank` stripes (the headline bench: 1 GiB of
source per GPU).  Strong scaling (a fixed total split over ranks) is provided by `shard()`.
"""


def shard(total, world, rank):
    """Contiguous [lo, hi) of `total` stripes owned by `rank` (balanced to within one stripe)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def global_offset(rank, stripes_per_rank, blocks, S):
    """Global source offset of a rank's first byte in the weak-scaling layout (each rank owns
    `stripes_per_rank` consecutive stripes of a job-wide stream)."""
    return rank * stripes_per_rank * blocks * S


def max_over_ranks(value, dist=None, device=None):
    """Max of a float over all ranks (the bench's elapsed-time rule); identity without a group."""
    if dist is None or not dist.is_available() or not dist.is_initialized():
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_gbps(bytes_per_rank, world, max_seconds):
    """Whole-job throughput: all ranks' bytes over the slowest rank's time."""
    return world * bytes_per_rank / max_seconds / 1e9


def distributed_repair(lost_id, helper_ids, owner, pieces, newcomer_out, project, combine, beta_like, dist=None,
                       rank=0):
    """Exact repair with the helpers and the newcomer on different ranks (the
    network step the codes exist to minimise, P:42, P:53 footnote): every rank projects the pieces
    of the helpers it owns onto phi_f / psi_f (``project(h, piece) -> beta``, the product's
    pmrc_repair_project on GPUs), ships each beta -- one block per stripe, d blocks in all instead
    of k*alpha for a decode-based repair -- to the newcomer's rank (point-to-point send/recv: NCCL
    over NVLink on GPUs, gloo in the CPU tests), and the newcomer's rank combines them
    (``combine(helper_ids, betas) -> piece``, pmrc_repair_combine).

    owner: node id -> rank; pieces: {node id: piece} for the helpers this rank owns;
    beta_like: an empty tensor of the beta shape/dtype/device (receive buffers);
    newcomer_out: the caller's output (written on the newcomer's rank only, via combine).
    Returns the number of bytes this rank sent to another rank."""
    new_rank = owner[lost_id]
    betas = {}
    sent = 0
    reqs = []
    for h in helper_ids:
        if owner[h] != rank:
            continue
        b = project(h, pieces[h])
        if rank == new_rank:
            betas[h] = b
        else:
            reqs.append(dist.isend(b, dst=new_rank))   # per (src, dst) pair in helper order
            sent += b.numel() * b.element_size()
    if rank == new_rank:
        recv = {}
        for h in helper_ids:
            if owner[h] != rank:
                buf = beta_like.clone()
                recv[h] = (buf, dist.irecv(buf, src=owner[h]))
        for h, (buf, rq) in recv.items():
            rq.wait()
            betas[h] = buf
        combine(helper_ids, [betas[h] for h in helper_ids], newcomer_out)
    for rq in reqs:
        rq.wait()
    return sent
