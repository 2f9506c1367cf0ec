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
