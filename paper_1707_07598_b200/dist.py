"""Multi-GPU plumbing for the benchmark: independent replicas, one process per
GPU (torch.distributed over NCCL on GPUs, gloo on CPU for tests).

The MSFV path does not shard in this tier ("replicas only"): each
rank runs the full forward+gradient on its own model; the only cross-rank
traffic is the barrier around the timed region and the max-reduction of the
device-measured step time.
"""

import os

import torch
import torch.distributed as dist


def world():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def init(backend=None):
    rank, size = world()
    if size > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        dist.init_process_group(backend, init_method="env://")
    return rank, size


def barrier():
    if dist.is_initialized():
        dist.barrier()


def max_over_ranks(value, device=None):
    """Max of a float over all ranks (the slowest replica sets the step time)."""
    if not dist.is_initialized():
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else ("cuda" if dist.get_backend() == "nccl" else "cpu"))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_seed(base_seed, rank):
    """Each replica inverts its own seeded model (independent units of work)."""
    return int(base_seed) + 1000 * int(rank)


def aggregate_seconds_per_iter(step_seconds_max, n_replicas):
    """Whole-job s/iter: n_replicas forward+gradient iterations finish every
    step_seconds_max seconds (weak scaling, fixed work per GPU)."""
    return float(step_seconds_max) / max(1, int(n_replicas))
