"""Particle sharding across GPUs: one process per GPU over torch.distributed.

The path shards naturally: particles are independent, the
volumes are replicated, and the only exchange per SMC iteration is one
all-gather of the per-particle likelihoods.  Every rank then runs the same
deterministic update (weights, ESS, resampling, estimate) on identical
inputs, so no broadcast is needed and results are GPU-count invariant.

The host logic here is backend-agnostic (NCCL on GPUs, gloo in the CPU
tests) and is exercised with world_size 2 on CPU by tests/test_dist.py.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class ShardPlan:
    """Contiguous, padded particle ranges: rank r owns [lo, hi) of n."""

    n: int
    world: int
    rank: int

    @property
    def shard(self) -> int:
        """Padded per-rank slot size (all_gather needs equal sizes)."""
        return -(-self.n // self.world)

    @property
    def lo(self) -> int:
        return min(self.n, self.rank * self.shard)

    @property
    def hi(self) -> int:
        return min(self.n, self.lo + self.shard)

    @property
    def count(self) -> int:
        return self.hi - self.lo


def world():
    """(world_size, rank, group-initialised) from torch.distributed."""
    try:
        import torch.distributed as td
    except Exception:  # pragma: no cover
        return 1, 0, False
    if td.is_available() and td.is_initialized():
        return td.get_world_size(), td.get_rank(), True
    return 1, 0, False


def plan(n: int) -> ShardPlan:
    w, r, _ = world()
    return ShardPlan(n, w, r)


def allgather_shards(local, plan: ShardPlan, out):
    """Gather every rank's padded shard of ``local`` (length plan.shard) into
    ``out`` (length plan.shard * world) and return the first n entries (on a
    single rank: ``local`` itself, no copy)."""
    import torch.distributed as td

    if plan.world == 1:
        return local[: plan.n]   # the local shard is the whole set: no copy
    td.all_gather_into_tensor(out, local)
    return out[: plan.n]


def packed_block_bytes(shard: int) -> int:
    """Bytes of one rank's packed block [z: shard f64 | flags: shard u8 | pad
    to 8] (er_smc_update_gathered)."""
    return -(-(9 * shard) // 8) * 8


def allgather_packed(local, out):
    """The one collective of an SMC iteration: every rank's packed uint8
    block into ``out`` (world blocks, rank order).  Under a host-staged
    process group (gloo, the CPU tests and the single-GPU multi-rank test)
    the device block is staged through host memory."""
    return allgather_tensor(local, out)


def allgather_tensor(local, out):
    """all_gather_into_tensor on the default group: NCCL directly on device
    tensors; other backends (gloo) through host memory."""
    import torch.distributed as td

    if td.get_backend() == "nccl" or local.device.type == "cpu":
        td.all_gather_into_tensor(out, local)
        return out
    host = local.cpu()
    gathered = host.new_empty(out.numel())
    td.all_gather_into_tensor(gathered, host)
    out.copy_(gathered)
    return out


def allgather_rows(local, plan: ShardPlan):
    """Gather every rank's padded (plan.shard, k) float64 block of host rows
    (numpy) and return the first plan.n rows, in rank order.  Used for the
    per-frame scores of the 4D pipeline: small, so the
    exchange goes through the default group's device (NCCL: the current CUDA
    device; gloo: host memory)."""
    import numpy as np

    local = np.ascontiguousarray(local, dtype=np.float64)
    if plan.world == 1:
        return local[: plan.n].copy()
    import torch
    import torch.distributed as td

    dev = torch.device("cuda", torch.cuda.current_device()) \
        if td.get_backend() == "nccl" else torch.device("cpu")
    src = torch.from_numpy(local).to(dev).reshape(-1)
    out = torch.empty(src.numel() * plan.world, dtype=torch.float64, device=dev)
    td.all_gather_into_tensor(out, src)
    return out.cpu().numpy().reshape(plan.world * plan.shard, -1)[: plan.n]
