"""Batched SVD across the GPUs of one node (BASELINE config 5).

A single SVD does not shard; a batch of independent matrices
does: rank r of W takes the contiguous slice ``shard_range(B, W, r)`` and
solves it on its own GPU with ``gesdd_batched`` -- no data-path collective.
The only communication is the optional final gather of (sigma, U, Vt) to the
owner rank.  Launch one process per GPU (torchrun); the process group backend
is NCCL on GPUs (gloo works for host-side tests).
"""

import torch
import torch.distributed as dist


def shard_range(total, world_size, rank):
    """[lo, hi) of `total` items owned by `rank` (contiguous, sizes differ by
    at most one, lower ranks take the remainder)."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError(f"bad rank {rank} for world size {world_size}")
    base, rem = divmod(total, world_size)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def gather_to_owner(local_items, dst=0, group=None):
    """Gather per-rank lists of tensors (each item a tuple of tensors) onto
    rank `dst` in global batch order.  Returns the full list on `dst`, None
    elsewhere.  Uses object gather (results are moved to CPU first), which is
    off the timed data path."""
    ws = dist.get_world_size(group)
    rank = dist.get_rank(group)
    payload = [tuple(t.detach().cpu() if isinstance(t, torch.Tensor) else t for t in item) for item in local_items]
    out = [None] * ws if rank == dst else None
    dist.gather_object(payload, out, dst=dst, group=group)
    if rank != dst:
        return None
    full = []
    for part in out:
        full.extend(part)
    return full


def gather_sigma(local_sigma, total, group=None):
    """All-gather the singular values of a sharded batch: ``local_sigma`` is
    this rank's (hi - lo) x k tensor for its ``shard_range`` slice; returns
    the total x k tensor in global batch order on every rank.  NCCL
    all-gather of device tensors (padded to the largest shard); with a gloo
    group the payload goes through host memory.  One 16 KiB row per SVD, off
    the timed path."""
    if not dist.is_initialized():
        return local_sigma
    ws = dist.get_world_size(group)
    k = int(local_sigma.shape[1]) if local_sigma.dim() == 2 else 0
    cap = -(-total // ws)
    on_gpu = dist.get_backend(group) == "nccl"
    buf = torch.zeros((cap, k), dtype=torch.float64, device=local_sigma.device if on_gpu else "cpu")
    buf[: local_sigma.shape[0]] = local_sigma.to(buf.device)
    out = torch.empty((ws * cap, k), dtype=torch.float64, device=buf.device)
    if on_gpu:
        dist.all_gather_into_tensor(out, buf, group=group)
    else:
        parts = [torch.empty_like(buf) for _ in range(ws)]
        dist.all_gather(parts, buf, group=group)
        out = torch.cat(parts)
    rows = []
    for r in range(ws):
        lo, hi = shard_range(total, ws, r)
        rows.append(out[r * cap: r * cap + (hi - lo)])
    return torch.cat(rows)


def batched_svd_sharded(make_matrix, total, options=None, gather=False):
    """Solve matrices [0, total) across the process group: this rank builds
    its slice with ``make_matrix(i)`` (returns an m x n array/tensor) and runs
    them on its GPU.  Returns this rank's results (and, with ``gather``, the
    full list on rank 0)."""
    from .svd import gesdd_batched

    ws = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    lo, hi = shard_range(total, ws, rank)
    mats = [make_matrix(i) for i in range(lo, hi)]
    res = gesdd_batched(mats, options) if mats else []
    if gather and ws > 1:
        return res, gather_to_owner([(r.sigma, r.u, r.vt) for r in res])
    return res, None
