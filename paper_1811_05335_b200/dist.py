"""Multi-GPU plumbing (torch.distributed; NCCL on GPUs, gloo on CPU tests).

The direct inverse NFFT is applied to many right-hand sides for FIXED nodes
(P:76), and the right-hand sides are independent, so the batch is sharded
across ranks with no collective on the data path (weak scaling: every rank
owns R_loc right-hand sides and a replica of the plan).  Collectives appear
only around the data path:
  * a checksum all-gather proving every rank built the same B_opt (setup),
  * the max-over-ranks reduction of the device time (measurement).
"""
import hashlib

import numpy as np


def shard(R_total, rank, world):
    """Contiguous shard [start, start + count) of R_total right-hand sides."""
    base, extra = divmod(R_total, world)
    count = base + (1 if rank < extra else 0)
    start = rank * base + min(rank, extra)
    return start, count


def bopt_digest(w):
    """64-bit digest of a B_opt weight array (bit-exact comparison across ranks)."""
    h = hashlib.sha256(np.ascontiguousarray(w).view(np.uint8)).digest()
    return int.from_bytes(h[:8], "little", signed=True)


def check_same_bopt(w, dist, device=None):
    """All ranks must hold bit-identical B_opt (deterministic setup); returns the digests."""
    import torch
    d = torch.tensor([bopt_digest(w)], dtype=torch.int64, device=device)
    out = [torch.zeros_like(d) for _ in range(dist.get_world_size())]
    dist.all_gather(out, d)
    vals = [int(t.item()) for t in out]
    if len(set(vals)) != 1:
        raise RuntimeError(f"B_opt differs across ranks: {vals}")
    return vals


def max_over_ranks(value, dist, device=None):
    """Max of a float over ranks (the bench's time is the slowest rank)."""
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
