"""Data parallelism for the DP backward.

Each rank owns a slice of the batch and produces, per layer, its clipped sum
scaled by 1/B_global (mean) plus noise on ITS slice of the layer's flat index
space only (fdp_noise_partition). One all-reduce (sum, fp32) per bucket then
yields exactly the single-GPU result: the clipped mean over the global batch
plus sigma*C*N(seed, layer, step, i) added once for every index i, so the
privacy accounting is unchanged. Per-sample norms and clip factors never cross
ranks.
"""

from __future__ import annotations

from typing import Iterable, Sequence

import torch
import torch.distributed as dist


def noise_partition(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous slice [lo, hi) of [0, n) whose noise `rank` adds (same arithmetic as fdp_noise_partition)."""
    if world < 1 or not (0 <= rank < world) or n < 0:
        raise ValueError("bad partition arguments")
    return n * rank // world, n * (rank + 1) // world


def flatten_bucket(tensors: Sequence[torch.Tensor]) -> torch.Tensor:
    return torch.cat([t.reshape(-1) for t in tensors])


def allreduce_grads_(grads: Iterable[torch.Tensor], group=None, bucket_bytes: int = 256 << 20) -> None:
    """Sum the per-rank DP gradients in place (NCCL over NVLink on B200, gloo in tests),
    in buckets of `bucket_bytes`."""
    grads = [g for g in grads if g is not None]
    bucket: list[torch.Tensor] = []
    size = 0

    def flush():
        nonlocal bucket, size
        if not bucket:
            return
        flat = flatten_bucket(bucket)
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
        off = 0
        for t in bucket:
            n = t.numel()
            t.copy_(flat[off:off + n].view_as(t))
            off += n
        bucket, size = [], 0

    for g in grads:
        bucket.append(g)
        size += g.numel() * g.element_size()
        if size >= bucket_bytes:
            flush()
    flush()
