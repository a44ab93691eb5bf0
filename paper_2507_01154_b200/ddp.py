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


class ChunkedAllReduceBackward:
    """The DP weight-gradient backward of a layer list as `n_chunks` fused
    persistent launches (PreparedGroup), each chunk's clipped + noised gradients
    summed over the ranks by an all-reduce on a communication stream while the
    next chunk computes (bucketed in layer order, overlapped with the
    rest of the backward). Under data parallelism each chunk's launch is capped
    at `sms - comm_sms` CTAs so the NCCL kernel has SMs to run on concurrently.

    layers: sequence of (x, dy, cfg); flat_grad: one fp32 buffer holding every
    layer's (D, P) gradient back to back in layer order (the all-reduce buckets
    are contiguous slices of it). `make_group(chunk_layers, grads, max_ctas)` can
    replace the device launch (tests on CPU pass a callable computing the same
    contribution)."""

    def __init__(self, layers, flat_grad: torch.Tensor, *, n_chunks: int = 4, comm_sms: int = 16,
                 noise_impl: str = "philox", rank: int = 0, world: int = 1, mean_batch: int = 0,
                 device_step: "torch.Tensor | None" = None, group=None, make_group=None):
        if n_chunks < 1:
            raise ValueError("n_chunks must be >= 1")
        self.world, self.group = world, group
        self.flat = flat_grad
        n = len(layers)
        n_chunks = min(n_chunks, n)
        bounds = [n * k // n_chunks for k in range(n_chunks + 1)]
        sizes = [dy.shape[2] * x.shape[2] for x, dy, _ in layers]
        offs = [0]
        for sz in sizes:
            offs.append(offs[-1] + sz)
        if offs[-1] > flat_grad.numel():
            raise ValueError("flat_grad is smaller than the layers' gradients")
        views = [flat_grad[offs[i]:offs[i + 1]].view(layers[i][1].shape[2], layers[i][0].shape[2])
                 for i in range(n)]
        cuda = flat_grad.is_cuda
        max_ctas = 0
        if cuda and world > 1:
            sms = torch.cuda.get_device_properties(flat_grad.device).multi_processor_count
            max_ctas = max(2, (sms - comm_sms) // 2 * 2)
        if make_group is None:
            from .workflows import PreparedGroup

            def make_group(chunk_layers, grads, cap):
                return PreparedGroup(chunk_layers, grads=grads, noise_impl=noise_impl, rank=rank, world=world,
                                     mean_batch=mean_batch, device_step=device_step, max_ctas=cap)
        self.chunks = []
        for k in range(n_chunks):
            lo, hi = bounds[k], bounds[k + 1]
            self.chunks.append((make_group(list(layers[lo:hi]), views[lo:hi], max_ctas),
                                flat_grad[offs[lo]:offs[hi]]))
        self.comm = torch.cuda.Stream(flat_grad.device) if cuda else None
        self.events = [torch.cuda.Event() for _ in self.chunks] if cuda else []
        self.max_ctas = max_ctas

    def __call__(self, stream=None) -> None:
        cuda = self.comm is not None
        if cuda and stream is None:
            stream = torch.cuda.current_stream(self.flat.device)
        for k, (grp, bucket) in enumerate(self.chunks):
            grp(stream) if cuda else grp()
            if self.world == 1:
                continue
            if cuda:
                self.events[k].record(stream)
                self.comm.wait_event(self.events[k])
                with torch.cuda.stream(self.comm):
                    dist.all_reduce(bucket, op=dist.ReduceOp.SUM, group=self.group)
            else:
                dist.all_reduce(bucket, op=dist.ReduceOp.SUM, group=self.group)
        if cuda and self.world > 1:
            stream.wait_stream(self.comm)
