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


def set_data_parallel(modules, rank: int, world: int) -> None:
    """Per-rank setup of every DP module of a model (DPLinear, DPLayerNorm,
    DPRMSNorm, DPEmbedding): each adds its noise only on the rank's slice of its
    group's index space. Pass the global batch as ``logical_batch`` to
    ``set_step`` so ``mean`` divides by it; then ``allreduce_grads_`` over the
    parameters' gradients gives the single-process DP gradients, noise once."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"rank {rank} out of range for world {world}")
    for m in modules:
        m.rank, m.world = rank, world


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

    def __init__(self, layers, flat_grad: torch.Tensor, *, n_chunks: int = 4, comm_sms: int = 4,
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


class ShardedDPAdam:
    """ZeRO-1 style data parallelism for the DP step (the 13B layout):
    every rank computes its clipped sums WITHOUT noise (scaled by 1/B_global), the
    per-layer gradients are reduce-scattered (sum) so rank r owns a contiguous
    shard of the flat parameter vector, rank r adds the DP noise of exactly that
    shard inside its Adam step (fdp_adam_step with the layer's noise key and the
    shard's flat offset within the layer) and updates its shard of the fp32
    master weights + moments, then the updated parameters are all-gathered.
    Noise is added exactly once per element, so the result equals the
    single-process DP-Adam step.

    layers: sequence of (n_elements, DPConfig) in flat order (the DPConfig keys the
    noise: seed, layer_id, step, sigma, clip_c); params: the flat fp32 master
    parameters (replicated), updated in place by step(grad_flat)."""

    def __init__(self, layers, params: torch.Tensor, *, eta: float, beta1: float = 0.9, beta2: float = 0.999,
                 eps: float = 1e-8, noise_impl: str = "philox", rank: int = 0, world: int = 1, group=None):
        self.layers = list(layers)
        self.params = params
        self.n = sum(n for n, _ in self.layers)
        if params.numel() != self.n:
            raise ValueError("params must hold every layer's elements")
        self.rank, self.world, self.group = rank, world, group
        self.noise_impl = noise_impl
        # equal (padded) shards for the collective: rank r owns [r*per, (r+1)*per) ∩ [0, n)
        self.per = -(-self.n // world)
        self.lo, self.hi = min(rank * self.per, self.n), min((rank + 1) * self.per, self.n)
        self.m = torch.zeros(self.hi - self.lo, dtype=params.dtype, device=params.device)
        self.v = torch.zeros_like(self.m)
        self.eta, self.beta1, self.beta2, self.eps = eta, beta1, beta2, eps

    def _shard_of(self, full: torch.Tensor) -> torch.Tensor:
        if self.world == 1:
            return full
        pad = torch.zeros(self.per * self.world, dtype=full.dtype, device=full.device)
        pad[:self.n] = full
        if dist.get_backend(self.group) == "nccl":
            out = torch.empty(self.per, dtype=full.dtype, device=full.device)
            dist.reduce_scatter_tensor(out, pad, op=dist.ReduceOp.SUM, group=self.group)
        else:  # gloo has no reduce-scatter: all-reduce and keep this rank's slice
            dist.all_reduce(pad, op=dist.ReduceOp.SUM, group=self.group)
            out = pad[self.rank * self.per:(self.rank + 1) * self.per].clone()
        return out

    def step(self, grad_flat: torch.Tensor, cfg_step: int) -> None:
        from dataclasses import replace

        from .dpcore import OptimizerState, dp_adam_step_

        own_lo, own_hi = self.lo, self.hi
        shard = self._shard_of(grad_flat)[:own_hi - own_lo]
        theta = self.params[own_lo:own_hi].clone()
        off = 0
        for n, cfg in self.layers:  # per (layer ∩ shard) segment: that layer's noise key and in-layer offset
            a, b = max(off, own_lo), min(off + n, own_hi)
            if a < b:
                st = OptimizerState(theta=theta[a - own_lo:b - own_lo], m=self.m[a - own_lo:b - own_lo],
                                    v=self.v[a - own_lo:b - own_lo], eta=self.eta, beta1=self.beta1,
                                    beta2=self.beta2, eps_adam=self.eps)
                dp_adam_step_(st, shard[a - own_lo:b - own_lo].contiguous(), noise=replace(cfg, step=cfg_step),
                              noise_offset=a - off, noise_impl=self.noise_impl, layer_numel=n)
            off += n
        if self.world == 1:
            self.params.copy_(theta)
            return
        pieces = [torch.empty(self.per, dtype=self.params.dtype, device=self.params.device)
                  for _ in range(self.world)]
        mine = torch.zeros(self.per, dtype=self.params.dtype, device=self.params.device)
        mine[:own_hi - own_lo] = theta
        dist.all_gather(pieces, mine, group=self.group)
        self.params.copy_(torch.cat(pieces)[:self.n])
