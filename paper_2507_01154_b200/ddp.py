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

import ctypes
import os
from typing import Iterable, Sequence

import torch
import torch.distributed as dist

from .dpcore import DPConfig


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


# ----------------------------------------------------------------------------- training-step data parallelism
#
# The pieces a multi-GPU DP training step needs beyond one layer list
# (SURVEY 8e): gradient buckets whose collectives
# are issued from the backward itself (reverse layer order, overlapped with the
# dX / DP kernels of the layers still to come), NCCL held to a CTA budget so the
# co-resident persistent DP kernels keep their SMs, and an Adam step on the
# bucket layout -- replicated after an all-reduce (DP-Adam, config 3) or ZeRO-1
# after a reduce-scatter (config 4), where each rank adds the DP noise of
# exactly the shard it owns.


def nccl_options(comm_sms: int = 4):
    """ProcessGroupNCCL options capping NCCL at `comm_sms` CTAs per collective
    (and NVLS at the same count), so NCCL kernels running under the backward
    take at most that many SMs; also exported as NCCL_MAX_CTAS / NCCL_NVLS_CTAS
    for communicators NCCL creates outside these options. None if the build has
    no NCCL."""
    if comm_sms < 1:
        raise ValueError("comm_sms must be >= 1")
    os.environ.setdefault("NCCL_MAX_CTAS", str(comm_sms))
    os.environ.setdefault("NCCL_NVLS_CTAS", str(comm_sms))
    try:
        opts = dist.ProcessGroupNCCL.Options()
    except AttributeError:  # pragma: no cover - torch built without NCCL
        return None
    opts.config.max_ctas = int(comm_sms)
    opts.config.min_ctas = 1
    try:
        opts.config.nvls_ctas = int(comm_sms)
    except AttributeError:  # pragma: no cover
        pass
    return opts


def init_distributed(backend: str = "nccl", comm_sms: int = 4, device: "torch.device | None" = None) -> None:
    """init_process_group with the NCCL CTA budget (nccl) or plain (gloo)."""
    if backend == "nccl":
        dist.init_process_group("nccl", pg_options=nccl_options(comm_sms), device_id=device)
    else:
        dist.init_process_group(backend)


def group_max_ctas(device: torch.device, comm_sms: int, world: int) -> int:
    """CTA cap of the persistent DP kernels under data parallelism: the SMs minus
    NCCL's budget, rounded down to whole CTA pairs (0 = uncapped when world == 1)."""
    if world <= 1 or device.type != "cuda":
        return 0
    sms = torch.cuda.get_device_properties(device).multi_processor_count
    return max(2, (sms - comm_sms) // 2 * 2)


class _Bucket:
    __slots__ = ("params", "offsets", "n", "per", "flat", "pflat", "shard", "pending", "launched", "deferred",
                 "m", "v", "marked", "scale", "scale_applied", "ready", "scale_buf")


class GradBuckets:
    """Gradient buckets of a model, filled by the backward and reduced as soon as
    they are complete.

    Parameters are taken in reverse registration order (the order the backward
    produces their gradients for a sequential model) and packed into buckets of
    about `bucket_bytes` fp32 bytes. Every parameter's ``.grad`` is a view of its
    bucket's flat fp32 buffer (padded to a multiple of `world`), so autograd, the
    DP kernels and the collective all work in place. When the last gradient of a
    bucket has been produced -- signalled by a post-accumulate-grad hook for
    autograd gradients and by ``mark_ready`` for the DP weight gradients that
    GroupedDPBackward writes -- the bucket's collective is issued on a separate
    communication stream and runs under the rest of the backward:

      mode "allreduce":      all_reduce(sum) of the flat buffer (every rank gets
                             the whole summed gradient; DP-Adam, config 3)
      mode "reduce_scatter": reduce_scatter(sum): rank r receives the slice
                             [r*per, (r+1)*per) of the bucket (ZeRO-1, config 4;
                             gloo has no reduce-scatter: all-reduce + slice)

    With ``flat_params`` the parameters' storage is moved into one flat buffer
    per bucket too (same layout), so an optimizer can step a bucket or a shard of
    it with one kernel and all-gather it in one collective.

    Bucket issue order is the backward's order, identical on every rank.

    Deferred clip (``isolate``): each listed parameter gets a bucket of its own,
    so a single-sample DP layer (B = 1 per rank) can hand its gradient over
    UNCLIPPED with its clip factor as a device scalar (``mark_ready(p, scale=)``,
    workflows fdp_dw_deferred): the bucket's collective then scales every rank's
    contribution inside the reduction (NCCL PreMulSum with the device scalar;
    gloo: an in-place multiply first) and at world 1 the optimizer step applies
    it -- the elementwise clip pass over the layer's gradient never runs."""

    def __init__(self, params, *, bucket_bytes: int = 512 << 20, mode: str = "allreduce", group=None,
                 rank: int = 0, world: int = 1, flat_params: bool = False, hooks: bool = True, isolate=()):
        if mode not in ("allreduce", "reduce_scatter"):
            raise ValueError(f"mode must be allreduce or reduce_scatter, got {mode!r}")
        if world < 1 or not (0 <= rank < world):
            raise ValueError(f"rank {rank} out of range for world {world}")
        self.mode, self.group, self.rank, self.world = mode, group, rank, world
        ps = [p for p in params if p.requires_grad]
        if not ps:
            raise ValueError("GradBuckets needs at least one trainable parameter")
        for p in ps:
            if p.dtype != torch.float32:
                raise ValueError(f"GradBuckets keeps fp32 master parameters and gradients, got {p.dtype}")
        self.device = ps[0].device
        self.buckets: list[_Bucket] = []
        iso = {id(p) for p in isolate}
        cur, size = [], 0
        for p in reversed(ps):
            if id(p) in iso:  # a bucket of its own (deferred clip), between its neighbours' buckets
                if cur:
                    self._close(cur, flat_params)
                    cur, size = [], 0
                self._close([p], flat_params)
                self.buckets[-1].scale_buf = True  # marks the isolated bucket: its factor slot follows
                continue
            cur.append(p)
            size += p.numel() * 4
            if size >= bucket_bytes:
                self._close(cur, flat_params)
                cur, size = [], 0
        if cur:
            self._close(cur, flat_params)
        # one persistent factor slot per isolated bucket (slices of one tensor: one fill resets
        # them all); a deferred layer's kernel writes its clip factor there, so the pointer the
        # collective / the optimizer table reads never changes (CUDA-graph capturable)
        iso_b = [b for b in self.buckets if b.scale_buf is True]
        self._scales = torch.ones(max(1, len(iso_b)), dtype=torch.float32, device=self.device) if iso_b else None
        for k, b in enumerate(iso_b):
            b.scale_buf = self._scales[k:k + 1]
        self._external: set = set()  # ids of parameters whose readiness is signalled explicitly
        self._written: set = set()  # ids of parameters whose .grad region was written since zero_grad
        self._where = {}
        for i, b in enumerate(self.buckets):
            for p in b.params:
                self._where[id(p)] = i
        cuda = self.device.type == "cuda"
        self.comm = torch.cuda.Stream(self.device) if cuda and world > 1 else None
        # deferred-clip buckets at N > 1 scale inside the collective (NCCL PreMulSum with a
        # device scalar); a one-time probe at construction (every rank builds its buckets)
        # checks that both collectives of the mode apply it, else each bucket is scaled in
        # place before a plain collective
        self.premul = bool(iso) and world > 1 and dist.is_initialized() and dist.get_backend(group) == "nccl" \
            and self._probe_premul()
        self._handles = []
        if hooks:
            import weakref

            from .baselines import register_inplace_grad_hook

            # the hooks live on the parameters (C++ side, invisible to the cycle collector):
            # they hold this object weakly, so dropping the buckets frees their buffers
            wself = weakref.ref(self)

            def _post_acc(p, wself=wself):
                me = wself()
                if me is not None:
                    me._hook(p)

            for p in ps:
                p.register_post_accumulate_grad_hook(_post_acc)
                register_inplace_grad_hook(p, self._inplace)  # gradients GEMMs write in place
        self.issued: list[int] = []  # bucket issue order of the last backward (tests / traces)
        self.enabled = True  # False while accumulating micro-batches (no collectives)
        self.trace = [] if os.environ.get("FDP_DDP_TRACE") == "1" else None  # (bucket, param, pending) per ready

    def _probe_premul(self) -> bool:
        w, dev = self.world, self.device
        want = float(sum(r + 2 for r in range(w)))
        s = torch.tensor([float(self.rank + 2)], device=dev)
        try:
            t = torch.ones(4 * w, device=dev)
            dist.all_reduce(t, op=dist._make_nccl_premul_sum(s), group=self.group)
            ok = bool(torch.all(t == want))
            if self.mode == "reduce_scatter":
                out = torch.empty(4, device=dev)
                dist.reduce_scatter_tensor(out, torch.ones(4 * w, device=dev), op=dist._make_nccl_premul_sum(s),
                                           group=self.group)
                ok = ok and bool(torch.all(out == want))
        except (RuntimeError, AttributeError, TypeError):
            ok = False
        flag = torch.tensor([1 if ok else 0], device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=self.group)  # one decision for every rank
        return bool(flag.item())

    def _close(self, params, flat_params):
        b = _Bucket()
        b.params = list(params)
        b.offsets = []
        off = 0
        for p in b.params:  # 16-byte aligned segments (vectorised optimizer kernels, quad-aligned noise)
            b.offsets.append(off)
            off += -(-p.numel() // 4) * 4
        b.n = off
        b.per = -(-off // (4 * self.world)) * 4
        dev = params[0].device
        b.flat = torch.zeros(b.per * self.world, dtype=torch.float32, device=dev)
        b.pflat = None
        if flat_params:
            b.pflat = torch.zeros(b.per * self.world, dtype=torch.float32, device=dev)
            for p, o in zip(b.params, b.offsets):
                b.pflat[o:o + p.numel()].copy_(p.detach().reshape(-1))
                p.data = b.pflat[o:o + p.numel()].view_as(p)
        for p, o in zip(b.params, b.offsets):
            p.grad = b.flat[o:o + p.numel()].view_as(p)
        b.shard = b.flat[self.rank * b.per:(self.rank + 1) * b.per]
        b.deferred = 0
        b.pending = len(b.params)
        b.launched = False
        b.marked = set()
        b.m = b.v = None
        b.scale, b.scale_applied = None, False
        b.ready = None  # event on the communication stream after this bucket's collective
        b.scale_buf = None  # isolated buckets: a persistent one-float factor slot (1 when nothing is deferred)
        self.buckets.append(b)

    def set_deferred(self, weights) -> None:
        """Weights whose gradient is written outside autograd (DPLinear under
        GroupedDPBackward): the per-bucket count GroupedDPBackward waits for
        before it runs a bucket's DP kernels."""
        for b in self.buckets:
            b.deferred = 0
        for w in weights:
            i = self._where.get(id(w))
            if i is not None:
                self.buckets[i].deferred += 1
                self._external.add(id(w))

    # ---- per step
    def zero_grad(self) -> None:
        """Zero every bucket and re-arm the readiness counters (call instead of
        optimizer.zero_grad(); the .grad views must stay in place)."""
        for b in self.buckets:
            b.flat.zero_()
            b.pending = len(b.params)
            b.launched = False
            b.marked = set()
            b.scale, b.scale_applied = None, False
            b.ready = None
            for p, o in zip(b.params, b.offsets):
                if p.grad is None or p.grad.data_ptr() != b.flat[o:].data_ptr():
                    p.grad = b.flat[o:o + p.numel()].view_as(p)
        self.issued = []
        self._written = set()
        if self._scales is not None:
            self._scales.fill_(1.0)

    def bucket_of(self, p) -> int:
        return self._where[id(p)]

    def fresh(self, p) -> bool:
        """p's .grad is still its zeroed bucket view (nothing written since
        zero_grad): a kernel may overwrite it instead of accumulating."""
        i = self._where.get(id(p))
        if i is None or id(p) in self._written:
            return False
        b = self.buckets[i]
        o = b.offsets[next(k for k, q in enumerate(b.params) if q is p)]
        return p.grad is not None and p.grad.data_ptr() == b.flat[o:].data_ptr()

    def scale_buffer(self, p) -> "torch.Tensor | None":
        """The persistent factor slot of p's bucket (isolated buckets only)."""
        i = self._where.get(id(p))
        return None if i is None else self.buckets[i].scale_buf

    def note_written(self, p) -> None:
        self._written.add(id(p))

    def can_defer(self, p) -> bool:
        """p may be handed over unclipped with a scale (mark_ready(p, scale=)): its
        bucket holds it alone (an isolated bucket, with a factor slot), its gradient is
        fresh and this is the step's last micro-batch (no later accumulation into it)."""
        i = self._where.get(id(p))
        return (i is not None and self.enabled and self.buckets[i].scale_buf is not None and self.fresh(p)
                and self.device.type == "cuda")

    def _hook(self, p):
        # autograd runs post-accumulate hooks even when a Function returned no
        # gradient for the parameter (a gradient written in place or deferred):
        # those parameters are signalled explicitly, never by this hook
        if id(p) not in self._external:
            self.mark_ready(p)

    def _inplace(self, p):
        self._external.add(id(p))
        self.mark_ready(p)

    def mark_ready(self, p, scale: "torch.Tensor | None" = None) -> None:
        """p's gradient is complete. ``scale`` (a (1,) fp32 device tensor, only for
        a parameter with can_defer(p)): the gradient is scale[0] * p.grad."""
        if not self.enabled:  # micro-batches before the last: gradients accumulate, no collective
            return
        i = self._where.get(id(p))
        if i is None:
            return
        b = self.buckets[i]
        if scale is not None:
            if len(b.params) != 1:
                raise RuntimeError("a scaled gradient needs a bucket of its own (GradBuckets(isolate=...))")
            b.scale = scale
        if id(p) in b.marked:  # one readiness signal per parameter and step
            return
        b.marked.add(id(p))
        if self.trace is not None:
            self.trace.append((i, next(k for k, q in enumerate(b.params) if q is p), b.pending))
        b.pending -= 1
        if b.pending == 0:
            self._launch(i)

    def _launch(self, i: int) -> None:
        b = self.buckets[i]
        if b.launched:
            return
        b.launched = True
        self.issued.append(i)
        if self.world == 1 or os.environ.get("FDP_DDP_NOCOMM") == "1":  # debug: local gradients only
            return
        if self.comm is not None:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(self.device))
            self.comm.wait_event(ev)
            with torch.cuda.stream(self.comm):
                self._collective(b)
                b.ready = torch.cuda.Event()
                b.ready.record(self.comm)
        else:
            self._collective(b)

    def _collective(self, b: _Bucket) -> None:
        nccl = dist.get_backend(self.group) == "nccl"
        op = dist.ReduceOp.SUM
        if b.scale is not None:  # deferred clip: each rank's contribution times its own factor
            if nccl and self.premul:
                op = dist._make_nccl_premul_sum(b.scale)
            else:  # gloo, or an NCCL whose PreMulSum failed the probe: scale in place first
                b.flat.mul_(b.scale.to(b.flat.device))
            b.scale_applied = True
            reset = b.scale_buf is not None and b.scale.data_ptr() == b.scale_buf.data_ptr()
        else:
            reset = False
        if self.mode == "allreduce":
            dist.all_reduce(b.flat, op=op, group=self.group)
        elif nccl:
            out = torch.empty_like(b.shard)
            dist.reduce_scatter_tensor(out, b.flat, op=op, group=self.group)
            b.shard.copy_(out)
        else:  # gloo: all-reduce, keep this rank's slice (b.shard is a view of it)
            dist.all_reduce(b.flat, op=op, group=self.group)
        if reset:  # the collective applied the factor: the slot the optimizer reads is 1 again
            b.scale_buf.fill_(1.0)

    def materialize_scales(self) -> None:
        """Apply every pending deferred-clip factor to its bucket in place (for a
        caller that reads .grad itself -- logging, clipping diagnostics -- instead of
        handing the buckets to BucketedAdam). After finish(); world 1 only has
        pending factors (at N > 1 the collective applied them)."""
        for b in self.buckets:
            if b.scale is not None and not b.scale_applied:
                b.flat.mul_(b.scale)
                b.scale_applied = True

    def finish(self, wait: bool = True) -> None:
        """After backward: issue any bucket not yet issued (parameters without a
        gradient this step), in bucket order, then order the current stream after
        the collectives (wait=False: the caller waits per bucket, wait_bucket)."""
        if not self.enabled:
            return
        for i, b in enumerate(self.buckets):
            if not b.launched:
                self._launch(i)
        if self.comm is not None and wait:
            torch.cuda.current_stream(self.device).wait_stream(self.comm)

    def wait_bucket(self, i: int) -> None:
        """Order the current stream after bucket i's collective (if it had one)."""
        b = self.buckets[i]
        if b.ready is not None:
            torch.cuda.current_stream(self.device).wait_event(b.ready)


def dp_noise_keys(model) -> dict:
    """{id(param): (DPConfig of the noise, offset in the group's index space,
    group length, noise_impl)} for every parameter of a DP module: the key under
    which the DP kernels would add sigma*C*N(seed, layer_id, step, i) to it
    (DPLinear weight: layer_id, flat d*P+p; its bias: layer_id + 2**32;
    RMSNorm gamma / LayerNorm [gamma, beta]: one group of D / 2D; embedding:
    v*D + c). ZeRO-1 draws the same noise on the owner's shard instead."""
    from .dplinear import DPLinear
    from .dpmodules import DPEmbedding, DPLayerNorm, DPRMSNorm

    keys = {}
    for m in model.modules():
        if isinstance(m, DPLinear):
            cfg = m.dp_config()
            keys[id(m.weight)] = (cfg, 0, m.weight.numel(), m.noise_impl)
            if m.bias is not None:
                bcfg = DPConfig(cfg.clip_c, cfg.sigma, cfg.reduction, cfg.seed, m.layer_id + (1 << 32), cfg.step)
                keys[id(m.bias)] = (bcfg, 0, m.bias.numel(), m.noise_impl)
        elif isinstance(m, (DPRMSNorm, DPLayerNorm)):
            cfg = m.dp_config()
            d = m.weight.numel()
            n = d * (2 if getattr(m, "bias", None) is not None else 1)
            keys[id(m.weight)] = (cfg, 0, n, m.noise_impl)
            if getattr(m, "bias", None) is not None:
                keys[id(m.bias)] = (cfg, d, n, m.noise_impl)
        elif isinstance(m, DPEmbedding):
            keys[id(m.weight)] = (m.dp_config(), 0, m.weight.numel(), m.noise_impl)
    return keys


def _torch_sgd_(theta, m, v, grad, eta, b1, b2, eps, noise_cfg, noise_offset, noise_impl, layer_numel,
                grad_scale=None):
    """Device-agnostic stand-in of fdp_sgd_step(_scaled) for CPU tests (no noise)."""
    if noise_cfg is not None and noise_cfg.sigma > 0:
        raise RuntimeError("the torch SGD stand-in does not draw DP noise")
    if grad_scale is not None:
        grad = grad * grad_scale.to(grad.device)
    theta.sub_(eta * grad)


def _torch_adam_(theta, m, v, grad, eta, b1, b2, eps, noise_cfg, noise_offset, noise_impl, layer_numel,
                 grad_scale=None):
    """Device-agnostic stand-in of fdp_adam_step(_scaled) for CPU tests (no noise)."""
    if noise_cfg is not None and noise_cfg.sigma > 0:
        raise RuntimeError("the torch Adam stand-in does not draw DP noise")
    if grad_scale is not None:
        grad = grad * grad_scale.to(grad.device)
    m.mul_(b1).add_(grad, alpha=1 - b1)
    v.mul_(b2).addcmul_(grad, grad, value=1 - b2)
    theta.sub_(eta * m / (v.sqrt() + eps))


class BucketedAdam:
    """Adam without bias correction and with the post-update v (the reference's
    DP-Adam, dpcore.py:139-156) on the GradBuckets layout (flat_params=True).

    mode "allreduce" (buckets were all-reduced): every rank steps every bucket
    whole -- one fused kernel per bucket; the noise was already added once by the
    rank partition of the DP kernels.
    mode "reduce_scatter" (ZeRO-1): rank r steps only its shard of every bucket,
    first adding the DP noise of exactly that shard (per parameter segment: that
    parameter's noise key and in-group offset, `noise_keys` from dp_noise_keys),
    then all-gathers the updated bucket; the moments exist for the shard only.

    `adam_fn(theta, m, v, grad, eta, b1, b2, eps, noise_cfg, noise_offset,
    noise_impl, layer_numel)` replaces the CUDA kernel in CPU tests."""

    def __init__(self, buckets: GradBuckets, *, lr: float, beta1: float = 0.9, beta2: float = 0.999,
                 eps: float = 1e-8, noise_keys: "dict | None" = None, adam_fn=None, kind: str = "adam"):
        if any(b.pflat is None for b in buckets.buckets):
            raise ValueError("BucketedAdam needs GradBuckets(flat_params=True)")
        if kind not in ("adam", "sgd"):
            raise ValueError(f"kind must be adam or sgd, got {kind!r}")
        self.kind = kind
        self.bk = buckets
        self.lr, self.beta1, self.beta2, self.eps = lr, beta1, beta2, eps
        self.noise_keys = noise_keys or {}
        self.adam_fn = adam_fn or (self._kernel if kind == "adam" else self._sgd_kernel)
        zero1 = buckets.mode == "reduce_scatter"
        for b in buckets.buckets:
            n = b.per if zero1 else b.n
            if kind == "adam":
                b.m = torch.zeros(n, dtype=torch.float32, device=b.flat.device)
                b.v = torch.zeros_like(b.m)
            else:  # plain DP-SGD (dpcore.py:131-136): no moments
                b.m = b.v = None
        # ZeRO-1 on CUDA at N > 1: each bucket's parameter all-gather runs on the buckets'
        # communication stream as soon as its shard is stepped; `gathered[i]` is the event a
        # reader of bucket i's parameters waits on (DataParallelStep: forward pre-hooks)
        self.gathered: dict = {}
        # a CUDA int64 scalar: the noise keys' step is read from it (captured CUDA graphs)
        self.device_step = None
        # multi-segment fast path (fdp_adam_step_multi): one launch per bucket (ZeRO-1 / N > 1)
        # or for the whole step, over a device table built once; the noise keys read the
        # step from a device counter (ours, or device_step under a graph)
        self.multi = adam_fn is None and buckets.device.type == "cuda"
        self._tables = None  # (key, [(bucket indices, table, n_seg, total_quads)], keepalive)
        self._own_step = None

    @staticmethod
    def _kernel(theta, m, v, grad, eta, b1, b2, eps, noise_cfg, noise_offset, noise_impl, layer_numel,
                grad_scale=None, device_step=None):
        from .dpcore import OptimizerState, dp_adam_step_

        st = OptimizerState(theta=theta, m=m, v=v, eta=eta, beta1=b1, beta2=b2, eps_adam=eps)
        dp_adam_step_(st, grad, noise=noise_cfg, noise_offset=noise_offset, noise_impl=noise_impl or "philox",
                      layer_numel=layer_numel, grad_scale=grad_scale, device_step=device_step)

    @staticmethod
    def _sgd_kernel(theta, m, v, grad, eta, b1, b2, eps, noise_cfg, noise_offset, noise_impl, layer_numel,
                    grad_scale=None, device_step=None):
        from .dpcore import dp_sgd_step_

        dp_sgd_step_(theta, grad, eta, noise=noise_cfg, noise_offset=noise_offset, noise_impl=noise_impl or "philox",
                     layer_numel=layer_numel, grad_scale=grad_scale, device_step=device_step)

    def _segments(self, b, lo: int, hi: int):
        """(a, z, noise key or None) pieces of [lo, hi) cut at parameter bounds;
        consecutive parameters without a noise key merge into one piece."""
        out = []
        for p, o in zip(b.params, b.offsets):
            a, z = max(o, lo), min(o + p.numel(), hi)
            if a >= z:
                continue
            key = self.noise_keys.get(id(p))
            if key is not None:
                cfg, goff, glen, impl = key
                out.append((a, z, (cfg, goff + (a - o), glen, impl)))
            elif out and out[-1][2] is None and out[-1][1] == a:
                out[-1] = (out[-1][0], z, None)
            else:
                out.append((a, z, None))
        return out

    def _multi_plan(self):
        """Device tables for fdp_adam_step_multi, or None when a segment does not fit it
        (keyed noise, an unaligned noise offset): then the per-segment launches run."""
        from dataclasses import replace

        from . import _lib

        bk = self.bk
        zero1 = bk.mode == "reduce_scatter"
        if self.device_step is None and self._own_step is None:
            self._own_step = torch.zeros(1, dtype=torch.int64, device=bk.device)
        step_t = self.device_step if self.device_step is not None else self._own_step
        key = (step_t.data_ptr(),)
        if self._tables is not None and self._tables[0] == key:
            return self._tables[1]
        groups = [[i] for i in range(len(bk.buckets))] if bk.world > 1 else [list(range(len(bk.buckets)))]
        lib = _lib.load()
        plan, keep = [], []
        for idx in groups:
            segs = []
            for i in idx:
                b = bk.buckets[i]
                lo = bk.rank * b.per if zero1 else 0
                hi = min(lo + b.per, b.n) if zero1 else b.n
                src = b.shard if zero1 else b.flat
                gs = b.scale_buf.data_ptr() if b.scale_buf is not None else None
                for a, z, nkey in self._segments(b, lo, hi):
                    adam = self.kind == "adam"
                    seg = _lib.FdpAdamSegment(theta=b.pflat[a:z].data_ptr(),
                                              m=b.m[a - lo:z - lo].data_ptr() if adam else None,
                                              v=b.v[a - lo:z - lo].data_ptr() if adam else None,
                                              grad=src[a - lo:z - lo].data_ptr(), grad_scale=gs, n=z - a, noise=None,
                                              noise_offset=0)
                    if nkey is not None:
                        cfg, off, glen, impl = nkey
                        if (impl or "philox") != "philox" or off % 4:
                            return None
                        desc = _lib.make_desc(B=1, T=1, P=glen, D=1, clip_c=cfg.clip_c, sigma=cfg.sigma,
                                              seed=cfg.seed, layer_id=cfg.layer_id, step=0, noise_impl="philox",
                                              device_step=step_t.data_ptr())
                        keep.append(desc)
                        seg.noise = ctypes.pointer(desc)
                        seg.noise_offset = off
                    segs.append(seg)
            arr = (_lib.FdpAdamSegment * max(1, len(segs)))(*segs)
            nb = ctypes.c_size_t()
            _lib.check(lib.fdp_adam_multi_table_bytes(len(segs), ctypes.byref(nb)))
            table = torch.empty(max(16, nb.value), dtype=torch.uint8, device=bk.device)
            tq = ctypes.c_int64()
            _lib.check(lib.fdp_adam_multi_prepare(len(segs), arr, table.data_ptr(), table.numel(), ctypes.byref(tq),
                                                  torch.cuda.current_stream(bk.device).cuda_stream))
            plan.append((idx, table, len(segs), tq.value))
            keep.append(arr)
        self._tables = (key, plan, keep)
        del replace
        return plan

    def step(self, dp_step: int = 0) -> None:
        from dataclasses import replace

        bk = self.bk
        plan = self._multi_plan() if self.multi else None
        if plan is not None:
            from . import _lib

            if self.device_step is None:
                self._own_step.fill_(int(dp_step))
            lib, st = _lib.load(), torch.cuda.current_stream(bk.device).cuda_stream
            order = range(len(plan) - 1, -1, -1) if bk.world > 1 and bk.mode == "reduce_scatter" else range(len(plan))
            for k in order:
                idx, table, n_seg, tq = plan[k]
                for i in idx:
                    bk.wait_bucket(i)
                if self.kind == "adam":
                    _lib.check(lib.fdp_adam_step_multi(n_seg, table.data_ptr(), tq, self.lr, self.beta1, self.beta2,
                                                       self.eps, st))
                else:
                    _lib.check(lib.fdp_sgd_step_multi(n_seg, table.data_ptr(), tq, self.lr, st))
                if bk.world > 1 and bk.mode == "reduce_scatter":
                    for i in idx:
                        self._gather(i, bk.buckets[i])
            return
        zero1_gather = bk.world > 1 and bk.mode == "reduce_scatter"
        # ZeRO-1: step the buckets in forward order (the last buckets hold the first layers), so
        # the all-gathers the next forward needs first are issued first
        order = range(len(bk.buckets) - 1, -1, -1) if zero1_gather else range(len(bk.buckets))
        for i in order:
            b = bk.buckets[i]
            bk.wait_bucket(i)  # this bucket's reduction is complete (later ones may still run)
            # a deferred clip factor no collective applied (world 1): the step multiplies it in
            kw = {"grad_scale": b.scale} if b.scale is not None and not b.scale_applied else {}
            if bk.mode == "allreduce" and not self.noise_keys:
                self.adam_fn(b.pflat[:b.n], b.m, b.v, b.flat[:b.n], self.lr, self.beta1, self.beta2, self.eps,
                             None, 0, None, 0, **kw)
                continue
            # ZeRO-1: this rank's shard; all-reduce with noise keys: the whole bucket on every
            # rank, each element's noise drawn once per rank from the same keys (counter-based,
            # so every replica adds the same noise and the parameters stay identical)
            lo = bk.rank * b.per if bk.mode == "reduce_scatter" else 0
            hi = min(lo + b.per, b.n) if bk.mode == "reduce_scatter" else b.n
            src = b.shard if bk.mode == "reduce_scatter" else b.flat
            for a, z, key in self._segments(b, lo, hi):
                th, g = b.pflat[a:z], src[a - lo:z - lo]
                mm = b.m[a - lo:z - lo] if b.m is not None else None
                vv = b.v[a - lo:z - lo] if b.v is not None else None
                if key is None:
                    self.adam_fn(th, mm, vv, g, self.lr, self.beta1, self.beta2, self.eps, None, 0, None, 0, **kw)
                else:
                    cfg, off, glen, impl = key
                    nkw = dict(kw, device_step=self.device_step) if self.device_step is not None else kw
                    self.adam_fn(th, mm, vv, g, self.lr, self.beta1, self.beta2, self.eps,
                                 replace(cfg, step=dp_step), off, impl, glen, **nkw)
            if zero1_gather:
                self._gather(i, b)

    def _gather(self, i: int, b) -> None:
        bk = self.bk
        mine = b.pflat[bk.rank * b.per:(bk.rank + 1) * b.per]

        def run():
            if dist.get_backend(bk.group) == "nccl":
                dist.all_gather_into_tensor(b.pflat, mine.clone(), group=bk.group)
            else:
                pieces = list(b.pflat.chunk(bk.world))
                dist.all_gather(pieces, mine.clone(), group=bk.group)

        if bk.comm is None:  # CPU: synchronous
            run()
            return
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(b.pflat.device))  # this shard's Adam step is enqueued
        bk.comm.wait_event(ev)
        with torch.cuda.stream(bk.comm):
            run()
            done = torch.cuda.Event()
            done.record(bk.comm)
        self.gathered[i] = done

    def wait_gathered(self, indices=None) -> None:
        """Order the current stream after the parameter all-gathers of the given buckets
        (all pending ones when None)."""
        keys = list(self.gathered) if indices is None else [i for i in indices if i in self.gathered]
        for i in keys:
            torch.cuda.current_stream(self.bk.device).wait_event(self.gathered.pop(i))


class DataParallelStep:
    """One data-parallel training step of a model, DP or non-DP, on the bucket
    layout: zero the buckets, forward + loss, backward with the buckets'
    collectives issued from inside it, Adam (no bias correction, dpcore.py:139-156)
    on the bucket layout.

      dp=True,  mode "allreduce":      DP-Adam (config 3): buckets all-reduced,
                                       replicated Adam; the noise is added inside the
                                       Adam step on every replica from the same keyed
                                       draws (noise_in_optimizer, default), or by the
                                       DP kernels on each rank's slice of every layer.
      dp=True,  mode "reduce_scatter": ZeRO-1 (config 4): the DP kernels run without
                                       noise, buckets reduce-scattered, each rank adds
                                       the noise of its shard inside its Adam step and
                                       all-gathers the parameters.
      dp=False: the same model's non-DP step with the same buckets, collectives and
                optimizer (the like-for-like baseline; give the model
                FP32GradLinear projections for the DP arm's fp32 gradient path).

    The loss must be the sum over samples of per-sample losses, scaled by
    1/global_batch for dp=False (the DP modules take the mean over the logical
    batch themselves), so the summed gradients are the global-batch ones.

    ``defer_clip`` (None = on when every rank holds one sample; DP only with the
    noise in the optimizer): weight matrices of >= isolate_min_numel elements get
    buckets of their own (in both arms: same layout)
    and a single-sample layer hands its gradient over unclipped with its clip
    factor (GradBuckets), so its elementwise clip pass never runs: the collective
    (PreMulSum) or, at world 1, the Adam step applies the factor.

    ``optimizer``: "adam" (the reference's DP-Adam, default) or "sgd" (plain DP-SGD,
    theta -= lr * g, dpcore.py:131-136: BASELINE config 2's optimizer)"""

    def __init__(self, model, *, dp: bool, mode: str = "allreduce", lr: float = 1e-5, beta1: float = 0.9,
                 beta2: float = 0.999, eps: float = 1e-8, rank: int = 0, world: int = 1, group=None,
                 comm_sms: int = 4, bucket_bytes: int = 512 << 20, global_batch: int = 1, adam_fn=None,
                 noise_in_optimizer: bool = True, defer_clip: "bool | None" = None,
                 isolate_min_numel: int = 1 << 22, optimizer: str = "adam"):
        from .dplinear import DPLinear

        self.model, self.dp, self.mode, self.world = model, dp, mode, world
        # where the DP noise is added: in the optimizer step (the finalize fused into Adam:
        # ZeRO-1 on the owner's shard, all-reduce on every replica with the same keyed draws)
        # or, all-reduce only, by the DP kernels on each rank's slice of every layer
        self.noise_in_optimizer = bool(noise_in_optimizer) or mode == "reduce_scatter"
        self.global_batch = global_batch
        if defer_clip is None:
            defer_clip = global_batch == world
        self.defer_clip = bool(defer_clip) and dp and self.noise_in_optimizer
        # the bucket layout follows the request for both arms (the non-DP baseline gets the same buckets)
        iso = [p for p in model.parameters() if p.dim() == 2 and p.numel() >= isolate_min_numel] if defer_clip else []
        self.buckets = GradBuckets(model.parameters(), bucket_bytes=bucket_bytes, mode=mode, group=group,
                                   rank=rank, world=world, flat_params=True, isolate=iso)
        self.dp_mods = model.dp_modules() if dp else []
        if dp:
            set_data_parallel(self.dp_mods, rank, world)
            self.buckets.set_deferred([m.weight for m in self.dp_mods if isinstance(m, DPLinear)])
        keys = dp_noise_keys(model) if dp and self.noise_in_optimizer else None
        self.opt = BucketedAdam(self.buckets, lr=lr, beta1=beta1, beta2=beta2, eps=eps, noise_keys=keys,
                                adam_fn=adam_fn, kind=optimizer)
        dev = next(model.parameters()).device
        self.max_ctas = group_max_ctas(dev, comm_sms, world)
        # ZeRO-1 at N > 1: the next forward overlaps the parameter all-gathers -- a module
        # waits only for the buckets holding its own parameters (parameters are first read
        # inside their own module's forward; whatever is left is waited for after the forward)
        if mode == "reduce_scatter" and world > 1 and dev.type == "cuda":
            import weakref

            wopt = weakref.ref(self.opt)
            for mod in model.modules():
                idx = sorted({self.buckets.bucket_of(p) for p in mod.parameters(recurse=False)
                              if id(p) in self.buckets._where})
                if idx:
                    def _pre(m, args, idx=tuple(idx), wopt=wopt):
                        o = wopt()
                        if o is not None and o.gathered:
                            o.wait_gathered(idx)
                    mod.register_forward_pre_hook(_pre)
        if world > 1:  # per-layer DP kernels leave NCCL's SMs free too (fdp_capi.cu reserved_sms)
            os.environ["FDP_RESERVE_SMS"] = str(int(comm_sms))
        self.last_flushes = 0
        self.last_deferred = 0  # layers whose clip was deferred to the collective / optimizer last step

    def finish(self) -> None:
        """Order the current stream after the last step's parameter all-gathers (ZeRO-1
        at N > 1 leaves them running under the next forward); call before reading the
        parameters outside a step."""
        if self.opt.gathered:
            self.opt.wait_gathered()

    def __call__(self, step: int, loss_fn):
        from .dplinear import GroupedDPBackward

        bk = self.buckets
        bk.zero_grad()
        for m in self.dp_mods:  # kernel noise only when the optimizer does not add it
            m.set_step(step, last_micro_batch=not self.noise_in_optimizer, logical_batch=self.global_batch)
        loss = loss_fn()
        if self.opt.gathered:  # parameter all-gathers no forward hook waited for
            self.opt.wait_gathered()
        if self.dp:
            with GroupedDPBackward(buckets=bk, max_ctas=self.max_ctas, defer_clip=self.defer_clip) as g:
                loss.backward()
            self.last_flushes = g.flushes
            self.last_deferred = g.deferred_clips
        else:
            loss.backward()
        bk.finish(wait=False)  # the Adam step waits bucket by bucket, under the remaining collectives
        self.opt.step(dp_step=step)
        return loss


class GraphedStep:
    """A DataParallelStep captured in ONE CUDA graph (one GPU): forward, the backward
    with its DP kernels and bucket hooks, and the bucketed Adam step replay as a
    single graph launch, so a small-batch step (hundreds of kernel launches, Python
    autograd and ctypes calls) is no longer bound by the host.

    ``loss_fn`` must read its batch from static tensors (copy each batch into them
    before the call). The optimizer's DP noise is keyed on a device step counter
    (BucketedAdam.device_step), so every replay draws the noise of its own step --
    which is why the DP kernels must not draw any (noise_in_optimizer, the default).
    ``warmup`` eager steps run first on a side stream (steps first_step ..
    first_step + warmup - 1; PyTorch's whole-network capture recipe), then step
    first_step + warmup is captured; each call replays the next step.

        g = GraphedStep(step, lambda: model.loss(x_static, y_static, reduction="sample_sum"))
        for i in range(g.next_step, n_steps):
            x_static.copy_(...); y_static.copy_(...)
            loss = g()"""

    def __init__(self, dstep: DataParallelStep, loss_fn, *, warmup: int = 3, first_step: int = 0):
        from .errors import UsageError

        if dstep.world != 1:
            raise UsageError("GraphedStep captures a one-GPU step (collectives stay eager)")
        if dstep.dp and not dstep.noise_in_optimizer:
            raise UsageError("GraphedStep needs the DP noise in the optimizer (kernel noise keys are host values)")
        if warmup < 1:
            raise UsageError("GraphedStep needs at least one warm-up step")
        dev = dstep.buckets.device
        self.dstep = dstep
        self.device_step = torch.zeros(1, dtype=torch.int64, device=dev)
        dstep.opt.device_step = self.device_step
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            for i in range(warmup):
                self.device_step.fill_(first_step + i)
                dstep(first_step + i, loss_fn)
        torch.cuda.current_stream(dev).wait_stream(side)
        self.next_step = first_step + warmup
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):  # recorded, not run: the first replay is this step
            self.loss = dstep(self.next_step, loss_fn)

    def __call__(self, step: "int | None" = None):
        i = self.next_step if step is None else int(step)
        self.device_step.fill_(i)
        self.graph.replay()
        self.next_step = i + 1
        return self.loss
