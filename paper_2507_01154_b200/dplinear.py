"""DPLinear: the per-layer clipping unit as a torch module (PAPER.md:161-163,
per-layer clipping PAPER.md:311-328).

Forward is a plain bf16 GEMM (Y = X W^T + b). Backward computes dX with the
standard GEMM and hands (X, dY) to the fused sm_100a kernel, which returns the
layer's finalized DP weight gradient -- per-sample clip at this layer's C,
sum (or mean over the logical batch), sigma*C keyed noise -- without ever
materialising per-sample gradients. The result lands in ``weight.grad``.

Gradient accumulation (dpcore.accumulate_micro_batches, dpcore.py:90-104):
call ``set_step(step, last_micro_batch=...)`` before each micro-batch; noise is
added only on the last micro-batch and ``mean`` divides by the logical batch.

The bias (if any) is clipped as its own per-layer group with the same C:
its per-sample gradient is sum_t dY_b (B x D, tiny), computed, clipped, summed
and noised by one fused CUDA pass pair (fdp_bias_dw), noise keyed on a
distinct layer id (layer_id + 2**32).
"""

from __future__ import annotations

from typing import Optional

import ctypes
import os
import weakref

import torch

from . import _lib
from .dpcore import DPConfig
from .workflows import WorkflowKind, _run


_CAST: list = [None]  # (source tensor, its version, dtype, the cast, its version) -- weak references


def _cast_shared(x: torch.Tensor, dtype) -> torch.Tensor:
    """x.to(dtype), reusing the previous call's cast when the same (unmodified) input
    comes again: projections fed by one activation (q/k/v, gate/up) then save ONE
    compute-dtype copy, which is also what lets their backward share the X Gram
    (fdp_backward_shared_x recognises the common input by its address)."""
    if x.dtype == dtype:
        return x
    c = _CAST[0]
    if c is not None and c[0]() is x and c[1] == x._version and c[2] == dtype:
        xc = c[3]()
        if xc is not None and xc._version == c[4]:
            return xc
    xc = x.to(dtype)
    _CAST[0] = (weakref.ref(x), x._version, dtype, weakref.ref(xc), xc._version)  # no reference kept alive
    return xc


class _DPLinearFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, weight, bias, module):
        ctx.module = module
        ctx.has_bias = bias is not None
        ctx.x_dtype = x.dtype
        # compute dtype: autocast's when enabled (bf16 GEMMs, bf16 saved input -- what
        # the DP kernel consumes, no second cast in backward), else the input's
        cdt = torch.get_autocast_dtype("cuda") if torch.is_autocast_enabled("cuda") else x.dtype
        with torch.autocast("cuda", enabled=False):
            xc = _cast_shared(x, cdt)
            wc = weight.to(cdt)
            y = torch.nn.functional.linear(xc, wc, None if bias is None else bias.to(cdt))
        ctx.save_for_backward(xc, wc)
        return y

    @staticmethod
    def backward(ctx, dy):
        x, wc = ctx.saved_tensors
        m: DPLinear = ctx.module
        weight = m.weight
        dx = (dy.to(wc.dtype) @ wc).to(ctx.x_dtype) if ctx.needs_input_grad[0] else None
        B = x.shape[0]
        P, D = weight.shape[1], weight.shape[0]
        x3 = x.reshape(B, -1, P)
        dy3 = dy.reshape(B, -1, D)
        cdt = torch.bfloat16 if m.compute_dtype == torch.bfloat16 else torch.float32
        cfg = m.dp_config()
        collector = _ACTIVE_GROUP[0]
        if collector is not None and cdt == torch.bfloat16:
            # deferred: the weight gradient comes from the collector's single multi-layer launch
            collector._record(m, x3.to(cdt).contiguous(), dy3.to(cdt).contiguous(), cfg, m._noise_now,
                              m.logical_batch or B)
            gb = m._bias_grad(dy3).to(weight.dtype) if ctx.has_bias else None
            return dx, None, gb, None
        res = _run(WorkflowKind.FLASHDP, x3.to(cdt).contiguous(), dy3.to(cdt).contiguous(), cfg, None, None,
                   add_noise=m._noise_now, mean_batch=m.logical_batch or B, rank=m.rank, world=m.world,
                   noise_impl=m.noise_impl)
        m.last_norms_sq = res.per_sample_norms_sq
        gw = res.grad_w.to(weight.dtype)
        gb = None
        if ctx.has_bias:
            gb = m._bias_grad(dy3).to(weight.dtype)
        return dx, gw, gb, None


_ACTIVE_GROUP: list = [None]


class GroupedDPBackward:
    """Context manager that defers the DP weight gradients of every DPLinear whose
    backward runs inside it and computes them in ONE persistent multi-layer launch
    (PreparedGroup / fdp_backward_group) -- the training-step form of Algorithm 1:
    no per-layer launch, pipelines that never drain between layers, small layers
    packed side by side on the SMs.

        with GroupedDPBackward():
            loss.backward()          # dX as usual; dW of DPLinear layers deferred
        # every DPLinear.weight.grad now holds its DP gradient (accumulated into an
        # existing .grad, as autograd would for micro-batches)

    Each layer keeps its own DPConfig (C, sigma, layer_id noise key, step). Layers
    the fused multi-layer launch cannot take (fp32 compute dtype, shapes over the
    co-resident grid) run through the per-layer kernels instead.

    Data parallel training (``buckets``: a ddp.GradBuckets over the model): the
    deferred layers are flushed bucket by bucket DURING the backward -- as soon as
    every DPLinear weight of a gradient bucket has recorded its (X, dY), that
    bucket's DP kernels run and the bucket is marked ready, so its collective
    starts on the communication stream while the backward continues with the
    earlier layers (reverse layer order). (X, dY) of a layer are released when its
    bucket flushes, not at the end of the backward. ``max_ctas`` caps the
    persistent launches so NCCL keeps its SMs.

    ``defer_finalize``: run the per-layer kernels through a DeferredChain (a B = 1
    layer's clip + noise pass carried by the next layer's GEMM). Off by default:
    measured slower on B200 (Llama-7B block, B = 1: 1174 vs 1074 us; the streamed
    pass slows the carrying GEMM more than the standalone pass costs).

    With ``buckets``, a layer whose bucket view is still fresh (nothing written
    since zero_grad) is written, not accumulated into: a B = 1 layer then takes the
    single-sample path (its GEMM is the sample's gradient) instead of ghost norms.
    ``defer_clip``: such a layer, alone in its bucket and without kernel noise,
    skips even the clip pass -- fdp_dw_deferred leaves the unclipped gradient and
    hands the factor to the bucket (GradBuckets.mark_ready(scale=)), applied by the
    collective or the optimizer step."""

    def __init__(self, *, noise_impl: Optional[str] = None, max_ctas: int = 0, buckets=None,
                 defer_finalize: bool = False, defer_clip: bool = False):
        self.noise_impl = noise_impl
        self.max_ctas = max_ctas
        self.buckets = buckets
        self._pending: list = []
        self.last_groups = 0
        self.flushes = 0
        self.shared_x_calls = 0  # fdp_backward_shared_x calls (layers reading one X) in the last backward
        self._ws = None
        self._waiting: dict = {}
        self.chain = None  # DeferredChain of the per-layer (solo) kernels; None: built on first use
        self.defer_finalize = defer_finalize
        self.defer_clip = defer_clip
        self.deferred_clips = 0  # layers handed over unclipped with a scale in the last backward

    def __enter__(self):
        if _ACTIVE_GROUP[0] is not None:
            raise RuntimeError("GroupedDPBackward contexts do not nest")
        _ACTIVE_GROUP[0] = self
        self._pending = []
        self._waiting = {}
        self.flushes = 0
        self.shared_x_calls = 0
        self.deferred_clips = 0
        return self

    def __exit__(self, exc_type, exc, tb):
        _ACTIVE_GROUP[0] = None
        if exc_type is None:
            for items in self._waiting.values():  # buckets whose other DP weights never ran
                self._flush_items(items)
            self._waiting = {}
            self.flush()
        self._pending = []
        return False

    def _record(self, module, x3, dy3, cfg, add_noise, mean_batch):
        item = (module, x3, dy3, cfg, add_noise, mean_batch)
        bk = self.buckets
        if bk is None or id(module.weight) not in bk._where:
            self._pending.append(item)
            return
        i = bk.bucket_of(module.weight)
        waiting = self._waiting.setdefault(i, [])
        waiting.append(item)
        if len(waiting) == bk.buckets[i].deferred:  # every DP weight of the bucket is here: run it now
            del self._waiting[i]
            self._flush_items(waiting)

    def flush(self) -> None:
        self._flush_items(self._pending)
        self._pending = []

    def _chain(self):
        if self.chain is None:
            from .workflows import DeferredChain

            self.chain = DeferredChain()
        return self.chain

    def _flush_items(self, pending) -> None:
        from .workflows import PreparedGroup, WorkflowKind, _run, _run_shared_x
        from .errors import CapacityError, UsageError

        if not pending:
            return
        self.flushes += 1

        bk = self.buckets

        def out_for(m):  # write straight into an fp32 .grad (bucket view / micro-batch sum)
            g = m.weight.grad
            if g is not None and g.dtype == torch.float32 and g.is_contiguous() and g.shape == m.weight.shape:
                return g
            return None

        claimed: set = set()  # weights already written by an earlier call of this flush

        def fresh(m):  # its bucket view holds zeros: overwrite instead of accumulating
            return (bk is not None and id(m.weight) not in claimed and out_for(m) is not None
                    and bk.fresh(m.weight))

        scales: dict = {}

        def deliver(m, gw, direct):
            if not direct:
                gw = gw.to(m.weight.dtype)
                if m.weight.grad is None:
                    m.weight.grad = gw
                else:
                    m.weight.grad += gw
            if bk is not None:
                bk.mark_ready(m.weight, scale=scales.get(id(m)))
                bk.note_written(m.weight)

        buckets: dict = {}
        for item in pending:  # one launch per (noise on/off, mean divisor, partition, noise generator)
            m, _, _, _, add_noise, mean_batch = item
            key = (add_noise, mean_batch, m.rank, m.world, self.noise_impl or m.noise_impl)
            buckets.setdefault(key, []).append(item)
        self.last_groups = 0
        for (add_noise, mean_batch, rank, world, impl), items in buckets.items():
            # layers whose tiles cannot all be co-resident (e.g. a 50K-row LM head) take the
            # per-layer two-phase kernels; the rest share the multi-layer launches
            solo = [it for it in items if not _fits_group(it[1].shape, it[2].shape)]
            items = [it for it in items if _fits_group(it[1].shape, it[2].shape)]
            # per-layer kernels in sequence through a deferred-finalize chain: a
            # single-sample layer's clip + noise pass runs inside the next layer's
            # GEMM (include/fdp.h fdp_dw_chained); the last one is flushed here
            done = []
            # layers reading the same X (q/k/v, gate/up) share the ghost phase's X Gram:
            # one fdp_backward_shared_x call per run of up to 3 of them
            runs: list = []
            for it in solo:
                x = it[1]
                if (not self.defer_finalize and runs and len(runs[-1]) < 3 and x.dtype == torch.bfloat16
                        and runs[-1][0][1].data_ptr() == x.data_ptr() and runs[-1][0][1].shape == x.shape):
                    runs[-1].append(it)
                else:
                    runs.append([it])
            for run in runs:
                if len(run) > 1:
                    self.shared_x_calls += 1
                    # fresh bucket views are written, not accumulated into (no read of the zeros)
                    specs = [(dy, cfg, out_for(m), not fresh(m)) for m, _, dy, cfg, _, _ in run]
                    gws = _run_shared_x(run[0][1], specs,
                                        noise_impl=impl, add_noise=add_noise, rank=rank, world=world,
                                        mean_batch=mean_batch)
                    done.extend((m, gw, out_for(m) is not None) for (m, *_), gw in zip(run, gws))
                    claimed.update(id(m.weight) for m, *_ in run)
                    continue
                m, x, dy, cfg, _, _ = run[0]
                g = out_for(m)
                new = fresh(m)
                claimed.add(id(m.weight))
                scale = None
                if (self.defer_clip and new and not add_noise and x.shape[0] == 1 and not self.defer_finalize
                        and bk.can_defer(m.weight)):
                    scale = bk.scale_buffer(m.weight)  # the bucket's persistent factor slot
                    if scale is None:
                        scale = torch.empty(1, dtype=torch.float32, device=x.device)
                    scales[id(m)] = scale
                    self.deferred_clips += 1
                gw = _run(WorkflowKind.FLASHDP, x, dy, cfg, None, None, add_noise=add_noise, mean_batch=mean_batch,
                          rank=rank, world=world, noise_impl=impl, grad_out=g, accumulate=g is not None and not new,
                          chain=self._chain() if self.defer_finalize else None, grad_scale_out=scale,
                          path=os.environ.get("FDP_SOLO_PATH", "auto")).grad_w
                done.append((m, gw, g is not None))
            if done and self.defer_finalize:
                self._chain().flush()
            for m, gw, direct in done:
                deliver(m, gw, direct)
            for lo in range(0, len(items), 48):  # fdp_backward_group takes up to 48 layers
                chunk = items[lo:lo + 48]
                direct = all(out_for(m) is not None for m, *_ in chunk)
                # zeroed bucket views (each weight once in the chunk): written, not accumulated into
                new = direct and all(fresh(m) for m, *_ in chunk) and len({id(m) for m, *_ in chunk}) == len(chunk)
                claimed.update(id(m.weight) for m, *_ in chunk)
                try:
                    # a fresh (non-accumulating) group output is written whole by the kernel: no
                    # zero-fill; existing fp32 .grad tensors are accumulated into in place
                    grads_out = ([out_for(m) for m, *_ in chunk] if direct else
                                 [torch.empty(dy.shape[2], x.shape[2], dtype=torch.float32, device=x.device)
                                  for _, x, dy, _, _, _ in chunk])
                    glayers = [(x, dy, cfg) for _, x, dy, cfg, _, _ in chunk]
                    kw = dict(grads=grads_out, noise_impl=impl, add_noise=add_noise, rank=rank, world=world,
                              mean_batch=mean_batch, max_ctas=self.max_ctas, accumulate=direct and not new)
                    try:
                        grp = PreparedGroup(glayers, workspace=self._ws, **kw)
                    except CapacityError:  # cached workspace too small for this layer list: grow it
                        grp = PreparedGroup(glayers, **kw)
                    self._ws = grp.workspace
                    grp()
                    grads = grp.grads
                    self.last_groups += 1
                except UsageError:  # per-layer kernels (two-phase for layers over the co-resident grid)
                    grads = []
                    for m, x, dy, cfg, _, _ in chunk:
                        g = out_for(m) if direct else None
                        grads.append(_run(WorkflowKind.FLASHDP, x, dy, cfg, None, None, add_noise=add_noise,
                                          mean_batch=mean_batch, rank=rank, world=world, noise_impl=impl,
                                          grad_out=g, accumulate=g is not None and not new).grad_w)
                for (m, _, _, _, _, _), gw in zip(chunk, grads):
                    deliver(m, gw, direct)


_FITS: dict = {}


def _fits_group(x_shape, dy_shape) -> bool:
    """Whether one layer's tiles fit the co-resident grid of the fused kernel (the
    multi-layer launch's per-layer condition); cached per shape."""
    if os.environ.get("FDP_NO_GROUP") == "1":  # debug / tests: every layer through the per-layer kernels
        return False
    key = (tuple(x_shape), tuple(dy_shape))
    v = _FITS.get(key)
    if v is None:
        from .errors import UsageError
        from .workflows import execution_plan
        try:
            v = execution_plan(key[0], key[1], path="fused")["path"] == "fused"
        except UsageError:  # no tensor-core path for this shape (e.g. D % 8 != 0): generic per-layer kernels
            v = False
        _FITS[key] = v
    return v


class DPLinear(torch.nn.Module):
    """Drop-in nn.Linear whose weight gradient is the per-layer DP gradient.

    Args mirror DPConfig (clip_c, sigma, reduction, seed) plus ``layer_id``
    (noise key); rank/world partition the noise under data parallelism."""

    def __init__(self, in_features: int, out_features: int, bias: bool = True, *, clip_c: float = 1.0,
                 sigma: float = 1.0, reduction: str = "mean", seed: int = 0, layer_id: int = 0,
                 noise_impl: str = "keyed_f32", compute_dtype=torch.bfloat16, device=None, dtype=None):
        super().__init__()
        self.weight = torch.nn.Parameter(torch.empty(out_features, in_features, device=device, dtype=dtype))
        self.bias = torch.nn.Parameter(torch.empty(out_features, device=device, dtype=dtype)) if bias else None
        torch.nn.init.kaiming_uniform_(self.weight, a=5 ** 0.5)
        if self.bias is not None:
            torch.nn.init.uniform_(self.bias, -1 / in_features ** 0.5, 1 / in_features ** 0.5)
        self.clip_c, self.sigma, self.reduction, self.seed = clip_c, sigma, reduction, seed
        self.layer_id = layer_id
        self.noise_impl = noise_impl
        self.compute_dtype = compute_dtype
        self.step = 0
        self._noise_now = True
        self.logical_batch: Optional[int] = None
        self.rank, self.world = 0, 1
        self.last_norms_sq = None
        DPConfig(clip_c, sigma, reduction)  # validate

    def dp_config(self) -> DPConfig:
        return DPConfig(self.clip_c, self.sigma, self.reduction, self.seed, self.layer_id, self.step)

    def set_step(self, step: int, *, last_micro_batch: bool = True, logical_batch: Optional[int] = None) -> None:
        self.step = step
        self._noise_now = last_micro_batch
        self.logical_batch = logical_batch

    def _bias_grad(self, dy3: torch.Tensor) -> torch.Tensor:
        """The bias as its own per-layer clipping group (fdp_bias_dw, one fused CUDA
        pass pair): per-sample g_b = sum_t dY_b, clip at C, sum / logical batch, +
        sigma*C noise keyed on layer_id + 2**32 over the rank's slice of [0, D)."""
        B, T, D = dy3.shape
        if dy3.dtype not in (torch.bfloat16, torch.float32):
            dy3 = dy3.float()
        dy3 = dy3.contiguous()
        lib = _lib.load()
        key = (B, T, D, dy3.dtype, self.reduction, self.clip_c, self.sigma, self.seed, self.rank, self.world,
               self.noise_impl)
        cached = getattr(self, "_bias_cache", None)
        if cached is None or cached[0] != key:  # descriptor + workspace size, rebuilt only when the shape changes
            desc = _lib.make_desc(B=B, T=T, P=8, D=D, in_dtype=_lib.DTYPE_BF16 if dy3.dtype == torch.bfloat16
                                  else _lib.DTYPE_F32, reduction=self.reduction, clip_c=self.clip_c,
                                  sigma=self.sigma, seed=self.seed, layer_id=self.layer_id + (1 << 32),
                                  rank=self.rank, world=self.world, noise_impl=self.noise_impl)
            nbytes = ctypes.c_size_t()
            _lib.check(lib.fdp_bias_workspace_bytes(ctypes.byref(desc), ctypes.byref(nbytes)))
            cached = (key, desc, nbytes.value)
            self._bias_cache = cached
        _, desc, ws_bytes = cached
        desc.step = _lib._wrap64(self.step)
        desc.layer_id = _lib._wrap64(self.layer_id + (1 << 32))
        desc.mean_batch = self.logical_batch or B
        desc.add_noise = int(bool(self._noise_now))
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dy3.device)
        out = torch.empty(D, dtype=torch.float32, device=dy3.device)
        _lib.check(lib.fdp_bias_dw(ctypes.byref(desc), dy3.data_ptr(), out.data_ptr(), None, ws.data_ptr(),
                                   ws.numel(), torch.cuda.current_stream(dy3.device).cuda_stream))
        return out

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        return _DPLinearFn.apply(x, self.weight, self.bias, self)

    def extra_repr(self) -> str:
        return (f"in_features={self.weight.shape[1]}, out_features={self.weight.shape[0]}, "
                f"bias={self.bias is not None}, clip_c={self.clip_c}, sigma={self.sigma}, layer_id={self.layer_id}")
