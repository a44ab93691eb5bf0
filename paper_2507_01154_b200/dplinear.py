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
its per-sample gradient is sum_t dY_b (B x D, tiny), handled with torch ops,
noise keyed on a distinct layer id (layer_id + 2**32).
"""

from __future__ import annotations

from typing import Optional

import torch

from .dpcore import DPConfig, noise_range
from .workflows import WorkflowKind, _run


class _DPLinearFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, weight, bias, module):
        ctx.module = module
        ctx.save_for_backward(x, weight)
        ctx.has_bias = bias is not None
        y = torch.nn.functional.linear(x, weight.to(x.dtype), None if bias is None else bias.to(x.dtype))
        return y

    @staticmethod
    def backward(ctx, dy):
        x, weight = ctx.saved_tensors
        m: DPLinear = ctx.module
        dx = dy @ weight.to(dy.dtype) if ctx.needs_input_grad[0] else None
        B = x.shape[0]
        P, D = weight.shape[1], weight.shape[0]
        x3 = x.reshape(B, -1, P)
        dy3 = dy.reshape(B, -1, D)
        cdt = torch.bfloat16 if m.compute_dtype == torch.bfloat16 else torch.float32
        cfg = m.dp_config()
        res = _run(WorkflowKind.FLASHDP, x3.to(cdt).contiguous(), dy3.to(cdt).contiguous(), cfg, None, None,
                   add_noise=m._noise_now, mean_batch=m.logical_batch or B, rank=m.rank, world=m.world,
                   noise_impl=m.noise_impl)
        m.last_norms_sq = res.per_sample_norms_sq
        gw = res.grad_w.to(weight.dtype)
        gb = None
        if ctx.has_bias:
            gb = m._bias_grad(dy3.float()).to(weight.dtype)
        return dx, gw, gb, None


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
        g = dy3.sum(dim=1)                                   # (B, D) per-sample bias gradients
        ns = (g.double() * g.double()).sum(dim=1)
        f = torch.where(ns <= self.clip_c ** 2, torch.ones_like(ns), self.clip_c / ns.clamp_min(1e-300).sqrt())
        s = (f.float()[:, None] * g).sum(dim=0)
        if self.reduction == "mean":
            s = s / float(self.logical_batch or g.shape[0])
        if self._noise_now and self.sigma > 0:
            cfg = DPConfig(self.clip_c, self.sigma, self.reduction, self.seed, self.layer_id + (1 << 32), self.step)
            n = s.numel()
            lo, hi = n * self.rank // self.world, n * (self.rank + 1) // self.world
            noise = torch.zeros_like(s)
            if hi > lo:
                noise[lo:hi] = noise_range(cfg, lo, hi, self.sigma * self.clip_c, noise_impl=self.noise_impl,
                                           device=s.device)
            s = s + noise
        return s

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        return _DPLinearFn.apply(x, self.weight, self.bias, self)

    def extra_repr(self) -> str:
        return (f"in_features={self.weight.shape[1]}, out_features={self.weight.shape[0]}, "
                f"bias={self.bias is not None}, clip_c={self.clip_c}, sigma={self.sigma}, layer_id={self.layer_id}")
