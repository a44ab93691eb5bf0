"""Non-DP baselines that match the DP path's gradient precision.

The DP kernels write every weight gradient in fp32 straight from the tensor-core
accumulator (include/fdp.h). Plain autocast autograd instead emits the dW GEMM
in bf16 and AccumulateGrad casts it into the fp32 ``.grad`` -- cheaper, and not
the same arithmetic. ``FP32GradLinear`` is the like-for-like non-DP linear
layer: bf16 forward GEMM under autocast, bf16 dX GEMM, and the weight gradient
from cuBLAS with fp32 output, accumulated in place into an fp32 ``.grad``
(beta = 1: no separate add pass), exactly the precision the DP arm writes.
"""

from __future__ import annotations

import weakref

import torch


def _dw_into(grad: torch.Tensor, dy2: torch.Tensor, x2: torch.Tensor) -> torch.Tensor:
    """grad += dy2^T x2 in fp32 (cuBLAS, bf16 operands, fp32 accumulate/output)."""
    try:
        return torch.addmm(grad, dy2.t(), x2, out_dtype=torch.float32, out=grad)
    except (RuntimeError, TypeError):  # builds without addmm.dtype_out
        return grad.add_(torch.mm(dy2.t(), x2, out_dtype=torch.float32))


class _FP32GradLinearFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, weight, bias):
        cdt = torch.get_autocast_dtype("cuda") if torch.is_autocast_enabled("cuda") else x.dtype
        with torch.autocast("cuda", enabled=False):
            xc, wc = x.to(cdt), weight.to(cdt)
            y = torch.nn.functional.linear(xc, wc, None if bias is None else bias.to(cdt))
        ctx.save_for_backward(xc, wc)
        ctx.weight = weight
        ctx.has_bias = bias is not None
        ctx.x_dtype = x.dtype
        return y

    @staticmethod
    def backward(ctx, dy):
        xc, wc = ctx.saved_tensors
        weight = ctx.weight
        dx = (dy.to(wc.dtype) @ wc).to(ctx.x_dtype) if ctx.needs_input_grad[0] else None
        x2 = xc.reshape(-1, xc.shape[-1])
        dy2 = dy.to(xc.dtype).reshape(-1, dy.shape[-1])
        gw = None
        g = weight.grad
        if g is not None and g.dtype == torch.float32 and g.is_contiguous() and g.is_cuda:
            _dw_into(g, dy2, x2)  # in place: autograd gets no weight gradient to add
            _notify(weight)
        else:
            gw = torch.mm(dy2.t(), x2, out_dtype=torch.float32) if dy2.is_cuda else (dy2.t().float() @ x2.float())
            gw = gw.to(weight.dtype)
        gb = dy.reshape(-1, dy.shape[-1]).float().sum(0).to(weight.dtype) if ctx.has_bias else None
        return dx, gw, gb


# id(weight) -> (weakref to the weight, weakref to the bound hook): weak on both ends, so
# a registry entry never keeps a model or its gradient buckets alive
_READY_HOOKS: dict = {}


def _notify(weight: torch.Tensor) -> None:
    """A gradient written in place bypasses AccumulateGrad (no post-accumulate
    hook): tell the gradient bucket (ddp.GradBuckets) directly."""
    entry = _READY_HOOKS.get(id(weight))
    if entry is None or entry[0]() is not weight:
        return
    fn = entry[1]()
    if fn is not None:
        fn(weight)


def register_inplace_grad_hook(weight: torch.Tensor, fn) -> None:
    if len(_READY_HOOKS) > 4096:  # drop entries whose weight or hook owner is gone
        for k in [k for k, (w, f) in _READY_HOOKS.items() if w() is None or f() is None]:
            del _READY_HOOKS[k]
    ref = weakref.WeakMethod(fn) if hasattr(fn, "__self__") else (lambda f=fn: f)
    _READY_HOOKS[id(weight)] = (weakref.ref(weight), ref)


class FP32GradLinear(torch.nn.Linear):
    """nn.Linear whose weight gradient is written in fp32 by the GEMM itself."""

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        return _FP32GradLinearFn.apply(x, self.weight, self.bias)
