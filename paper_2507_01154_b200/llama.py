"""Llama-2 (7B / 13B shapes) with DP parameters: BASELINE configs 3/4 as a
training step on one GPU (SURVEY 8d E2E inputs).

``dp=True`` makes every parameter DP with per-layer clipping: the seven
projections of each block and the untied LM head are ``DPLinear`` (bias-free),
the RMSNorms ``DPRMSNorm``, the token embedding ``DPEmbedding``. ``dp=False``
builds the same model from torch modules (the non-DP baseline). Attention is
torch SDPA (causal) with rotary position embeddings; the MLP is SwiGLU.
Random-init weights, synthetic token ids; bf16 autocast, fp32 master weights.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.nn.functional as F

from .dplinear import DPLinear
from .dpmodules import DPEmbedding, DPRMSNorm, _DPGroupModule


@dataclass
class LlamaConfig:
    vocab: int = 32000
    d: int = 4096
    heads: int = 32
    layers: int = 32
    mlp: int = 11008
    seq: int = 2048
    eps: float = 1e-5

    @staticmethod
    def named(name: str, **kw) -> "LlamaConfig":
        base = {"llama-7b": dict(d=4096, heads=32, layers=32, mlp=11008),
                "llama-13b": dict(d=5120, heads=40, layers=40, mlp=13824)}[name]
        base.update(kw)
        return LlamaConfig(**base)


class _RMSNorm(torch.nn.Module):
    def __init__(self, d: int, eps: float):
        super().__init__()
        self.weight = torch.nn.Parameter(torch.ones(d))
        self.eps = eps

    def forward(self, x):
        xf = x.float()
        return xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + self.eps) * self.weight


def _rope(q, k, cos, sin):
    def rot(t):
        t1, t2 = t[..., : t.shape[-1] // 2], t[..., t.shape[-1] // 2:]
        return torch.cat((-t2, t1), dim=-1)

    return q * cos + rot(q) * sin, k * cos + rot(k) * sin


class Block(torch.nn.Module):
    def __init__(self, cfg: LlamaConfig, idx: int, dp: bool, clip_c: float, sigma: float, noise_impl: str,
                 linear_cls=torch.nn.Linear):
        super().__init__()
        self.heads = cfg.heads

        def lin(cin, cout, j):
            if dp:
                return DPLinear(cin, cout, bias=False, clip_c=clip_c, sigma=sigma, reduction="mean",
                                layer_id=7 * idx + j, noise_impl=noise_impl)
            return linear_cls(cin, cout, bias=False)

        def norm(j):
            if dp:
                return DPRMSNorm(cfg.d, cfg.eps, clip_c=clip_c, sigma=sigma, layer_id=100000 + 2 * idx + j,
                                 noise_impl=noise_impl)
            return _RMSNorm(cfg.d, cfg.eps)

        self.attn_norm, self.mlp_norm = norm(0), norm(1)
        self.q, self.k, self.v, self.o = (lin(cfg.d, cfg.d, j) for j in range(4))
        self.gate, self.up = lin(cfg.d, cfg.mlp, 4), lin(cfg.d, cfg.mlp, 5)
        self.down = lin(cfg.mlp, cfg.d, 6)

    def forward(self, x, cos, sin):
        B, T, C = x.shape
        h = self.attn_norm(x)
        hd = C // self.heads
        q = self.q(h).view(B, T, self.heads, hd).transpose(1, 2)
        k = self.k(h).view(B, T, self.heads, hd).transpose(1, 2)
        v = self.v(h).view(B, T, self.heads, hd).transpose(1, 2)
        q, k = _rope(q, k, cos.to(q.dtype), sin.to(q.dtype))
        y = F.scaled_dot_product_attention(q, k, v, is_causal=True)
        x = x + self.o(y.transpose(1, 2).reshape(B, T, C))
        h = self.mlp_norm(x)
        return x + self.down(F.silu(self.gate(h)) * self.up(h))


class Llama(torch.nn.Module):
    """``nondp_linear``: the non-DP model's projection class -- "torch" (nn.Linear:
    bf16 dW GEMM cast into the fp32 .grad by autograd) or "fp32grad"
    (baselines.FP32GradLinear: cuBLAS writes the fp32 weight gradient directly,
    the DP kernels' precision; the like-for-like baseline)."""

    def __init__(self, cfg: LlamaConfig, *, dp: bool = True, clip_c: float = 1.0, sigma: float = 1.0,
                 noise_impl: str = "philox", nondp_linear: str = "torch"):
        super().__init__()
        self.cfg = cfg
        self.dp = dp
        if nondp_linear == "fp32grad":
            from .baselines import FP32GradLinear as linear_cls
        elif nondp_linear == "torch":
            linear_cls = torch.nn.Linear
        else:
            raise ValueError(f"nondp_linear must be torch or fp32grad, got {nondp_linear!r}")
        # registration order = forward order (embedding, blocks, final norm, LM head), so
        # reversed(parameters()) is the order the backward produces the gradients
        # (ddp.GradBuckets fills and reduces its buckets in that order)
        if dp:
            self.embed = DPEmbedding(cfg.vocab, cfg.d, clip_c=clip_c, sigma=sigma, layer_id=200000,
                                     noise_impl=noise_impl)
        else:
            self.embed = torch.nn.Embedding(cfg.vocab, cfg.d)
        self.blocks = torch.nn.ModuleList(Block(cfg, i, dp, clip_c, sigma, noise_impl, linear_cls)
                                          for i in range(cfg.layers))
        if dp:
            self.norm = DPRMSNorm(cfg.d, cfg.eps, clip_c=clip_c, sigma=sigma, layer_id=200001, noise_impl=noise_impl)
            self.lm_head = DPLinear(cfg.d, cfg.vocab, bias=False, clip_c=clip_c, sigma=sigma, reduction="mean",
                                    layer_id=200002, noise_impl=noise_impl)
        else:
            self.norm = _RMSNorm(cfg.d, cfg.eps)
            self.lm_head = linear_cls(cfg.d, cfg.vocab, bias=False)
        for p in self.parameters():
            if p.dim() >= 2:
                torch.nn.init.normal_(p, std=0.02)
        hd = cfg.d // cfg.heads
        inv = 1.0 / (10000 ** (torch.arange(0, hd, 2).float() / hd))
        ang = torch.outer(torch.arange(cfg.seq).float(), inv)
        ang = torch.cat((ang, ang), dim=-1)
        self.register_buffer("cos", ang.cos()[None, None], persistent=False)
        self.register_buffer("sin", ang.sin()[None, None], persistent=False)

    def dp_modules(self):
        return [m for m in self.modules() if isinstance(m, (DPLinear, _DPGroupModule))]

    def forward(self, idx):
        T = idx.shape[1]
        x = self.embed(idx)
        cos, sin = self.cos[:, :, :T], self.sin[:, :, :T]
        for blk in self.blocks:
            x = blk(x, cos, sin)
        return self.lm_head(self.norm(x))

    def loss(self, idx, targets, reduction: str = "mean"):
        """reduction "mean": over every token of the batch. "sample_sum": sum over
        samples of each sample's mean token loss -- the per-sample loss whose
        gradient is the sample's own, independent of how the batch is split over
        ranks (the DP modules then take the mean over the logical batch)."""
        with torch.autocast("cuda", dtype=torch.bfloat16, cache_enabled=False):  # CUDA-graph capturable
            logits = self(idx)
        if reduction == "mean":
            return F.cross_entropy(logits.float().view(-1, logits.shape[-1]), targets.view(-1))
        if reduction == "sample_sum":
            tok = F.cross_entropy(logits.float().view(-1, logits.shape[-1]), targets.view(-1), reduction="none")
            return tok.view(idx.shape[0], -1).mean(1).sum()
        raise ValueError(f"unknown reduction {reduction!r}")
