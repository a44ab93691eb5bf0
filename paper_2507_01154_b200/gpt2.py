"""GPT-2 small with DP linear layers: the consumer of the hot path in a training step.

``dp="full"`` makes every parameter DP: token and position
embeddings are ``DPEmbedding``, the LayerNorms ``DPLayerNorm``, and the LM head
an untied ``DPLinear`` over the vocabulary padded to a multiple of 64 (the
non-DP baseline of that mode is built with ``tied=False`` and the same padding).

Only the four linear layers of every block (attention c_attn / c_proj, MLP c_fc /
c_proj) are the reference's hot path (per-layer DP weight gradients,
workflows.py:340-421); they are ``DPLinear`` modules whose weight gradients
come from ONE multi-layer persistent launch per backward
(``GroupedDPBackward``). Everything else (embeddings, LayerNorm, attention core,
LM head) is plain PyTorch and, like in the reference, not clipped
per sample. ``dp=False`` builds the same model with ``nn.Linear`` -- the non-DP
baseline of "% of non-DP training throughput".

Random-init weights, synthetic token ids; bf16 compute, fp32 master weights.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.nn.functional as F

from .dplinear import DPLinear
from .dpmodules import DPEmbedding, DPLayerNorm, _DPGroupModule


@dataclass
class GPT2Config:
    vocab: int = 50257
    seq: int = 1024
    d: int = 768
    heads: int = 12
    layers: int = 12
    mlp: int = 3072


def _linear(cin: int, cout: int, dp: bool, layer_id: int, clip_c: float, sigma: float, noise_impl: str,
            nondp_cls=torch.nn.Linear):
    if dp:
        return DPLinear(cin, cout, bias=True, clip_c=clip_c, sigma=sigma, reduction="mean", layer_id=layer_id,
                        noise_impl=noise_impl)
    return nondp_cls(cin, cout, bias=True)


def _nondp_cls(name: str):
    """non-DP projections: "torch" (nn.Linear: autocast bf16 dW cast into the fp32
    .grad) or "fp32grad" (baselines.FP32GradLinear: cuBLAS writes the fp32 weight
    gradient, the DP kernels' output precision -- the like-for-like baseline)."""
    if name == "torch":
        return torch.nn.Linear
    if name == "fp32grad":
        from .baselines import FP32GradLinear
        return FP32GradLinear
    raise ValueError(f"nondp_linear must be torch or fp32grad, got {name!r}")


def _layernorm(d: int, dp_full: bool, layer_id: int, clip_c: float, sigma: float, noise_impl: str):
    if dp_full:
        return DPLayerNorm(d, clip_c=clip_c, sigma=sigma, reduction="mean", layer_id=layer_id, noise_impl=noise_impl)
    return torch.nn.LayerNorm(d)


class Block(torch.nn.Module):
    def __init__(self, cfg: GPT2Config, idx: int, dp, clip_c: float, sigma: float, noise_impl: str,
                 nondp_cls=torch.nn.Linear):
        super().__init__()
        full = dp == "full"
        self.ln1 = _layernorm(cfg.d, full, 1002 + 2 * idx, clip_c, sigma, noise_impl)
        self.ln2 = _layernorm(cfg.d, full, 1003 + 2 * idx, clip_c, sigma, noise_impl)
        dp = bool(dp)
        base = 4 * idx
        self.c_attn = _linear(cfg.d, 3 * cfg.d, dp, base + 0, clip_c, sigma, noise_impl, nondp_cls)
        self.attn_proj = _linear(cfg.d, cfg.d, dp, base + 1, clip_c, sigma, noise_impl, nondp_cls)
        self.c_fc = _linear(cfg.d, cfg.mlp, dp, base + 2, clip_c, sigma, noise_impl, nondp_cls)
        self.mlp_proj = _linear(cfg.mlp, cfg.d, dp, base + 3, clip_c, sigma, noise_impl, nondp_cls)
        self.heads = cfg.heads

    def forward(self, x):
        B, T, C = x.shape
        qkv = self.c_attn(self.ln1(x))
        q, k, v = qkv.split(C, dim=2)
        q = q.view(B, T, self.heads, C // self.heads).transpose(1, 2)
        k = k.view(B, T, self.heads, C // self.heads).transpose(1, 2)
        v = v.view(B, T, self.heads, C // self.heads).transpose(1, 2)
        y = F.scaled_dot_product_attention(q, k, v, is_causal=True)
        x = x + self.attn_proj(y.transpose(1, 2).reshape(B, T, C))
        return x + self.mlp_proj(F.gelu(self.c_fc(self.ln2(x)), approximate="tanh"))


class GPT2(torch.nn.Module):
    def __init__(self, cfg: GPT2Config, *, dp=True, clip_c: float = 1.0, sigma: float = 1.0,
                 noise_impl: str = "philox", tied: bool = True, nondp_linear: str = "torch"):
        super().__init__()
        self.cfg = cfg
        nondp_cls = _nondp_cls(nondp_linear)
        full = dp == "full"
        self.tied = tied and not full
        if full:
            self.wte = DPEmbedding(cfg.vocab, cfg.d, clip_c=clip_c, sigma=sigma, layer_id=1000, noise_impl=noise_impl)
            self.wpe = DPEmbedding(cfg.seq, cfg.d, clip_c=clip_c, sigma=sigma, layer_id=1001, noise_impl=noise_impl)
        else:
            self.wte = torch.nn.Embedding(cfg.vocab, cfg.d)
            self.wpe = torch.nn.Embedding(cfg.seq, cfg.d)
        self.blocks = torch.nn.ModuleList(Block(cfg, i, dp, clip_c, sigma, noise_impl, nondp_cls)
                                          for i in range(cfg.layers))
        self.ln_f = _layernorm(cfg.d, full, 1100, clip_c, sigma, noise_impl)
        self.vocab_padded = (cfg.vocab + 63) // 64 * 64
        self.lm_head = None
        if not self.tied:
            self.lm_head = (DPLinear(cfg.d, self.vocab_padded, bias=False, clip_c=clip_c, sigma=sigma,
                                     reduction="mean", layer_id=4 * cfg.layers, noise_impl=noise_impl)
                            if full else nondp_cls(cfg.d, self.vocab_padded, bias=False))
        self.dp = dp
        for p in self.parameters():
            if p.dim() >= 2:
                torch.nn.init.normal_(p, std=0.02 / math.sqrt(2 * cfg.layers) if p.shape[0] == cfg.d else 0.02)

    def dp_layers(self):
        return [m for m in self.modules() if isinstance(m, DPLinear)]

    def dp_modules(self):
        """Every module with a per-layer DP gradient (set_step each step)."""
        return [m for m in self.modules() if isinstance(m, (DPLinear, _DPGroupModule))]

    def forward(self, idx):
        B, T = idx.shape
        pos = torch.arange(T, device=idx.device)
        if self.dp == "full":  # per-sample position ids: the sample dimension stays first
            x = self.wte(idx) + self.wpe(pos.expand(B, T))
        else:
            x = self.wte(idx) + self.wpe(pos)[None]
        for blk in self.blocks:
            x = blk(x)
        h = self.ln_f(x)
        if self.tied:
            return F.linear(h, self.wte.weight)  # tied LM head
        return self.lm_head(h)[..., :self.cfg.vocab]

    def loss(self, idx, targets):
        with torch.autocast("cuda", dtype=torch.bfloat16, cache_enabled=False):  # CUDA-graph capturable
            logits = self(idx)
        return F.cross_entropy(logits.float().view(-1, logits.shape[-1]), targets.view(-1))
