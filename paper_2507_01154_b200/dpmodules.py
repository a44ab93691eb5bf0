"""DP gradients of the non-linear parameters of a model.

The reference clips linear-layer weights only; full-model DP
training also needs every other parameter clipped per sample. Each module here
is its own per-layer clipping group with the reference's arithmetic -- own C,
sigma, ``layer_id`` noise key, clip factor dpcore.py:41-47, sum or mean over the
logical batch + sigma*C*N(seed, layer_id, step, i) (dpcore.py:60-73) -- computed
by the CUDA kernels of ``csrc/fdp_params.cu`` through the C ABI:

* ``DPLayerNorm`` / ``DPRMSNorm``: per-sample gamma gradient sum_t dY * xhat
  (and beta sum_t dY); gamma and beta form one group (``fdp_vec_dw``).
* ``DPEmbedding``: per-sample table gradient = scatter of dY rows onto the
  sample's token rows; its norm is the token-equality Gram, computed from
  sorted (token, position) runs without materialising the (V, d) per-sample
  gradient (``fdp_embedding_dw``). Every row gets its noise.
* ``vector_dp_grad`` / ``embedding_dp_grad``: the functional forms.

The first dimension of every input is the sample dimension (B, T, ...).
"""

from __future__ import annotations

import ctypes
from typing import Optional

import torch
import torch.nn.functional as F

from . import _lib
from .dpcore import DPConfig
from .errors import ShapeError, UsageError


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return _lib.DTYPE_BF16
    if t.dtype == torch.float32:
        return _lib.DTYPE_F32
    raise UsageError(f"parameter-group gradients take bfloat16 or float32 CUDA tensors, got {t.dtype}")


def _desc(cfg: DPConfig, B, T, P, D, dtype_code, *, rank, world, mean_batch, add_noise, noise_impl, accumulate):
    return _lib.make_desc(B=B, T=T, P=P, D=D, in_dtype=dtype_code, reduction=cfg.reduction, clip_c=cfg.clip_c,
                          sigma=cfg.sigma, seed=cfg.seed, layer_id=cfg.layer_id, step=cfg.step, rank=rank,
                          world=world, mean_batch=mean_batch, accumulate=accumulate, add_noise=add_noise,
                          noise_impl=noise_impl)


_WS: dict = {}
_DESCS: dict = {}


def _cached_desc(tag, cfg: DPConfig, B, T, P, D, dtype_code, *, size_fn, **kw):
    """Descriptor + workspace size per call signature (a training loop repeats the
    same shapes every step; only the step key changes): validated once by the C
    library, then reused with the step patched in."""
    key = (tag, B, T, P, D, dtype_code, cfg.clip_c, cfg.sigma, cfg.reduction, cfg.seed, cfg.layer_id,
           tuple(sorted(kw.items())))
    hit = _DESCS.get(key)
    if hit is None:
        desc = _desc(cfg, B, T, P, D, dtype_code, **kw)
        nb = ctypes.c_size_t()
        _lib.check(size_fn(ctypes.byref(desc), ctypes.byref(nb)))
        if len(_DESCS) > 4096:
            _DESCS.clear()
        hit = _DESCS[key] = (desc, nb)
    desc, nb = hit
    desc.step = _lib._wrap64(cfg.step)
    return desc, nb


def _workspace(device: torch.device, nbytes: int) -> torch.Tensor:
    """A per-(device, stream) scratch buffer grown on demand (stream-ordered reuse)."""
    key = (device, torch.cuda.current_stream(device).cuda_stream)
    ws = _WS.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.empty(max(nbytes, 4096), dtype=torch.uint8, device=device)
        _WS[key] = ws
    return ws


def vector_dp_grad(kind: str, dy: torch.Tensor, xhat: Optional[torch.Tensor], cfg: DPConfig, *, rank: int = 0,
                   world: int = 1, mean_batch: int = 0, add_noise: bool = True, noise_impl: str = "keyed_f32",
                   out: Optional[torch.Tensor] = None, accumulate: bool = False,
                   norms_sq: Optional[torch.Tensor] = None) -> torch.Tensor:
    """DP gradient of a bias / RMSNorm gamma / LayerNorm [gamma, beta] group.

    dy, xhat: (B, T, D) (xhat unused for "bias"). Returns (D,) or, for
    "layernorm", (2 D,) = [gamma grad, beta grad], fp32."""
    if kind not in _lib.VEC_KIND:
        raise UsageError(f"kind must be one of {tuple(_lib.VEC_KIND)}, got {kind!r}")
    if dy.dim() != 3:
        raise ShapeError(f"dy must be (B, T, D), got {tuple(dy.shape)}")
    B, T, D = dy.shape
    if kind != "bias":
        if xhat is None or tuple(xhat.shape) != (B, T, D):
            raise ShapeError(f"xhat must match dy's shape {tuple(dy.shape)}")
        if xhat.dtype != dy.dtype:
            dy, xhat = dy.float(), xhat.float()
        xhat = xhat.contiguous()
    dy = dy.contiguous()
    if not dy.is_cuda:
        raise UsageError("vector_dp_grad needs CUDA tensors")
    L = 2 * D if kind == "layernorm" else D
    lib = _lib.load()
    k = _lib.VEC_KIND[kind]
    desc, nb = _cached_desc(("vec", k), cfg, B, T, 8, D, _dtype_code(dy), rank=rank, world=world,
                            mean_batch=mean_batch, add_noise=add_noise, noise_impl=noise_impl, accumulate=accumulate,
                            size_fn=lambda d, out: lib.fdp_vec_workspace_bytes(d, k, out))
    if out is None:
        out = (torch.zeros if accumulate else torch.empty)(L, dtype=torch.float32, device=dy.device)
    elif out.dtype != torch.float32 or out.numel() != L or not out.is_contiguous():
        raise ShapeError(f"out must be a contiguous fp32 tensor of {L} elements")
    if norms_sq is not None and (norms_sq.dtype != torch.float32 or norms_sq.numel() != B):
        raise ShapeError(f"norms_sq must be an fp32 tensor of {B} elements")
    ws = _workspace(dy.device, nb.value)
    _lib.check(lib.fdp_vec_dw(ctypes.byref(desc), k, dy.data_ptr(), None if xhat is None else xhat.data_ptr(),
                              out.data_ptr(), None if norms_sq is None else norms_sq.data_ptr(), ws.data_ptr(),
                              ws.numel(), torch.cuda.current_stream(dy.device).cuda_stream))
    return out


def embedding_dp_grad(tokens: torch.Tensor, dy: torch.Tensor, vocab: int, cfg: DPConfig, *, rank: int = 0,
                      world: int = 1, mean_batch: int = 0, add_noise: bool = True, noise_impl: str = "keyed_f32",
                      out: Optional[torch.Tensor] = None, accumulate: bool = False,
                      norms_sq: Optional[torch.Tensor] = None) -> torch.Tensor:
    """DP gradient of an embedding table (vocab, d) from tokens (B, T) and dY (B, T, d); fp32."""
    if tokens.dim() != 2 or dy.dim() != 3 or tuple(tokens.shape) != tuple(dy.shape[:2]):
        raise ShapeError(f"tokens (B, T) and dy (B, T, d) expected, got {tuple(tokens.shape)} and {tuple(dy.shape)}")
    if not (tokens.is_cuda and dy.is_cuda):
        raise UsageError("embedding_dp_grad needs CUDA tensors")
    B, T, D = dy.shape
    if dy.dtype not in (torch.bfloat16, torch.float32):
        dy = dy.float()
    dy = dy.contiguous()
    tokens = tokens.to(torch.int64).contiguous()
    lib = _lib.load()
    desc, nb = _cached_desc(("emb",), cfg, B, T, int(vocab), D, _dtype_code(dy), rank=rank, world=world,
                            mean_batch=mean_batch, add_noise=add_noise, noise_impl=noise_impl, accumulate=accumulate,
                            size_fn=lib.fdp_embedding_workspace_bytes)
    if out is None:
        out = (torch.zeros if accumulate else torch.empty)((vocab, D), dtype=torch.float32, device=dy.device)
    elif out.dtype != torch.float32 or tuple(out.shape) != (vocab, D) or not out.is_contiguous():
        raise ShapeError(f"out must be a contiguous fp32 tensor of shape {(vocab, D)}")
    if norms_sq is not None and (norms_sq.dtype != torch.float32 or norms_sq.numel() != B):
        raise ShapeError(f"norms_sq must be an fp32 tensor of {B} elements")
    ws = _workspace(dy.device, nb.value)
    _lib.check(lib.fdp_embedding_dw(ctypes.byref(desc), tokens.data_ptr(), dy.data_ptr(), out.data_ptr(),
                                    None if norms_sq is None else norms_sq.data_ptr(), ws.data_ptr(), ws.numel(),
                                    torch.cuda.current_stream(dy.device).cuda_stream))
    return out


class _DPGroupModule(torch.nn.Module):
    """Shared per-layer DP state (mirrors DPLinear: DPConfig fields, layer_id,
    set_step for micro-batching, rank / world noise partition)."""

    def _init_dp(self, clip_c, sigma, reduction, seed, layer_id, noise_impl):
        DPConfig(clip_c, sigma, reduction)  # validate
        self.clip_c, self.sigma, self.reduction, self.seed = clip_c, sigma, reduction, seed
        self.layer_id = layer_id
        self.noise_impl = noise_impl
        self.step = 0
        self._noise_now = True
        self.logical_batch: Optional[int] = None
        self.rank, self.world = 0, 1
        self.last_norms_sq: Optional[torch.Tensor] = None

    def dp_config(self) -> DPConfig:
        return DPConfig(self.clip_c, self.sigma, self.reduction, self.seed, self.layer_id, self.step)

    def set_step(self, step: int, *, last_micro_batch: bool = True, logical_batch: Optional[int] = None) -> None:
        self.step = step
        self._noise_now = last_micro_batch
        self.logical_batch = logical_batch

    def _dp_kw(self, B: int) -> dict:
        return dict(rank=self.rank, world=self.world, mean_batch=self.logical_batch or B,
                    add_noise=self._noise_now, noise_impl=self.noise_impl)


class _DPAffineFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, xhat, weight, bias, module):
        ctx.module = module
        ctx.has_bias = bias is not None
        ctx.save_for_backward(xhat, weight)
        y = xhat * weight.to(xhat.dtype)
        return y + bias.to(xhat.dtype) if bias is not None else y

    @staticmethod
    def backward(ctx, dy):
        xhat, weight = ctx.saved_tensors
        m = ctx.module
        dxhat = (dy * weight.to(dy.dtype)) if ctx.needs_input_grad[0] else None
        D = weight.numel()
        B = xhat.shape[0] if xhat.dim() > 1 else 1
        kind = "layernorm" if ctx.has_bias else "rmsnorm"
        norms = torch.empty(B, dtype=torch.float32, device=dy.device)
        g = vector_dp_grad(kind, dy.reshape(B, -1, D), xhat.reshape(B, -1, D), m.dp_config(), norms_sq=norms,
                           **m._dp_kw(B))
        m.last_norms_sq = norms
        gw = g[:D].view_as(weight).to(weight.dtype)
        gb = g[D:].view_as(weight).to(weight.dtype) if ctx.has_bias else None
        return dxhat, gw, gb, None


class DPLayerNorm(_DPGroupModule):
    """nn.LayerNorm over the last dimension whose (gamma, beta) gradient is the
    per-layer DP gradient of the pair as one clipping group."""

    def __init__(self, normalized_shape: int, eps: float = 1e-5, bias: bool = True, *, clip_c: float = 1.0,
                 sigma: float = 1.0, reduction: str = "mean", seed: int = 0, layer_id: int = 0,
                 noise_impl: str = "keyed_f32", device=None, dtype=None):
        super().__init__()
        self.normalized_shape = (int(normalized_shape),)
        self.eps = eps
        self.weight = torch.nn.Parameter(torch.ones(normalized_shape, device=device, dtype=dtype))
        self.bias = torch.nn.Parameter(torch.zeros(normalized_shape, device=device, dtype=dtype)) if bias else None
        self._init_dp(clip_c, sigma, reduction, seed, layer_id, noise_impl)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        xhat = F.layer_norm(x, self.normalized_shape, None, None, self.eps)
        if self.bias is None:  # gamma only: the RMSNorm-shaped group over the centred input
            return _DPAffineFn.apply(xhat, self.weight, None, self)
        return _DPAffineFn.apply(xhat, self.weight, self.bias, self)


class DPRMSNorm(_DPGroupModule):
    """RMSNorm (x / rms(x) * gamma) with the per-layer DP gamma gradient."""

    def __init__(self, dim: int, eps: float = 1e-6, *, clip_c: float = 1.0, sigma: float = 1.0,
                 reduction: str = "mean", seed: int = 0, layer_id: int = 0, noise_impl: str = "keyed_f32",
                 device=None, dtype=None):
        super().__init__()
        self.eps = eps
        self.weight = torch.nn.Parameter(torch.ones(dim, device=device, dtype=dtype))
        self._init_dp(clip_c, sigma, reduction, seed, layer_id, noise_impl)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        xf = x.float()
        xhat = xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + self.eps)
        return _DPAffineFn.apply(xhat, self.weight, None, self)


class _DPEmbeddingFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, tokens, weight, module):
        ctx.module = module
        ctx.save_for_backward(tokens)
        ctx.shape = weight.shape
        ctx.wdtype = weight.dtype
        return F.embedding(tokens, weight)

    @staticmethod
    def backward(ctx, dy):
        (tokens,) = ctx.saved_tensors
        m = ctx.module
        V, D = ctx.shape
        B = tokens.shape[0]
        t2 = tokens.reshape(B, -1)
        norms = torch.empty(B, dtype=torch.float32, device=dy.device)
        g = embedding_dp_grad(t2, dy.reshape(B, t2.shape[1], D), V, m.dp_config(), norms_sq=norms, **m._dp_kw(B))
        m.last_norms_sq = norms
        return None, g.to(ctx.wdtype), None


class DPEmbedding(_DPGroupModule):
    """nn.Embedding whose table gradient is the per-layer DP gradient. Inputs are
    (B, T) token ids (sample dimension first; expand shared positions per sample)."""

    def __init__(self, num_embeddings: int, embedding_dim: int, *, clip_c: float = 1.0, sigma: float = 1.0,
                 reduction: str = "mean", seed: int = 0, layer_id: int = 0, noise_impl: str = "keyed_f32",
                 device=None, dtype=None):
        super().__init__()
        self.num_embeddings, self.embedding_dim = num_embeddings, embedding_dim
        self.weight = torch.nn.Parameter(torch.empty(num_embeddings, embedding_dim, device=device, dtype=dtype))
        torch.nn.init.normal_(self.weight)
        self._init_dp(clip_c, sigma, reduction, seed, layer_id, noise_impl)

    def forward(self, tokens: torch.Tensor) -> torch.Tensor:
        if tokens.dim() < 2:
            raise ShapeError("DPEmbedding takes (B, T) token ids: the first dimension is the sample dimension")
        return _DPEmbeddingFn.apply(tokens, self.weight, self)
