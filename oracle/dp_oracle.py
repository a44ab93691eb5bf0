"""CPU oracle for the FlashDP hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module, and only as the checker or the timed
CPU baseline. The product (paper_2507_01154_b200) never routes through it.

A float64 numpy restatement of the reference algorithm
(/root/reference/pkg/src/dpflows), written from its semantics:

  keyed RNG            rng.py:35-94   splitmix64 absorb, salted words, Box-Muller
  clip factor          dpcore.py:41-47, workflows.py:59-65
  finalize             dpcore.py:60-73  (sum | sum/B) + sigma*C*draw(flat index)
  per-sample G         oracle.py:16-36, tensor.py:64-73  G_b = dY_b^T X_b
  dp backward          oracle.py:49-65  clip-sum-noise
  flashdp workflow     workflows.py:340-421 (same arithmetic, tiling-invariant)
  micro-batching       dpcore.py:90-104, bench.py:244-271
  optimizer steps      dpcore.py:131-156 (SGD; Adam without bias correction, post-update v)
  training demo        bench.py:409-458 train_demo (least-squares linear layer)
  input generator      bench.py:234-241 cell_inputs, rng.py:88-94

Parity is pinned: tests/test_oracle_golden.py checks every function here
against golden vectors produced by the reference itself
(tools/gen_golden.py -> tests/golden/*.npz).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

M64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB
SALT_A = 0xD1B54A32D192ED03
SALT_B = 0x8BB84B93962EACC9
TWO_NEG53 = 2.0 ** -53
TWO_PI = 2.0 * math.pi


# ------------------------------------------------------------------ keyed RNG (rng.py:35-94)

def mix64(z: int) -> int:
    z &= M64
    z = ((z ^ (z >> 30)) * MIX1) & M64
    z = ((z ^ (z >> 27)) * MIX2) & M64
    return z ^ (z >> 31)


def absorb(*parts: int) -> int:
    h = mix64(parts[0] & M64) if parts else mix64(0)
    for v in parts[1:]:
        h = mix64((h + GAMMA) ^ (v & M64))
    return h


def _vmix(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * np.uint64(MIX1)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(MIX2)
    return z ^ (z >> np.uint64(31))


def keyed_words(seed: int, layer_id: int, step: int, idx) -> tuple[np.ndarray, np.ndarray]:
    """The two 53-bit words behind each draw (rng.py:51-54, vector form rng.py:75-79)."""
    idx = np.ascontiguousarray(idx, dtype=np.uint64)
    base = absorb(seed, layer_id, step)
    with np.errstate(over="ignore"):
        h = _vmix(np.uint64((base + GAMMA) & M64) ^ idx)
        w1 = _vmix(h ^ np.uint64(SALT_A)) >> np.uint64(11)
        w2 = _vmix(h ^ np.uint64(SALT_B)) >> np.uint64(11)
    return w1, w2


def keyed_normal(seed: int, layer_id: int, step: int, flat_index: int) -> float:
    """Scalar canonical draw with libm transcendentals (rng.py:50-60)."""
    state = absorb(seed, layer_id, step, flat_index)
    w1 = mix64(state ^ SALT_A)
    w2 = mix64(state ^ SALT_B)
    u1 = ((w1 >> 11) + 1) * TWO_NEG53
    u2 = (w2 >> 11) * TWO_NEG53
    return math.sqrt(-2.0 * math.log(u1)) * math.cos(TWO_PI * u2)


def keyed_normal_array(seed: int, layer_id: int, step: int, flat_indices, exact: bool = True) -> np.ndarray:
    """Vector draws. exact=True applies libm per element (bitwise = reference);
    exact=False uses numpy ufuncs (within ~1 ulp, for large oracle runs)."""
    w1, w2 = keyed_words(seed, layer_id, step, flat_indices)
    if exact:
        a, b = w1.ravel().tolist(), w2.ravel().tolist()
        out = np.fromiter((math.sqrt(-2.0 * math.log((x + 1) * TWO_NEG53)) * math.cos(TWO_PI * (y * TWO_NEG53))
                           for x, y in zip(a, b)), dtype=np.float64, count=len(a))
        return out.reshape(w1.shape)
    u1 = (w1.astype(np.float64) + 1.0) * TWO_NEG53
    u2 = w2.astype(np.float64) * TWO_NEG53
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(TWO_PI * u2)


def keyed_uniform_array(key_parts, count: int, low: float = -1.0, high: float = 1.0) -> np.ndarray:
    """Deterministic U[low, high) input generator (rng.py:88-94)."""
    base = absorb(*key_parts)
    idx = np.arange(count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = _vmix(np.uint64((base + GAMMA) & M64) ^ idx)
    u = (h >> np.uint64(11)).astype(np.float64) * TWO_NEG53
    return low + (high - low) * u


# ------------------------------------------------------------------ DP arithmetic

@dataclass(frozen=True)
class Cfg:
    clip_c: float
    sigma: float
    reduction: str = "sum"
    seed: int = 0
    layer_id: int = 0
    step: int = 0


def clip_factor(norm_sq: float, clip_c: float) -> float:
    """dpcore.py:41-47."""
    if norm_sq < 0:
        raise ValueError("norm_sq must be >= 0")
    if norm_sq == 0.0:
        return 1.0
    return min(1.0, clip_c / math.sqrt(norm_sq))


def clip_factors(norms_sq: np.ndarray, clip_c: float) -> np.ndarray:
    """workflows.py:59-65."""
    ns = np.asarray(norms_sq, dtype=np.float64)
    f = np.ones_like(ns)
    pos = ns > 0.0
    f[pos] = np.minimum(1.0, clip_c / np.sqrt(ns[pos]))
    return f


def noise(cfg: Cfg, n: int, lo: int = 0, hi: int | None = None, exact: bool = True) -> np.ndarray:
    hi = n if hi is None else hi
    return keyed_normal_array(cfg.seed, cfg.layer_id, cfg.step, np.arange(lo, hi), exact=exact)


def finalize(acc: np.ndarray, batch: int, cfg: Cfg, exact_noise: bool = True, lo: int = 0,
             hi: int | None = None, add_noise: bool = True) -> np.ndarray:
    """dpcore.py:60-73 on a (D,P) accumulator; noise only on flat indices [lo, hi)."""
    base = acc if cfg.reduction == "sum" else acc / batch
    if cfg.sigma == 0.0 or not add_noise:
        return base.copy()
    flat = base.reshape(-1).copy()
    hi = flat.size if hi is None else hi
    flat[lo:hi] += (cfg.sigma * cfg.clip_c) * noise(cfg, flat.size, lo, hi, exact=exact_noise)
    return flat.reshape(base.shape)


def per_sample_grads(x: np.ndarray, dy: np.ndarray) -> np.ndarray:
    """(B,D,P) float64: G_b = dY_b^T X_b (oracle.py:16-36)."""
    x = np.asarray(x, dtype=np.float64)
    dy = np.asarray(dy, dtype=np.float64)
    return np.matmul(dy.transpose(0, 2, 1), x)


def dp_backward(x: np.ndarray, dy: np.ndarray, cfg: Cfg, exact_noise: bool = True, *, mean_batch: int | None = None,
                noise_lo: int = 0, noise_hi: int | None = None, add_noise: bool = True):
    """Clip-sum-noise (oracle.py:49-65). Returns (grad_w (D,P), norms_sq (B,))."""
    g = per_sample_grads(x, dy)
    norms = np.einsum("bdp,bdp->b", g, g)
    f = clip_factors(norms, cfg.clip_c)
    acc = np.einsum("b,bdp->dp", f, g)
    batch = g.shape[0] if mean_batch is None else mean_batch
    return finalize(acc, batch, cfg, exact_noise, noise_lo, noise_hi, add_noise), norms


def dp_backward_streaming(x: np.ndarray, dy: np.ndarray, cfg: Cfg, exact_noise: bool = False):
    """Same result, one sample at a time (bounded memory for large layers):
    the flashdp dataflow of workflows.py:371-418 with whole-layer blocks."""
    B = x.shape[0]
    D, P = dy.shape[2], x.shape[2]
    acc = np.zeros((D, P))
    norms = np.zeros(B)
    for b in range(B):
        gb = np.asarray(dy[b], dtype=np.float64).T @ np.asarray(x[b], dtype=np.float64)
        norms[b] = float(np.einsum("dp,dp->", gb, gb))
        acc += clip_factor(norms[b], cfg.clip_c) * gb
    return finalize(acc, B, cfg, exact_noise), norms


def per_sample_accumulate(x: np.ndarray, dy: np.ndarray, clip_c: float, scale: float = 1.0):
    """Per-sample G_b, norm, clip, accumulate (workflows.py:381-407 with whole-layer
    blocks); no finalize. Returns (acc (D,P), norms (B,))."""
    B = x.shape[0]
    acc = np.zeros((dy.shape[2], x.shape[2]))
    norms = np.zeros(B)
    for b in range(B):
        gb = np.asarray(dy[b], dtype=np.float64).T @ np.asarray(x[b], dtype=np.float64)
        norms[b] = float(np.einsum("dp,dp->", gb, gb))
        acc += (clip_factor(norms[b], clip_c) * scale) * gb
    return acc, norms


def nondp_backward(x: np.ndarray, dy: np.ndarray) -> np.ndarray:
    """workflows.py:121-150."""
    return per_sample_grads(x, dy).sum(axis=0)


# ------------------------------------------------------------------ non-linear parameter groups
# SURVEY 8f rank 3. Not in the reference (SPEC.md:8 clips linear weights only); the
# per-sample gradients below are the textbook ones and everything after them (norm,
# clip_factors, sum / mean, keyed noise on [lo, hi) of the group's own index space)
# is the reference's per-layer arithmetic (oracle.py:49-65, dpcore.py:41-73).

def vector_per_sample_grads(dy: np.ndarray, xhat: np.ndarray | None, kind: str) -> np.ndarray:
    """(B, L): bias g_b = sum_t dY; rmsnorm g_b = sum_t dY * xhat (gamma);
    layernorm g_b = [sum_t dY * xhat (gamma), sum_t dY (beta)] (L = 2 D)."""
    dy = np.asarray(dy, dtype=np.float64)
    if kind == "bias":
        return dy.sum(axis=1)
    gam = (dy * np.asarray(xhat, dtype=np.float64)).sum(axis=1)
    if kind == "rmsnorm":
        return gam
    if kind == "layernorm":
        return np.concatenate([gam, dy.sum(axis=1)], axis=1)
    raise ValueError(kind)


def dp_vector_backward(dy, xhat, kind: str, cfg: Cfg, exact_noise: bool = True, *, noise_lo: int = 0,
                       noise_hi: int | None = None, mean_batch: int | None = None):
    """Clip-sum-noise of a bias / RMSNorm / LayerNorm parameter group. Returns (grad (L,), norms_sq (B,))."""
    g = vector_per_sample_grads(dy, xhat, kind)
    norms = (g * g).sum(axis=1)
    acc = (clip_factors(norms, cfg.clip_c)[:, None] * g).sum(axis=0)
    batch = g.shape[0] if mean_batch is None else mean_batch
    return finalize(acc, batch, cfg, exact_noise, noise_lo, noise_hi), norms


def embedding_per_sample_grads(tokens: np.ndarray, dy: np.ndarray, vocab: int) -> np.ndarray:
    """(B, V, d): G_b[v] = sum over positions t with tokens[b, t] == v of dY[b, t]."""
    tokens = np.asarray(tokens)
    dy = np.asarray(dy, dtype=np.float64)
    B, T, d = dy.shape
    g = np.zeros((B, vocab, d))
    for b in range(B):
        np.add.at(g[b], tokens[b], dy[b])
    return g


def embedding_norms_gram(tokens: np.ndarray, dy: np.ndarray) -> np.ndarray:
    """||G_b||^2 without G: sum over position pairs with equal tokens of <dY_t, dY_s>
    (the token-equality Gram of SURVEY 8f rank 3) -- a cross-check of the above."""
    dy = np.asarray(dy, dtype=np.float64)
    out = np.zeros(dy.shape[0])
    for b in range(dy.shape[0]):
        eq = (tokens[b][:, None] == tokens[b][None, :]).astype(np.float64)
        out[b] = float(np.einsum("ts,td,sd->", eq, dy[b], dy[b]))
    return out


def dp_embedding_backward(tokens, dy, vocab: int, cfg: Cfg, exact_noise: bool = True, *, noise_lo: int = 0,
                          noise_hi: int | None = None, mean_batch: int | None = None):
    """Clip-sum-noise of an embedding table (V, d): noise on every row (untouched
    rows included), flat index v * d + col. Returns (grad (V, d), norms_sq (B,))."""
    g = embedding_per_sample_grads(tokens, dy, vocab)
    norms = np.einsum("bvd,bvd->b", g, g)
    acc = np.einsum("b,bvd->vd", clip_factors(norms, cfg.clip_c), g)
    batch = g.shape[0] if mean_batch is None else mean_batch
    return finalize(acc, batch, cfg, exact_noise, noise_lo, noise_hi), norms


def micro_batched(x: np.ndarray, dy: np.ndarray, cfg: Cfg, size: int, exact_noise: bool = True) -> np.ndarray:
    """bench.py:244-271: sigma=0/sum micro runs, one finalize for the logical batch."""
    B = x.shape[0]
    acc = np.zeros((dy.shape[2], x.shape[2]))
    for i in range(0, B, size):
        micro = Cfg(cfg.clip_c, 0.0, "sum", cfg.seed, cfg.layer_id, cfg.step)
        part, _ = dp_backward(x[i:i + size], dy[i:i + size], micro)
        acc += part
    return finalize(acc, B, cfg, exact_noise)


def sgd_step(theta: np.ndarray, grad: np.ndarray, eta: float) -> np.ndarray:
    """dpcore.py:131-136."""
    return theta - eta * grad


def adam_step(theta, m, v, grad, eta, beta1=0.9, beta2=0.999, eps=1e-8):
    """dpcore.py:139-156: no bias correction, post-update v. Returns (theta, m, v)."""
    m = beta1 * m + (1.0 - beta1) * grad
    v = beta2 * v + (1.0 - beta2) * (grad * grad)
    theta = theta - (eta / (np.sqrt(v) + eps)) * m
    return theta, m, v


def train_demo(x, w0, y_target, sigma: float, steps: int, eta: float, optimizer: str = "sgd", clip_c: float = 1.0,
               seed: int = 2024, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8) -> np.ndarray:
    """bench.py:409-458: least-squares training of one linear layer; the loss is
    recorded before each update; the DP gradient is clip-sum-noise (reduction sum)
    keyed on (seed, layer 0, step)."""
    B, T, _ = x.shape
    D = w0.shape[0]
    denom = B * T * D
    theta = np.array(w0, dtype=np.float64)
    m = np.zeros_like(theta)
    v = np.zeros_like(theta)
    losses = []
    for step in range(steps):
        resid = np.einsum("btp,dp->btd", x, theta) - y_target
        losses.append(float((resid * resid).sum() / denom))
        dy = (2.0 / denom) * resid
        grad, _ = dp_backward(x, dy, Cfg(clip_c, sigma, "sum", seed, 0, step))
        if optimizer == "adam":
            theta, m, v = adam_step(theta, m, v, grad, eta, beta1, beta2, eps)
        else:
            theta = sgd_step(theta, grad, eta)
    return np.array(losses)


def cell_inputs(seed: int, layer_index: int, B: int, T: int, P: int, D: int) -> tuple[np.ndarray, np.ndarray]:
    """bench.py:234-241 (streams 101 / 202)."""
    x = keyed_uniform_array((seed, 101, layer_index, B), B * T * P).reshape(B, T, P)
    dy = keyed_uniform_array((seed, 202, layer_index, B), B * T * D).reshape(B, T, D)
    return x, dy


def noise_partition(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous rank slice of [0, n) (noise-once under data parallelism)."""
    return n * rank // world, n * (rank + 1) // world


# ------------------------------------------------------------------ ledgers (memmodel counters)

def ledger(kind: str, B: int, T: int, P: int, D: int, width: int, n_b=1, n_d=1, n_p=1) -> dict:
    """Closed forms of the reference TrafficReport counters."""
    inputs, g, dp = B * T * (P + D), B * D * P, D * P
    if kind == "non_dp":
        return {"bytes_loaded": inputs * width, "bytes_stored": dp * width, "flops": 2 * B * T * D * P}
    if kind == "explicit_dp":
        return {"bytes_loaded": (inputs + 3 * g + B) * width, "bytes_stored": (2 * g + B + dp) * width,
                "flops": 2 * B * T * D * P + 4 * g + dp}
    if kind == "implicit_dp":
        return {"bytes_loaded": (2 * inputs + B) * width, "bytes_stored": (B + dp) * width,
                "flops": 4 * B * T * D * P + 4 * g + dp}
    return {"bytes_loaded": (inputs + n_p * n_d * B + dp) * width,
            "bytes_stored": (n_p * n_d * B + n_b * dp + dp) * width,
            "flops": 2 * B * T * D * P + 4 * g + dp}


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float64 (what the GPU sees)."""
    f = np.asarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)
