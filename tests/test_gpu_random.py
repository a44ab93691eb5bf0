"""Randomised GPU parity sweep: many (B, T, P, D, C, sigma, reduction, path,
noise) draws through the drop-in API against the CPU oracle on the same
bf16-rounded inputs (rel <= 1e-3), reference-keyed noise so sigma > 0 is exact.
Shapes include ragged T (not a multiple of 64/128/256), P/D multiples of 8 that
are not multiples of the tile, single samples, and clip levels that clip some,
all or none of the samples. The seed is fixed: the draws are reproducible."""

import numpy as np
import pytest
import torch

import paper_2507_01154_b200 as fdp
from oracle import dp_oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-3
N_CASES = 120


def _rel(got, want):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    return float(np.max(np.abs(got - want))) / max(float(np.max(np.abs(want))), 1e-30)


def _cases():
    rng = np.random.default_rng(20261017)
    out = []
    for i in range(N_CASES):
        B = int(rng.choice([1, 2, 3, 5, 8]))
        T = int(rng.choice([1, 7, 64, 100, 130, 256, 300]))
        P = int(8 * rng.integers(1, 72))     # 8 .. 568
        D = int(8 * rng.integers(1, 72))
        path = str(rng.choice(["auto", "fused", "two_phase"]))
        norm_phase = str(rng.choice(["auto", "ghost", "recompute"])) if path == "two_phase" else "auto"
        if path == "two_phase" and B == 1 and rng.random() < 0.5:
            norm_phase = "single"
        red = str(rng.choice(["sum", "mean"]))
        sigma = float(rng.choice([0.0, 0.5, 1.0]))
        out.append((i, B, T, P, D, path, norm_phase, red, sigma, int(rng.integers(0, 1 << 30))))
    return out


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"c{c[0]}-B{c[1]}T{c[2]}P{c[3]}D{c[4]}-{c[5]}-{c[6]}")
def test_random_parity(case):
    i, B, T, P, D, path, norm_phase, red, sigma, seed = case
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(B, T, P, generator=g).to(torch.bfloat16).cuda()
    dy = (torch.randn(B, T, D, generator=g) * 0.05).to(torch.bfloat16).cuda()
    xh, yh = x.double().cpu().numpy(), dy.double().cpu().numpy()
    norms = np.einsum("bdp,bdp->b", *(2 * [O.per_sample_grads(xh, yh)]))
    # clip level: below, around or above the per-sample norms (some / all / no samples clipped)
    C = float(np.sqrt(np.quantile(norms, [0.0, 0.5, 1.0][i % 3])) * [0.5, 1.0, 2.0][i % 3]) or 1.0
    cfg = fdp.DPConfig(C, sigma, red, seed=seed % 1000, layer_id=i, step=i % 7)
    r = fdp.backward_flashdp(x, dy, cfg, path=path, norm_phase=norm_phase, noise_impl="keyed_f64")
    want, wn = O.dp_backward(xh, yh, O.Cfg(C, sigma, red, cfg.seed, cfg.layer_id, cfg.step), exact_noise=True)
    assert _rel(r.grad_w.double().cpu().numpy(), want) < TOL
    assert _rel(r.per_sample_norms_sq.double().cpu().numpy(), wn) < TOL


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_random_group_parity(seed):
    """A random layer list (2-6 layers, mixed shapes and DP configs) in ONE
    persistent multi-layer launch (PreparedGroup) against the oracle per layer."""
    rng = np.random.default_rng(seed)
    B = int(rng.choice([2, 4, 8]))
    T = int(rng.choice([64, 100, 256]))
    layers, host = [], []
    for li in range(int(rng.integers(2, 7))):
        P, D = int(8 * rng.integers(4, 64)), int(8 * rng.integers(4, 64))
        g = torch.Generator().manual_seed(seed * 100 + li)
        x = torch.randn(B, T, P, generator=g).to(torch.bfloat16).cuda()
        dy = (torch.randn(B, T, D, generator=g) * 0.05).to(torch.bfloat16).cuda()
        cfg = fdp.DPConfig(float(rng.uniform(0.1, 3.0)), float(rng.choice([0.0, 1.0])),
                           str(rng.choice(["sum", "mean"])), seed=seed, layer_id=li, step=seed)
        layers.append((x, dy, cfg))
        host.append((x.double().cpu().numpy(), dy.double().cpu().numpy(), cfg))
    try:
        grp = fdp.PreparedGroup(layers, noise_impl="keyed_f64")
    except fdp.UsageError:
        pytest.skip("layer list does not fit the co-resident fused grid")
    grp()
    torch.cuda.synchronize()
    for (xh, yh, c), gw, nrm in zip(host, grp.grads, grp.norms):
        want, wn = O.dp_backward(xh, yh, O.Cfg(c.clip_c, c.sigma, c.reduction, c.seed, c.layer_id, c.step),
                                 exact_noise=True)
        assert _rel(gw.double().cpu().numpy(), want) < TOL
        assert _rel(nrm.double().cpu().numpy(), wn) < TOL


@pytest.mark.parametrize("B,T,P,D,path", [
    (64, 1, 256, 256, "fused"), (64, 3, 512, 128, "two_phase"), (1, 4096, 8, 8, "auto"),
    (3, 5000, 64, 72, "auto"), (2, 33, 8, 4096, "auto"), (2, 33, 4096, 8, "auto"),
    (128, 16, 128, 128, "fused"), (96, 8, 384, 256, "two_phase"), (1, 1, 8, 8, "auto")])
def test_extreme_shapes(B, T, P, D, path):
    """Degenerate and extreme extents: single tokens, one sample, very long or very
    short sequences, skinny layers, many samples per tile (several sample groups)."""
    g = torch.Generator().manual_seed(B * 7 + T)
    x = torch.randn(B, T, P, generator=g).to(torch.bfloat16).cuda()
    dy = (torch.randn(B, T, D, generator=g) * 0.05).to(torch.bfloat16).cuda()
    cfg = fdp.DPConfig(0.2, 1.0, "mean", seed=4, layer_id=1, step=2)
    r = fdp.backward_flashdp(x, dy, cfg, path=path, noise_impl="keyed_f64")
    want, wn = O.dp_backward(x.double().cpu().numpy(), dy.double().cpu().numpy(),
                             O.Cfg(0.2, 1.0, "mean", 4, 1, 2), exact_noise=True)
    assert _rel(r.grad_w.double().cpu().numpy(), want) < TOL
    assert _rel(r.per_sample_norms_sq.double().cpu().numpy(), wn) < TOL


def _group_cases():
    rng = np.random.default_rng(20261018)
    out = []
    for i in range(40):
        kind = str(rng.choice(["bias", "rmsnorm", "layernorm", "embedding"]))
        B = int(rng.choice([1, 2, 3, 7, 16]))
        T = int(rng.choice([1, 5, 33, 64, 130, 257]))
        D = int(rng.choice([8, 24, 96, 130, 256, 770]))
        V = int(rng.choice([1, 3, 40, 300]))
        dtype = torch.bfloat16 if rng.random() < 0.5 else torch.float32
        world = int(rng.choice([1, 1, 2, 3]))
        rank = int(rng.integers(0, world))
        red = str(rng.choice(["sum", "mean"]))
        sigma = float(rng.choice([0.0, 0.7]))
        clip_q = float(rng.choice([0.25, 0.5, 2.0]))  # C as a quantile multiple of the median norm
        out.append((i, kind, B, T, D, V, dtype, rank, world, red, sigma, clip_q))
    return out


@pytest.mark.parametrize("case", _group_cases(), ids=lambda c: f"g{c[0]}-{c[1]}")
def test_random_parameter_groups_against_oracle(case):
    """Random bias / RMSNorm / LayerNorm / embedding groups (shapes, dtypes, rank
    slices, reductions, clip levels) against the oracle's restatements, keyed noise."""
    i, kind, B, T, D, V, dtype, rank, world, red, sigma, clip_q = case
    g = torch.Generator().manual_seed(1000 + i)
    dy = (torch.randn(B, T, D, generator=g) * 0.1).to(dtype)
    if kind == "embedding":
        tok = torch.randint(0, V, (B, T), generator=g)
        G = O.embedding_per_sample_grads(tok.numpy(), dy.double().numpy(), V)
        ns = np.einsum("bvd,bvd->b", G, G)
    else:
        xh = torch.randn(B, T, D, generator=g).to(dtype)
        ns = (O.vector_per_sample_grads(dy.double().numpy(), xh.double().numpy(), kind) ** 2).sum(1)
    C = max(float(np.median(np.sqrt(ns))) * clip_q, 1e-6)
    cfg = fdp.DPConfig(C, sigma, red, seed=7, layer_id=i, step=3)
    ocfg = O.Cfg(C, sigma, red, 7, i, 3)
    norms = torch.empty(B, device="cuda")
    if kind == "embedding":
        n = V * D
        lo, hi = n * rank // world, n * (rank + 1) // world
        got = fdp.embedding_dp_grad(tok.cuda(), dy.cuda(), V, cfg, noise_impl="keyed_f64", rank=rank, world=world,
                                    norms_sq=norms)
        want, wn = O.dp_embedding_backward(tok.numpy(), dy.double().numpy(), V, ocfg, noise_lo=lo, noise_hi=hi)
    else:
        n = 2 * D if kind == "layernorm" else D
        lo, hi = n * rank // world, n * (rank + 1) // world
        got = fdp.vector_dp_grad(kind, dy.cuda(), xh.cuda(), cfg, noise_impl="keyed_f64", rank=rank, world=world,
                                 norms_sq=norms)
        want, wn = O.dp_vector_backward(dy.double().numpy(), xh.double().numpy(), kind, ocfg, noise_lo=lo,
                                        noise_hi=hi)
    assert _rel(got.double().cpu().numpy(), want) < 1e-5, case
    assert _rel(norms.double().cpu().numpy(), wn) < 1e-5, case
