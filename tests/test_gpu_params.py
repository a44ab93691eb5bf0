"""GPU parity of the non-linear parameter groups (csrc/fdp_params.cu):
bias / RMSNorm / LayerNorm vector groups and embedding tables against the oracle's
restatements (oracle/dp_oracle.py: per-sample gradients materialised in fp64,
the reference's clip / sum / keyed-noise arithmetic), plus the modules against
torch's own non-DP gradients in the C -> inf, sigma = 0, sum limit.

Tolerance: rel 1e-5 (fp32 accumulation of bf16- or fp32-exact inputs; the oracle
gets the same rounded values); reference-keyed noise (keyed_f64) makes sigma > 0
deterministic, Philox noise is checked as out(sigma) - out(0) == noise_range.
"""

import numpy as np
import pytest
import torch

import paper_2507_01154_b200 as fdp
from oracle import dp_oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-5


def rel(got, want):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    scale = max(float(np.max(np.abs(want))), 1e-30)
    return float(np.max(np.abs(got - want))) / scale


def host(t):
    return t.double().cpu().numpy()


def ocfg(c: fdp.DPConfig) -> O.Cfg:
    return O.Cfg(c.clip_c, c.sigma, c.reduction, c.seed, c.layer_id, c.step)


@pytest.mark.parametrize("kind", ["bias", "rmsnorm", "layernorm"])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("B,T,D", [(5, 70, 777), (1, 1, 64), (3, 200, 256), (16, 9, 1030), (2, 65, 8), (4, 33, 1028)])
@pytest.mark.parametrize("sched", ["auto", "three_pass"])
def test_vector_groups_against_oracle(kind, dtype, B, T, D, sched, monkeypatch):
    """auto: aligned rows take the column-slice kernel (k_vec_cols + finalize), unaligned
    ones (D not a multiple of the vector width) the three passes."""
    if sched == "three_pass":
        monkeypatch.setenv("FDP_VEC_COLS", "0")
    g = torch.Generator().manual_seed(B * 1000 + T + D)
    dy = (torch.randn(B, T, D, generator=g) * 0.1).to(dtype).cuda()
    xh = torch.randn(B, T, D, generator=g).to(dtype).cuda()
    # C at the median norm: some samples clip, some pass
    gb = O.vector_per_sample_grads(host(dy), host(xh), kind)
    c = float(np.median(np.sqrt((gb * gb).sum(1)))) or 1.0
    cfg = fdp.DPConfig(c, 1.3, "mean", seed=11, layer_id=3, step=4)
    norms = torch.empty(B, device="cuda")
    out = fdp.vector_dp_grad(kind, dy, xh, cfg, noise_impl="keyed_f64", norms_sq=norms)
    want, wn = O.dp_vector_backward(host(dy), host(xh), kind, ocfg(cfg))
    assert out.shape == ((2 * D,) if kind == "layernorm" else (D,))
    assert rel(host(out), want) < TOL
    assert rel(host(norms), wn) < TOL


@pytest.mark.parametrize("rank,world", [(0, 2), (1, 2), (2, 3)])
def test_vector_group_noise_partition_and_accumulate(rank, world):
    """Rank slices of [0, 2D) partition the noise; accumulate adds onto grad; sum reduction."""
    B, T, D = 4, 33, 300
    g = torch.Generator().manual_seed(5)
    dy = torch.randn(B, T, D, generator=g).cuda()
    xh = torch.randn(B, T, D, generator=g).cuda()
    cfg = fdp.DPConfig(2.0, 0.7, "sum", seed=3, layer_id=8, step=1)
    base = torch.randn(2 * D, generator=g).cuda()
    out = base.clone()
    fdp.vector_dp_grad("layernorm", dy, xh, cfg, noise_impl="keyed_f64", rank=rank, world=world, out=out,
                       accumulate=True)
    L = 2 * D
    lo, hi = L * rank // world, L * (rank + 1) // world
    want, _ = O.dp_vector_backward(host(dy), host(xh), "layernorm", ocfg(cfg), noise_lo=lo, noise_hi=hi)
    assert rel(host(out), want + host(base)) < TOL


def test_vector_group_unaligned_view():
    """A dY view starting 4 bytes into its storage takes the scalar-load variant."""
    B, T, D = 3, 40, 64
    g = torch.Generator().manual_seed(9)
    big = (torch.randn(B * T * D + 1, generator=g) * 0.1).cuda()
    dy = big[1:].view(B, T, D)
    xh = torch.randn(B, T, D, generator=g).cuda()
    cfg = fdp.DPConfig(0.2, 0.0, "sum", seed=1, layer_id=1)
    out = fdp.vector_dp_grad("rmsnorm", dy, xh, cfg)
    want, _ = O.dp_vector_backward(host(dy), host(xh), "rmsnorm", ocfg(cfg))
    assert rel(host(out), want) < TOL


@pytest.mark.parametrize("kind", ["bias", "layernorm", "rmsnorm"])
@pytest.mark.parametrize("B,T,D", [(1, 1024, 768), (1, 1024, 3072), (2, 4096, 4096), (8, 1000, 1536), (1, 7, 40)])
def test_vector_group_column_slices_match_three_pass(kind, B, T, D, monkeypatch):
    """The column-slice schedule (one CTA per 32-byte column slice over all T rows) against
    the three-pass one at model shapes: same values to fp32 reordering, bitwise
    repeatable, and unchanged under CUDA-graph replay."""
    g = torch.Generator().manual_seed(B + T + D)
    dy = (torch.randn(B, T, D, generator=g) * 0.05).to(torch.bfloat16).cuda()
    xh = torch.randn(B, T, D, generator=g).to(torch.bfloat16).cuda()
    cfg = fdp.DPConfig(0.3, 0.9, "mean", seed=4, layer_id=2, step=5)
    xa = None if kind == "bias" else xh
    fused = fdp.vector_dp_grad(kind, dy, xa, cfg, noise_impl="keyed_f64")
    again = fdp.vector_dp_grad(kind, dy, xa, cfg, noise_impl="keyed_f64")
    assert torch.equal(fused, again)
    monkeypatch.setenv("FDP_VEC_COLS", "0")
    three = fdp.vector_dp_grad(kind, dy, xa, cfg, noise_impl="keyed_f64")
    monkeypatch.delenv("FDP_VEC_COLS")
    assert rel(host(fused), host(three)) < 1e-5
    out = torch.zeros_like(fused)
    fdp.vector_dp_grad(kind, dy, xa, cfg, noise_impl="keyed_f64", out=out)  # warm the workspace cache
    gr = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(gr, stream=s):
            fdp.vector_dp_grad(kind, dy, xa, cfg, noise_impl="keyed_f64", out=out)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(3):
        out.zero_()
        gr.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, fused)


def test_bias_dw_is_the_bias_vector_group():
    B, T, D = 6, 40, 500
    dy = torch.randn(B, T, D, device="cuda").to(torch.bfloat16)
    cfg = fdp.DPConfig(0.5, 1.0, "mean", seed=2, layer_id=4, step=3)
    a = fdp.vector_dp_grad("bias", dy, None, cfg, noise_impl="philox")
    b = fdp.vector_dp_grad("bias", dy, None, cfg, noise_impl="philox")
    assert torch.equal(a, b)  # deterministic
    want, _ = O.dp_vector_backward(host(dy), None, "bias", ocfg(fdp.DPConfig(0.5, 0.0, "mean")))
    n = fdp.noise_range(cfg, 0, D, 0.5, noise_impl="philox")
    assert rel(host(a - n), want) < TOL


def _tokens(B, T, V, seed, bad=False):
    g = torch.Generator().manual_seed(seed)
    t = torch.randint(0, V, (B, T), generator=g)
    if bad and T > 3:
        t[0, 1] = -1
        t[-1, 2] = V  # out of range: contributes nothing
    return t


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("B,T,V,D", [(4, 100, 37, 64), (3, 1500, 500, 70), (1, 1, 5, 8), (8, 257, 1000, 256),
                                     (2, 64, 3, 1030), (2, 2000, 2, 40)])
def test_embedding_against_oracle(dtype, B, T, V, D):
    """Repeated tokens (small vocabularies), ragged d (per-element noise), T > 1024
    (2048-key sort), single token, multiple column chunks, runs of one token longer
    than a norm block's key stage (V = 2, T = 2000)."""
    tok = _tokens(B, T, V, seed=T + V, bad=True)
    g = torch.Generator().manual_seed(D)
    dy = (torch.randn(B, T, D, generator=g) * 0.1).to(dtype)
    valid = (tok >= 0) & (tok < V)
    tk = np.where(valid.numpy(), tok.numpy(), 0)
    dyh = host(dy) * valid.numpy()[:, :, None]
    G = O.embedding_per_sample_grads(tk, dyh, V)
    ns = np.einsum("bvd,bvd->b", G, G)
    assert np.allclose(O.embedding_norms_gram(tk, dyh), ns, rtol=1e-10)
    c = float(np.median(np.sqrt(ns))) or 1.0
    cfg = fdp.DPConfig(c, 0.9, "mean", seed=4, layer_id=12, step=6)
    norms = torch.empty(B, device="cuda")
    out = fdp.embedding_dp_grad(tok.cuda(), dy.cuda(), V, cfg, noise_impl="keyed_f64", norms_sq=norms)
    want, wn = O.dp_embedding_backward(tk, dyh, V, ocfg(cfg))
    assert out.shape == (V, D)
    assert rel(host(out), want) < TOL
    assert rel(host(norms), wn) < TOL


@pytest.mark.parametrize("rank,world", [(0, 1), (1, 2), (3, 4)])
def test_embedding_philox_noise_partition(rank, world):
    B, T, V, D = 3, 50, 80, 96
    tok = _tokens(B, T, V, seed=1).cuda()
    dy = torch.randn(B, T, D, device="cuda")
    c0 = fdp.DPConfig(1.0, 0.0, "mean", seed=9, layer_id=1, step=2)
    c1 = fdp.DPConfig(1.0, 2.0, "mean", seed=9, layer_id=1, step=2)
    kw = dict(noise_impl="philox", rank=rank, world=world)
    g0 = fdp.embedding_dp_grad(tok, dy, V, c0, **kw)
    g1 = fdp.embedding_dp_grad(tok, dy, V, c1, **kw)
    n = fdp.noise_range(c1, 0, V * D, 2.0, noise_impl="philox")
    lo, hi = V * D * rank // world, V * D * (rank + 1) // world
    mask = torch.zeros(V * D, device="cuda")
    mask[lo:hi] = 1.0
    assert rel(host((g1 - g0).reshape(-1)), host(n * mask)) < 1e-5


def test_embedding_accumulate_and_usage_errors():
    B, T, V, D = 2, 20, 30, 16
    tok = _tokens(B, T, V, seed=3).cuda()
    dy = torch.randn(B, T, D, device="cuda")
    cfg = fdp.DPConfig(1.0, 0.0, "sum", seed=1, layer_id=1)
    a = fdp.embedding_dp_grad(tok, dy, V, cfg)
    acc = torch.ones(V, D, device="cuda")
    fdp.embedding_dp_grad(tok, dy, V, cfg, out=acc, accumulate=True)
    assert torch.allclose(acc, a + 1.0, rtol=0, atol=1e-6)
    with pytest.raises(fdp.ShapeError):
        fdp.embedding_dp_grad(tok, dy[:, :5], V, cfg)
    with pytest.raises(fdp.ShapeError):  # T over the single-CTA sort
        fdp.embedding_dp_grad(torch.zeros(1, 20000, dtype=torch.int64, device="cuda"),
                              torch.zeros(1, 20000, 8, device="cuda"), V, cfg)


def test_modules_match_torch_in_the_no_clip_limit():
    """C -> inf, sigma = 0, reduction sum: each DP module's parameter gradient is the
    ordinary gradient (torch's own modules), and its input gradient is unchanged."""
    torch.manual_seed(0)
    B, T, D, V = 4, 30, 96, 50
    big = dict(clip_c=1e30, sigma=0.0, reduction="sum")
    ln, ln_ref = fdp.DPLayerNorm(D, **big).cuda(), torch.nn.LayerNorm(D).cuda()
    with torch.no_grad():
        ln.weight.uniform_(0.5, 1.5)
        ln.bias.uniform_(-0.5, 0.5)
        ln_ref.weight.copy_(ln.weight)
        ln_ref.bias.copy_(ln.bias)
    x = torch.randn(B, T, D, device="cuda", requires_grad=True)
    x2 = x.detach().clone().requires_grad_(True)
    w = torch.randn(B, T, D, device="cuda")
    (ln(x) * w).sum().backward()
    (ln_ref(x2) * w).sum().backward()
    assert torch.allclose(ln.weight.grad, ln_ref.weight.grad, rtol=1e-4, atol=1e-4)
    assert torch.allclose(ln.bias.grad, ln_ref.bias.grad, rtol=1e-4, atol=1e-4)
    assert torch.allclose(x.grad, x2.grad, rtol=1e-4, atol=1e-5)

    rms = fdp.DPRMSNorm(D, **big).cuda()
    x3 = torch.randn(B, T, D, device="cuda", requires_grad=True)
    (rms(x3) * w).sum().backward()
    xf = x3.detach()
    xhat = xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + rms.eps)
    assert torch.allclose(rms.weight.grad, (w * xhat).sum((0, 1)), rtol=1e-4, atol=1e-4)

    emb, emb_ref = fdp.DPEmbedding(V, D, **big).cuda(), torch.nn.Embedding(V, D).cuda()
    with torch.no_grad():
        emb_ref.weight.copy_(emb.weight)
    tok = torch.randint(0, V, (B, T), device="cuda")
    (emb(tok) * w).sum().backward()
    (emb_ref(tok) * w).sum().backward()
    assert torch.allclose(emb.weight.grad, emb_ref.weight.grad, rtol=1e-4, atol=1e-5)


def test_module_norms_and_clip():
    """A DP module's per-sample norms are those of its per-sample gradients, and the
    result is the clipped mean + keyed noise (oracle)."""
    torch.manual_seed(1)
    B, T, D = 3, 17, 40
    ln = fdp.DPLayerNorm(D, clip_c=0.3, sigma=0.5, reduction="mean", layer_id=77, noise_impl="keyed_f64").cuda()
    ln.set_step(5)
    x = torch.randn(B, T, D, device="cuda")
    dy = torch.randn(B, T, D, device="cuda")
    ln(x).backward(dy)
    xhat = torch.nn.functional.layer_norm(x, (D,))
    want, wn = O.dp_vector_backward(host(dy), host(xhat), "layernorm", O.Cfg(0.3, 0.5, "mean", 0, 77, 5))
    got = torch.cat([ln.weight.grad, ln.bias.grad])
    assert rel(host(got), want) < 1e-4
    assert rel(host(ln.last_norms_sq), wn) < 1e-4
