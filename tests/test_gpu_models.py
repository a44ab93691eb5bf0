"""The model consumers of the DP kernels (gpt2.py full-DP mode, llama.py): in the
no-clip limit (C -> inf, sigma = 0) every DP parameter gradient, times the batch
(the DP reduction is the mean over samples), equals plain autograd's gradient of
the same model with the same weights; with clipping on, every per-sample
gradient norm the DP modules report is finite and a step runs end to end."""

import pytest
import torch

from paper_2507_01154_b200.dplinear import GroupedDPBackward
from paper_2507_01154_b200.gpt2 import GPT2, GPT2Config
from paper_2507_01154_b200.llama import Llama, LlamaConfig

pytestmark = pytest.mark.gpu


def _grads_match(dp_model, ref_model, x, y, B, tol=3e-2):
    ref_model.load_state_dict(dp_model.state_dict(), strict=True)
    ref_model.zero_grad(set_to_none=True)
    ref_model.loss(x, y).backward()
    dp_model.zero_grad(set_to_none=True)
    with GroupedDPBackward():
        dp_model.loss(x, y).backward()
    ref = dict(ref_model.named_parameters())
    n = 0
    for name, p in dp_model.named_parameters():
        g_ref = ref[name].grad
        assert p.grad is not None, name
        scale = float(g_ref.abs().max()) + 1e-12
        err = float((p.grad * B - g_ref).abs().max()) / scale
        assert err < tol, (name, err)
        n += 1
    return n


def test_gpt2_full_dp_equals_autograd_without_clipping():
    torch.manual_seed(0)
    cfg = GPT2Config(vocab=1000, seq=64, d=128, heads=4, layers=2, mlp=512)
    kw = dict(clip_c=1e30, sigma=0.0, tied=False)
    dp = GPT2(cfg, dp="full", **kw).cuda()
    ref = GPT2(cfg, dp=False, **kw).cuda()
    B = 3
    idx = torch.randint(0, cfg.vocab, (B, cfg.seq + 1), device="cuda")
    n = _grads_match(dp, ref, idx[:, :-1].contiguous(), idx[:, 1:].contiguous(), B)
    assert n == len(list(ref.parameters()))


def test_llama_dp_equals_autograd_without_clipping():
    torch.manual_seed(0)
    cfg = LlamaConfig(vocab=1000, d=256, heads=4, layers=2, mlp=512, seq=128)
    dp = Llama(cfg, dp=True, clip_c=1e30, sigma=0.0).cuda()
    ref = Llama(cfg, dp=False).cuda()
    B = 2
    idx = torch.randint(0, cfg.vocab, (B, cfg.seq + 1), device="cuda")
    n = _grads_match(dp, ref, idx[:, :-1].contiguous(), idx[:, 1:].contiguous(), B)
    assert n == len(list(ref.parameters()))


def test_llama_dp_step_with_clipping_and_noise():
    torch.manual_seed(1)
    cfg = LlamaConfig(vocab=500, d=256, heads=4, layers=1, mlp=384, seq=64)
    m = Llama(cfg, dp=True, clip_c=0.5, sigma=1.0).cuda()
    opt = torch.optim.AdamW(m.parameters(), lr=1e-3, fused=True)
    idx = torch.randint(0, cfg.vocab, (4, cfg.seq + 1), device="cuda")
    for step in range(2):
        for mod in m.dp_modules():
            mod.set_step(step)
        opt.zero_grad(set_to_none=True)
        with GroupedDPBackward():
            m.loss(idx[:, :-1].contiguous(), idx[:, 1:].contiguous()).backward()
        opt.step()
    for p in m.parameters():
        assert p.grad is not None and torch.isfinite(p.grad).all()
    norms = [mod.last_norms_sq for mod in m.dp_modules() if getattr(mod, "last_norms_sq", None) is not None]
    assert norms and all(torch.isfinite(t).all() and (t >= 0).all() for t in norms)


def test_full_dp_gpt2_micro_batches_equal_one_batch():
    """SURVEY 8f rank 1 with every parameter group: two micro-batches (noise only on
    the last, mean over the logical batch, gradients accumulated by autograd) equal
    one step on the whole batch (reference-keyed noise: exact draws)."""
    torch.manual_seed(0)
    cfg = GPT2Config(vocab=512, seq=32, d=128, heads=4, layers=1, mlp=256)
    model = GPT2(cfg, dp="full", clip_c=0.3, sigma=0.5, noise_impl="keyed_f64", tied=False).cuda()
    g = torch.Generator().manual_seed(5)
    idx = torch.randint(0, cfg.vocab, (4, cfg.seq + 1), generator=g).cuda()
    B = idx.shape[0]
    mods = model.dp_modules()

    def run(chunks):
        model.zero_grad(set_to_none=True)
        for i, (lo, hi) in enumerate(chunks):
            for m in mods:
                m.set_step(7, last_micro_batch=(i == len(chunks) - 1), logical_batch=B)
            x, y = idx[lo:hi, :-1].contiguous(), idx[lo:hi, 1:].contiguous()
            with GroupedDPBackward():
                (model.loss(x, y) * ((hi - lo) / B)).backward()
        return [p.grad.detach().clone() for p in model.parameters()]

    whole = run([(0, 4)])
    micro = run([(0, 2), (2, 4)])
    for a, b in zip(whole, micro):
        assert float((a - b).abs().max()) <= 2e-2 * max(float(a.abs().max()), 1e-6)
