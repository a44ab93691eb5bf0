"""GPT-2 small training step, DP (DPLinear + GroupedDPBackward) vs non-DP, one GPU.

    python tools/train_gpt2.py [--batch 8] [--seq 1024] [--steps 20] [--warmup 5]

Prints one JSON line: tokens/s of both and DP as % of non-DP. Same model,
same optimizer (torch fused AdamW), random init, synthetic token ids; the only
difference is how the 48 linear layers' weight gradients are computed.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_01154_b200.dplinear import GroupedDPBackward  # noqa: E402
from paper_2507_01154_b200.gpt2 import GPT2, GPT2Config  # noqa: E402


def run(dp, a) -> dict:
    torch.manual_seed(0)
    cfg = GPT2Config(seq=a.seq)
    model = GPT2(cfg, dp=dp, clip_c=1.0, sigma=1.0, tied=not a.full,
                 nondp_linear=getattr(a, "nondp_linear", "fp32grad")).cuda()
    opt = torch.optim.AdamW(model.parameters(), lr=1e-4, fused=True)
    g = torch.Generator(device="cuda").manual_seed(1)
    idx = torch.randint(0, cfg.vocab, (a.batch, a.seq + 1), device="cuda", generator=g)
    x, y = idx[:, :-1].contiguous(), idx[:, 1:].contiguous()
    layers = model.dp_modules()

    def step(i):
        for m in layers:
            m.set_step(i)
        opt.zero_grad(set_to_none=True)
        loss = model.loss(x, y)
        if dp:
            with GroupedDPBackward():
                loss.backward()
        else:
            loss.backward()
        opt.step()
        return loss

    for i in range(a.warmup):
        step(i)
    torch.cuda.synchronize()
    time.sleep(1.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(a.steps):
        loss = step(a.warmup + i)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    return {"ms_per_step": ms, "tokens_per_s": a.batch * a.seq / (ms * 1e-3), "loss": float(loss.detach()),
            "dp_modules": len(layers)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--seq", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--nondp-linear", default="fp32grad", choices=["fp32grad", "torch"],
                    help="non-DP projections: fp32grad = cuBLAS writes fp32 weight gradients (like-for-like with the "
                         "DP kernels); torch = nn.Linear under autocast (bf16 dW cast into fp32 .grad)")
    ap.add_argument("--full", action="store_true", help="every parameter DP (embeddings, LayerNorms, untied LM "
                    "head); the non-DP baseline is then untied too")
    a = ap.parse_args()
    nd = run(False, a)
    dp = run("full" if a.full else True, a)
    print(json.dumps({"model": "gpt2-small (124M), random init, synthetic tokens", "batch": a.batch, "seq": a.seq,
                      "nondp_linear": a.nondp_linear,
                      "dp_scope": "every parameter (untied LM head)" if a.full else "the 48 linear layers",
                      "dp": dp, "non_dp": nd, "dp_pct_of_non_dp": 100.0 * dp["tokens_per_s"] / nd["tokens_per_s"],
                      "note": ("DP = per-layer clipped + noised gradients of every parameter: the 48 linear layers "
                               "(one fdp_backward_group launch), biases, LayerNorms, token / position embeddings "
                               "and the LM head (per-layer two-phase)") if a.full else
                              ("DP = per-layer clipped + noised weight and bias gradients of the 48 linear layers "
                               "(one fdp_backward_group launch per step); embeddings / LayerNorm / LM head not DP")}))


if __name__ == "__main__":
    main()
