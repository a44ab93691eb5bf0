"""Llama-2 training step on one GPU, every parameter DP vs non-DP (BASELINE
configs 3/4 shapes, SURVEY 8d E2E inputs, N=1).

    python tools/train_llama.py --model llama-7b [--layers 32] [--batch 1] [--seq 2048]

Same model twice: torch modules (non-DP) and DPLinear / DPRMSNorm / DPEmbedding
with GroupedDPBackward (DP: per-layer clip C=1, sigma=1, Philox noise), fused
AdamW on fp32 master weights, bf16 autocast, random init, synthetic token ids.
Prints one JSON line. --layers below the model's depth measures a shallower
stack of the same blocks (stated in the line): the per-block ratio is what the
depth does not change.
"""
import argparse
import gc
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_01154_b200.dplinear import GroupedDPBackward  # noqa: E402
from paper_2507_01154_b200.llama import Llama, LlamaConfig  # noqa: E402


def run(dp: bool, a) -> dict:
    torch.manual_seed(0)
    cfg = LlamaConfig.named(a.model, seq=a.seq, **({"layers": a.layers} if a.layers else {}))
    with torch.device("cuda"):
        model = Llama(cfg, dp=dp, clip_c=1.0, sigma=1.0)
    opt = torch.optim.AdamW(model.parameters(), lr=1e-5, fused=True)
    g = torch.Generator(device="cuda").manual_seed(1)
    idx = torch.randint(0, cfg.vocab, (a.batch, a.seq + 1), device="cuda", generator=g)
    x, y = idx[:, :-1].contiguous(), idx[:, 1:].contiguous()
    mods = model.dp_modules() if dp else []

    def step(i):
        for m in mods:
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

    torch.cuda.reset_peak_memory_stats()
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
    out = {"ms_per_step": ms, "tokens_per_s": a.batch * a.seq / (ms * 1e-3), "loss": float(loss.detach()),
           "dp_modules": len(mods), "params": sum(p.numel() for p in model.parameters()),
           "peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9}
    del model, opt, mods
    gc.collect()
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama-7b", choices=["llama-7b", "llama-13b"])
    ap.add_argument("--layers", type=int, default=0, help="0 = the model's depth")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--seq", type=int, default=2048)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    nd = run(False, a)
    dp = run(True, a)
    print(json.dumps({"model": a.model, "layers": a.layers or LlamaConfig.named(a.model).layers, "batch": a.batch,
                      "seq": a.seq, "dp": dp, "non_dp": nd,
                      "dp_pct_of_non_dp": 100.0 * dp["tokens_per_s"] / nd["tokens_per_s"],
                      "note": "one GPU; every parameter DP (7 projections per block + LM head: DPLinear; RMSNorms; "
                              "token embedding), per-layer clip C=1, sigma=1, Philox; fused AdamW; random init, "
                              "synthetic tokens"}))


if __name__ == "__main__":
    main()
