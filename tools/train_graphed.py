"""GPT-2 small training step through ddp.DataParallelStep, eager vs captured in one
CUDA graph (ddp.GraphedStep), DP (every parameter) vs non-DP (FP32GradLinear), one GPU.
At small batches the eager step is bound by the host (hundreds of launches, Python
autograd); the graph removes that from both arms.

    python tools/train_graphed.py [--batches 1,2,4,8] [--steps 50]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2507_01154_b200.ddp import DataParallelStep, GraphedStep  # noqa: E402
from paper_2507_01154_b200.gpt2 import GPT2, GPT2Config  # noqa: E402


def run(dp: bool, graphed: bool, B: int, steps: int, optimizer: str = "adam") -> dict:
    torch.manual_seed(0)
    cfg = GPT2Config(seq=1024)
    model = GPT2(cfg, dp="full" if dp else False, clip_c=1.0, sigma=1.0, tied=False, nondp_linear="fp32grad").cuda()
    step = DataParallelStep(model, dp=dp, lr=1e-4, global_batch=B, optimizer=optimizer)
    g = torch.Generator(device="cuda").manual_seed(1)
    idx = torch.randint(0, cfg.vocab, (B, cfg.seq + 1), device="cuda", generator=g)
    x, y = idx[:, :-1].contiguous(), idx[:, 1:].contiguous()
    scale = float(B) if dp else 1.0  # DP modules: sum of per-sample (token-mean) losses; non-DP: the batch mean

    def loss_fn():
        return model.loss(x, y) * scale

    if graphed:
        gs = GraphedStep(step, loss_fn, warmup=3)
        call = gs
    else:
        it = [0]

        def call():
            it[0] += 1
            return step(it[0], loss_fn)
        for _ in range(3):
            call()
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    time.sleep(0.5)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        loss = call()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    out = {"ms_per_step": round(ms, 3), "tokens_per_s": round(B * cfg.seq / (ms * 1e-3)),
           "loss": float(loss.detach())}
    del model, step
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--optimizer", default="adam", choices=["adam", "sgd"],
                    help="sgd: plain DP-SGD (BASELINE config 2's optimizer)")
    a = ap.parse_args()
    for B in (int(b) for b in a.batches.split(",")):
        row = {"model": "gpt2-small, every parameter DP (untied LM head, vocab padded to 50304) vs FP32GradLinear "
                        "non-DP, DataParallelStep + bucketed " + a.optimizer, "batch": B, "seq": 1024}
        for graphed in (False, True):
            tag = "graphed" if graphed else "eager"
            nd = run(False, graphed, B, a.steps, a.optimizer)
            dp = run(True, graphed, B, a.steps, a.optimizer)
            row[tag] = {"dp": dp, "non_dp": nd, "dp_pct_of_non_dp": round(100.0 * dp["tokens_per_s"] /
                                                                          nd["tokens_per_s"], 1)}
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
