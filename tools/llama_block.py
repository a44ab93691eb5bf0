"""Llama-7B / Llama-13B transformer-block DP weight gradients on one B200 (BASELINE
configs 3/4, per GPU): the 7 linear layers of a block (q, k, v, o, gate, up,
down) through the auto-selected path vs cuBLAS non-DP dW, B in {1, 2, 4}, T=2048.

Also the implied training-step ratio if dW is one third of the step's flops
(forward 2, dX 2, dW 2 flops per parameter per token): (1 + 1 + 1) / (1 + 1 + r)
with r = DP dW time / non-DP dW time.

    python tools/llama_block.py > profiles/r1_llama_blocks.jsonl
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_01154_b200 as fdp  # noqa: E402

MODELS = {"llama-7b": (4096, 11008), "llama-13b": (5120, 13824)}


def timed(fn, n=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3  # us


def main():
    T = 2048
    g = torch.Generator(device="cuda").manual_seed(0)
    variants = {"separate": lambda d, ff: [("q", d, d), ("k", d, d), ("v", d, d), ("o", d, d), ("gate", d, ff),
                                           ("up", d, ff), ("down", ff, d)],
                # fused projections (one clip group each, like GPT-2's c_attn): qkv and gate_up
                "fused_qkv_gateup": lambda d, ff: [("qkv", d, 3 * d), ("o", d, d), ("gate_up", d, 2 * ff),
                                                   ("down", ff, d)]}
    for (name, (d, ff)), (vname, vshapes) in [(m, v) for m in MODELS.items() for v in variants.items()]:
        shapes = vshapes(d, ff)
        for B in (1, 2, 4):
            row = {"model": name, "projections": vname, "B": B, "T": T, "layers": {}}
            dp_total = nd_total = 0.0
            flops = 0.0
            for lname, P, D in shapes:
                x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
                dy = (torch.randn(B, T, D, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
                cfg = fdp.DPConfig(1.0, 1.0, "mean", seed=1, layer_id=0)
                c = fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x, dy, cfg, noise_impl="philox")
                dp_us = timed(c)
                x2, y2 = x.view(-1, P), dy.view(-1, D)
                nd_us = timed(lambda: torch.mm(y2.t(), x2, out_dtype=torch.float32))
                plan = fdp._lib.PATH_NAMES[c.plan.path] + (
                    "/" + fdp._lib.NORM_PHASE_NAMES.get(c.plan.norm_phase, "") if c.plan.path == 2 else "")
                row["layers"][lname] = {"dp_us": round(dp_us, 1), "nondp_us": round(nd_us, 1), "path": plan}
                dp_total += dp_us
                nd_total += nd_us
                flops += 2.0 * B * T * P * D
                del x, dy, c
                torch.cuda.empty_cache()
            r = dp_total / nd_total
            row.update({"dp_us": round(dp_total, 1), "nondp_us": round(nd_total, 1),
                        "dp_tflops": round(flops / dp_total / 1e6, 1), "dw_ratio": round(r, 3),
                        "implied_step_pct_of_nondp": round(100.0 * 3.0 / (2.0 + r), 1)})
            print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
