"""Llama-7B / Llama-13B transformer-block DP weight gradients on one B200 (BASELINE
configs 3/4, per GPU): the 7 linear layers of a block (q, k, v, o, gate, up,
down) vs cuBLAS non-DP dW with fp32 output (the like-for-like baseline: the DP
kernels write fp32 gradients too), B in {1, 2, 4}, T=2048.

Each block is timed as the SEQUENCE the backward runs (down, up, gate, o, v, k,
q), back to back on one stream:
  dp_chained  per-layer DP kernels through a DeferredChain: a single-sample
              layer's clip + noise pass is carried by the next layer's GEMM kernel
              (B = 1), the last one flushed at the end of the block
  dp          the same calls unchained (every layer's pass standalone)
  dp_shared_x the unchained calls with q/k/v and gate/up each through ONE
              fdp_backward_shared_x call (they read the same X: one X Gram per tile
              pair in the ghost phase)
  dp_deferred B = 1: the unchained calls through fdp_dw_deferred (no noise in the
              call; the clip factor is left for the optimizer step / collective,
              which adds the noise too -- what ddp.DataParallelStep runs at B = 1)
  nondp       cuBLAS torch.mm(dY^T, X, out_dtype=fp32) per layer
and each layer alone (dp_us / nondp_us per layer).

Implied training-step ratio if dW is one third of the step's flops (forward 2,
dX 2, dW 2 flops per parameter per token): 3 / (2 + r), r = DP dW / non-DP dW.

    python tools/llama_block.py [--models llama-7b,llama-13b] [--batches 1,2,4] > profiles/rNN_llama_blocks.jsonl
"""
import argparse
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
    ap = argparse.ArgumentParser()
    ap.add_argument("--models", default="llama-7b,llama-13b")
    ap.add_argument("--batches", default="1,2,4")
    ap.add_argument("--T", type=int, default=2048)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    T = a.T
    g = torch.Generator(device="cuda").manual_seed(0)
    for name in a.models.split(","):
        d, ff = MODELS[name]
        # backward order of a block
        shapes = [("down", ff, d), ("up", d, ff), ("gate", d, ff), ("o", d, d), ("v", d, d), ("k", d, d),
                  ("q", d, d)]
        for B in (int(b) for b in a.batches.split(",")):
            row = {"model": name, "B": B, "T": T, "layers": {}}
            ins, chained, plain, nd, own, deferred = [], [], [], [], [], []
            shared_x = {}
            chain = fdp.DeferredChain()
            ws = torch.zeros(256 << 20, dtype=torch.uint8, device="cuda")
            flops = 0.0
            for j, (lname, P, D) in enumerate(shapes):
                # up/gate read the MLP norm's output, v/k/q the attention norm's: one X each
                if lname in ("up", "v"):
                    shared_x[lname] = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
                if lname in ("up", "gate"):
                    x = shared_x["up"]
                elif lname in ("v", "k", "q"):
                    x = shared_x["v"]
                else:
                    x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
                dy = (torch.randn(B, T, D, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
                cfg = fdp.DPConfig(1.0, 1.0, "mean", seed=1, layer_id=j)
                gw = torch.zeros(D, P, device="cuda")
                nrm = torch.zeros(B, device="cuda")
                plain.append(fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x, dy, cfg, noise_impl="philox",
                                                  grad_w=gw, norms_sq=nrm, workspace=ws))
                chained.append(fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x, dy, cfg, noise_impl="philox",
                                                    grad_w=gw, norms_sq=nrm, workspace=ws, chain=chain))
                if B == 1:
                    deferred.append(fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x, dy, cfg, noise_impl="philox",
                                                         grad_w=gw, norms_sq=nrm, workspace=ws, add_noise=False,
                                                         grad_scale=torch.zeros(1, device="cuda")))
                own.append(fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x, dy, cfg, noise_impl="philox",
                                                grad_w=gw, norms_sq=nrm))  # own workspace (shared-X arm)
                x2, y2 = x.view(-1, P), dy.view(-1, D)
                nd.append((x2, y2))
                ins.append((x, dy))
                flops += 2.0 * B * T * P * D
                c = plain[-1]
                path = fdp._lib.PATH_NAMES[c.plan.path] + (
                    "/" + fdp._lib.NORM_PHASE_NAMES.get(c.plan.norm_phase, "") if c.plan.path == 2 else "")
                row["layers"][lname] = {"dp_us": round(timed(c, a.reps), 1),
                                        "nondp_us": round(timed(lambda: torch.mm(y2.t(), x2, out_dtype=torch.float32),
                                                                a.reps), 1),
                                        "path": path}

            def dp_chained():
                for c in chained:
                    c()
                chain.flush()

            def dp_plain():
                for c in plain:
                    c()

            names = [sn[0] for sn in shapes]
            sx_calls = [own[names.index("down")], fdp.PreparedSharedX([own[names.index("up")], own[names.index("gate")]]),
                        own[names.index("o")],
                        fdp.PreparedSharedX([own[names.index("v")], own[names.index("k")], own[names.index("q")]])]

            def dp_shared_x():
                for c in sx_calls:
                    c()

            def dp_deferred():
                for c in deferred:
                    c()

            def nondp():
                for x2, y2 in nd:
                    torch.mm(y2.t(), x2, out_dtype=torch.float32)

            res = {}
            for _ in range(2):  # alternate, keep the best
                arms = [("dp_chained", dp_chained), ("dp", dp_plain), ("dp_shared_x", dp_shared_x), ("nondp", nondp)]
                for k, fn in arms + ([("dp_deferred", dp_deferred)] if deferred else []):
                    t = timed(fn, a.reps)
                    res[k] = min(res.get(k, 1e30), t)
            st = chain.stats()
            r = res["dp_chained"] / res["nondp"]
            row.update({"dp_chained_us": round(res["dp_chained"], 1), "dp_us": round(res["dp"], 1),
                        "nondp_us": round(res["nondp"], 1), "dp_tflops": round(flops / res["dp_chained"] / 1e6, 1),
                        "dw_ratio": round(r, 3), "dw_ratio_unchained": round(res["dp"] / res["nondp"], 3),
                        "dp_shared_x_us": round(res["dp_shared_x"], 1),
                        "dw_ratio_shared_x": round(res["dp_shared_x"] / res["nondp"], 3),
                        "implied_step_pct_of_nondp": round(100.0 * 3.0 / (2.0 + r), 1), "chain": st})
            if deferred:
                rd = res["dp_deferred"] / res["nondp"]
                row.update({"dp_deferred_us": round(res["dp_deferred"], 1), "dw_ratio_deferred": round(rd, 3),
                            "implied_step_pct_deferred": round(100.0 * 3.0 / (2.0 + rd), 1)})
            print(json.dumps(row), flush=True)
            del ins, chained, plain, nd, chain, ws, own, sx_calls, shared_x, deferred
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
