"""Non-linear parameter groups at GPT-2 small shapes (B=8, T=1024, d=768, V=50257):
DP kernels (csrc/fdp_params.cu) vs torch's non-DP gradient of the same parameter,
plus the untied LM head (768 -> 50304) through the two-phase path vs cuBLAS.

    python tools/params_bench.py > profiles/r1_params_bench.jsonl
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_01154_b200 as fdp  # noqa: E402


def timed(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


def main():
    B, T, D, V = 8, 1024, 768, 50257
    cfg = fdp.DPConfig(1.0, 1.0, "mean", seed=1, layer_id=5)
    g = torch.Generator(device="cuda").manual_seed(0)
    dy = torch.randn(B, T, D, device="cuda", generator=g)
    xh = torch.randn(B, T, D, device="cuda", generator=g)
    rows = []
    # LayerNorm (gamma, beta): DP group vs the plain reductions torch's LN backward performs
    us = timed(lambda: fdp.vector_dp_grad("layernorm", dy, xh, cfg, noise_impl="philox"))
    nd = timed(lambda: ((dy * xh).sum((0, 1)), dy.sum((0, 1))))
    rows.append({"group": "layernorm gamma+beta (fp32 in)", "B": B, "T": T, "D": D, "dp_us": round(us, 1),
                 "nondp_us": round(nd, 1), "hbm_gbs": round(2 * B * T * D * 4 / us / 1e3, 1)})
    dyb = dy.to(torch.bfloat16)
    us = timed(lambda: fdp.vector_dp_grad("bias", dyb, None, cfg, noise_impl="philox"))
    nd = timed(lambda: dyb.sum((0, 1), dtype=torch.float32))
    rows.append({"group": "bias (bf16 in)", "B": B, "T": T, "D": 768, "dp_us": round(us, 1), "nondp_us": round(nd, 1),
                 "hbm_gbs": round(B * T * D * 2 / us / 1e3, 1)})
    # token embedding: DP (sort, run norms, every row written with noise) vs dense embedding backward
    tok = torch.randint(0, V, (B, T), device="cuda", generator=g)
    us = timed(lambda: fdp.embedding_dp_grad(tok, dy, V, cfg, noise_impl="philox"))
    nd = timed(lambda: torch.ops.aten.embedding_dense_backward(dy, tok, V, -1, False))
    rows.append({"group": "token embedding (fp32 dY)", "B": B, "T": T, "V": V, "D": D, "dp_us": round(us, 1),
                 "nondp_us": round(nd, 1), "table_write_gbs": round(V * D * 4 / us / 1e3, 1)})
    # untied LM head 768 -> 50304 (bf16 autocast): two-phase DP vs cuBLAS dW
    Vp = 50304
    x = torch.randn(B, T, D, device="cuda", generator=g).to(torch.bfloat16)
    dyl = (torch.randn(B, T, Vp, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
    c = fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x, dyl, cfg, noise_impl="philox")
    us = timed(c, n=5)
    nd = timed(lambda: torch.mm(dyl.view(-1, Vp).t(), x.view(-1, D), out_dtype=torch.float32), n=5)
    plan = fdp.execution_plan(tuple(x.shape), tuple(dyl.shape))
    rows.append({"group": "lm head 768->50304 (bf16)", "B": B, "T": T, "P": D, "D": Vp, "dp_us": round(us, 1),
                 "nondp_us": round(nd, 1), "path": plan["path"] + "/" + plan["norm_phase"]})
    for r in rows:
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
