"""Timing experiments on the multi-layer fused launch (PreparedGroup).

    python tools/group_exp.py [B] [T]

Times (CUDA events, back-to-back launches) the grouped kernel over: all 48
GPT-2 layers, and 12 copies of each layer type alone; with and without noise;
and cuBLAS non-DP dW of the same layers. Env toggles of the native layer (e.g.
FDP_DEBUG_NOSYNC=1) are applied by the caller. Prints one JSON line per case.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_01154_b200 as fdp  # noqa: E402

TYPES = [("c_attn", 768, 2304), ("attn_proj", 768, 768), ("c_fc", 768, 3072), ("mlp_proj", 3072, 768)]
B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
T = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
TAG = os.environ.get("EXP_TAG", "")


def timed(fn, n=30):
    for _ in range(3):
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
    g = torch.Generator(device="cuda").manual_seed(0)
    inputs = {}
    for name, P, D in TYPES:
        inputs[name] = [(torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16),
                         (torch.randn(B, T, D, device="cuda", generator=g) * 1e-3).to(torch.bfloat16))
                        for _ in range(12)]
    cases = {"all48": [(name, blk) for blk in range(12) for name, _, _ in TYPES]}
    if os.environ.get("EXP_ONLY48"):
        TYPES_ = []
    else:
        TYPES_ = TYPES
    for name, _, _ in TYPES_:
        cases[name + "x12"] = [(name, blk) for blk in range(12)]
    for case, items in cases.items():
        flops = sum(2 * B * T * inputs[n][b][0].shape[2] * inputs[n][b][1].shape[2] for n, b in items)
        for sigma in [float(v) for v in os.environ.get("EXP_SIGMAS", "0,1").split(",")]:
            layers = [(inputs[n][b][0], inputs[n][b][1], fdp.DPConfig(1.0, sigma, "mean", seed=1, layer_id=i))
                      for i, (n, b) in enumerate(items)]
            grp = fdp.PreparedGroup(layers, noise_impl="philox")
            us = timed(grp)
            print(json.dumps({"tag": TAG, "case": case, "sigma": sigma, "us": round(us, 1),
                              "tflops": round(flops / us / 1e6, 1)}), flush=True)

        def nd():
            for n, b in items:
                x, y = inputs[n][b]
                torch.mm(y.view(-1, y.shape[2]).t(), x.view(-1, x.shape[2]), out_dtype=torch.float32)
        us = timed(nd)
        print(json.dumps({"tag": TAG, "case": case, "variant": "cublas_nondp", "us": round(us, 1),
                          "tflops": round(flops / us / 1e6, 1)}), flush=True)


if __name__ == "__main__":
    main()
