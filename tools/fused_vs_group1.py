"""Single-layer fused DP backward: the per-layer fused kernel (dpdw_tc_kernel) vs the
multi-layer group kernel given a one-layer list, vs cuBLAS non-DP dW.

    python tools/fused_vs_group1.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_01154_b200 as fdp  # noqa: E402

SHAPES = [(8, 1024, 2048, 2048), (32, 512, 2048, 2048), (4, 2048, 2048, 2048), (8, 1024, 1024, 1024),
          (8, 1024, 768, 3072), (8, 1024, 3072, 768), (16, 512, 1024, 1024), (4, 2048, 1024, 1024)]


def timed(fn, n=20):
    time.sleep(0.3)
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
    g = torch.Generator(device="cuda").manual_seed(0)
    for B, T, P, D in SHAPES:
        x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
        dy = (torch.randn(B, T, D, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
        cfg = fdp.DPConfig(1.0, 1.0, "mean", seed=1, layer_id=0)
        row = {"shape": [B, T, P, D]}
        try:
            c = fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x, dy, cfg, path="fused", noise_impl="philox")
            row["fused_us"] = round(timed(c), 1)
        except Exception as e:  # noqa: BLE001
            row["fused_us"] = repr(e)[:60]
        grp = fdp.PreparedGroup([(x, dy, cfg)], noise_impl="philox")
        row["group1_us"] = round(timed(grp), 1)
        x2, y2 = x.view(-1, P), dy.view(-1, D)
        row["cublas_us"] = round(timed(lambda: torch.mm(y2.t(), x2, out_dtype=torch.float32)), 1)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
