"""Fused vs two-phase (ghost / recompute / single) timings for planner calibration.

    python tools/path_cal.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_01154_b200 as fdp  # noqa: E402


def timed(fn, n=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


POINTS = [(64, 128, 1024, 1024), (32, 512, 1024, 1024), (8, 1024, 1024, 1024), (32, 512, 2048, 2048),
          (8, 1024, 2048, 2048), (4, 2048, 2048, 2048), (64, 128, 2048, 2048), (1, 4096, 2048, 2048),
          (8, 1024, 768, 3072), (16, 256, 1024, 4096), (2, 1024, 4096, 4096), (64, 256, 4096, 4096)]
g = torch.Generator(device="cuda").manual_seed(0)
for B, T, P, D in POINTS:
    x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
    dy = (torch.randn(B, T, D, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
    F = 2.0 * B * T * P * D
    cfg = fdp.DPConfig(1.0, 1.0, "mean", seed=1, layer_id=0)
    row = {"B": B, "T": T, "P": P, "D": D, "auto": fdp.execution_plan((B, T, P), (B, T, D))["path"]}
    for name, kw in (("fused", dict(path="fused")), ("ghost", dict(path="two_phase", norm_phase="ghost")),
                     ("recompute", dict(path="two_phase", norm_phase="recompute")),
                     ("auto", dict(path="auto"))):
        try:
            c = fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x, dy, cfg, noise_impl="philox", **kw)
            row[name + "_us"] = round(timed(c), 1)
        except Exception as e:  # noqa: BLE001
            row[name + "_us"] = None
    x2, y2 = x.view(-1, P), dy.view(-1, D)
    row["cublas_us"] = round(timed(lambda: torch.mm(y2.t(), x2, out_dtype=torch.float32)), 1)
    print(json.dumps(row), flush=True)
    del x, dy
    torch.cuda.empty_cache()
