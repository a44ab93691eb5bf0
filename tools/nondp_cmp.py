"""Non-DP stream-K GEMM vs cuBLAS (fp32 out) vs the DP two-phase path on small-T shapes.

    python tools/nondp_cmp.py ["B,T,P,D;..."]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_01154_b200 as fdp  # noqa: E402


def timed(fn, n=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


shapes = sys.argv[1] if len(sys.argv) > 1 else "64,128,1024,1024;64,128,2048,2048;32,256,2048,2048;4,2048,4096,4096"
g = torch.Generator(device="cuda").manual_seed(0)
for s in shapes.split(";"):
    B, T, P, D = (int(v) for v in s.split(","))
    x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
    dy = (torch.randn(B, T, D, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
    x2, y2 = x.view(-1, P), dy.view(-1, D)
    row = {"shape": [B, T, P, D]}
    row["cublas_us"] = round(timed(lambda: torch.mm(y2.t(), x2, out_dtype=torch.float32)), 1)
    nd = fdp.PreparedBackward(fdp.WorkflowKind.NON_DP, x, dy, None)
    row["nondp_us"] = round(timed(nd), 1)
    cfg = fdp.DPConfig(1.0, 1.0, "mean", seed=1, layer_id=0)
    for path in ("auto", "fused", "two_phase"):
        try:
            c = fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x, dy, cfg, noise_impl="philox", path=path)
            row[f"dp_{path}_us"] = round(timed(c), 1)
        except Exception as e:  # noqa: BLE001
            row[f"dp_{path}_us"] = None
    row["plan_auto"] = fdp.execution_plan((B, T, P), (B, T, D))["path"]
    print(json.dumps(row), flush=True)
    del x, dy
    torch.cuda.empty_cache()
