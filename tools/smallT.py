"""Small-T shapes: fused / two-phase with each forced tile shape (planner calibration)."""
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


g = torch.Generator(device="cuda").manual_seed(0)
for B, T, P, D in [(64, 128, 1024, 1024), (64, 128, 2048, 2048), (32, 256, 2048, 2048), (64, 128, 4096, 4096),
                   (32, 512, 2048, 2048)]:
    x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
    dy = (torch.randn(B, T, D, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
    cfg = fdp.DPConfig(1.0, 1.0, "mean", seed=1, layer_id=0)
    row = {"shape": [B, T, P, D]}
    x2, y2 = x.view(-1, P), dy.view(-1, D)
    row["cublas"] = round(timed(lambda: torch.mm(y2.t(), x2, out_dtype=torch.float32)), 1)
    for bn, cg in (("0", "0"), ("256", "2"), ("128", "2"), ("256", "1"), ("128", "1")):
        os.environ["FDP_FORCE_BN"], os.environ["FDP_FORCE_CG"] = bn, cg
        for path, ph in (("fused", "auto"), ("two_phase", "ghost")):
            try:
                c = fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x, dy, cfg, path=path, norm_phase=ph,
                                         noise_impl="philox")
                row[f"{path}_{bn}x{cg}"] = round(timed(c), 1)
            except Exception as e:  # noqa: BLE001
                row[f"{path}_{bn}x{cg}"] = None
    os.environ.pop("FDP_FORCE_BN")
    os.environ.pop("FDP_FORCE_CG")
    print(json.dumps(row), flush=True)
