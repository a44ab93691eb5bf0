"""Per-kernel breakdown of the two-phase path on Llama shapes (run under
ncu --metrics gpu__time_duration.sum, or plain for wall timings).

    python tools/phase_times.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_01154_b200 as fdp  # noqa: E402

POINTS = [(4, 2048, 4096, 4096), (4, 2048, 4096, 11008), (2, 2048, 5120, 13824), (8, 1024, 4096, 4096)]
SIGMA = float(os.environ.get("PT_SIGMA", "1.0"))
PHASES = os.environ.get("PT_PHASES", "ghost,recompute").split(",")
if os.environ.get("PT_POINTS"):
    POINTS = [tuple(int(v) for v in p.split("x")) for p in os.environ["PT_POINTS"].split(",")]
g = torch.Generator(device="cuda").manual_seed(0)
for B, T, P, D in POINTS:
    x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
    dy = (torch.randn(B, T, D, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
    cfg = fdp.DPConfig(1.0, SIGMA, "mean", seed=1, layer_id=0)
    for ph in PHASES:
        c = fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x, dy, cfg, noise_impl="philox", norm_phase=ph)
        c()
    nd = fdp.PreparedBackward(fdp.WorkflowKind.NON_DP, x, dy, None)
    nd()
    torch.mm(dy.view(-1, D).t(), x.view(-1, P), out_dtype=torch.float32)
    torch.cuda.synchronize()
    print("point", B, T, P, D, flush=True)
