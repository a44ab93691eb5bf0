"""Small cases of every native path, for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("FDP_NO_COOP", "1")  # sanitizers cannot replay cooperative cluster launches
import torch  # noqa: E402

import paper_2507_01154_b200 as fdp  # noqa: E402

g = torch.Generator().manual_seed(0)


def inputs(B, T, P, D, dtype=torch.bfloat16):
    return (torch.randn(B, T, P, generator=g).to(dtype).cuda(), (torch.randn(B, T, D, generator=g) * 0.1).to(dtype).cuda())


cfg = fdp.DPConfig(0.5, 1.0, "mean", seed=3, layer_id=1, step=2)
x, dy = inputs(3, 100, 256, 512)
for path in ("fused", "two_phase"):
    fdp.backward_flashdp(x, dy, cfg, path=path, noise_impl="philox")
fdp.backward_flashdp(x, dy, cfg, path="two_phase", norm_phase="recompute")
for kind in (fdp.WorkflowKind.NON_DP, fdp.WorkflowKind.EXPLICIT_DP, fdp.WorkflowKind.IMPLICIT_DP):
    fdp.run_backward(kind, x, dy, cfg)
x1, dy1 = inputs(1, 300, 512, 256)
fdp.backward_flashdp(x1, dy1, cfg, path="two_phase")  # single-sample path
xf, dyf = inputs(2, 40, 24, 40, torch.float32)
fdp.backward_flashdp(xf, dyf, cfg)  # SIMT fp32
xd, dyd = inputs(2, 20, 16, 8, torch.float64)
fdp.backward_flashdp(xd, dyd, cfg)  # fp64 parity path
grp = fdp.PreparedGroup([(x, dy, cfg), inputs(3, 100, 512, 256) + (cfg,)], noise_impl="philox")
grp()
st = fdp.OptimizerState.fresh(torch.zeros(1000, device="cuda"), eta=0.1)
fdp.dp_adam_step_(st, torch.ones(1000, device="cuda"))
torch.cuda.synchronize()
print("sanitize cases done")
