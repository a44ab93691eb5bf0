"""Mainloop rate of the tcgen05 pipeline: NON_DP mode on a GEMM with many more
tiles than SMs (persistent grid), BN=128 and 256, vs cuBLAS."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_01154_b200 as fdp  # noqa: E402
from perf_sweep import timed  # noqa: E402

for (B, T, P, D) in [(8, 1024, 4096, 4096), (4, 2048, 5120, 13824), (8, 1024, 768, 3072)]:
    x = torch.randn(B, T, P, device="cuda").to(torch.bfloat16)
    dy = torch.randn(B, T, D, device="cuda").to(torch.bfloat16)
    fl = 2 * B * T * P * D
    x2, y2 = x.view(-1, P), dy.view(-1, D)
    us = timed(lambda: torch.mm(y2.t(), x2, out_dtype=torch.float32))
    print(f"{B}x{T} {P}->{D} cublas {us:.1f}us {fl/us/1e6:.0f} TF", flush=True)
    for bn, cg in (("128", "1"), ("256", "1"), ("128", "2"), ("256", "2")):
        os.environ["FDP_FORCE_BN"] = bn
        os.environ["FDP_FORCE_CG"] = cg
        c = fdp.PreparedBackward(fdp.WorkflowKind.NON_DP, x, dy, None)
        us = timed(c)
        print(f"{B}x{T} {P}->{D} tcgen05 nondp bn{bn} cg{cg} grid{c.plan.grid} {us:.1f}us {fl/us/1e6:.0f} TF", flush=True)
        c = fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x, dy, fdp.DPConfig(1.0, 0.0), path="two_phase")
        us = timed(c)
        print(f"{B}x{T} {P}->{D} two_phase bn{bn} cg{cg} {us:.1f}us {fl/us/1e6:.0f} TF(dW-equiv)", flush=True)
    os.environ.pop("FDP_FORCE_BN")
    os.environ.pop("FDP_FORCE_CG")
