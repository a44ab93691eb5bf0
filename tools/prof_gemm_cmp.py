"""Our stream-K non-DP dW GEMM vs cuBLAS on one Llama projection (ncu captures).

    ncu ... python tools/prof_gemm_cmp.py P D [B] [T]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_01154_b200 as fdp  # noqa: E402

P, D = int(sys.argv[1]), int(sys.argv[2])
B = int(sys.argv[3]) if len(sys.argv) > 3 else 1
T = int(sys.argv[4]) if len(sys.argv) > 4 else 2048
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
dy = torch.randn(B, T, D, device="cuda", generator=g).to(torch.bfloat16)
ours = fdp.PreparedBackward(fdp.WorkflowKind.NON_DP, x, dy, None)
single = fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x, dy, fdp.DPConfig(1.0, 1.0), noise_impl="philox")
x2, y2 = x.view(-1, P), dy.view(-1, D)
for _ in range(2):
    ours()
    torch.mm(y2.t(), x2, out_dtype=torch.float32)
    single()
torch.cuda.synchronize()
print("plan", single.plan.path, single.plan.norm_phase, single.plan.grid)
