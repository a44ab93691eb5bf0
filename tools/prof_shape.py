"""Launch one layer's DP backward a few times at an arbitrary shape (ncu captures).

    python tools/prof_shape.py B T P D [path] [reps] [kind]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_01154_b200 as fdp  # noqa: E402

B, T, P, D = (int(v) for v in sys.argv[1:5])
path = sys.argv[5] if len(sys.argv) > 5 else "auto"
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 3
kind = fdp.WorkflowKind(sys.argv[7]) if len(sys.argv) > 7 else fdp.WorkflowKind.FLASHDP
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
dy = (torch.randn(B, T, D, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
cfg = fdp.DPConfig(clip_c=1.0, sigma=1.0, reduction="mean", seed=1, layer_id=2, step=0)
call = fdp.PreparedBackward(kind, x, dy, cfg if kind != fdp.WorkflowKind.NON_DP else None, path=path,
                            noise_impl="philox")
for _ in range(reps):
    call()
torch.cuda.synchronize()
print("plan", fdp.execution_plan((B, T, P), (B, T, D), path=path))
