"""Launch one GPT-2 layer's fused DP backward a few times (for ncu captures).

    python tools/prof_one.py [c_fc|c_attn|attn_proj|mlp_proj] [reps] [kind] [B] [T]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_01154_b200 as fdp  # noqa: E402

SHAPES = {"c_attn": (768, 2304), "attn_proj": (768, 768), "c_fc": (768, 3072), "mlp_proj": (3072, 768)}
name = sys.argv[1] if len(sys.argv) > 1 else "c_fc"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
kind = fdp.WorkflowKind(sys.argv[3]) if len(sys.argv) > 3 else fdp.WorkflowKind.FLASHDP
B = int(sys.argv[4]) if len(sys.argv) > 4 else 8
T = int(sys.argv[5]) if len(sys.argv) > 5 else 1024
P, D = SHAPES[name]
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
dy = (torch.randn(B, T, D, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
cfg = fdp.DPConfig(clip_c=1.0, sigma=1.0, reduction="mean", seed=1, layer_id=2, step=0)
call = fdp.PreparedBackward(kind, x, dy, cfg if kind != fdp.WorkflowKind.NON_DP else None)
for _ in range(reps):
    call()
torch.cuda.synchronize()
print("plan", call.plan.path, call.plan.tile_p, call.plan.groups, call.plan.grid)
