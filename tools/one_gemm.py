import os, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2507_01154_b200 as fdp
g = torch.Generator(device="cuda").manual_seed(0)
B, T, P, D = 1, 2048, 5120, 5120
x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
dy = (torch.randn(B, T, D, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
c = fdp.PreparedBackward(fdp.WorkflowKind.NON_DP, x, dy, None)
for _ in range(3): c()
torch.mm(dy.view(-1, D).t(), x.view(-1, P), out_dtype=torch.float32)
torch.mm(dy.view(-1, D).t(), x.view(-1, P), out_dtype=torch.float32)
torch.cuda.synchronize()
