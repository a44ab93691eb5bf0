import sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_2507_01154_b200 as fdp
def timed(fn, n=50):
    time.sleep(0.5)
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
g = torch.Generator(device="cuda").manual_seed(0)
for B, T, P, D in [(8, 1024, 768, 3072), (8, 1024, 768, 2304), (8, 1024, 768, 768), (8, 1024, 3072, 768),
                   (4, 2048, 2048, 2048), (8, 1024, 1024, 1024)]:
    x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
    dy = (torch.randn(B, T, D, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
    cfg = fdp.DPConfig(1.0, 1.0, "mean", seed=1, layer_id=0)
    a = fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x, dy, cfg, noise_impl="philox", path="fused")
    b = fdp.PreparedGroup([(x, dy, cfg)], noise_impl="philox")
    x2, y2 = x.view(-1, P), dy.view(-1, D)
    print((B, T, P, D), "per-layer", round(timed(a), 1), "group(n=1)", round(timed(b), 1),
          "cublas", round(timed(lambda: torch.mm(y2.t(), x2, out_dtype=torch.float32)), 1), "plan", a.plan.groups, a.plan.grid)
