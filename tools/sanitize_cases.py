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
# ghost norms with K slices (single CTA and pair), multicast stream layout (down projection)
for pair, split in (("0", "3"), ("1", "2")):
    os.environ["FDP_GHOST_PAIR"], os.environ["FDP_GHOST_SPLIT"] = pair, split
    fdp.backward_flashdp(*inputs(2, 300, 192, 1600), cfg, path="two_phase", norm_phase="ghost")
os.environ.pop("FDP_GHOST_PAIR")
os.environ.pop("FDP_GHOST_SPLIT")
xm, dym = inputs(3, 130, 1536, 640)
fdp.backward_flashdp(xm, dym, cfg, path="two_phase", noise_impl="philox")  # P >= 2D: 4-CTA multicast layout
# non-linear parameter groups
for kind in ("bias", "rmsnorm", "layernorm"):
    for dt in (torch.bfloat16, torch.float32):
        a, b = inputs(3, 70, 8, 777, dt)
        fdp.vector_dp_grad(kind, b, b, cfg, noise_impl="philox")
        a, b = inputs(2, 33, 8, 1024, dt)
        fdp.vector_dp_grad(kind, b, b, cfg, noise_impl="keyed_f32")
tok = torch.randint(-1, 51, (3, 300), device="cuda")
for d in (70, 256):
    fdp.embedding_dp_grad(tok, torch.randn(3, 300, d, device="cuda"), 50, cfg, noise_impl="philox")
fdp.embedding_dp_grad(torch.zeros(2, 700, dtype=torch.int64, device="cuda"), torch.randn(2, 700, 40, device="cuda"),
                      3, cfg)  # one run longer than a norm block's key stage
# round 2: shared-X ghost (3 layers, partial 256-row Gram tiles), spill norm phase, deferred chain,
# stream-K reweight with split tiles (opening-segment stores, continuation reduce-adds), accumulate
xs = inputs(2, 300, 384, 8)[0]
pbs = [fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, xs, inputs(2, 300, 8, D)[1], cfg, path="two_phase",
                            norm_phase="ghost", noise_impl="philox") for D in (256, 512, 384)]
fdp.PreparedSharedX(pbs)()
fdp.backward_flashdp(*inputs(3, 200, 512, 256), cfg, path="two_phase", norm_phase="spill", noise_impl="philox")
chain = fdp.DeferredChain()
for D in (256, 384):
    fdp.workflows._run(fdp.WorkflowKind.FLASHDP, *inputs(1, 256, 512, D), cfg, None, None, path="two_phase",
                       noise_impl="philox", chain=chain)
chain.flush()
xk, dyk = inputs(40, 64, 512, 512)
for acc in (False, True):
    gout = torch.zeros(512, 512, device="cuda")
    fdp.workflows._run(fdp.WorkflowKind.FLASHDP, xk, dyk, cfg, None, None, path="two_phase", noise_impl="philox",
                       grad_out=gout, accumulate=acc)
st = fdp.OptimizerState.fresh(torch.zeros(1000, device="cuda"), eta=0.1)
fdp.dp_adam_step_(st, torch.ones(1000, device="cuda"))
# session 2: deferred clip (single-sample GEMM + PDL factor kernel; fallback scale 1), scaled Adam / SGD,
# PDL ghost -> factor reduce -> reweight (the default two-phase launches above already use it)
sc = torch.zeros(1, device="cuda")
fdp.workflows._run(fdp.WorkflowKind.FLASHDP, *inputs(1, 256, 512, 384), cfg, None, None, path="two_phase",
                   noise_impl="philox", add_noise=False, grad_scale_out=sc)
fdp.workflows._run(fdp.WorkflowKind.FLASHDP, *inputs(2, 256, 512, 384), cfg, None, None, path="two_phase",
                   noise_impl="philox", add_noise=False, grad_scale_out=sc)
st = fdp.OptimizerState.fresh(torch.zeros(1003, device="cuda"), eta=0.1)
fdp.dp_adam_step_(st, torch.ones(1003, device="cuda"), grad_scale=sc, noise=cfg, layer_numel=1003)
fdp.dp_sgd_step_(torch.zeros(1003, device="cuda"), torch.ones(1003, device="cuda"), 0.1, grad_scale=sc)
# session 2 (cont.): mixed ghost schedule (whole items + K-split last wave), multi-segment Adam / SGD
os.environ["FDP_GHOST_PAIR"] = "1"
fdp.backward_flashdp(*inputs(8, 256, 256, 256), cfg, path="two_phase", norm_phase="ghost")  # 8 items, few clusters
os.environ.pop("FDP_GHOST_PAIR")
from paper_2507_01154_b200.ddp import BucketedAdam, GradBuckets  # noqa: E402

for kind in ("adam", "sgd"):
    ps = [torch.nn.Parameter(torch.randn(n, device="cuda")) for n in (1001, 3, 4096)]
    bk = GradBuckets(ps, flat_params=True, hooks=False, isolate=[ps[2]])
    bk.zero_grad()
    for p_ in ps:
        p_.grad.copy_(torch.randn_like(p_))
    keys = {id(ps[0]): (cfg, 0, 1001, "philox"), id(ps[2]): (cfg, 0, 4096, "philox")}
    opt = BucketedAdam(bk, lr=1e-3, noise_keys=keys, kind=kind)
    opt.step(3)
torch.cuda.synchronize()
print("sanitize cases done")
