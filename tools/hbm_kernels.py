"""The HBM-bound kernels of the path, for an ncu launch list (achieved DRAM GB/s):
the single-sample clip + noise finalize (Llama-13B up projection, B = 1), the fp32
DP-Adam step with shard noise (67 M parameters) and with a deferred clip factor,
and the bias / RMSNorm parameter-group passes.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum python tools/hbm_kernels.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_01154_b200 as fdp  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
cfg = fdp.DPConfig(1.0, 1.0, "mean", seed=1, layer_id=2)
x = torch.randn(1, 2048, 5120, device="cuda", generator=g).to(torch.bfloat16)
dy = (torch.randn(1, 2048, 13824, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
call = fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x, dy, cfg, noise_impl="philox")  # GEMM + finalize
for _ in range(2):
    call()
n = 67_108_864
st = fdp.OptimizerState.fresh(torch.zeros(n, device="cuda"), eta=1e-4)
grad = torch.randn(n, device="cuda", generator=g)
scale = torch.full((1,), 0.5, device="cuda")
for _ in range(2):
    fdp.dp_adam_step_(st, grad, noise=cfg, layer_numel=n)
    fdp.dp_adam_step_(st, grad, grad_scale=scale)
# the one-launch DP-Adam over a bucket table (noise + deferred factor slot), and the
# deferred single-sample path (GEMM + one-warp factor kernel, no pass)
from paper_2507_01154_b200.ddp import BucketedAdam, GradBuckets  # noqa: E402

ps = [torch.nn.Parameter(torch.randn(n, device="cuda", generator=g)) for n in (16_777_216, 45_088_768, 4096)]
bk = GradBuckets(ps, flat_params=True, hooks=False, isolate=ps[:2])
bk.zero_grad()
keys = {id(p_): (cfg, 0, p_.numel(), "philox") for p_ in ps}
opt = BucketedAdam(bk, lr=1e-4, noise_keys=keys)
for i in range(2):
    opt.step(i)
sc = torch.zeros(1, device="cuda")
dfr = fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x, dy, cfg, noise_impl="philox", add_noise=False, grad_scale=sc)
for _ in range(2):
    dfr()
dyv = torch.randn(8, 1024, 4096, device="cuda", generator=g).to(torch.bfloat16)
for kind in ("bias", "rmsnorm"):
    fdp.vector_dp_grad(kind, dyv, dyv, cfg, noise_impl="philox")
torch.cuda.synchronize()
print("done")
