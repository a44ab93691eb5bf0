"""q/k/v (or gate/up) of one Llama block: per-layer calls vs one fdp_backward_shared_x call
(run under ncu for the per-kernel times, or plainly for CUDA-event times).

    python tools/shared_x_prof.py [P] [D,D,...] [B] [T]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_01154_b200 as fdp  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 5120
Ds = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "5120,5120,5120").split(",")]
B = int(sys.argv[3]) if len(sys.argv) > 3 else 2
T = int(sys.argv[4]) if len(sys.argv) > 4 else 2048
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
solo, own = [], []
for k, D in enumerate(Ds):
    dy = (torch.randn(B, T, D, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
    cfg = fdp.DPConfig(1.0, 1.0, "mean", seed=1, layer_id=k)
    solo.append(fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x, dy, cfg, noise_impl="philox"))
    own.append(fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x, dy, cfg, noise_impl="philox"))
shared = fdp.PreparedSharedX(own)


def timed(fn, n=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


def run_solo():
    for c in solo:
        c()


res = {"P": P, "Ds": Ds, "B": B, "T": T}
for _ in range(2):
    for k, fn in (("solo_us", run_solo), ("shared_us", shared)):
        res[k] = round(min(res.get(k, 1e30), timed(fn)), 1)
print(json.dumps(res), flush=True)
