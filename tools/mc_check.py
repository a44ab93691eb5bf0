"""Quick correctness + timing check of the multicast stream kernel (FDP_STREAM_MC=1)
against the default layout on the same inputs (non-DP GEMM, B=1 path, two-phase)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_01154_b200 as fdp  # noqa: E402


def timed(fn, n=10):
    fn()
    torch.cuda.synchronize()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


g = torch.Generator(device="cuda").manual_seed(0)
for (B, T, P, D) in [(1, 512, 1024, 768), (1, 2048, 5120, 5120), (2, 2048, 5120, 13824), (3, 1000, 1536, 2560),
                     (4, 2048, 13824, 5120)]:
    x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
    dy = (torch.randn(B, T, D, device="cuda", generator=g) * 1e-2).to(torch.bfloat16)
    cfg = fdp.DPConfig(1.0, 1.0, "mean", seed=1, layer_id=0)
    out = {}
    for mc in ("0", "1"):
        os.environ["FDP_STREAM_MC"] = mc
        nd = fdp.PreparedBackward(fdp.WorkflowKind.NON_DP, x, dy, None)
        dp = fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x, dy, cfg, noise_impl="philox", path="two_phase")
        nd()
        dp()
        torch.cuda.synchronize()
        out[mc] = (nd.grad_w.clone(), dp.grad_w.clone(), dp.norms_sq.clone(), timed(nd), timed(dp))
    a, b = out["0"], out["1"]
    err_nd = float((a[0] - b[0]).abs().max() / a[0].abs().max())
    err_dp = float((a[1] - b[1]).abs().max() / a[1].abs().max())
    err_n = float((a[2] - b[2]).abs().max() / a[2].abs().max())
    print(f"B={B} T={T} P={P} D={D}: nondp err {err_nd:.2e} dp err {err_dp:.2e} norms err {err_n:.2e} | "
          f"nondp {a[3]:.1f} -> {b[3]:.1f} us, dp {a[4]:.1f} -> {b[4]:.1f} us", flush=True)
