"""Per-CTA wait totals of the stream-K kernel (FDP_STREAM_TRACE=1 prints one JSON line per
launch on stderr): where the reweight / non-DP launches spend their time.

    FDP_STREAM_TRACE=1 python tools/stream_trace.py "B,T,P,D;..." 2> trace.jsonl
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2507_01154_b200 as fdp  # noqa: E402

shapes = sys.argv[1] if len(sys.argv) > 1 else "64,128,1024,1024;64,128,2048,2048;4,2048,4096,4096"
g = torch.Generator(device="cuda").manual_seed(0)
for s in shapes.split(";"):
    B, T, P, D = (int(v) for v in s.split(","))
    x = torch.randn(B, T, P, device="cuda", generator=g).to(torch.bfloat16)
    dy = (torch.randn(B, T, D, device="cuda", generator=g) * 1e-3).to(torch.bfloat16)
    cfg = fdp.DPConfig(1.0, 1.0, "mean", seed=1, layer_id=0)
    for name, call in (("nondp", fdp.PreparedBackward(fdp.WorkflowKind.NON_DP, x, dy, None)),
                       ("dp", fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, x, dy, cfg, noise_impl="philox",
                                                   path="two_phase"))):
        for i in range(3):
            print(f'{{"shape": [{B}, {T}, {P}, {D}], "call": "{name}", "rep": {i}}}', file=sys.stderr, flush=True)
            call()
            torch.cuda.synchronize()
