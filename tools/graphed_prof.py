"""Kernel-time breakdown (CUPTI) of the graphed GPT-2 small step (every parameter DP vs
non-DP, DP-SGD, B = 1): what the DP arm's extra GPU time is.

    python tools/graphed_prof.py [B]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2507_01154_b200.ddp import DataParallelStep, GraphedStep  # noqa: E402
from paper_2507_01154_b200.gpt2 import GPT2, GPT2Config  # noqa: E402

GROUPS = [("dp_dW", ("dpdw_", "ghost_norm", "k_single", "k_reduce_norms")), ("dp_vec", ("k_vec_",)),
          ("dp_emb", ("k_emb_",)), ("optimizer", ("k_adam", "k_sgd")), ("gemm", ("nvjet", "gemm", "cutlass", "sm100")),
          ("attention", ("flash", "fmha", "attention")), ("layernorm", ("layer_norm", "LayerNorm")),
          ("embedding", ("embedding", "index")), ("reduce", ("reduce",)), ("elementwise", ("elementwise",))]


def grp(name):
    for g, keys in GROUPS:
        if any(k in name for k in keys):
            return g
    return "other"


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    for dp in (False, True):
        torch.manual_seed(0)
        cfg = GPT2Config(seq=1024)
        model = GPT2(cfg, dp="full" if dp else False, tied=False, nondp_linear="fp32grad").cuda()
        step = DataParallelStep(model, dp=dp, lr=1e-4, global_batch=B, optimizer="sgd")
        idx = torch.randint(0, cfg.vocab, (B, cfg.seq + 1), device="cuda")
        x, y = idx[:, :-1].contiguous(), idx[:, 1:].contiguous()
        gs = GraphedStep(step, lambda: model.loss(x, y) * (B if dp else 1.0), warmup=3)
        for _ in range(3):
            gs()
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(5):
                gs()
            torch.cuda.synchronize()
        tot, cnt, per = {}, {}, {}
        for ev in prof.events():
            if ev.device_type != torch.autograd.DeviceType.CUDA:
                continue
            g = grp(ev.name)
            if g in ("dp_dW", "dp_vec", "gemm"):
                k = (g, ev.name[:70])
                per[k] = per.get(k, 0.0) + ev.time_range.elapsed_us() / 5
            tot[g] = tot.get(g, 0.0) + ev.time_range.elapsed_us() / 5
            cnt[g] = cnt.get(g, 0) + 1 / 5
        print(json.dumps({"dp": dp, "B": B, "us_per_step": {k: round(v, 1) for k, v in sorted(tot.items(), key=lambda kv: -kv[1])},
                          "launches_per_step": {k: round(v) for k, v in cnt.items()},
                          "top_kernels_us": [[g, n, round(v, 1)] for (g, n), v in
                                             sorted(per.items(), key=lambda kv: -kv[1])[:12]]}), flush=True)
        del model, step, gs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
