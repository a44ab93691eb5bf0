"""torch.profiler breakdown of the Llama training step (DP vs non-DP), GPU kernel
time grouped by what it does (tools/train_llama.py's model and step).

    python tools/train_llama_prof.py [--model llama-7b] [--layers 4]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2507_01154_b200.ddp import DataParallelStep  # noqa: E402
from paper_2507_01154_b200.llama import Llama, LlamaConfig  # noqa: E402

GROUPS = [("fdp_dp_dW", ("dpdw_", "ghost_norm", "k_single_finalize", "k_reduce_norms", "k_single_factor")),
          ("fdp_optimizer", ("k_adam", "k_sgd")),
          ("fdp_param_groups", ("k_vec_", "k_emb_")),
          ("gemm (cuBLAS)", ("nvjet", "gemm", "cutlass", "sm90_", "sm100_")),
          ("attention", ("flash", "fmha", "attention")),
          ("adam", ("adam", "Adam", "multi_tensor")),
          ("cast / copy", ("copy", "cast", "to_copy", "bfloat16")),
          ("reduce", ("reduce",)),
          ("elementwise", ("elementwise", "vectorized")),
          ]


def group_of(name):
    for g, keys in GROUPS:
        if any(k in name for k in keys):
            return g
    return "other"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama-7b")
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--seq", type=int, default=2048)
    ap.add_argument("--zero1", action="store_true")
    a = ap.parse_args()
    for dp in (False, True):
        torch.manual_seed(0)
        cfg = LlamaConfig.named(a.model, seq=a.seq, layers=a.layers)
        with torch.device("cuda"):
            model = Llama(cfg, dp=dp, nondp_linear="fp32grad")
        dstep = DataParallelStep(model, dp=dp, mode="reduce_scatter" if a.zero1 else "allreduce", lr=1e-5,
                                 global_batch=a.batch)
        idx = torch.randint(0, cfg.vocab, (a.batch, a.seq + 1), device="cuda")
        x, y = idx[:, :-1].contiguous(), idx[:, 1:].contiguous()
        it = [0]

        def step():
            it[0] += 1
            dstep(it[0], lambda: model.loss(x, y, reduction="sample_sum") * (1.0 if dp else 1.0 / a.batch))

        for _ in range(3):
            step()
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(3):
                step()
            torch.cuda.synchronize()
        tot = {}
        top = {}
        for ev in prof.key_averages():
            t = ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
            if t <= 0:
                continue
            g = group_of(ev.key)
            tot[g] = tot.get(g, 0.0) + t / 3 / 1e3
            top[ev.key[:80]] = t / 3 / 1e3
        print(json.dumps({"dp": dp, "model": a.model, "layers": a.layers, "ms_per_step_by_group":
                          {k: round(v, 3) for k, v in sorted(tot.items(), key=lambda kv: -kv[1])},
                          "top_kernels_ms": {k: round(v, 3) for k, v in
                                             sorted(top.items(), key=lambda kv: -kv[1])[:14]}}), flush=True)
        del model, dstep, step
        import gc
        gc.collect()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
