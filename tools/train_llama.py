"""Llama-2 DP pre-training step vs the same model's non-DP step, on 1..N GPUs
(BASELINE configs 3 and 4; PAPER.md:6, :37, :247 -- FlashDP at 90 % of non-DP on
Llama-13B; setup PAPER.md:535-537).

    python tools/train_llama.py --model llama-7b [--layers L] [--batch B] [--seq 2048]
    torchrun --nnodes 1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29511 \
        tools/train_llama.py --model llama-7b                       # config 3: DP-Adam, all-reduce
    torchrun --nnodes 1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29511 \
        tools/train_llama.py --model llama-13b --zero1              # config 4: ZeRO-1

One process per GPU (NCCL capped at --comm-sms CTAs). Both arms run the SAME
data-parallel machinery (ddp.DataParallelStep): fp32 master weights in flat
per-bucket buffers, gradient buckets reduced from inside the backward on a
communication stream, Adam without bias correction on the bucket layout
(replicated after an all-reduce, or ZeRO-1 after a reduce-scatter with the DP
noise added on the owner's shard). They differ only in the gradients:

  DP:     every parameter DP -- DPLinear (7 projections per block + LM head),
          DPRMSNorm, DPEmbedding -- per-layer clip C, sigma, Philox noise added
          once per element; the DP linear weight gradients run bucket by bucket
          inside the backward (GroupedDPBackward(buckets=...)).
  non-DP: nn.Linear replaced by FP32GradLinear (cuBLAS writes the fp32 weight
          gradient, the DP kernels' precision), torch RMSNorm / Embedding.

Random-init weights (same seed on every rank), synthetic token ids (different
per rank), bf16 autocast. Timing: CUDA events over --steps steps after
--warmup, barrier + synchronize on both sides, max over ranks. Rank 0 prints
one JSON line with global tokens/s of both arms and DP as % of non-DP.
"""
import argparse
import gc
import json
import os
import sys
import time

# full-depth models: parameters move into per-bucket flat buffers after construction;
# expandable segments let the freed per-parameter blocks serve the bucket-sized optimizer state
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2507_01154_b200.ddp import DataParallelStep, init_distributed  # noqa: E402
from paper_2507_01154_b200.llama import Llama, LlamaConfig  # noqa: E402


def run(dp: bool, a, rank: int, world: int, dev: torch.device) -> dict:
    torch.manual_seed(0)  # identical initial weights on every rank
    cfg = LlamaConfig.named(a.model, seq=a.seq, **({"layers": a.layers} if a.layers else {}))
    with torch.device(dev):
        model = Llama(cfg, dp=dp, clip_c=a.clip, sigma=a.sigma, noise_impl="philox", nondp_linear=a.nondp_linear)
    gB = a.batch * world
    step = DataParallelStep(model, dp=dp, mode="reduce_scatter" if a.zero1 else "allreduce", lr=1e-5,
                            rank=rank, world=world, comm_sms=a.comm_sms, bucket_bytes=a.bucket_mb << 20,
                            global_batch=gB, defer_clip={"auto": None, "on": True, "off": False}[a.defer_clip])
    g = torch.Generator(device=dev).manual_seed(1 + rank)
    idx = torch.randint(0, cfg.vocab, (a.batch, a.seq + 1), device=dev, generator=g)
    x, y = idx[:, :-1].contiguous(), idx[:, 1:].contiguous()
    scale = 1.0 if dp else 1.0 / gB  # DP modules take the mean over the logical batch themselves

    def one(i):
        return step(i, lambda: model.loss(x, y, reduction="sample_sum") * scale)

    torch.cuda.reset_peak_memory_stats(dev)
    for i in range(a.warmup):
        one(i)
    torch.cuda.synchronize(dev)
    time.sleep(1.0)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(a.steps):
        loss = one(a.warmup + i)
    e1.record()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1) / a.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    out = {"ms_per_step": ms, "tokens_per_s": gB * a.seq / (ms * 1e-3),
           "loss_per_sample": float(loss.detach()) / (a.batch if dp else a.batch / gB),
           "dp_modules": len(step.dp_mods), "params": sum(p.numel() for p in model.parameters()),
           "buckets": len(step.buckets.buckets), "deferred_clips": step.last_deferred, "peak_mem_gb": torch.cuda.max_memory_allocated(dev) / 1e9}
    return out


def run_arm(dp: bool, a, rank: int, world: int, dev: torch.device) -> dict:
    out = run(dp, a, rank, world, dev)
    gc.collect()  # the arm's model, buckets and optimizer state are unreachable now
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="llama-7b", choices=["llama-7b", "llama-13b"])
    ap.add_argument("--layers", type=int, default=0, help="0 = the model's depth")
    ap.add_argument("--batch", type=int, default=1, help="sequences per rank")
    ap.add_argument("--seq", type=int, default=2048)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--zero1", action="store_true", help="reduce-scatter + ZeRO-1 Adam (config 4)")
    ap.add_argument("--comm-sms", type=int, default=4)
    ap.add_argument("--bucket-mb", type=int, default=512)
    ap.add_argument("--clip", type=float, default=1.0)
    ap.add_argument("--sigma", type=float, default=1.0)
    ap.add_argument("--nondp-linear", default="fp32grad", choices=["fp32grad", "torch"])
    ap.add_argument("--arms", default="nondp,dp")
    ap.add_argument("--defer-clip", default="auto", choices=["auto", "on", "off"],
                    help="B = 1 per rank: clip factor applied by the collective / Adam (ddp.DataParallelStep)")
    a = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        init_distributed("nccl", comm_sms=a.comm_sms, device=dev)
    res = {}
    for arm in a.arms.split(","):
        res[arm] = run_arm(arm == "dp", a, rank, world, dev)
    if rank == 0:
        line = {"model": a.model, "layers": a.layers or LlamaConfig.named(a.model).layers, "gpus": world,
                "batch_per_gpu": a.batch, "global_batch": a.batch * world, "seq": a.seq,
                "parallelism": ("zero1" if a.zero1 else "allreduce") + f"-dp{world}",
                "comm_sms": a.comm_sms, "bucket_mb": a.bucket_mb, "nondp_linear": a.nondp_linear,
                "defer_clip": a.defer_clip}
        line.update(res)
        if "dp" in res and "nondp" in res:
            line["dp_pct_of_non_dp"] = 100.0 * res["dp"]["tokens_per_s"] / res["nondp"]["tokens_per_s"]
        line["note"] = ("every parameter DP (7 projections per block + LM head: DPLinear; RMSNorms; token "
                        "embedding), per-layer clip C, sigma, Philox; non-DP: FP32GradLinear projections (fp32 "
                        "weight gradients from cuBLAS); both arms: same buckets, collectives and Adam; random init, "
                        "synthetic tokens")
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
