#!/usr/bin/env python
"""Benchmark of the FlashDP hot path on B200: the fused per-layer DP-SGD
weight-gradient backward of every linear layer of GPT-2 small.

A "step" is one pass of the hot path over one batch of synthetic activations:
for each of the 48 linear layers of GPT-2 small (12 blocks x c_attn 768->2304,
attn c_proj 768->768, mlp c_fc 768->3072, mlp c_proj 3072->768) the DP weight
gradient  mean_b clip_C(dY_b^T X_b) + sigma*C*N(seed, layer, step, idx)  with
per-sample per-layer clipping (reference workflows.py:340-421), at B=8
sequences x T=1024 tokens, bf16 inputs, fp32 accumulate/output.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N>1 (under torchrun): data parallel over ranks, weak scaling (B=8 per rank);
each rank adds noise only on its slice of every layer's index space and the
clipped sums are summed with one NCCL all-reduce per step.

Prints ONE JSON line (rank 0).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GPT2_LAYERS = [("c_attn", 768, 2304), ("attn_proj", 768, 768), ("c_fc", 768, 3072), ("mlp_proj", 3072, 768)]
N_BLOCKS = 12
METRIC = "DP-train tokens/sec + % of non-DP at 1/2/4/8 B200; fused DP-linear TFLOP/s vs peak"
UNIT = "tokens/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--seq", type=int, default=1024)
    ap.add_argument("--clip", type=float, default=1.0)
    ap.add_argument("--sigma", type=float, default=1.0)
    ap.add_argument("--noise", default="philox", choices=["keyed_f32", "keyed_f64", "philox"],
                    help="production noise: Philox (north star); keyed_f32 reproduces the reference draws")
    ap.add_argument("--path", default="auto")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-nondp", action="store_true")
    ap.add_argument("--no-train", action="store_true",
                    help="skip the GPT-2 training-step comparison (DP linear layers vs nn.Linear)")
    ap.add_argument("--graph", action="store_true", help="replay the step as a CUDA graph")
    ap.add_argument("--no-llama", action="store_true", help="skip the Llama-13B-shape training-step comparison")
    ap.add_argument("--llama-layers", type=int, default=8)
    ap.add_argument("--per-layer", action="store_true",
                    help="one fused launch per layer instead of one multi-layer launch per step")
    ap.add_argument("--chunks", type=int, default=4,
                    help="N>1: layer chunks whose all-reduce overlaps the next chunk's launch")
    ap.add_argument("--comm-sms", type=int, default=4,
                    help="N>1: SMs left free for the NCCL kernel (the GPT-2 packing uses 144 of 148 SMs anyway)")
    return ap.parse_args()


def layer_list():
    out = []
    for blk in range(N_BLOCKS):
        for j, (name, P, D) in enumerate(GPT2_LAYERS):
            out.append((blk * len(GPT2_LAYERS) + j, f"h{blk}.{name}", P, D))
    return out


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return pk, "measured"
    except Exception:  # noqa: BLE001
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:  # noqa: BLE001
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:  # noqa: BLE001
            self.proc.kill()
        sm, mx, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
                power.append(float(parts[3]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm), "power_w_max": max(power) if power else None}


# ----------------------------------------------------------------------------- reference (CPU) arm

def bench_config(a, world: int, global_B: int, T: int, graph: bool) -> dict:
    """The workload dict both arms print (identical, so the driver can pair them)."""
    return {"workload": "gpt2-small: DP weight-gradient backward of all 48 linear layers "
                        "(per-sample per-layer clip, mean, keyed noise)",
            "global_batch": global_B, "seq_len": T, "parallelism": f"dp{world}",
            "clip_c": a.clip, "sigma": a.sigma, "noise": a.noise,
            "l2": "inputs larger than L2 (%.2f GB of X/dY per rank per step)" % (
                sum((global_B // world) * T * (P + D) * 2 for _, _, P, D in layer_list()) / 1e9),
            "graph": graph}


def cpu_whole_steps(a, warmup: int, steps: int):
    """The reference's CPU implementation of the path, WHOLE steps: every step runs
    the flashdp arithmetic of workflows.py:340-421 (per-sample G_b = dY_b^T X_b,
    ||G_b||^2, clip factor, clipped sum, mean + sigma*C*keyed noise over D*P) for
    all 48 layers at the full batch, in float64 (the reference's precision), as
    the oracle port (oracle/dp_oracle.py; the reference is pure numpy and does not
    travel to the GPU box). The layers of a step run on a thread pool with one
    BLAS thread per worker, one worker per host core. -> (seconds per timed step,
    cores, sample description)."""
    import numpy as np
    from concurrent.futures import ThreadPoolExecutor

    from oracle import dp_oracle as O

    try:
        from threadpoolctl import threadpool_limits
    except ImportError:  # pragma: no cover
        threadpool_limits = None
    B, T = a.batch, a.seq
    cores = os.cpu_count() or 1
    rng = np.random.default_rng(7)
    # one (X, dY) pair per layer type, float32 storage (the math is float64), reused by the 12 blocks
    data = [(rng.standard_normal((B, T, P)).astype(np.float32),
             (rng.standard_normal((B, T, D)) * 1e-3).astype(np.float32)) for _, P, D in GPT2_LAYERS]
    layers = layer_list()

    def one_layer(item, step_idx):
        lid = item[0]
        x, dy = data[lid % len(GPT2_LAYERS)]
        acc, norms = O.per_sample_accumulate(x, dy, a.clip)
        out = O.finalize(acc, B, O.Cfg(a.clip, a.sigma, "mean", 1234, lid, step_idx), exact_noise=False)
        return float(out[0, 0]) + float(norms[0])

    per = []
    ctx = threadpool_limits(1) if threadpool_limits else None
    try:
        with ThreadPoolExecutor(max_workers=cores) as pool:
            for i in range(warmup + steps):
                t0 = time.perf_counter()
                sum(pool.map(lambda it: one_layer(it, i), layers))
                if i >= warmup:
                    per.append(time.perf_counter() - t0)
    finally:
        if ctx is not None:
            ctx.unregister()
    sample = (f"whole steps: all {len(layers)} layers x {B} sequences x T={T} per step, float64 numpy "
              f"(oracle/dp_oracle.py restating workflows.py:340-421: per-sample G_b, norm, clip, sum, mean, "
              f"sigma*C*noise over every D*P index with the reference's own keyed construction), "
              f"{cores} worker threads x 1 BLAS thread; {warmup} warm-up + {steps} timed steps")
    return sum(per) / len(per), cores, sample, sum(per)


def run_reference_arm(a, rank: int, world: int):
    """--impl reference: rank 0 alone times whole CPU steps (cpu_whole_steps)."""
    if rank != 0:
        return
    B, T = a.batch, a.seq
    step_s, cores, sample, timed = cpu_whole_steps(a, a.warmup, a.steps)
    value = B * T / step_s  # one rank's workload; under torchrun only rank 0 runs this arm
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(a, world, B * world, T, False),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "timed_s": timed}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm

def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    import torch
    import torch.distributed as dist

    if a.impl == "reference":
        if world > 1:
            dist.init_process_group("gloo")
        run_reference_arm(a, rank, world)
        if world > 1:
            dist.destroy_process_group()
        return

    # test hooks: run the N>1 code path on a one-GPU box (every rank on cuda:0, gloo);
    # the driver's multi-GPU runs use one GPU per rank and NCCL
    same_gpu = os.environ.get("FDP_BENCH_SAME_GPU") == "1"
    backend = os.environ.get("FDP_BENCH_BACKEND", "nccl")
    dev_index = 0 if same_gpu else local_rank
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    if world > 1:
        if backend == "nccl":  # NCCL held to comm_sms CTAs: it runs beside the capped group launches
            from paper_2507_01154_b200.ddp import init_distributed

            init_distributed("nccl", comm_sms=a.comm_sms, device=dev)
        else:
            dist.init_process_group(backend)

    import paper_2507_01154_b200 as fdp

    B, T = a.batch, a.seq
    layers = layer_list()
    g = torch.Generator(device=dev).manual_seed(1000 + rank)
    xs, dys = {}, {}
    for _, name, P, D in layers:
        # activations O(1), upstream gradients small (typical backward magnitudes)
        xs[name] = torch.randn(B, T, P, device=dev, generator=g, dtype=torch.float32).to(torch.bfloat16)
        dys[name] = (torch.randn(B, T, D, device=dev, generator=g, dtype=torch.float32) * 1e-3).to(torch.bfloat16)
    n_params = sum(P * D for _, _, P, D in layers)
    flat = torch.zeros(n_params, dtype=torch.float32, device=dev)
    device_step = torch.zeros(1, dtype=torch.int64, device=dev)
    calls, off = [], 0
    global_B = B * world
    # one workspace shared by all layers (they run in order on one stream)
    shared_ws = torch.zeros(64 << 20, dtype=torch.uint8, device=dev)
    for lid, name, P, D in layers:
        grad = flat[off:off + P * D].view(D, P)
        off += P * D
        cfg = fdp.DPConfig(clip_c=a.clip, sigma=a.sigma, reduction="mean", seed=1234, layer_id=lid, step=0)
        c = fdp.PreparedBackward(fdp.WorkflowKind.FLASHDP, xs[name], dys[name], cfg, grad_w=grad, path=a.path,
                                 noise_impl=a.noise, rank=rank, world=world, mean_batch=global_B,
                                 device_step=device_step, workspace=shared_ws)
        calls.append((name, c))
    plans = {n: c.plan for n, c in calls[:4]}
    group = None
    if not a.per_layer:
        glayers = [(xs[name], dys[name], fdp.DPConfig(clip_c=a.clip, sigma=a.sigma, reduction="mean", seed=1234,
                                                      layer_id=lid, step=0)) for lid, name, P, D in layers]
        if world > 1:
            from paper_2507_01154_b200.ddp import ChunkedAllReduceBackward

            group = ChunkedAllReduceBackward(glayers, flat, n_chunks=a.chunks, comm_sms=a.comm_sms,
                                             noise_impl=a.noise, rank=rank, world=world, mean_batch=global_B,
                                             device_step=device_step)
        else:
            group = fdp.PreparedGroup(glayers, grads=[c.grad_w for _, c in calls], noise_impl=a.noise, rank=rank,
                                      world=world, mean_batch=global_B, device_step=device_step)

    stream = torch.cuda.current_stream(dev)
    dominant = "h0.c_fc"  # largest per-launch work; every block's c_fc is timed
    dom_events = []

    def step(record=False):
        # launch on the CURRENT stream: inside torch.cuda.graph() that is the capture stream
        st = torch.cuda.current_stream(dev)
        if group is not None:
            if record:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                group(st)
                e1.record(st)
                dom_events.append((e0, e1))
            else:
                group(st)
            device_step.add_(1)  # N>1: the chunked group already all-reduced every bucket
            return
        for name, c in calls:
            if record and name.endswith(".c_fc"):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                c(st)
                e1.record(st)
                dom_events.append((e0, e1))
            else:
                c(st)
        device_step.add_(1)
        if world > 1:
            dist.all_reduce(flat, op=dist.ReduceOp.SUM)

    graph = None
    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    if a.graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        graph.replay()
        torch.cuda.synchronize()

    clocks = ClockSampler(dev_index)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0e.record(stream)
    for _ in range(a.steps):
        if graph is not None:
            graph.replay()
        else:
            step(record=True)
    t1e.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    elapsed_ms = t0e.elapsed_time(t1e)
    if world > 1:
        tt = torch.tensor([elapsed_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed_ms = float(tt.item())
    ms_per_step = elapsed_ms / a.steps
    tokens_per_step = global_B * T
    value = tokens_per_step / (ms_per_step * 1e-3)
    flops_per_step_rank = sum(2 * B * T * P * D for _, _, P, D in layers)

    # dominant kernel: fused DP-dW launch of the c_fc layers, CUDA events on the launch stream
    dom_ms = [e0.elapsed_time(e1) for e0, e1 in dom_events] if dom_events else []
    dom_flops = flops_per_step_rank if group is not None else 2 * B * T * 768 * 3072
    peaks, peak_kind = load_peaks()
    dom_avg_s = (statistics.mean(dom_ms) * 1e-3) if dom_ms else None
    achieved = dom_flops / dom_avg_s / 1e12 if dom_avg_s else None
    # algorithmic bytes of the same launch: bf16 X and dY read once, fp32 grad_w written, fp32 norms
    dom_layers = layers if group is not None else [(0, "c_fc", 768, 3072)]
    dom_bytes = sum(2 * B * T * (P + D) + 4 * D * P + 4 * B for _, _, P, D in dom_layers)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("group_kernel_dram_bytes" if group is not None
                                                 else "fused_c_fc_dram_bytes")
        except Exception:  # noqa: BLE001
            traffic = None
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
                "frac": (achieved / peaks["bf16_tflops"]) if achieved else None, "traffic": traffic,
                "peak_source": f"{peak_kind} bf16 burst (MEASURED_PEAKS.json)",
                "frac_of_spec_2250": (achieved / 2250.0) if achieved else None,
                "frac_of_sustained": (achieved / peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]))
                if achieved else None,
                "kernel": ("dpdw_group_kernel: fused DP backward of all 48 layers in one launch, B=%d T=%d" % (B, T))
                if group is not None else "dpdw_tc_kernel (MODE_FUSED) on c_fc: B=%d T=%d P=768 D=3072" % (B, T),
                "algorithmic_flops_per_launch": dom_flops, "algorithmic_bytes_per_launch": dom_bytes,
                "avg_launch_ms": dom_avg_s * 1e3 if dom_avg_s else None,
                "launches_timed": len(dom_ms)}

    extra = {}
    if group is not None:
        def per_layer_step():
            for _, c in calls:
                c(stream)
        for _ in range(3):
            per_layer_step()
        torch.cuda.synchronize()
        p0e, p1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0e.record(stream)
        n_pl = max(10, a.steps // 4)
        for _ in range(n_pl):
            per_layer_step()
        p1e.record(stream)
        torch.cuda.synchronize()
        extra["per_layer_launches_ms_per_step"] = p0e.elapsed_time(p1e) / n_pl
    # ---- non-DP baseline (same layers, plain bf16 dW GEMM): cuBLAS and our tcgen05 kernel
    if not a.no_nondp:
        def nondp_cublas():
            for _, name, P, D in layers:
                x2 = xs[name].view(-1, P)
                y2 = dys[name].view(-1, D)
                torch.mm(y2.t(), x2, out_dtype=torch.float32)
            if world > 1:  # non-DP data parallelism sums the same gradient bytes (the DP arm's chunks do too)
                dist.all_reduce(flat, op=dist.ReduceOp.SUM)

        nd_calls = [fdp.PreparedBackward(fdp.WorkflowKind.NON_DP, xs[n], dys[n], None, grad_w=c.grad_w)
                    for n, c in calls]

        def nondp_ours():
            for c in nd_calls:
                c(stream)

        def timeit(fn, n):
            time.sleep(1.0)  # same idle start for every arm (clock / power state)
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(n):
                fn()
            e1.record(stream)
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / n

        # paired comparison: DP step and non-DP dW timed alike, alternating, best of 3
        n_cmp = max(20, a.steps // 2)
        dp_t, nd_t, nd_own_t = [], [], []
        nd_err = None
        def dp_kernels():  # the DP backward alone (collectives excluded on both sides)
            if group is not None:
                group(stream)
            else:
                for _, c in calls:
                    c(stream)
            device_step.add_(1)

        for _ in range(3):
            dp_t.append(timeit(dp_kernels, n_cmp))
            try:
                nd_t.append(timeit(nondp_cublas, n_cmp))
            except Exception as e:  # noqa: BLE001
                nd_err = repr(e)[:200]
            nd_own_t.append(timeit(nondp_ours, n_cmp))
        nd_ms = min(nd_t) if nd_t else None
        dp_ms = min(dp_t)
        nd_ours_ms = min(nd_own_t)
        if nd_err:
            extra["nondp_cublas_error"] = nd_err
        extra["nondp"] = {
            "method": "DP step, cuBLAS non-DP dW and our non-DP dW each timed over %d steps after 1 s idle, "
                      "alternating, best of 3%s" % (n_cmp, "; N>1: both arms include the gradient all-reduce"
                                                    if world > 1 else ""),
            "dp_ms_per_step": dp_ms, "cublas_ms_per_step": nd_ms, "tcgen05_nondp_ms_per_step": nd_ours_ms,
            "dp_over_nondp_pct_vs_cublas": (100.0 * nd_ms / dp_ms) if nd_ms else None,
            "dp_over_nondp_pct_vs_own": 100.0 * nd_ours_ms / dp_ms,
            "nondp_tflops_cublas": flops_per_step_rank / (nd_ms * 1e-3) / 1e12 if nd_ms else None,
        }
        # restore DP grads (non-DP calls overwrote them); not part of any timing
        for _ in range(1):
            step()
        torch.cuda.synchronize()

    # ---- end to end through the public API with host buffers (H2D in, D2H out)
    e2e = None
    if not a.no_e2e:
        host = {}
        for _, name, P, D in layers[:4]:
            host[name.split(".")[1]] = (xs[name].cpu().pin_memory(), dys[name].cpu().pin_memory())
        h2d = sum(B * T * (P + D) * 2 for _, _, P, D in layers)
        d2h = sum(P * D * 4 + B * 4 for _, _, P, D in layers)

        streamer = fdp.HostStreamedBackward(dev, noise_impl=a.noise, rank=rank, world=world, mean_batch=global_B)

        def e2e_step(step_idx):
            batch = []
            for lid, name, P, D in layers:
                xh, yh = host[name.split(".")[1]]
                batch.append((xh, yh, fdp.DPConfig(clip_c=a.clip, sigma=a.sigma, reduction="mean", seed=1234,
                                                    layer_id=lid, step=step_idx)))
            res = streamer(batch)
            assert res[-1].grad_w.device.type == "cpu"

        e2e_step(0)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for i in range(a.e2e_steps):
            e2e_step(i + 1)
        torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - t0) / a.e2e_steps
        if world > 1:
            tt = torch.tensor([e2e_s], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_s = float(tt.item())
        e2e = {"value": tokens_per_step / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": e2e_s * 1e3,
               "api": "paper_2507_01154_b200.HostStreamedBackward (per-layer fdp_backward; pinned host bf16 X/dY in, fp32 grad_w + norms out; H2D/kernel/D2H overlapped on 3 streams)"}

    # ---- CPU baseline (rank 0, N=1 only): oracle port on a bounded sample
    cpu = None
    if not a.no_cpu and world == 1 and rank == 0:
        s, cores, sample, _ = cpu_whole_steps(a, 1, 2)  # ~10-20 s of CPU work on the box's host cores
        cpu = {"value": tokens_per_step / s, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample}

    # ---- whole training step of the same model (N=1): DP linear layers through
    # GroupedDPBackward vs plain nn.Linear, same optimizer (tools/train_gpt2.py)
    train = None
    if not a.no_train and world == 1:
        try:
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            import train_gpt2 as tg

            targs = argparse.Namespace(batch=B, seq=T, steps=10, warmup=3, full=False, nondp_linear="fp32grad")
            nd_t = tg.run(False, targs)
            dp_t = tg.run(True, targs)
            train = {"model": "gpt2-small (124M) training step, random init, synthetic tokens, bf16 autocast, "
                              "fused AdamW",
                     "nondp_baseline": "FP32GradLinear projections: cuBLAS writes the fp32 weight gradients "
                                       "directly (the DP kernels' output precision; no bf16 dW + cast pass)",
                     "dp_tokens_per_s": dp_t["tokens_per_s"],
                     "non_dp_tokens_per_s": nd_t["tokens_per_s"], "dp_ms_per_step": dp_t["ms_per_step"],
                     "non_dp_ms_per_step": nd_t["ms_per_step"],
                     "dp_pct_of_non_dp": 100.0 * dp_t["tokens_per_s"] / nd_t["tokens_per_s"],
                     "dp_scope": "per-layer clipped + noised weight gradients of the 48 linear layers (+ their "
                                 "biases); embeddings / LayerNorm not DP (as in the reference, SPEC.md:8)"}
            # every parameter DP: embeddings, LayerNorms, untied LM head too;
            # the non-DP baseline of this line is the same untied model with nn modules
            fargs = argparse.Namespace(batch=B, seq=T, steps=10, warmup=3, full=True, nondp_linear="fp32grad")
            nd_f = tg.run(False, fargs)
            dp_f = tg.run("full", fargs)
            train["full_dp"] = {"dp_tokens_per_s": dp_f["tokens_per_s"], "non_dp_tokens_per_s": nd_f["tokens_per_s"],
                                "dp_pct_of_non_dp": 100.0 * dp_f["tokens_per_s"] / nd_f["tokens_per_s"],
                                "dp_modules": dp_f["dp_modules"],
                                "dp_scope": "every parameter: 48 linear weights + biases, 25 LayerNorms, token and "
                                            "position embeddings, untied LM head (vocab padded to 50304)"}
            # BASELINE config 2 as stated (DP-SGD): the step through DataParallelStep(optimizer="sgd")
            # captured in ONE CUDA graph (ddp.GraphedStep), every parameter DP vs non-DP, at the
            # paper's smallest batch (host-bound eager) and at the bench's B
            import train_graphed as tgr

            graphed = {"optimizer": "DP-SGD (one fdp_sgd_step_multi launch; noise keyed on a device step)"}
            for gb in sorted({1, B}):
                nd_g = tgr.run(False, True, gb, 20, "sgd")
                dp_g = tgr.run(True, True, gb, 20, "sgd")
                graphed[f"B{gb}"] = {"dp_tokens_per_s": dp_g["tokens_per_s"], "non_dp_tokens_per_s":
                                     nd_g["tokens_per_s"], "dp_pct_of_non_dp":
                                     100.0 * dp_g["tokens_per_s"] / nd_g["tokens_per_s"]}
            train["graphed_every_param_dp"] = graphed
        except Exception as e:  # noqa: BLE001
            train = {"error": repr(e)[:300]}

    # ---- BASELINE config 4 (the paper's headline): Llama-13B-shape DP pre-training step vs
    # the same model's non-DP step, every parameter DP, ZeRO-1 DP-Adam, one GPU, a reduced
    # depth (stated); tools/train_llama.py is the full driver (torchrun for N GPUs)
    llama = None
    if not a.no_train and not a.no_llama and world == 1:
        try:
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            import gc

            import train_llama as tl

            largs = argparse.Namespace(model="llama-13b", layers=a.llama_layers, batch=1, seq=2048, steps=3,
                                       warmup=2, zero1=True, comm_sms=4, bucket_mb=512, clip=1.0, sigma=1.0,
                                       nondp_linear="fp32grad", defer_clip="auto")
            gc.collect()
            torch.cuda.empty_cache()
            nd_l = tl.run_arm(False, largs, 0, 1, dev)
            dp_l = tl.run_arm(True, largs, 0, 1, dev)
            llama = {"model": f"llama-13b shapes (d=5120, 40 heads, MLP 13824, vocab 32000), {a.llama_layers} of 40 "
                              f"blocks, B=1, T=2048, every parameter DP, ZeRO-1 DP-Adam (noise on the owner's shard), "
                              f"random init, synthetic tokens; non-DP = the same model with FP32GradLinear projections, "
                              f"same buckets / optimizer; B=1: the projections' clip factors applied in the "
                              f"Adam step (deferred clip, fdp_dw_deferred)",
                     "deferred_clips": dp_l.get("deferred_clips"),
                     "dp_tokens_per_s": dp_l["tokens_per_s"], "non_dp_tokens_per_s": nd_l["tokens_per_s"],
                     "dp_ms_per_step": dp_l["ms_per_step"], "non_dp_ms_per_step": nd_l["ms_per_step"],
                     "dp_pct_of_non_dp": 100.0 * dp_l["tokens_per_s"] / nd_l["tokens_per_s"],
                     "params": dp_l["params"]}
        except Exception as e:  # noqa: BLE001
            llama = {"error": repr(e)[:300]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic",
            "config": bench_config(a, world, global_B, T, bool(graph is not None)),
            "tflops_per_gpu": flops_per_step_rank / (ms_per_step * 1e-3) / 1e12,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
            # + the pre-drawn noise pass the group launch runs before itself at B <= 2
            # (fdp_capi.cu, FDP_GROUP_PRENOISE_MAXB) when a layer has one sample group:
            # every layer at B = 1, most of the 48 at B = 2 (the planner's packing)
            "gpu_launches": ((a.steps * (2 if (a.sigma > 0 and B <= int(os.environ.get("FDP_GROUP_PRENOISE_MAXB", "2")))
                                         else 1))
                             if group is not None else len(calls) * a.steps),
            "plans": {k: {"path": fdp._lib.PATH_NAMES[v.path], "tile": [v.tile_d, v.tile_p], "groups": v.groups,
                          "grid": v.grid} for k, v in plans.items()},
        }
        line.update(extra)
        if train is not None:
            line["train_step"] = train
        if llama is not None:
            line["llama13b_train_step"] = llama
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
