"""Generate golden vectors from the REAL reference package (run in the dev container).

    PYTHONPATH=/root/reference/pkg/src python tools/gen_golden.py

Imports dpflows from /root/reference/pkg/src (read-only) and writes small
.npz fixtures under tests/golden/. The GPU box never needs the reference: the
tests read only these fixtures and the oracle.
"""

from __future__ import annotations

import json
import math
import random
import sys
from dataclasses import replace
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from dpflows import rng  # noqa: E402
from dpflows.bench import LayerSpec, cell_inputs  # noqa: E402
from dpflows.dpcore import DPConfig, accumulate_micro_batches  # noqa: E402
from dpflows.memmodel import MemSpec  # noqa: E402
from dpflows.tensor import Tensor  # noqa: E402
from dpflows.tiling import BlockPlan, LayerDims, footprint, plan_blocks  # noqa: E402
from dpflows.workflows import WorkflowKind, backward_flashdp, run_backward  # noqa: E402

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"
KINDS = ["non_dp", "explicit_dp", "implicit_dp", "flashdp"]


def gen_rng():
    keys = [(0, 0, 0), (9, 5, 2), (42, 3, 7), (-1, 2**40 + 3, -7), (2**63 + 11, 1, 2**62), (7, 3, 11)]
    idx = np.concatenate([np.arange(4096, dtype=np.uint64),
                          np.array([2**40 + k for k in range(16)] + [2**63 - 5, 2**64 - 1], dtype=np.uint64)])
    out = {"keys": np.array([[k & ((1 << 64) - 1) for k in key] for key in keys], dtype=np.uint64), "idx": idx}
    for i, (s, l, t) in enumerate(keys):
        out[f"draws{i}"] = rng.keyed_normal_array(s, l, t, idx)
    out["uniform"] = rng.keyed_uniform_array((3, 101, 0, 4), 4096)
    out["absorb"] = np.array([rng.absorb(*k) for k in keys], dtype=np.uint64)
    np.savez_compressed(OUT / "rng.npz", **out)


def gen_worked():
    x = Tensor.from_nested([[[1.0, 2.0]], [[1.0, 1.0]]])
    dy = Tensor.from_nested([[[3.0]], [[10.0]]])
    spec = MemSpec(4096, 8)
    out = {"x": x.array, "dy": dy.array}
    for tag, cfg in {"c10_sum": DPConfig(10.0, 0.0), "c10_mean": DPConfig(10.0, 0.0, "mean"),
                     "c1e9": DPConfig(1e9, 0.0), "c10_s07": DPConfig(10.0, 0.7, seed=11, layer_id=2, step=5)}.items():
        for k in KINDS:
            r = run_backward(WorkflowKind(k), x, dy, cfg, spec)
            out[f"{tag}_{k}_grad"] = r.grad_w.array
            out[f"{tag}_{k}_norms"] = r.per_sample_norms_sq
            out[f"{tag}_{k}_report"] = np.array(list(r.report.to_dict().values()), dtype=np.int64)
    np.savez_compressed(OUT / "worked.npz", **out)


def gen_config1():
    """BASELINE config 1: B=4, T=128, 256->256, cell_inputs (bench.py:234-241)."""
    layer = LayerSpec("l", 128, 256, 256)
    spec = MemSpec(228 * 1024, 2)
    x, dy = cell_inputs(DPConfig(clip_c=1.0, sigma=0.0, seed=0), 0, layer, 4)
    out = {"x_head": x.data[:64], "dy_head": dy.data[:64], "x_sum": np.array([x.data.sum()]),
           "dy_sum": np.array([dy.data.sum()])}
    base = run_backward(WorkflowKind.NON_DP, x, dy, None, spec)
    r0 = run_backward(WorkflowKind.FLASHDP, x, dy, DPConfig(1.0, 0.0), spec)
    med = float(np.median(np.sqrt(r0.per_sample_norms_sq)))
    out["median_norm"] = np.array([med])
    out["nondp_grad"] = base.grad_w.array
    cases = {
        "c1_s0": DPConfig(1.0, 0.0),
        "c1_s1": DPConfig(1.0, 1.0),
        "cmed_s0": DPConfig(med, 0.0),
        "c1e9_s0": DPConfig(1e9, 0.0),
        "c1_s1_mean_l3": DPConfig(1.0, 1.0, "mean", seed=0, layer_id=3, step=7),
    }
    for tag, cfg in cases.items():
        r = run_backward(WorkflowKind.FLASHDP, x, dy, cfg, spec)
        out[f"{tag}_grad"] = r.grad_w.array
        out[f"{tag}_norms"] = r.per_sample_norms_sq
        out[f"{tag}_cfg"] = np.array([cfg.clip_c, cfg.sigma, cfg.reduction == "mean", cfg.seed, cfg.layer_id,
                                      cfg.step], dtype=np.float64)
    np.savez_compressed(OUT / "config1.npz", **out)


def gen_report():
    """The reference's own scenario report (run_scenario + render_report, bench.py:274-335)
    for the config-1 cell, whole batch and 2x2 micro-batches."""
    from dpflows.bench import MicroBatchSpec, ScenarioConfig, render_report, run_scenario
    for tag, micro in (("report_c1", None), ("report_c1_micro", MicroBatchSpec(2, 2))):
        cfg = ScenarioConfig(layers=(LayerSpec("l", 128, 256, 256),), batch_sizes=(4,),
                             workflows=tuple(WorkflowKind(k) for k in KINDS), mem=MemSpec(228 * 1024, 2),
                             dp=DPConfig(clip_c=1.0, sigma=0.0, seed=0), micro_batch=micro)
        (OUT / f"{tag}.csv").write_text(render_report(run_scenario(cfg), "csv"))


def gen_random():
    """Small random instances with random valid plans (test_acceptance.py:38-58 style)."""
    r = random.Random(20817)
    out = {}
    n = 60
    for i in range(n):
        B, T = r.randint(1, 4), r.randint(1, 4)
        P, D = r.randint(1, 8), r.randint(1, 8)
        x = Tensor((B, T, P), [r.uniform(-2, 2) for _ in range(B * T * P)])
        dy = Tensor((B, T, D), [r.uniform(-2, 2) for _ in range(B * T * D)])
        b, t, d, p = r.randint(1, B), r.randint(1, T), r.randint(1, D), r.randint(1, P)
        plan = BlockPlan(b=b, t=t, d=d, p=p, n_b=math.ceil(B / b), n_t=math.ceil(T / t), n_d=math.ceil(D / d),
                         n_p=math.ceil(P / p))
        cfg = DPConfig(clip_c=r.choice([0.1, 1.0, 10.0, 1e9]), sigma=r.choice([0.0, 1.0]),
                       reduction=r.choice(["sum", "mean"]), seed=i, layer_id=i % 7, step=i % 13)
        res = backward_flashdp(x, dy, cfg, plan, MemSpec(footprint(b, t, d, p) * 8, 8))
        out[f"x{i}"] = x.array
        out[f"dy{i}"] = dy.array
        out[f"cfg{i}"] = np.array([cfg.clip_c, cfg.sigma, cfg.reduction == "mean", cfg.seed, cfg.layer_id, cfg.step])
        out[f"plan{i}"] = np.array([b, t, d, p, plan.n_b, plan.n_t, plan.n_d, plan.n_p])
        out[f"grad{i}"] = res.grad_w.array
        out[f"norms{i}"] = res.per_sample_norms_sq
        out[f"report{i}"] = np.array(list(res.report.to_dict().values()), dtype=np.int64)
    out["count"] = np.array([n])
    np.savez_compressed(OUT / "random.npz", **out)


def gen_ledgers():
    """Reference TrafficReport counters over a grid of shapes/specs for the closed forms."""
    r = random.Random(77)
    rows = []
    for _ in range(40):
        B, T, P, D = r.randint(1, 5), r.randint(1, 8), r.randint(1, 16), r.randint(1, 16)
        spec = MemSpec(r.choice([64, 256, 1024, 4096, 65536]), r.choice([2, 4, 8]))
        try:
            plan = plan_blocks(LayerDims(B, T, P, D), spec)
        except Exception:  # infeasible
            continue
        x = Tensor((B, T, P), [r.uniform(-1, 1) for _ in range(B * T * P)])
        dy = Tensor((B, T, D), [r.uniform(-1, 1) for _ in range(B * T * D)])
        cfg = DPConfig(1.0, 0.5, seed=1)
        for k in KINDS:
            rep = run_backward(WorkflowKind(k), x, dy, cfg, spec).report.to_dict()
            rows.append({"kind": k, "B": B, "T": T, "P": P, "D": D, "cap": spec.scratchpad_capacity_bytes,
                         "width": spec.dtype_width_bytes, "plan": plan.to_dict(), "report": rep})
    (OUT / "ledgers.json").write_text(json.dumps(rows, indent=0))


def gen_micro():
    """Micro-batch accumulation (bench.py:244-271 / dpcore.py:90-104)."""
    layer = LayerSpec("m", 8, 16, 12)
    dp = DPConfig(clip_c=0.5, sigma=0.7, reduction="mean", seed=5)
    x, dy = cell_inputs(dp, 1, layer, 6)
    cell_cfg = replace(dp, layer_id=1, step=0)
    parts = []
    for i in range(3):
        sl = np.s_[i * 2:(i + 1) * 2]
        xs = Tensor((2, 8, 16), x.array[sl].ravel())
        ys = Tensor((2, 8, 12), dy.array[sl].ravel())
        parts.append(run_backward(WorkflowKind.FLASHDP, xs, ys, replace(cell_cfg, sigma=0.0, reduction="sum"),
                                  MemSpec(4096, 8)).grad_w)
    grad = accumulate_micro_batches(parts, 6, cell_cfg)
    np.savez_compressed(OUT / "micro.npz", x=x.array, dy=dy.array, grad=grad.array,
                        cfg=np.array([0.5, 0.7, 1, 5, 1, 0]))


def gen_train():
    """The reference's train_demo (bench.py:409-458) with SGD and Adam: inputs,
    initial weights, targets and the per-step loss curves of explicit_dp and
    flashdp at three noise levels (acceptance criterion 9, test_acceptance.py:231-251)."""
    from dpflows.bench import TrainDemoConfig, train_demo

    out = {}
    for opt in ("sgd", "adam"):
        train = {"dims": {"B": 4, "T": 4, "P": 8, "D": 4}, "steps": 50, "workflows": ["explicit_dp", "flashdp"],
                 "sigmas": [0.1, 0.5, 1.0], "eta": 0.05}
        if opt == "adam":
            train.update({"optimizer": "adam", "eta": 0.02, "beta1": 0.9, "beta2": 0.999, "eps_adam": 1e-8})
        cfg = TrainDemoConfig.from_dict({"train": train, "mem": {"scratchpad_capacity_bytes": 8192},
                                         "dp": {"clip_c": 1.0, "sigma": 0.0, "seed": 2024}})
        res = train_demo(cfg)
        for sigma, per_wf in res.items():
            for wf, losses in per_wf.items():
                out[f"{opt}_{sigma}_{wf}"] = np.array(losses)
    d = (4, 4, 8, 4)
    out["x"] = rng.keyed_uniform_array((2024, 11), d[0] * d[1] * d[2]).reshape(d[0], d[1], d[2])
    out["w0"] = rng.keyed_uniform_array((2024, 12), d[3] * d[2], -0.5, 0.5).reshape(d[3], d[2])
    out["y"] = rng.keyed_uniform_array((2024, 13), d[0] * d[1] * d[3]).reshape(d[0], d[1], d[3])
    np.savez_compressed(OUT / "train.npz", **out)


def gen_dpcore():
    """dpcore.finalize_gradient / per_layer_process / accumulate_micro_batches on
    float64 inputs (dpcore.py:60-104): the drop-ins must match at 1e-12."""
    from dpflows.dpcore import finalize_gradient, per_layer_process

    out = {}
    g = rng.keyed_uniform_array((77, 1), 6 * 10).reshape(6, 10)
    out["g"] = g
    cfgs = {"sum_s0": DPConfig(0.8, 0.0, "sum", 3, 4, 5), "sum_s07": DPConfig(0.8, 0.7, "sum", 3, 4, 5),
            "mean_s13": DPConfig(2.5, 1.3, "mean", 9, 1, 2)}
    for tag, cfg in cfgs.items():
        out[f"cfg_{tag}"] = np.array([cfg.clip_c, cfg.sigma, cfg.reduction == "mean", cfg.seed, cfg.layer_id,
                                      cfg.step])
        out[f"finalize_{tag}"] = finalize_gradient(Tensor((6, 10), g.ravel()), 3, cfg).array
        ps = [Tensor((6, 10), (rng.keyed_uniform_array((77, 2, i), 60) * (i + 1)).ravel()) for i in range(4)]
        out["per_sample"] = np.stack([t.array for t in ps])
        out[f"per_layer_{tag}"] = per_layer_process(ps, cfg).array
        parts = [Tensor((6, 10), rng.keyed_uniform_array((77, 3, i), 60)) for i in range(3)]
        out["partials"] = np.stack([t.array for t in parts])
        out[f"micro_{tag}"] = accumulate_micro_batches(parts, 5, cfg).array
    np.savez_compressed(OUT / "dpcore.npz", **out)


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    gen_dpcore()
    gen_train()
    gen_rng()
    gen_worked()
    gen_config1()
    gen_report()
    gen_random()
    gen_ledgers()
    gen_micro()
    for p in sorted(OUT.iterdir()):
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    main()
