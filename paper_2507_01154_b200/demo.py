"""The reference's training demo on the GPU (bench.py:355-458).

``train_demo(cfg)`` trains one linear layer by least squares under each DP
workflow with identical data, noise keys and optimizer settings, returning
``{sigma: {workflow: [loss per step]}}`` (losses recorded before each update),
like ``dpflows.bench.train_demo``. Here every backward is a ``run_backward``
call on float64 CUDA tensors (the fp64 parity path of the C ABI, agreement
1e-12 with the reference) and every update an ``fdp_sgd_step`` /
``fdp_adam_step`` kernel, so the loss curves reproduce the reference's own
(tests/test_gpu_parity.py checks them against its golden curves).

``keyed_uniform`` restates the reference's input generator (rng.py:88-94:
splitmix64 absorb of the key parts, one mix per index, 53-bit uniforms).
"""

from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Iterable

import numpy as np
import torch

from .dpcore import DPConfig, OptimizerState, dp_adam_step_, dp_sgd_step_
from .errors import ConfigError, TrainingDivergedError
from .memmodel import MemSpec
from .tiling import LayerDims
from .workflows import WorkflowKind, run_backward

_M64 = (1 << 64) - 1
_GAMMA = 0x9E3779B97F4A7C15
_TWO_NEG53 = 2.0 ** -53


def _mix64(z: int) -> int:
    z &= _M64
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9 & _M64
    z = (z ^ (z >> 27)) * 0x94D049BB133111EB & _M64
    return z ^ (z >> 31)


def _absorb(*parts: int) -> int:  # rng.absorb (rng.py:42-47)
    h = _mix64(parts[0] & _M64) if parts else _mix64(0)
    for p in parts[1:]:
        h = _mix64((h + _GAMMA) ^ (p & _M64))
    return h


def _vmix(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def keyed_uniform(key_parts: Iterable[int], count: int, low: float = -1.0, high: float = 1.0) -> np.ndarray:
    """Deterministic U[low, high) draws (rng.keyed_uniform_array, rng.py:88-94)."""
    base = _absorb(*key_parts)
    idx = np.arange(count, dtype=np.uint64)
    h = _vmix(np.uint64((base + _GAMMA) & _M64) ^ idx)
    return low + (high - low) * ((h >> np.uint64(11)).astype(np.float64) * _TWO_NEG53)


@dataclass(frozen=True)
class TrainDemoConfig:
    """bench.TrainDemoConfig (bench.py:355-407): same fields and JSON schema."""
    dims: LayerDims
    steps: int
    workflows: tuple
    sigmas: tuple
    optimizer: str
    eta: float
    beta1: float
    beta2: float
    eps_adam: float
    mem: MemSpec
    dp: DPConfig

    @classmethod
    def from_dict(cls, doc: dict) -> "TrainDemoConfig":
        try:
            train, mem, dp = doc["train"], doc["mem"], doc["dp"]
            dims = LayerDims(**{k: int(train["dims"][k]) for k in ("B", "T", "P", "D")})
            workflows = tuple(WorkflowKind(w) for w in train["workflows"])
            sigmas = tuple(float(s) for s in train["sigmas"])
            steps, eta = int(train["steps"]), float(train["eta"])
        except (KeyError, TypeError, ValueError) as e:
            raise ConfigError(f"bad train-demo config: {e!r}") from None
        if sum(1 for w in workflows if w != WorkflowKind.NON_DP) < 2:
            raise ConfigError("$.train.workflows must name at least two DP workflows")
        if not sigmas:
            raise ConfigError("$.train.sigmas must be a non-empty list")
        optimizer = train.get("optimizer", "sgd")
        if optimizer not in ("sgd", "adam"):
            raise ConfigError(f"$.train.optimizer must be 'sgd' or 'adam', got {optimizer!r}")
        return cls(dims=dims, steps=steps, workflows=workflows, sigmas=sigmas, optimizer=optimizer, eta=eta,
                   beta1=float(train.get("beta1", 0.9)), beta2=float(train.get("beta2", 0.999)),
                   eps_adam=float(train.get("eps_adam", 1e-8)),
                   mem=MemSpec(int(mem["scratchpad_capacity_bytes"]), int(mem.get("dtype_width_bytes", 8))),
                   dp=DPConfig(float(dp["clip_c"]), float(dp.get("sigma", 0.0)), dp.get("reduction", "sum"),
                               int(dp.get("seed", 0)), int(dp.get("layer_id", 0)), int(dp.get("step", 0))))


def train_demo(cfg: TrainDemoConfig, device="cuda") -> dict:
    """bench.train_demo (bench.py:409-458) with the GPU backward and optimizer."""
    d = cfg.dims
    dev = torch.device(device)
    x = torch.tensor(keyed_uniform((cfg.dp.seed, 11), d.B * d.T * d.P).reshape(d.B, d.T, d.P), device=dev)
    w0 = torch.tensor(keyed_uniform((cfg.dp.seed, 12), d.D * d.P, -0.5, 0.5).reshape(d.D, d.P), device=dev)
    y_target = torch.tensor(keyed_uniform((cfg.dp.seed, 13), d.B * d.T * d.D).reshape(d.B, d.T, d.D), device=dev)
    denom = d.B * d.T * d.D
    out: dict = {}
    for sigma in cfg.sigmas:
        per_wf: dict = {}
        for kind in cfg.workflows:
            theta = w0.clone()
            state = None
            if cfg.optimizer == "adam":
                state = OptimizerState.fresh(theta, cfg.eta, beta1=cfg.beta1, beta2=cfg.beta2, eps_adam=cfg.eps_adam)
            losses = []
            for step in range(cfg.steps):
                th = state.theta if state is not None else theta
                resid = torch.einsum("btp,dp->btd", x, th) - y_target
                loss = float((resid * resid).sum() / denom)
                if not np.isfinite(loss):
                    raise TrainingDivergedError(step, loss)
                losses.append(loss)
                dy = ((2.0 / denom) * resid).contiguous()
                step_cfg = replace(cfg.dp, sigma=sigma, layer_id=0, step=step)
                grad = run_backward(kind, x, dy, step_cfg, cfg.mem, noise_impl="keyed_f64").grad_w
                if state is not None:
                    state = dp_adam_step_(state, grad.contiguous())
                else:
                    dp_sgd_step_(theta, grad.contiguous(), cfg.eta)
            per_wf[kind.value] = losses
        out[sigma] = per_wf
    return out
