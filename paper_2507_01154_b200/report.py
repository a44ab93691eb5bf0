"""Comparison rows in the reference's report schema.

The reference tabulates one ``ComparisonRow`` per (workflow, layer, batch) cell
from its simulator counters (``bench.py:206-231`` schema, ``run_scenario``
``bench.py:274-315``, ``render_report`` ``bench.py:325-335``). Here the same
columns come from the closed-form ledger of the path actually taken
(``memmodel.ledger``, pinned to the reference simulator in the host tests), and
the GPU run adds what the simulator could only model: the measured launch time
and, when an ncu capture is supplied, the measured DRAM bytes. A CSV written by
``render_report(rows)`` is column-for-column the reference's CSV; the measured
columns are appended only with ``measured=True``.
"""

from __future__ import annotations

import csv
import io
import json
from dataclasses import dataclass, fields
from pathlib import Path
from typing import Mapping, Optional, Sequence

import torch

from .dpcore import DPConfig, accumulate_micro_batches
from .errors import UsageError
from .workflows import BackwardResult, WorkflowKind, backward_nondp, run_backward

REPORT_FIELDNAMES = [
    "workflow", "layer", "B",
    "bytes_loaded", "bytes_stored", "per_sample_grad_bytes_stored",
    "flops", "redundant_flops", "kernel_launches", "barriers",
    "peak_scratch_bytes", "relative_traffic", "grad_checksum",
]
MEASURED_FIELDNAMES = ["gpu_ms", "measured_dram_bytes"]


@dataclass(frozen=True)
class ComparisonRow:
    workflow: str
    layer: str
    B: int
    bytes_loaded: int
    bytes_stored: int
    per_sample_grad_bytes_stored: int
    flops: int
    redundant_flops: int
    kernel_launches: int
    barriers: int
    peak_scratch_bytes: int
    relative_traffic: float
    grad_checksum: float
    gpu_ms: Optional[float] = None
    measured_dram_bytes: Optional[int] = None

    def to_dict(self, measured: bool = False) -> dict:
        names = REPORT_FIELDNAMES + (MEASURED_FIELDNAMES if measured else [])
        return {name: getattr(self, name) for name in names}


def _timed(fn, reps: int) -> tuple[BackwardResult, float]:
    res = fn()  # warm-up (workspace allocation, plan)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        res = fn()
    e1.record()
    torch.cuda.synchronize()
    return res, e0.elapsed_time(e1) / reps


def _run_cell(kind: WorkflowKind, x, dy, cfg: DPConfig, micro_batch: Optional[tuple[int, int]], opts: dict):
    """One cell, optionally as micro-batches with noise and `mean` applied once
    (reference ``bench._run_cell`` ``bench.py:244-271``)."""
    if micro_batch is None:
        if kind == WorkflowKind.NON_DP:
            return backward_nondp(x, dy, **opts)
        return run_backward(kind, x, dy, cfg, **opts)
    size, steps = micro_batch
    if size * steps != x.shape[0]:
        raise UsageError(f"micro_batch {size}x{steps} does not cover B={x.shape[0]}")
    from .memmodel import merge_reports
    parts, reports, refs, norms = [], [], [], []
    micro_cfg = DPConfig(clip_c=cfg.clip_c, sigma=0.0, reduction="sum", seed=cfg.seed, layer_id=cfg.layer_id,
                         step=cfg.step)
    for i in range(steps):
        xs, dys = x[i * size:(i + 1) * size], dy[i * size:(i + 1) * size]
        res = backward_nondp(xs, dys, **opts) if kind == WorkflowKind.NON_DP else run_backward(kind, xs, dys, micro_cfg,
                                                                                               **opts)
        parts.append(res.grad_w)
        reports.append(res.report)
        refs.append(res.reference_report)
        norms.append(res.per_sample_norms_sq)
    report, ref = merge_reports(reports), merge_reports(refs)
    if kind == WorkflowKind.NON_DP:
        return BackwardResult(sum(parts[1:], parts[0].clone()), report, torch.zeros(0, device=x.device), ref)
    grad = accumulate_micro_batches(parts, x.shape[0], cfg, noise_impl=opts.get("noise_impl", "keyed_f32"))
    return BackwardResult(grad, report, torch.cat(norms), ref)


def compare_workflows(x: torch.Tensor, dy: torch.Tensor, cfg: DPConfig, *, layer: str = "layer",
                      workflows: Sequence[WorkflowKind] = tuple(WorkflowKind), micro_batch: Optional[tuple[int, int]] = None,
                      time_reps: int = 0, dram_bytes: Optional[Mapping[str, int]] = None,
                      **opts) -> list[ComparisonRow]:
    """All requested workflows on one (layer, batch) cell, the non-DP cell always
    computed as the traffic baseline (reference ``run_scenario`` ``bench.py:283-290``).

    ``time_reps > 0`` times each cell with CUDA events (mean of `time_reps`
    launches after one warm-up); ``dram_bytes`` maps workflow names to measured
    ncu ``dram__bytes_read.sum + dram__bytes_write.sum``.
    """
    results, times = {}, {}
    kinds = [WorkflowKind.NON_DP] + [k for k in workflows if k != WorkflowKind.NON_DP]
    for kind in kinds:
        fn = lambda k=kind: _run_cell(k, x, dy, cfg, micro_batch, opts)  # noqa: E731
        if time_reps > 0:
            results[kind], times[kind] = _timed(fn, time_reps)
        else:
            results[kind] = fn()
    # the rows are the reference's schema and ledgers (what dpflows would print);
    # the executed-path ledgers stay on each BackwardResult.report
    base = results[WorkflowKind.NON_DP].reference_report
    base_traffic = base.bytes_loaded + base.bytes_stored
    rows = []
    for kind in workflows:
        res = results[kind]
        rep = res.reference_report
        rows.append(ComparisonRow(
            workflow=kind.value, layer=layer, B=int(x.shape[0]),
            bytes_loaded=rep.bytes_loaded, bytes_stored=rep.bytes_stored,
            per_sample_grad_bytes_stored=rep.per_sample_grad_bytes_stored,
            flops=rep.flops, redundant_flops=rep.redundant_flops, kernel_launches=rep.kernel_launches,
            barriers=rep.barriers, peak_scratch_bytes=rep.peak_scratch_bytes,
            relative_traffic=(rep.bytes_loaded + rep.bytes_stored) / base_traffic,
            grad_checksum=float(res.grad_w.double().sum()),
            gpu_ms=times.get(kind),
            measured_dram_bytes=None if dram_bytes is None else dram_bytes.get(kind.value),
        ))
    return rows


def _fmt(value) -> str:
    if isinstance(value, float):
        return repr(value)
    return "" if value is None else str(value)


def render_report(rows: Sequence[ComparisonRow], fmt: str = "csv", *, measured: bool = False) -> str:
    """CSV or JSON text; the reference's columns first (``bench.py:325-335``)."""
    if not rows:
        raise UsageError("no rows to emit")
    names = REPORT_FIELDNAMES + (MEASURED_FIELDNAMES if measured else [])
    if fmt == "csv":
        buf = io.StringIO()
        writer = csv.writer(buf, lineterminator="\n")
        writer.writerow(names)
        for row in rows:
            writer.writerow([_fmt(getattr(row, n)) for n in names])
        return buf.getvalue()
    if fmt == "json":
        return json.dumps([row.to_dict(measured) for row in rows], indent=2) + "\n"
    raise UsageError(f"format must be 'csv' or 'json', got {fmt!r}")


def emit_report(rows: Sequence[ComparisonRow], fmt: str = "csv", path=None, stream=None, *,
                measured: bool = False) -> str:
    text = render_report(rows, fmt, measured=measured)
    if path is not None:
        Path(path).write_text(text, encoding="utf-8")
    if stream is not None:
        stream.write(text)
    return text


assert [f.name for f in fields(ComparisonRow)][:len(REPORT_FIELDNAMES)] == REPORT_FIELDNAMES
