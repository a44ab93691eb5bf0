"""Report schema: rows in the reference's ComparisonRow/CSV
format (bench.py:206-231, 274-335), pinned to CSVs the reference itself wrote
for the config-1 cell (tools/gen_golden.py: gen_report)."""

import csv
import io
from pathlib import Path

import numpy as np
import pytest

import paper_2507_01154_b200 as fdp
from paper_2507_01154_b200 import report as R

GOLDEN = Path(__file__).parent / "golden"
KINDS = ["non_dp", "explicit_dp", "implicit_dp", "flashdp"]
SPEC = fdp.MemSpec(228 * 1024, 2)
B, T, P, D = 4, 128, 256, 256


def golden_rows(tag):
    return list(csv.DictReader(io.StringIO((GOLDEN / f"{tag}.csv").read_text())))


def ledger_cell(kind, micro):
    """Ledger of one cell exactly as the GPU path reports it (plan from the spec)."""
    sizes = [B] if micro is None else [micro[0]] * micro[1]
    reps = []
    for b in sizes:
        plan = fdp.plan_blocks(fdp.LayerDims(B=b, T=T, P=P, D=D), SPEC)
        reps.append(fdp.ledger(kind, b, T, P, D, SPEC.dtype_width_bytes, plan=plan))
    return fdp.merge_reports(reps)


@pytest.mark.parametrize("tag,micro", [("report_c1", None), ("report_c1_micro", (2, 2))])
def test_ledger_rows_render_the_reference_csv(tag, micro):
    """Our ledger + the reference's checksums, rendered by render_report, is the
    reference's CSV byte for byte (schema, column order, float formatting)."""
    gold = golden_rows(tag)
    base = ledger_cell("non_dp", micro)
    rows = []
    for g in gold:
        rep = ledger_cell(g["workflow"], micro)
        rows.append(R.ComparisonRow(
            workflow=g["workflow"], layer="l", B=B, bytes_loaded=rep.bytes_loaded, bytes_stored=rep.bytes_stored,
            per_sample_grad_bytes_stored=rep.per_sample_grad_bytes_stored, flops=rep.flops,
            redundant_flops=rep.redundant_flops, kernel_launches=rep.kernel_launches, barriers=rep.barriers,
            peak_scratch_bytes=rep.peak_scratch_bytes,
            relative_traffic=(rep.bytes_loaded + rep.bytes_stored) / (base.bytes_loaded + base.bytes_stored),
            grad_checksum=float(g["grad_checksum"])))
    assert R.render_report(rows, "csv") == (GOLDEN / f"{tag}.csv").read_text()
    js = R.render_report(rows, "json", measured=True)
    assert '"gpu_ms": null' in js and '"measured_dram_bytes": null' in js
    with pytest.raises(fdp.UsageError):
        R.render_report(rows, "xml")
    with pytest.raises(fdp.UsageError):
        R.render_report([], "csv")


@pytest.mark.gpu
@pytest.mark.parametrize("tag,micro", [("report_c1", None), ("report_c1_micro", (2, 2))])
def test_gpu_comparison_matches_reference_report(tag, micro):
    """compare_workflows on the GPU (fp32 inputs): integer columns and relative
    traffic equal the reference's, grad checksums within fp32 error."""
    import torch
    from oracle import dp_oracle as O
    x64, dy64 = O.cell_inputs(0, 0, B, T, P, D)
    x = torch.tensor(x64, dtype=torch.float32).cuda()
    dy = torch.tensor(dy64, dtype=torch.float32).cuda()
    cfg = fdp.DPConfig(clip_c=1.0, sigma=0.0, seed=0, layer_id=0, step=0)
    rows = R.compare_workflows(x, dy, cfg, layer="l", workflows=[fdp.WorkflowKind(k) for k in KINDS],
                               micro_batch=micro, time_reps=2, spec=SPEC)
    gold = golden_rows(tag)
    scale = float(np.abs(np.load(GOLDEN / "config1.npz")["nondp_grad"]).sum())
    for row, g in zip(rows, gold):
        assert row.workflow == g["workflow"]
        for k in R.REPORT_FIELDNAMES[2:11]:
            assert getattr(row, k) == int(g[k]), (row.workflow, k)
        assert row.relative_traffic == float(g["relative_traffic"])
        assert abs(row.grad_checksum - float(g["grad_checksum"])) <= 1e-6 * scale, row.workflow
        assert row.gpu_ms is not None and row.gpu_ms > 0
    text = R.render_report(rows, "csv", measured=True)
    assert text.splitlines()[0].endswith("gpu_ms,measured_dram_bytes")
