"""Memory-spec and traffic-ledger types of the reference API.

``MemSpec``/``TrafficReport``/``merge_reports`` keep the reference's fields
and serialisation order (memmodel.py:30-79). On B200 nothing is simulated: the
kernels run on the device, and the report attached to a result is the
reference's exact ledger for the workflow evaluated in closed form
(``ledger``), in elements x ``dtype_width_bytes``. The closed forms are pinned
against the reference simulator by tests/test_ledger.py; measured DRAM bytes
(ncu) are reported next to them by bench.py.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable

from .errors import UsageError

_ALLOWED_WIDTHS = (2, 4, 8)


@dataclass(frozen=True)
class MemSpec:
    scratchpad_capacity_bytes: int
    dtype_width_bytes: int = 8

    def __post_init__(self):
        if self.dtype_width_bytes not in _ALLOWED_WIDTHS:
            raise UsageError(f"dtype_width_bytes must be one of {_ALLOWED_WIDTHS}, got {self.dtype_width_bytes}")
        if self.scratchpad_capacity_bytes < 1:
            raise UsageError(f"scratchpad_capacity_bytes must be positive, got {self.scratchpad_capacity_bytes}")


# Per-SM shared memory of a B200 (227 KB usable per CTA + 1 KB reserved) with
# bf16 elements: the default spec when a caller passes none.
B200_SPEC = MemSpec(228 * 1024, 2)


@dataclass
class TrafficReport:
    bytes_loaded: int = 0
    bytes_stored: int = 0
    flops: int = 0
    redundant_flops: int = 0
    barriers: int = 0
    kernel_launches: int = 0
    peak_scratch_bytes: int = 0
    per_sample_grad_bytes_stored: int = 0

    def to_dict(self) -> dict:
        return {
            "bytes_loaded": self.bytes_loaded,
            "bytes_stored": self.bytes_stored,
            "flops": self.flops,
            "redundant_flops": self.redundant_flops,
            "barriers": self.barriers,
            "kernel_launches": self.kernel_launches,
            "peak_scratch_bytes": self.peak_scratch_bytes,
            "per_sample_grad_bytes_stored": self.per_sample_grad_bytes_stored,
        }


def merge_reports(reports: Iterable[TrafficReport]) -> TrafficReport:
    """Sum counters; the peak is a max (memmodel.py:67-79)."""
    out = TrafficReport()
    for r in reports:
        out.bytes_loaded += r.bytes_loaded
        out.bytes_stored += r.bytes_stored
        out.flops += r.flops
        out.redundant_flops += r.redundant_flops
        out.barriers += r.barriers
        out.kernel_launches += r.kernel_launches
        out.peak_scratch_bytes = max(out.peak_scratch_bytes, r.peak_scratch_bytes)
        out.per_sample_grad_bytes_stored += r.per_sample_grad_bytes_stored
    return out


def ledger(kind: str, B: int, T: int, P: int, D: int, width: int, plan=None, dp: bool = True) -> TrafficReport:
    """Closed-form traffic ledger of one workflow (elements x width).

    Derived from the dataflow of workflows.py (loads of X/dY once per fused
    pass, norm/accumulator round trips, per-sample G materialisation); the
    formulas are cross-checked against the reference simulator in the tests.
    ``plan`` (a BlockPlan) sets the flashdp norm reloads per (p,d) block and
    accumulator spills per batch chunk, and every kind's peak scratch: the
    simulator's high-water mark is one input tile pair b·t·(p+d), plus the
    per-sample tile b·d·p where one is materialised (explicit, implicit,
    flashdp) and flashdp's b norm partials, or the d·p output tile when that is
    larger (pinned on all golden ledgers). Without a plan, peak scratch is 0.
    ``dp`` False drops the finalize flops (non-DP has no emit step).
    """
    inputs = B * T * (P + D)
    g = B * D * P
    dp_elems = D * P
    grad_flops = 2 * B * T * D * P
    tile_in = tile_g = tile_out = 0
    if plan is not None:
        tile_in, tile_g, tile_out = plan.b * plan.t * (plan.p + plan.d), plan.b * plan.d * plan.p, plan.d * plan.p
    if kind == "non_dp":
        return TrafficReport(bytes_loaded=inputs * width, bytes_stored=dp_elems * width, flops=grad_flops,
                             kernel_launches=1, peak_scratch_bytes=max(tile_in, tile_out) * width)
    emit = dp_elems
    if kind == "explicit_dp":
        return TrafficReport(bytes_loaded=(inputs + 3 * g + B) * width,
                             bytes_stored=(2 * g + B + dp_elems) * width,
                             flops=grad_flops + 4 * g + emit, kernel_launches=4,
                             per_sample_grad_bytes_stored=2 * g * width,
                             peak_scratch_bytes=max(tile_in + tile_g, tile_out) * width)
    if kind == "implicit_dp":
        return TrafficReport(bytes_loaded=(2 * inputs + B) * width, bytes_stored=(B + dp_elems) * width,
                             flops=2 * grad_flops + 4 * g + emit, redundant_flops=grad_flops,
                             kernel_launches=2, peak_scratch_bytes=max(tile_in + tile_g, tile_out) * width)
    if kind == "flashdp":
        if plan is None:
            raise UsageError("flashdp ledger needs the block plan")
        blocks = plan.n_p * plan.n_d
        return TrafficReport(bytes_loaded=(inputs + blocks * B + dp_elems) * width,
                             bytes_stored=(blocks * B + plan.n_b * dp_elems + dp_elems) * width,
                             flops=grad_flops + 4 * g + emit, barriers=plan.n_b + 1,
                             kernel_launches=plan.n_b,
                             peak_scratch_bytes=(plan.b * plan.t * (plan.p + plan.d) + plan.b * plan.d * plan.p
                                                 + plan.b) * width)
    raise UsageError(f"unknown workflow kind {kind!r}")


def device_ledger(kind: str, path: str, norm_phase: str, launches: int, B: int, T: int, P: int, D: int,
                  in_width: int, out_width: int, *, n_tiles: int = 1, groups: int = 1, accumulate: bool = False,
                  add_noise: bool = True, deferred: bool = False) -> TrafficReport:
    """Ledger of the path the device actually executed (the report
    describes the path taken), in BYTES of the real element types: X / dY of
    `in_width` bytes, grad_w and norms of `out_width` bytes.

      fused      one launch: X, dY read once; per (sample, CTA tile) one norm
                 partial (8-byte tagged slot) published and polled (barriers: one
                 block-wise all-reduce per sample); grad_w written once, plus one
                 pre-fill write and one reduce-add read+write per extra sample group
      two_phase  ghost:     X, dY read by the Gram norm pass AND the reweight pass
                            (inputs twice), Gram flops T^2 (P+D) per sample redundant
                 recompute: inputs twice, the per-sample contraction computed twice
                 single:    B == 1, the GEMM writes G, one pass reads it and writes
                            c * G + noise (grad_w written twice, read once);
                            deferred (fdp_dw_deferred): no pass, G written once and
                            the factor left to the consumer
      simt       partial-norm pass + weighted pass: inputs twice, contraction twice
      explicit   G and G' materialised (2 B D P out_width bytes), 5 launches
      non_dp     inputs once, grad_w once
    Peak scratch is the device workspace's per-sample state (norm slots), not a
    simulated scratchpad."""
    inputs = B * T * (P + D) * in_width
    gw = D * P * out_width
    grad_flops = 2 * B * T * D * P
    clip_flops = 4 * B * D * P
    emit = D * P if add_noise else 0
    acc_read = gw if accumulate else 0
    if kind == "non_dp":
        return TrafficReport(bytes_loaded=inputs + acc_read, bytes_stored=gw, flops=grad_flops,
                             kernel_launches=launches)
    if kind == "explicit_dp":
        g = B * D * P * out_width
        return TrafficReport(bytes_loaded=inputs + 3 * g + B * out_width + acc_read,
                             bytes_stored=2 * g + B * out_width + gw, flops=grad_flops + clip_flops + emit,
                             kernel_launches=launches, barriers=launches - 1, per_sample_grad_bytes_stored=2 * g,
                             peak_scratch_bytes=2 * g)
    norm_slots = B * n_tiles * 8
    if kind == "flashdp" and path == "fused":
        extra = (groups - 1) * gw  # sample groups: rows pre-filled once, every group reduce-adds onto them
        return TrafficReport(bytes_loaded=inputs + norm_slots + extra + acc_read,
                             bytes_stored=gw + norm_slots + extra + B * out_width,
                             flops=grad_flops + clip_flops + emit, barriers=B, kernel_launches=launches,
                             peak_scratch_bytes=norm_slots)
    if kind == "flashdp" and path == "two_phase" and norm_phase == "single" and deferred:
        return TrafficReport(bytes_loaded=inputs + n_tiles * 4, bytes_stored=gw + n_tiles * 4 + B * out_width + 4,
                             flops=grad_flops + 2 * D * P, barriers=launches - 1, kernel_launches=launches,
                             peak_scratch_bytes=n_tiles * 4)
    if kind == "flashdp" and path == "two_phase" and norm_phase == "single":
        return TrafficReport(bytes_loaded=inputs + gw + acc_read, bytes_stored=2 * gw + B * out_width,
                             flops=grad_flops + 2 * D * P + emit, barriers=launches - 1, kernel_launches=launches,
                             peak_scratch_bytes=n_tiles * 4)
    if kind == "flashdp" and path == "two_phase" and norm_phase == "spill":
        g = B * D * P * out_width  # per-sample gradients written once, read once by the combine pass
        return TrafficReport(bytes_loaded=inputs + g + acc_read, bytes_stored=g + gw + B * out_width,
                             flops=grad_flops + 2 * B * D * P + emit, barriers=launches - 1,
                             kernel_launches=launches, per_sample_grad_bytes_stored=g, peak_scratch_bytes=g)
    if kind == "flashdp" and path == "two_phase" and norm_phase == "ghost":
        ghost = B * T * T * (P + D)
        return TrafficReport(bytes_loaded=2 * inputs + acc_read, bytes_stored=gw + B * out_width,
                             flops=grad_flops + ghost + B * D * P + emit, redundant_flops=ghost,
                             barriers=launches - 1, kernel_launches=launches, peak_scratch_bytes=norm_slots)
    # recompute norm phase (flashdp two-phase / implicit) and the generic SIMT path
    return TrafficReport(bytes_loaded=2 * inputs + acc_read, bytes_stored=gw + B * out_width,
                         flops=2 * grad_flops + clip_flops + emit, redundant_flops=grad_flops,
                         barriers=launches - 1, kernel_launches=launches, peak_scratch_bytes=norm_slots)
