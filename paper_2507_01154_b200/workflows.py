"""Drop-in replacement of the reference workflow API (workflows.py:33-440).

``run_backward(kind, x, dy, cfg, spec, plan=None, *, sim=None)`` and
``backward_{flashdp,explicit,implicit,nondp}`` keep the reference names,
argument meaning, result type and exceptions. The body of every workflow is
one C-ABI call (include/fdp.h) that launches sm_100a kernels:

  flashdp      fused tcgen05 kernel (per-sample tiles in TMEM, in-kernel norm
               all-reduce + grid barrier, clip, batch sum, noise), or the
               two-phase tcgen05 path for layers too large for on-chip tiles
  implicit_dp  norm pass + recompute pass (GhostClip-style, workflows.py:246-324)
  explicit_dp  G materialised in HBM, then norms / clip / sum+noise stages
               (Opacus-style, workflows.py:156-240)
  non_dp       plain sum_b dY_b^T X_b (workflows.py:121-150)

Inputs may be torch tensors on the GPU (the hot path: no copies), or host
objects (reference ``Tensor``, numpy, CPU torch) which are copied to the GPU
and whose results come back as reference-style host objects.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass
from enum import Enum
from typing import Optional

import numpy as np
import torch

from . import _lib
from .dpcore import DPConfig
from .errors import OrderingFault, ShapeError, UsageError
from .memmodel import B200_SPEC, MemSpec, TrafficReport, device_ledger, ledger
from .tensor import Tensor
from .tiling import BlockPlan, LayerDims, check_plan, plan_blocks


class WorkflowKind(Enum):
    NON_DP = "non_dp"
    EXPLICIT_DP = "explicit_dp"
    IMPLICIT_DP = "implicit_dp"
    FLASHDP = "flashdp"


@dataclass
class BackwardResult:
    grad_w: object             # torch (D,P) fp32 on the GPU, or Tensor for host callers
    report: TrafficReport      # ledger of the path the device executed (memmodel.device_ledger)
    per_sample_norms_sq: object  # torch (B,) fp32, or np.ndarray for host callers
    # the reference simulator's ledger of the same call and block plan
    # (memmodel.ledger, workflows.py:340-440 semantics; what dpflows itself returns)
    reference_report: Optional[TrafficReport] = None


# ---------------------------------------------------------------- workspaces

class _WorkspacePool:
    """One zero-initialised device workspace per (device, stream); grows on demand.

    The kernels leave their counters zeroed, so a workspace is reused without a
    memset; distinct streams get distinct workspaces (include/fdp.h)."""

    def __init__(self):
        self._lock = threading.Lock()
        self._bufs: dict = {}

    def get(self, nbytes: int, device: torch.device, stream: torch.cuda.Stream, slot=None) -> torch.Tensor:
        # `slot`: a separate buffer for callers that need several workspaces at once
        # (each buffer is always used from its start, so the C library's per-address
        # layout signature keeps its counters valid)
        key = (device.index, stream.cuda_stream, slot)
        with self._lock:
            buf = self._bufs.get(key)
            if buf is None or buf.numel() < nbytes:
                buf = torch.zeros(max(nbytes, 4096), dtype=torch.uint8, device=device)
                self._bufs[key] = buf
            return buf


_POOL = _WorkspacePool()


def _dims(x, dy) -> LayerDims:
    xs, ys = tuple(x.shape), tuple(dy.shape)
    if len(xs) != 3 or len(ys) != 3:
        raise ShapeError(f"expected (B,T,P) and (B,T,D), got {xs} and {ys}")
    if xs[0] != ys[0] or xs[1] != ys[1]:
        raise ShapeError(f"batch/time extents differ: {xs} vs {ys}")
    return LayerDims(B=xs[0], T=xs[1], P=xs[2], D=ys[2])


def _to_device(t, dtype, device) -> tuple[torch.Tensor, bool]:
    """-> (contiguous device tensor, came_from_host)."""
    if isinstance(t, torch.Tensor) and t.is_cuda:
        if dtype is not None and t.dtype != dtype:
            t = t.to(dtype)
        return t.contiguous(), False
    # host inputs keep their precision: float64 (the reference's Tensor / numpy
    # arrays) takes the fp64 parity path, bf16 / fp32 the fast paths
    keep = (torch.bfloat16, torch.float32, torch.float64)
    if isinstance(t, torch.Tensor):  # host torch tensor: one H2D copy
        target = dtype if dtype is not None else (t.dtype if t.dtype in keep else torch.float32)
        return t.detach().to(device=device, dtype=target, non_blocking=t.is_pinned()).contiguous(), True
    arr = t.array if isinstance(t, Tensor) else np.asarray(t)
    host = torch.from_numpy(np.ascontiguousarray(arr))
    target = dtype if dtype is not None else (host.dtype if host.dtype in keep else torch.float32)
    return host.to(device=device, dtype=target, non_blocking=False).contiguous(), True


def _input_dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return _lib.DTYPE_BF16
    if t.dtype == torch.float32:
        return _lib.DTYPE_F32
    if t.dtype == torch.float64:
        return _lib.DTYPE_F64
    raise UsageError(f"inputs must be bfloat16, float32 or float64 on the device, got {t.dtype}")


def _run(kind: WorkflowKind, x, dy, cfg: Optional[DPConfig], spec: Optional[MemSpec], plan: Optional[BlockPlan], *,
         path: str = "auto", noise_impl: str = "keyed_f32", dtype: Optional[torch.dtype] = None,
         grad_out: Optional[torch.Tensor] = None, norms_out: Optional[torch.Tensor] = None,
         accumulate: bool = False, add_noise: bool = True, rank: int = 0, world: int = 1, mean_batch: int = 0,
         skip_barrier: bool = False, short_timeout: bool = False, workspace: Optional[torch.Tensor] = None,
         device_step: Optional[torch.Tensor] = None, norm_phase: str = "auto",
         deterministic: bool = False, chain: Optional[DeferredChain] = None,
         grad_scale_out: Optional[torch.Tensor] = None) -> BackwardResult:
    """``grad_scale_out`` (a (1,) fp32 device tensor, FLASHDP only): fdp_dw_deferred --
    on the single-sample path without noise the result holds the UNCLIPPED gradient
    and grad_scale_out[0] its clip factor / mean divisor (else 1); the consumer forms
    the product (include/fdp.h)."""
    dims = _dims(x, dy)
    if kind != WorkflowKind.NON_DP and cfg is None:
        raise UsageError("DP workflows need a DPConfig")
    device = x.device if isinstance(x, torch.Tensor) and x.is_cuda else torch.device("cuda", torch.cuda.current_device())
    xd, host_x = _to_device(x, dtype, device)
    yd, host_y = _to_device(dy, xd.dtype, device)
    host = host_x or host_y
    host_torch = host and isinstance(x, torch.Tensor)
    if xd.dtype != yd.dtype:
        raise UsageError(f"x and dy must share a dtype, got {xd.dtype} and {yd.dtype}")
    in_dtype = _input_dtype_code(xd)

    c = cfg or DPConfig(clip_c=1.0, sigma=0.0)
    flags = ((_lib.FLAG_SKIP_BARRIER if skip_barrier else 0) | (_lib.FLAG_TIMEOUT_SHORT if short_timeout else 0)
             | (_lib.FLAG_DETERMINISTIC if deterministic else 0))
    desc = _lib.make_desc(B=dims.B, T=dims.T, P=dims.P, D=dims.D, in_dtype=in_dtype, reduction=c.reduction,
                          clip_c=c.clip_c, sigma=c.sigma, seed=c.seed, layer_id=c.layer_id, step=c.step, rank=rank,
                          world=world, mean_batch=mean_batch, accumulate=accumulate, add_noise=add_noise,
                          noise_impl=noise_impl, path=path, flags=flags, norm_phase=norm_phase,
                          device_step=_step_ptr(device_step))
    lib = _lib.load()
    k = _lib.KIND[kind.value]
    ws_bytes = ctypes.c_size_t()
    _lib.check(lib.fdp_workspace_bytes(ctypes.byref(desc), k, ctypes.byref(ws_bytes)))

    out_dtype = torch.float64 if in_dtype == _lib.DTYPE_F64 else torch.float32  # fp64 path: fp64 outputs
    if grad_out is None:
        grad = (torch.zeros if accumulate else torch.empty)((dims.D, dims.P), dtype=out_dtype, device=device)
    else:
        _check_out(grad_out, (dims.D, dims.P), out_dtype, device, "grad_out")
        grad = grad_out
    if kind == WorkflowKind.NON_DP:
        norms = None
    elif norms_out is not None:
        _check_out(norms_out, (dims.B,), out_dtype, device, "norms_out")
        norms = norms_out
    else:
        norms = torch.empty(dims.B, dtype=out_dtype, device=device)

    stream = torch.cuda.current_stream(device)
    if workspace is not None:
        if workspace.numel() * workspace.element_size() < ws_bytes.value:
            raise fdp_capacity(ws_bytes.value, workspace.numel() * workspace.element_size())
        ws = workspace.view(torch.uint8) if workspace.dtype != torch.uint8 else workspace
    else:
        ws = _POOL.get(ws_bytes.value, device, stream)
    if grad_scale_out is not None:
        if kind != WorkflowKind.FLASHDP or chain is not None or host:
            raise UsageError("grad_scale_out needs kind FLASHDP, device inputs and no chain")
        _check_out(grad_scale_out, (1,), torch.float32, device, "grad_scale_out")
        _lib.check(lib.fdp_dw_deferred(ctypes.byref(desc), xd.data_ptr(), yd.data_ptr(), grad.data_ptr(),
                                       norms.data_ptr(), grad_scale_out.data_ptr(), ws.data_ptr(), ws.numel(),
                                       stream.cuda_stream))
    elif chain is not None:
        if host:
            raise UsageError("chain= needs device inputs (the pending finalize writes device memory later)")
        rc = lib.fdp_backward_chained(k, ctypes.byref(desc), xd.data_ptr(), yd.data_ptr(), grad.data_ptr(),
                                      norms.data_ptr() if norms is not None else None, ws.data_ptr(), ws.numel(),
                                      chain.handle, stream.cuda_stream)
        _lib.check(rc)
        if chain.stats()["pending"]:
            chain.hold(grad, norms)  # this call's finalize is pending: keep its outputs alive
    else:
        rc = lib.fdp_backward(k, ctypes.byref(desc), xd.data_ptr(), yd.data_ptr(), grad.data_ptr(),
                              norms.data_ptr() if norms is not None else None, ws.data_ptr(), ws.numel(),
                              stream.cuda_stream)
        _lib.check(rc)

    if skip_barrier:
        # The kernel records whether a clip read the norm accumulator before every
        # tile had published (device fault word, workspace word 1).
        word = ws[4:8].view(torch.int32)
        fault = int(word.item())
        word.zero_()
        if fault & 0x200:
            raise OrderingFault("clip read the per-sample norm accumulator before the block-wise all-reduce "
                                "completed (barrier skipped)")

    wplan = plan
    if wplan is None:  # the reference plans every kind from the spec (workflows.py:437-438)
        wplan = plan_blocks(dims, spec or B200_SPEC)
    width = (spec or B200_SPEC).dtype_width_bytes
    ref_report = ledger(kind.value, dims.B, dims.T, dims.P, dims.D, width, plan=wplan)
    report = _executed_ledger(kind, desc, dims, xd.element_size(), out_dtype, accumulate, add_noise and c.sigma > 0,
                              deferred=grad_scale_out is not None)

    if host_torch:
        return BackwardResult(grad.cpu(), report, norms.cpu() if norms is not None else torch.zeros(0), ref_report)
    if host:
        g_host = Tensor((dims.D, dims.P), grad.double().cpu().numpy())
        n_host = norms.double().cpu().numpy() if norms is not None else np.zeros(0)
        return BackwardResult(g_host, report, n_host, ref_report)
    return BackwardResult(grad, report, norms if norms is not None else torch.zeros(0, device=device), ref_report)


def _run_shared_x(x: torch.Tensor, layers: list, *, noise_impl: str = "keyed_f32", add_noise: bool = True,
                  rank: int = 0, world: int = 1, mean_batch: int = 0) -> list:
    """FLASHDP backward of 1..3 layers that read the same device input X through ONE
    fdp_backward_shared_x call (include/fdp.h: the ghost phase computes X X^T once for
    all of them). `layers`: (dy, cfg, grad_out or None[, accumulate]) per layer; returns
    the grads (grad_out, accumulated into when given unless accumulate is False)."""
    n = len(layers)
    if not 1 <= n <= 3:
        raise UsageError(f"_run_shared_x takes 1..3 layers, got {n}")
    lib = _lib.load()
    device = x.device
    descs = (_lib.FdpDesc * n)()
    grads, norms, sizes = [], [], []
    for k, entry in enumerate(layers):
        dy, cfg, g = entry[:3]
        acc = bool(entry[3]) if len(entry) > 3 else g is not None
        dims = _dims(x, dy)
        descs[k] = _lib.make_desc(B=dims.B, T=dims.T, P=dims.P, D=dims.D, in_dtype=_input_dtype_code(x),
                                  reduction=cfg.reduction, clip_c=cfg.clip_c, sigma=cfg.sigma, seed=cfg.seed,
                                  layer_id=cfg.layer_id, step=cfg.step, rank=rank, world=world,
                                  mean_batch=mean_batch, accumulate=acc and g is not None, add_noise=add_noise,
                                  noise_impl=noise_impl)
        nb = ctypes.c_size_t()
        _lib.check(lib.fdp_workspace_bytes(ctypes.byref(descs[k]), _lib.KIND["flashdp"], ctypes.byref(nb)))
        sizes.append(nb.value)
        if g is not None:
            _check_out(g, (dims.D, dims.P), torch.float32, device, "grad_out")
        grads.append(g if g is not None else torch.empty((dims.D, dims.P), dtype=torch.float32, device=device))
        norms.append(torch.empty(dims.B, dtype=torch.float32, device=device))
    stream = torch.cuda.current_stream(device)
    # one workspace per layer (the ghost phase fills every layer's partials before any reweight)
    wss = [_POOL.get(sizes[k], device, stream, slot=("shared_x", k)) for k in range(n)]
    ptrs = ctypes.c_void_p * n
    rc = lib.fdp_backward_shared_x(n, descs, x.data_ptr(), ptrs(*[e[0].data_ptr() for e in layers]),
                                   ptrs(*[g.data_ptr() for g in grads]), ptrs(*[t.data_ptr() for t in norms]),
                                   ptrs(*[w.data_ptr() for w in wss]),
                                   (ctypes.c_size_t * n)(*[w.numel() for w in wss]), stream.cuda_stream)
    _lib.check(rc)
    return grads


_PLAN_CACHE: dict = {}


def _executed_ledger(kind: WorkflowKind, desc, dims: LayerDims, in_width: int, out_dtype, accumulate: bool,
                     add_noise: bool, deferred: bool = False) -> TrafficReport:
    """device_ledger of the plan the C library resolved for this descriptor."""
    key = (kind.value, dims.B, dims.T, dims.P, dims.D, desc.in_dtype, desc.path, desc.norm_phase, desc.flags,
           torch.cuda.current_device())
    info = _PLAN_CACHE.get(key)
    if info is None:
        info = _lib.plan(desc, kind.value)
        if len(_PLAN_CACHE) > 4096:
            _PLAN_CACHE.clear()
        _PLAN_CACHE[key] = info
    path = _lib.PATH_NAMES[info.path]
    phase = _lib.NORM_PHASE_NAMES.get(info.norm_phase, "auto")
    out_w = 8 if out_dtype == torch.float64 else 4
    n_tiles = max(1, info.n_d * info.n_p)
    return device_ledger(kind.value, path, phase, info.launches, dims.B, dims.T, dims.P, dims.D, in_width, out_w,
                         n_tiles=n_tiles, groups=info.groups, accumulate=accumulate, add_noise=add_noise,
                         deferred=deferred and path == "two_phase" and phase == "single" and not add_noise)


def _check_out(t: torch.Tensor, shape: tuple, dtype: torch.dtype, device: torch.device, name: str) -> None:
    """Caller-supplied outputs are written by the kernels through raw pointers:
    shape, dtype (float64 on the fp64 path), contiguity and device must match."""
    if not isinstance(t, torch.Tensor) or tuple(t.shape) != tuple(shape) or t.dtype != dtype \
            or not t.is_contiguous() or t.device != device:
        got = (tuple(t.shape), t.dtype, t.device) if isinstance(t, torch.Tensor) else type(t)
        raise ShapeError(f"{name} must be a contiguous {dtype} {tuple(shape)} tensor on {device}, got {got}")


class DeferredChain:
    """A deferred-finalize chain (include/fdp.h fdp_chain): pass it as ``chain=``
    to consecutive DP backward calls on one stream. A single-sample layer's
    clip + noise pass (B == 1) is then carried by the next call's GEMM kernel,
    whose idle warps stream it under the tensor-core work, instead of running as
    its own HBM-bound pass; ``flush()`` runs the last pending one. Until a later
    call or ``flush()``, the pending layer's grad_w holds the unclipped G and its
    norms are unwritten. Results equal the unchained calls."""

    def __init__(self):
        self._lib = _lib.load()
        h = ctypes.c_void_p()
        _lib.check(self._lib.fdp_chain_create(ctypes.byref(h)))
        self._h = h
        self._keep = []  # tensors the pending job writes (kept alive until it ran)

    @property
    def handle(self):
        return self._h

    def hold(self, *tensors) -> None:
        self._keep = [t for t in tensors if t is not None]

    def flush(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        s = stream if stream is not None else torch.cuda.current_stream()
        _lib.check(self._lib.fdp_chain_flush(self._h, s.cuda_stream))
        self._keep = []

    def stats(self) -> dict:
        c, f, p = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
        _lib.check(self._lib.fdp_chain_stats(self._h, ctypes.byref(c), ctypes.byref(f), ctypes.byref(p)))
        return {"carried": c.value, "standalone": f.value, "pending": bool(p.value)}

    def __del__(self):
        try:
            if self._h:
                if self.stats()["pending"]:
                    self.flush()
                self._lib.fdp_chain_destroy(self._h)
                self._h = None
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


def _step_ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not (t.is_cuda and t.dtype == torch.int64 and t.numel() >= 1):
        raise UsageError("device_step must be a CUDA int64 tensor")
    return t.data_ptr()


def fdp_capacity(need: int, have: int):
    from .errors import CapacityError
    return CapacityError(need, have, have, message=f"workspace of {have} bytes is smaller than the {need} bytes "
                                                   "this call needs")


class PreparedBackward:
    """One layer's DP backward bound to fixed device buffers: calling it is a
    single C-ABI call (no per-call planning or allocation in Python), which is
    what a training loop or a CUDA graph capture wants.

    grad_w / norms_sq are written in place; `device_step` (CUDA int64 scalar)
    keys the noise so replays of a captured graph draw fresh noise."""

    def __init__(self, kind: WorkflowKind, x: torch.Tensor, dy: torch.Tensor, cfg: Optional[DPConfig], *,
                 grad_w: Optional[torch.Tensor] = None, norms_sq: Optional[torch.Tensor] = None,
                 path: str = "auto", noise_impl: str = "keyed_f32", accumulate: bool = False,
                 add_noise: bool = True, rank: int = 0, world: int = 1, mean_batch: int = 0,
                 device_step: Optional[torch.Tensor] = None, workspace: Optional[torch.Tensor] = None,
                 norm_phase: str = "auto", deterministic: bool = False, chain: Optional["DeferredChain"] = None,
                 grad_scale: Optional[torch.Tensor] = None):
        dims = _dims(x, dy)
        if not (x.is_cuda and dy.is_cuda and x.is_contiguous() and dy.is_contiguous() and x.dtype == dy.dtype):
            raise UsageError("PreparedBackward needs contiguous CUDA inputs of one dtype")
        if grad_scale is not None:  # fdp_dw_deferred (include/fdp.h): the consumer applies grad_scale[0]
            if kind != WorkflowKind.FLASHDP or chain is not None:
                raise UsageError("grad_scale needs kind FLASHDP and no chain")
            _check_out(grad_scale, (1,), torch.float32, x.device, "grad_scale")
        self.grad_scale = grad_scale
        self.chain = chain
        c = cfg or DPConfig(clip_c=1.0, sigma=0.0)
        self.kind = kind
        self.x, self.dy = x, dy
        self.desc = _lib.make_desc(B=dims.B, T=dims.T, P=dims.P, D=dims.D, in_dtype=_input_dtype_code(x),
                                   reduction=c.reduction, clip_c=c.clip_c, sigma=c.sigma, seed=c.seed,
                                   layer_id=c.layer_id, step=c.step, rank=rank, world=world, mean_batch=mean_batch,
                                   accumulate=accumulate, add_noise=add_noise, noise_impl=noise_impl, path=path,
                                   norm_phase=norm_phase, device_step=_step_ptr(device_step),
                                   flags=_lib.FLAG_DETERMINISTIC if deterministic else 0)
        self._device_step = device_step
        lib = _lib.load()
        self._lib = lib
        self._k = _lib.KIND[kind.value]
        nbytes = ctypes.c_size_t()
        _lib.check(lib.fdp_workspace_bytes(ctypes.byref(self.desc), self._k, ctypes.byref(nbytes)))
        dev = x.device
        # the fp64 parity path writes float64 outputs (include/fdp.h FDP_DTYPE_F64)
        out_dtype = torch.float64 if x.dtype == torch.float64 else torch.float32
        if grad_w is not None:
            _check_out(grad_w, (dims.D, dims.P), out_dtype, dev, "grad_w")
        self.grad_w = grad_w if grad_w is not None else torch.zeros((dims.D, dims.P), dtype=out_dtype, device=dev)
        if kind == WorkflowKind.NON_DP:
            self.norms_sq = None
        else:
            if norms_sq is not None:
                _check_out(norms_sq, (dims.B,), out_dtype, dev, "norms_sq")
            self.norms_sq = norms_sq if norms_sq is not None else torch.zeros(dims.B, dtype=out_dtype, device=dev)
        if workspace is None:
            workspace = torch.zeros(max(nbytes.value, 4096), dtype=torch.uint8, device=dev)
        elif workspace.numel() * workspace.element_size() < nbytes.value:
            raise fdp_capacity(nbytes.value, workspace.numel() * workspace.element_size())
        self.workspace = workspace
        self.workspace_bytes = nbytes.value
        self._args = (self._k, ctypes.byref(self.desc), x.data_ptr(), dy.data_ptr(), self.grad_w.data_ptr(),
                      self.norms_sq.data_ptr() if self.norms_sq is not None else None, workspace.data_ptr(),
                      workspace.numel() * workspace.element_size())
        self.plan = _lib.plan(self.desc, kind.value)

    def set_step(self, step: int) -> None:
        self.desc.step = _lib._wrap64(step)

    def __call__(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        s = stream if stream is not None else torch.cuda.current_stream(self.x.device)
        if self.chain is not None:  # single-sample finalize deferred into the next chained call
            _lib.check(self._lib.fdp_backward_chained(*self._args, self.chain.handle, s.cuda_stream))
        elif self.grad_scale is not None:
            a = self._args
            _lib.check(self._lib.fdp_dw_deferred(a[1], a[2], a[3], a[4], a[5], self.grad_scale.data_ptr(), a[6], a[7],
                                                 s.cuda_stream))
        else:
            _lib.check(self._lib.fdp_backward(*self._args, s.cuda_stream))


class PreparedSharedX:
    """Two or three prepared FLASHDP layers that read the same input X (q/k/v of an
    attention block, gate/up of a SwiGLU MLP) run through ONE C-ABI call
    (`fdp_backward_shared_x`): when each takes the two-phase ghost path, the X Gram
    of every tile pair is computed once for all of them; per-layer clipping, noise
    and outputs are those of the individual calls (include/fdp.h)."""

    def __init__(self, layers: list):
        if not 1 <= len(layers) <= 3:
            raise UsageError(f"PreparedSharedX takes 1..3 layers, got {len(layers)}")
        x0 = layers[0].x
        for pb in layers:
            if pb.kind != WorkflowKind.FLASHDP or pb.chain is not None:
                raise UsageError("PreparedSharedX layers must be unchained FLASHDP PreparedBackward calls")
            if pb.x.data_ptr() != x0.data_ptr() or pb.x.shape != x0.shape:
                raise UsageError("PreparedSharedX layers must share one X tensor")
        self.layers = layers
        self.x = x0
        n = len(layers)
        self._descs = (_lib.FdpDesc * n)(*[pb.desc for pb in layers])
        ptrs = ctypes.c_void_p * n
        self._dy = ptrs(*[pb.dy.data_ptr() for pb in layers])
        self._gw = ptrs(*[pb.grad_w.data_ptr() for pb in layers])
        self._ns = ptrs(*[pb.norms_sq.data_ptr() for pb in layers])
        self._ws = ptrs(*[pb.workspace.data_ptr() for pb in layers])
        self._wsb = (ctypes.c_size_t * n)(*[pb.workspace.numel() * pb.workspace.element_size() for pb in layers])
        self._lib = _lib.load()

    def set_step(self, step: int) -> None:
        for k, pb in enumerate(self.layers):
            pb.set_step(step)
            self._descs[k].step = pb.desc.step

    def __call__(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        s = stream if stream is not None else torch.cuda.current_stream(self.x.device)
        _lib.check(self._lib.fdp_backward_shared_x(len(self.layers), self._descs, self.x.data_ptr(), self._dy,
                                                   self._gw, self._ns, self._ws, self._wsb, s.cuda_stream))


class PreparedGroup:
    """The fused DP backward of several layers in ONE persistent launch
    (fdp_backward_group): e.g. every linear layer of a model after the
    activation-gradient pass. Each layer keeps its own DPConfig (clip C, sigma,
    noise key = layer_id), norms and outputs; results equal per-layer
    backward_flashdp calls (up to fp32 summation order across sample groups).

    layers: sequence of (x, dy, cfg) with contiguous bf16 CUDA tensors.
    max_ctas > 0 caps the launch (SMs left free for a concurrent collective)."""

    def __init__(self, layers, *, grads=None, norms=None, noise_impl: str = "keyed_f32", accumulate: bool = False,
                 add_noise: bool = True, rank: int = 0, world: int = 1, mean_batch: int = 0,
                 device_step: Optional[torch.Tensor] = None, workspace: Optional[torch.Tensor] = None,
                 max_ctas: int = 0):
        n = len(layers)
        if max_ctas < 0:
            raise UsageError(f"max_ctas must be >= 0, got {max_ctas}")
        self.max_ctas = int(max_ctas)
        if n < 1:
            raise UsageError("PreparedGroup needs at least one layer")
        self.layers = list(layers)
        descs = (_lib.FdpDesc * n)()
        self.grads, self.norms = [], []
        xs, dys, gs, ns = [], [], [], []
        for i, (x, dy, cfg) in enumerate(self.layers):
            dims = _dims(x, dy)
            if not (x.is_cuda and dy.is_cuda and x.dtype == torch.bfloat16 and dy.dtype == torch.bfloat16
                    and x.is_contiguous() and dy.is_contiguous()):
                raise UsageError(f"layer {i}: PreparedGroup needs contiguous bf16 CUDA inputs")
            descs[i] = _lib.make_desc(B=dims.B, T=dims.T, P=dims.P, D=dims.D, reduction=cfg.reduction,
                                      clip_c=cfg.clip_c, sigma=cfg.sigma, seed=cfg.seed, layer_id=cfg.layer_id,
                                      step=cfg.step, rank=rank, world=world, mean_batch=mean_batch,
                                      accumulate=accumulate, add_noise=add_noise, noise_impl=noise_impl,
                                      device_step=_step_ptr(device_step))
            if grads is not None:
                _check_out(grads[i], (dims.D, dims.P), torch.float32, x.device, f"grads[{i}]")
            if norms is not None:
                _check_out(norms[i], (dims.B,), torch.float32, x.device, f"norms[{i}]")
            g = grads[i] if grads is not None else torch.zeros((dims.D, dims.P), dtype=torch.float32, device=x.device)
            nrm = norms[i] if norms is not None else torch.zeros(dims.B, dtype=torch.float32, device=x.device)
            self.grads.append(g)
            self.norms.append(nrm)
            xs.append(x.data_ptr())
            dys.append(dy.data_ptr())
            gs.append(g.data_ptr())
            ns.append(nrm.data_ptr())
        self.descs = descs
        arr = ctypes.c_void_p * n
        self._ptrs = (arr(*xs), arr(*dys), arr(*gs), arr(*ns))
        lib = _lib.load()
        self._lib = lib
        nbytes = ctypes.c_size_t()
        _lib.check(lib.fdp_group_workspace_bytes_ex(n, descs, self.max_ctas, ctypes.byref(nbytes)))
        if workspace is None:
            workspace = torch.zeros(max(nbytes.value, 4096), dtype=torch.uint8, device=self.layers[0][0].device)
        elif workspace.numel() * workspace.element_size() < nbytes.value:
            raise fdp_capacity(nbytes.value, workspace.numel() * workspace.element_size())
        self.workspace = workspace
        self._n = n

    def __call__(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        s = stream if stream is not None else torch.cuda.current_stream(self.layers[0][0].device)
        xs, dys, gs, ns = self._ptrs
        _lib.check(self._lib.fdp_backward_group_ex(self._n, self.descs, xs, dys, gs, ns, self.workspace.data_ptr(),
                                                   self.workspace.numel(), self.max_ctas, s.cuda_stream))


class HostStreamedBackward:
    """DP backward of a list of layers whose inputs live in HOST memory (the
    reference's calling convention: run_backward on host arrays, once per layer,
    workflows.py:427-440), pipelined over three CUDA streams:

        copy-in   layer i+1's X/dY host->device into one of two device slots
        compute   layer i's fused DP backward (fdp_backward, one launch)
        copy-out  layer i-1's grad_w / norms device->host

    so the PCIe transfers in both directions overlap each other and the kernels;
    the step costs ~max(H2D bytes / PCIe bandwidth, kernel time). Results are
    identical to per-layer run_backward calls (same kernels, same descriptors).

    layers: sequence of (x_host, dy_host, cfg); x_host (B,T,P) / dy_host (B,T,D)
    CPU torch tensors (bf16 or fp32; pinned for asynchronous copies). Returns one
    BackwardResult per layer with host grad_w (D,P) fp32 and norms (B,) fp32."""

    def __init__(self, device: Optional[torch.device] = None, *, noise_impl: str = "keyed_f32", path: str = "auto",
                 rank: int = 0, world: int = 1, mean_batch: int = 0, deterministic: bool = False):
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.opts = dict(noise_impl=noise_impl, path=path, rank=rank, world=world, mean_batch=mean_batch,
                         flags=_lib.FLAG_DETERMINISTIC if deterministic else 0)
        self._in = torch.cuda.Stream(self.device)
        self._out = torch.cuda.Stream(self.device)
        self._slots: list = [None, None]
        self._lib = _lib.load()

    def _slot(self, i: int, nx: int, ny: int, dtype: torch.dtype):
        s = self._slots[i]
        if s is None or s[0].numel() < nx or s[1].numel() < ny or s[0].dtype != dtype:
            s = (torch.empty(nx, dtype=dtype, device=self.device), torch.empty(ny, dtype=dtype, device=self.device))
            self._slots[i] = s
        return s

    def __call__(self, layers, kind: WorkflowKind = WorkflowKind.FLASHDP, spec: Optional[MemSpec] = None):
        dev = self.device
        comp = torch.cuda.current_stream(dev)
        lib = self._lib
        k = _lib.KIND[kind.value]
        n = len(layers)
        in_done = [torch.cuda.Event() for _ in range(n)]
        comp_done = [torch.cuda.Event() for _ in range(n)]
        results = []
        pending = []  # device tensors kept alive until the copy-out stream is synchronised
        # the copy-in stream writes device slots that earlier work on the compute stream may
        # still read (slots of a previous call, blocks the caching allocator recycled)
        self._in.wait_stream(comp)
        for i, (x, dy, cfg) in enumerate(layers):
            dims = _dims(x, dy)
            if not (isinstance(x, torch.Tensor) and isinstance(dy, torch.Tensor)) or x.is_cuda or dy.is_cuda:
                raise UsageError("HostStreamedBackward takes host (CPU) torch tensors")
            if x.dtype != dy.dtype or x.dtype not in (torch.bfloat16, torch.float32):
                raise UsageError(f"x and dy must share a dtype in (bfloat16, float32), got {x.dtype}, {dy.dtype}")
            if kind != WorkflowKind.NON_DP and cfg is None:
                raise UsageError("DP workflows need a DPConfig")
            xs, ys = x.contiguous(), dy.contiguous()
            xd, yd = self._slot(i % 2, xs.numel(), ys.numel(), xs.dtype)
            xd, yd = xd[:xs.numel()], yd[:ys.numel()]
            with torch.cuda.stream(self._in):
                if i >= 2:  # slot reuse: layer i-2's kernel has consumed it
                    self._in.wait_event(comp_done[i - 2])
                xd.copy_(xs.view(-1), non_blocking=True)
                yd.copy_(ys.view(-1), non_blocking=True)
                in_done[i].record(self._in)
            c = cfg or DPConfig(clip_c=1.0, sigma=0.0)
            desc = _lib.make_desc(B=dims.B, T=dims.T, P=dims.P, D=dims.D, in_dtype=_input_dtype_code(xd),
                                  reduction=c.reduction, clip_c=c.clip_c, sigma=c.sigma, seed=c.seed,
                                  layer_id=c.layer_id, step=c.step, **self.opts)
            ws_bytes = ctypes.c_size_t()
            _lib.check(lib.fdp_workspace_bytes(ctypes.byref(desc), k, ctypes.byref(ws_bytes)))
            ws = _POOL.get(ws_bytes.value, dev, comp)
            grad = torch.empty((dims.D, dims.P), dtype=torch.float32, device=dev)
            norms = torch.empty(dims.B, dtype=torch.float32, device=dev)
            comp.wait_event(in_done[i])
            _lib.check(lib.fdp_backward(k, ctypes.byref(desc), xd.data_ptr(), yd.data_ptr(), grad.data_ptr(),
                                        norms.data_ptr() if kind != WorkflowKind.NON_DP else None, ws.data_ptr(),
                                        ws.numel(), comp.cuda_stream))
            comp_done[i].record(comp)
            g_host = torch.empty((dims.D, dims.P), dtype=torch.float32, pin_memory=True)
            n_host = torch.empty(dims.B, dtype=torch.float32, pin_memory=True)
            with torch.cuda.stream(self._out):
                self._out.wait_event(comp_done[i])
                g_host.copy_(grad, non_blocking=True)
                if kind != WorkflowKind.NON_DP:
                    n_host.copy_(norms, non_blocking=True)
            pending.append((grad, norms))
            width = (spec or B200_SPEC).dtype_width_bytes
            ref = ledger(kind.value, dims.B, dims.T, dims.P, dims.D, width, plan=plan_blocks(dims, spec or B200_SPEC))
            report = _executed_ledger(kind, desc, dims, xd.element_size(), torch.float32, False,
                                      c.sigma > 0)
            results.append(BackwardResult(g_host, report, n_host if kind != WorkflowKind.NON_DP else torch.zeros(0),
                                          ref))
        self._out.synchronize()
        comp.wait_stream(self._out)  # later device work on these buffers (caching allocator reuse) orders after
        del pending
        return results


def backward_nondp(x, dy, spec: Optional[MemSpec] = None, *, sim=None, **opts) -> BackwardResult:
    """grad_w = sum_b sum_t dY^T X; no per-sample quantity (workflows.py:121-150)."""
    return _run(WorkflowKind.NON_DP, x, dy, None, spec, None, **opts)


def backward_explicit(x, dy, cfg: DPConfig, spec: Optional[MemSpec] = None, *, sim=None, **opts) -> BackwardResult:
    """Opacus-style: materialise G, norms, clip into G', sum + noise (workflows.py:156-240)."""
    return _run(WorkflowKind.EXPLICIT_DP, x, dy, cfg, spec, None, **opts)


def backward_implicit(x, dy, cfg: DPConfig, spec: Optional[MemSpec] = None, *, sim=None, **opts) -> BackwardResult:
    """Norm pass, then recompute + clip + sum + noise (workflows.py:246-324)."""
    return _run(WorkflowKind.IMPLICIT_DP, x, dy, cfg, spec, None, **opts)


def backward_flashdp(x, dy, cfg: DPConfig, plan: Optional[BlockPlan] = None, spec: Optional[MemSpec] = None, *,
                     sim=None, skip_barrier: bool = False, **opts) -> BackwardResult:
    """Fused DP backward (workflows.py:340-421), one sm_100a launch on the fused path.

    ``plan`` is validated against the extents (UsageError, workflows.py:330-337)
    and recorded in the ledger; the device tiling is fixed by the tcgen05 shape.
    ``skip_barrier=True`` removes the in-kernel wait of the norm all-reduce and
    delays one CTA; the kernel detects the premature read and the call raises
    ``OrderingFault`` like the reference simulator."""
    dims = _dims(x, dy)
    if plan is not None:
        check_plan(plan, dims)
    if skip_barrier:
        opts.setdefault("path", "fused")
    return _run(WorkflowKind.FLASHDP, x, dy, cfg, spec, plan, skip_barrier=skip_barrier, **opts)


def run_backward(kind: WorkflowKind, x, dy, cfg: DPConfig, spec: Optional[MemSpec] = None,
                 plan: Optional[BlockPlan] = None, *, sim=None, **opts) -> BackwardResult:
    """Run one workflow; flashdp derives a block plan if none is given (workflows.py:427-440)."""
    if kind == WorkflowKind.NON_DP:
        return backward_nondp(x, dy, spec, **opts)
    if kind == WorkflowKind.EXPLICIT_DP:
        return backward_explicit(x, dy, cfg, spec, **opts)
    if kind == WorkflowKind.IMPLICIT_DP:
        return backward_implicit(x, dy, cfg, spec, **opts)
    if kind == WorkflowKind.FLASHDP:
        return backward_flashdp(x, dy, cfg, plan, spec, **opts)
    raise UsageError(f"unknown workflow kind {kind!r}")


def execution_plan(x_shape, dy_shape, kind: WorkflowKind = WorkflowKind.FLASHDP, *, dtype=torch.bfloat16,
                   path: str = "auto") -> dict:
    """The device plan the native layer will take (path, tiles, groups, grid, workspace)."""
    B, T, P = x_shape
    D = dy_shape[2]
    desc = _lib.make_desc(B=B, T=T, P=P, D=D, in_dtype=_lib.DTYPE_BF16 if dtype == torch.bfloat16 else _lib.DTYPE_F32,
                          path=path)
    info = _lib.plan(desc, kind.value)
    return {"path": _lib.PATH_NAMES[info.path], "norm_phase": _lib.NORM_PHASE_NAMES.get(info.norm_phase, "auto"),
            "tile_d": info.tile_d, "tile_p": info.tile_p, "tile_t": info.tile_t,
            "n_d": info.n_d, "n_p": info.n_p, "groups": info.groups, "grid": info.grid, "launches": info.launches,
            "sms": info.sms, "workspace_bytes": info.workspace_bytes}
