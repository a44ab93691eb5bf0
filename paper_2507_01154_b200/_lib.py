"""ctypes binding of the C ABI declared in include/fdp.h.

This is the one place the Python mirror of the reference API touches native
code. There is no fallback: if the shared library is missing or no CUDA device
is present, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import CapacityError, ShapeError, UsageError

_HERE = Path(__file__).resolve().parent
# FDP_LIB_PATH: an alternative build of the same sources (A/B of compile-time variants only)
LIB_PATH = Path(os.environ["FDP_LIB_PATH"]) if os.environ.get("FDP_LIB_PATH") else _HERE / "_fdp.so"

FDP_OK, FDP_ERR_SHAPE, FDP_ERR_USAGE, FDP_ERR_CAPACITY, FDP_ERR_CUDA = range(5)
DTYPE_BF16, DTYPE_F32, DTYPE_F64 = 0, 1, 2
REDUCE = {"sum": 0, "mean": 1}
NOISE = {"keyed_f32": 0, "keyed_f64": 1, "philox": 2}
PATH = {"auto": 0, "fused": 1, "two_phase": 2, "simt": 3}
PATH_NAMES = {v: k for k, v in PATH.items()}
KIND = {"non_dp": 0, "explicit_dp": 1, "implicit_dp": 2, "flashdp": 3}
NORM_PHASE = {"auto": 0, "ghost": 1, "recompute": 2, "single": 3, "spill": 4}
NORM_PHASE_NAMES = {v: k for k, v in NORM_PHASE.items()}
FLAG_SKIP_BARRIER = 1
FLAG_TIMEOUT_SHORT = 2
FLAG_TRACE = 4
FLAG_DETERMINISTIC = 8

# Every symbol include/fdp.h declares (checked by the CPU test suite).
EXPORTED_SYMBOLS = (
    "fdp_abi_version", "fdp_last_error", "fdp_device_info", "fdp_plan", "fdp_workspace_bytes",
    "fdp_workspace_init", "fdp_backward", "fdp_dw", "fdp_noise", "fdp_noise_f64", "fdp_noise_partition",
    "fdp_group_workspace_bytes", "fdp_backward_group", "fdp_group_workspace_bytes_ex", "fdp_backward_group_ex",
    "fdp_sgd_step", "fdp_adam_step", "fdp_bias_workspace_bytes", "fdp_bias_dw", "fdp_vec_workspace_bytes",
    "fdp_vec_dw", "fdp_embedding_workspace_bytes", "fdp_embedding_dw",
    "fdp_chain_create", "fdp_chain_destroy", "fdp_chain_flush", "fdp_chain_stats", "fdp_dw_chained",
    "fdp_backward_chained", "fdp_backward_shared_x", "fdp_dw_deferred", "fdp_sgd_step_scaled",
    "fdp_adam_step_scaled", "fdp_adam_multi_table_bytes", "fdp_adam_multi_prepare", "fdp_adam_step_multi",
    "fdp_sgd_step_multi",
)
VEC_KIND = {"bias": 0, "rmsnorm": 1, "layernorm": 2}


class FdpDesc(ctypes.Structure):
    _fields_ = [
        ("B", ctypes.c_int64), ("T", ctypes.c_int64), ("P", ctypes.c_int64), ("D", ctypes.c_int64),
        ("in_dtype", ctypes.c_int32), ("reduction", ctypes.c_int32),
        ("clip_c", ctypes.c_double), ("sigma", ctypes.c_double),
        ("seed", ctypes.c_int64), ("layer_id", ctypes.c_int64), ("step", ctypes.c_int64),
        ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
        ("mean_batch", ctypes.c_int64),
        ("accumulate", ctypes.c_int32), ("add_noise", ctypes.c_int32),
        ("noise_impl", ctypes.c_int32), ("path", ctypes.c_int32),
        ("flags", ctypes.c_int32), ("norm_phase", ctypes.c_int32),
        ("device_step", ctypes.c_void_p),
    ]


class FdpAdamSegment(ctypes.Structure):
    _fields_ = [
        ("theta", ctypes.c_void_p), ("m", ctypes.c_void_p), ("v", ctypes.c_void_p), ("grad", ctypes.c_void_p),
        ("grad_scale", ctypes.c_void_p), ("n", ctypes.c_int64), ("noise", ctypes.POINTER(FdpDesc)),
        ("noise_offset", ctypes.c_int64),
    ]


class FdpPlanInfo(ctypes.Structure):
    _fields_ = [
        ("path", ctypes.c_int32), ("norm_phase", ctypes.c_int32),
        ("tile_d", ctypes.c_int32), ("tile_p", ctypes.c_int32), ("tile_t", ctypes.c_int32),
        ("n_d", ctypes.c_int32), ("n_p", ctypes.c_int32), ("groups", ctypes.c_int32),
        ("grid", ctypes.c_int32), ("launches", ctypes.c_int32), ("sms", ctypes.c_int32),
        ("workspace_bytes", ctypes.c_int64),
    ]


_lib = None


def _wrap64(v: int) -> int:
    """Two's-complement view of any Python int as int64 (the reference masks keys
    with & (2**64-1), rng.py:42-47)."""
    v &= (1 << 64) - 1
    return v - (1 << 64) if v >= (1 << 63) else v


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"native library {LIB_PATH} is missing; build it with `python -m paper_2507_01154_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(str(LIB_PATH))
    lib.fdp_abi_version.restype = ctypes.c_int
    lib.fdp_last_error.restype = ctypes.c_char_p
    lib.fdp_device_info.argtypes = [ctypes.POINTER(ctypes.c_int32)] * 3
    lib.fdp_plan.argtypes = [ctypes.POINTER(FdpDesc), ctypes.c_int32, ctypes.POINTER(FdpPlanInfo)]
    lib.fdp_workspace_bytes.argtypes = [ctypes.POINTER(FdpDesc), ctypes.c_int32, ctypes.POINTER(ctypes.c_size_t)]
    lib.fdp_workspace_init.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
    lib.fdp_backward.argtypes = [ctypes.c_int32, ctypes.POINTER(FdpDesc), ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                 ctypes.c_void_p]
    lib.fdp_dw.argtypes = [ctypes.POINTER(FdpDesc), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
    lib.fdp_noise.argtypes = [ctypes.POINTER(FdpDesc), ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                              ctypes.c_double, ctypes.c_void_p]
    lib.fdp_noise_f64.argtypes = [ctypes.POINTER(FdpDesc), ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                  ctypes.c_double, ctypes.c_void_p]
    lib.fdp_noise_partition.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                        ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
    lib.fdp_group_workspace_bytes.argtypes = [ctypes.c_int32, ctypes.POINTER(FdpDesc),
                                              ctypes.POINTER(ctypes.c_size_t)]
    lib.fdp_backward_group.argtypes = [ctypes.c_int32, ctypes.POINTER(FdpDesc)] + [ctypes.POINTER(ctypes.c_void_p)] * 4 + [
        ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
    lib.fdp_group_workspace_bytes_ex.argtypes = [ctypes.c_int32, ctypes.POINTER(FdpDesc), ctypes.c_int32,
                                                 ctypes.POINTER(ctypes.c_size_t)]
    lib.fdp_backward_group_ex.argtypes = [ctypes.c_int32, ctypes.POINTER(FdpDesc)] + [
        ctypes.POINTER(ctypes.c_void_p)] * 4 + [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int32, ctypes.c_void_p]
    lib.fdp_sgd_step.argtypes = [ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_double,
                                 ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
    lib.fdp_adam_step.argtypes = [ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                  ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
    lib.fdp_bias_workspace_bytes.argtypes = [ctypes.POINTER(FdpDesc), ctypes.POINTER(ctypes.c_size_t)]
    lib.fdp_bias_dw.argtypes = [ctypes.POINTER(FdpDesc), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
    lib.fdp_vec_workspace_bytes.argtypes = [ctypes.POINTER(FdpDesc), ctypes.c_int32, ctypes.POINTER(ctypes.c_size_t)]
    lib.fdp_vec_dw.argtypes = [ctypes.POINTER(FdpDesc), ctypes.c_int32] + [ctypes.c_void_p] * 5 + [
        ctypes.c_size_t, ctypes.c_void_p]
    lib.fdp_embedding_workspace_bytes.argtypes = [ctypes.POINTER(FdpDesc), ctypes.POINTER(ctypes.c_size_t)]
    lib.fdp_embedding_dw.argtypes = [ctypes.POINTER(FdpDesc)] + [ctypes.c_void_p] * 5 + [ctypes.c_size_t,
                                                                                        ctypes.c_void_p]
    lib.fdp_chain_create.argtypes = [ctypes.POINTER(ctypes.c_void_p)]
    lib.fdp_chain_destroy.argtypes = [ctypes.c_void_p]
    lib.fdp_chain_flush.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    lib.fdp_chain_stats.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
                                    ctypes.POINTER(ctypes.c_int32)]
    lib.fdp_dw_chained.argtypes = [ctypes.POINTER(FdpDesc), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p]
    lib.fdp_backward_chained.argtypes = [ctypes.c_int32, ctypes.POINTER(FdpDesc), ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                         ctypes.c_void_p, ctypes.c_void_p]
    lib.fdp_backward_shared_x.argtypes = [ctypes.c_int32, ctypes.POINTER(FdpDesc), ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_void_p]
    lib.fdp_dw_deferred.argtypes = [ctypes.POINTER(FdpDesc)] + [ctypes.c_void_p] * 6 + [ctypes.c_size_t,
                                                                                       ctypes.c_void_p]
    lib.fdp_sgd_step_scaled.argtypes = [ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_int64, ctypes.c_double, ctypes.c_void_p, ctypes.c_int64,
                                        ctypes.c_void_p]
    lib.fdp_adam_step_scaled.argtypes = [ctypes.c_int32] + [ctypes.c_void_p] * 5 + [
        ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_void_p,
        ctypes.c_int64, ctypes.c_void_p]
    lib.fdp_adam_multi_table_bytes.argtypes = [ctypes.c_int32, ctypes.POINTER(ctypes.c_size_t)]
    lib.fdp_adam_multi_prepare.argtypes = [ctypes.c_int32, ctypes.POINTER(FdpAdamSegment), ctypes.c_void_p,
                                           ctypes.c_size_t, ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p]
    lib.fdp_adam_step_multi.argtypes = [ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_void_p]
    lib.fdp_sgd_step_multi.argtypes = [ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64, ctypes.c_double,
                                       ctypes.c_void_p]
    for name in ("fdp_sgd_step_multi", "fdp_adam_multi_table_bytes", "fdp_adam_multi_prepare", "fdp_adam_step_multi",
                 "fdp_dw_deferred", "fdp_sgd_step_scaled", "fdp_adam_step_scaled", "fdp_backward_shared_x", "fdp_chain_create", "fdp_chain_destroy", "fdp_chain_flush", "fdp_chain_stats", "fdp_dw_chained",
                 "fdp_backward_chained", "fdp_vec_workspace_bytes", "fdp_vec_dw", "fdp_embedding_workspace_bytes", "fdp_embedding_dw",
                 "fdp_bias_workspace_bytes", "fdp_bias_dw", "fdp_sgd_step", "fdp_adam_step", "fdp_group_workspace_bytes_ex", "fdp_backward_group_ex", "fdp_group_workspace_bytes",
                 "fdp_backward_group", "fdp_device_info", "fdp_plan", "fdp_workspace_bytes", "fdp_workspace_init", "fdp_backward",
                 "fdp_dw", "fdp_noise", "fdp_noise_f64", "fdp_noise_partition"):
        getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def check(rc: int) -> None:
    """Map a C status to the reference exception types (errors.py)."""
    if rc == FDP_OK:
        return
    msg = load().fdp_last_error().decode("utf-8", "replace")
    if rc == FDP_ERR_SHAPE:
        raise ShapeError(msg)
    if rc == FDP_ERR_CAPACITY:
        raise CapacityError.from_message(msg)
    if rc == FDP_ERR_USAGE:
        raise UsageError(msg)
    raise RuntimeError(f"CUDA failure in native FlashDP call: {msg}")


def make_desc(*, B, T, P, D, in_dtype=DTYPE_BF16, reduction="sum", clip_c=1.0, sigma=0.0, seed=0, layer_id=0,
              step=0, rank=0, world=1, mean_batch=0, accumulate=False, add_noise=True, noise_impl="keyed_f32",
              path="auto", flags=0, norm_phase="auto", device_step=None) -> FdpDesc:
    if reduction not in REDUCE:
        raise UsageError(f"reduction must be one of {tuple(REDUCE)}, got {reduction!r}")
    if noise_impl not in NOISE:
        raise UsageError(f"noise_impl must be one of {tuple(NOISE)}, got {noise_impl!r}")
    if path not in PATH:
        raise UsageError(f"path must be one of {tuple(PATH)}, got {path!r}")
    if isinstance(norm_phase, str):
        if norm_phase not in NORM_PHASE:
            raise UsageError(f"norm_phase must be one of {tuple(NORM_PHASE)}, got {norm_phase!r}")
        norm_phase = NORM_PHASE[norm_phase]
    return FdpDesc(B=B, T=T, P=P, D=D, in_dtype=in_dtype, reduction=REDUCE[reduction], clip_c=float(clip_c),
                   sigma=float(sigma), seed=_wrap64(seed), layer_id=_wrap64(layer_id), step=_wrap64(step),
                   rank=rank, world=world, mean_batch=mean_batch, accumulate=int(bool(accumulate)),
                   add_noise=int(bool(add_noise)), noise_impl=NOISE[noise_impl], path=PATH[path], flags=flags,
                   norm_phase=norm_phase, device_step=device_step)


def plan(desc: FdpDesc, kind: str) -> FdpPlanInfo:
    info = FdpPlanInfo()
    check(load().fdp_plan(ctypes.byref(desc), KIND[kind], ctypes.byref(info)))
    return info


def device_info() -> tuple[int, int, int]:
    a, b, c = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    check(load().fdp_device_info(ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
    return a.value, b.value, c.value


def library_path() -> str:
    return os.fspath(LIB_PATH)
