"""The C ABI exactly as INTEGRATION.md's ctypes stub binds it (its own fdp_desc
Structure, raw ctypes calls, no package helpers): fp64 reference inputs through
fdp_workspace_bytes + fdp_dw, results vs the reference's golden outputs at its
1e-12 bar; error codes for bad calls."""

import ctypes
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class fdp_desc(ctypes.Structure):  # noqa: N801 -- the C struct's name, as in INTEGRATION.md
    _fields_ = [("B", ctypes.c_int64), ("T", ctypes.c_int64), ("P", ctypes.c_int64), ("D", ctypes.c_int64),
                ("in_dtype", ctypes.c_int32), ("reduction", ctypes.c_int32),
                ("clip_c", ctypes.c_double), ("sigma", ctypes.c_double),
                ("seed", ctypes.c_int64), ("layer_id", ctypes.c_int64), ("step", ctypes.c_int64),
                ("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("mean_batch", ctypes.c_int64),
                ("accumulate", ctypes.c_int32), ("add_noise", ctypes.c_int32), ("noise_impl", ctypes.c_int32),
                ("path", ctypes.c_int32), ("flags", ctypes.c_int32), ("norm_phase", ctypes.c_int32),
                ("device_step", ctypes.c_void_p)]


def _lib():
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2507_01154_b200", "_fdp.so"))
    lib.fdp_last_error.restype = ctypes.c_char_p
    return lib


def _call(lib, d, x, dy):
    nbytes = ctypes.c_size_t()
    rc = lib.fdp_workspace_bytes(ctypes.byref(d), 3, ctypes.byref(nbytes))
    if rc:
        return rc, None, None
    ws = torch.zeros(max(nbytes.value, 1), dtype=torch.uint8, device="cuda")
    g = torch.empty(int(d.D), int(d.P), dtype=torch.float64, device="cuda")
    n = torch.empty(int(d.B), dtype=torch.float64, device="cuda")
    rc = lib.fdp_dw(ctypes.byref(d), ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(dy.data_ptr()),
                    ctypes.c_void_p(g.data_ptr()), ctypes.c_void_p(n.data_ptr()), ctypes.c_void_p(ws.data_ptr()),
                    ctypes.c_size_t(ws.numel()), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    return rc, g, n


def test_integration_stub_fp64_reference_parity():
    g = np.load(os.path.join(ROOT, "tests", "golden", "random.npz"))
    lib = _lib()
    for i in range(int(g["count"][0])):
        x = torch.tensor(g[f"x{i}"], dtype=torch.float64, device="cuda")
        dy = torch.tensor(g[f"dy{i}"], dtype=torch.float64, device="cuda")
        c, s, mean, seed, layer, step = g[f"cfg{i}"].tolist()
        B, T, P = x.shape
        d = fdp_desc(B=B, T=T, P=P, D=dy.shape[2], in_dtype=2, reduction=int(mean), clip_c=c, sigma=s,
                     seed=int(seed), layer_id=int(layer), step=int(step), rank=0, world=1, add_noise=1, noise_impl=1)
        rc, gw, nrm = _call(lib, d, x, dy)
        assert rc == 0, lib.fdp_last_error()
        want = g[f"grad{i}"]
        assert np.max(np.abs(gw.cpu().numpy() - want)) <= 1e-12 * max(1.0, np.max(np.abs(want))), i
        assert np.max(np.abs(nrm.cpu().numpy() - g[f"norms{i}"])) <= 1e-12 * max(1.0, np.max(g[f"norms{i}"])), i


def test_integration_stub_error_codes():
    lib = _lib()
    x = torch.zeros(2, 4, 8, dtype=torch.float64, device="cuda")
    dy = torch.zeros(2, 4, 8, dtype=torch.float64, device="cuda")
    bad = [fdp_desc(B=0, T=4, P=8, D=8, in_dtype=2, clip_c=1.0, world=1),            # SHAPE
           fdp_desc(B=2, T=4, P=8, D=8, in_dtype=2, clip_c=-1.0, world=1),           # USAGE: clip_c <= 0
           fdp_desc(B=2, T=4, P=8, D=8, in_dtype=7, clip_c=1.0, world=1),            # USAGE: dtype
           fdp_desc(B=2, T=4, P=8, D=8, in_dtype=2, clip_c=1.0, world=2, rank=2)]    # USAGE: rank
    want = [1, 2, 2, 2]
    for d, w in zip(bad, want):
        rc, _, _ = _call(lib, d, x, dy)
        assert rc == w, (rc, w, lib.fdp_last_error())
        assert lib.fdp_last_error()
    # CAPACITY: workspace smaller than fdp_workspace_bytes
    d = fdp_desc(B=2, T=4, P=8, D=8, in_dtype=2, clip_c=1.0, world=1)
    g = torch.empty(8, 8, dtype=torch.float64, device="cuda")
    n = torch.empty(2, dtype=torch.float64, device="cuda")
    ws = torch.zeros(16, dtype=torch.uint8, device="cuda")
    rc = lib.fdp_dw(ctypes.byref(d), ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(dy.data_ptr()),
                    ctypes.c_void_p(g.data_ptr()), ctypes.c_void_p(n.data_ptr()), ctypes.c_void_p(ws.data_ptr()),
                    ctypes.c_size_t(16), None)
    assert rc == 3
