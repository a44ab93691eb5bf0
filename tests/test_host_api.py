"""Host-side logic of the drop-in API (CPU only): planning types, ledgers,
config validation, error mapping, and the C-ABI library's exported symbols."""

import ctypes
import json
import os
import random
import re

import numpy as np
import pytest

import paper_2507_01154_b200 as fdp
from paper_2507_01154_b200 import _lib
from paper_2507_01154_b200.memmodel import ledger
from paper_2507_01154_b200.tiling import check_plan

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ---------------------------------------------------------------- C ABI

def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "fdp.h")).read()
    declared = set(re.findall(r"FDP_API\s+[\w\s\*]+?\b(fdp_\w+)\s*\(", header))
    assert declared == set(_lib.EXPORTED_SYMBOLS)
    lib = _lib.load()
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.fdp_abi_version() == 1


def test_desc_layout_matches_header():
    # 4 x int64, 2 x int32, 2 x double, 3 x int64, 2 x int32, int64, 6 x int32, pointer
    assert ctypes.sizeof(_lib.FdpDesc) == 4 * 8 + 2 * 4 + 2 * 8 + 3 * 8 + 2 * 4 + 8 + 6 * 4 + 8
    assert _lib.FdpDesc.device_step.offset == ctypes.sizeof(_lib.FdpDesc) - 8
    assert ctypes.sizeof(_lib.FdpPlanInfo) == 11 * 4 + 4 + 8


def test_noise_partition_is_disjoint_and_complete():
    lib = _lib.load()
    for n in (1, 7, 65536, 5120 * 13824):
        for world in (1, 2, 3, 4, 8):
            edges = []
            for r in range(world):
                lo, hi = ctypes.c_int64(), ctypes.c_int64()
                assert lib.fdp_noise_partition(n, r, world, ctypes.byref(lo), ctypes.byref(hi)) == 0
                edges.append((lo.value, hi.value))
            assert edges[0][0] == 0 and edges[-1][1] == n
            for a, b in zip(edges, edges[1:]):
                assert a[1] == b[0]
    assert lib.fdp_noise_partition(10, 2, 2, None, None) == _lib.FDP_ERR_USAGE


def test_validation_errors_without_gpu():
    lib = _lib.load()
    info = _lib.FdpPlanInfo()
    bad = _lib.make_desc(B=0, T=1, P=1, D=1)
    assert lib.fdp_plan(ctypes.byref(bad), 3, ctypes.byref(info)) == _lib.FDP_ERR_SHAPE
    with pytest.raises(fdp.ShapeError):
        _lib.check(_lib.FDP_ERR_SHAPE)
    bad = _lib.make_desc(B=1, T=1, P=1, D=1, clip_c=0.0)
    assert lib.fdp_plan(ctypes.byref(bad), 3, ctypes.byref(info)) == _lib.FDP_ERR_USAGE
    assert b"clip_c" in lib.fdp_last_error()
    bad = _lib.make_desc(B=1, T=1, P=1, D=1, sigma=-1.0)
    assert lib.fdp_plan(ctypes.byref(bad), 3, ctypes.byref(info)) == _lib.FDP_ERR_USAGE
    bad = _lib.make_desc(B=1, T=1, P=1, D=1, rank=2, world=2)
    assert lib.fdp_plan(ctypes.byref(bad), 3, ctypes.byref(info)) == _lib.FDP_ERR_USAGE
    with pytest.raises(fdp.UsageError):
        _lib.make_desc(B=1, T=1, P=1, D=1, reduction="median")
    err = fdp.CapacityError.from_message("workspace of 10 bytes is smaller than the 4096 bytes this call needs")
    assert isinstance(err, fdp.UsageError) and err.requested_bytes == 4096


def test_key_wrapping_matches_reference_masking():
    assert _lib._wrap64(-1) == -1
    assert _lib._wrap64(2**64 - 1) == -1
    assert _lib._wrap64(2**63 + 11) == -(2**63) + 11
    assert _lib._wrap64(5) == 5


# ---------------------------------------------------------------- reference-mirroring host types

def test_dpconfig_validation():
    with pytest.raises(fdp.UsageError):
        fdp.DPConfig(clip_c=0.0, sigma=0.0)
    with pytest.raises(fdp.UsageError):
        fdp.DPConfig(clip_c=1.0, sigma=-0.1)
    with pytest.raises(fdp.UsageError):
        fdp.DPConfig(clip_c=1.0, sigma=0.0, reduction="median")
    assert fdp.clip_factor(2.0, 1.0) == 0.7071067811865475
    assert fdp.clip_factor(0.0, 1.0) == 1.0
    with pytest.raises(fdp.UsageError):
        fdp.clip_factor(-1.0, 1.0)


def test_footprint_and_halving_chain():
    assert fdp.footprint(2, 4, 8, 8) == 258
    plan = fdp.plan_blocks(fdp.LayerDims(B=2, T=4, P=8, D=8), fdp.MemSpec(1024, 8))
    assert (plan.b, plan.t, plan.d, plan.p) == (2, 2, 4, 8)
    assert (plan.n_b, plan.n_t, plan.n_d, plan.n_p) == (1, 2, 2, 1)
    plan = fdp.plan_blocks(fdp.LayerDims(B=3, T=5, P=7, D=9), fdp.MemSpec(640, 8))
    assert (plan.b, plan.t, plan.d, plan.p) == (3, 1, 2, 7)
    with pytest.raises(fdp.InfeasiblePlanError):
        fdp.plan_blocks(fdp.LayerDims(2, 4, 8, 8), fdp.MemSpec(24, 8))
    with pytest.raises(fdp.UsageError):
        fdp.LayerDims(0, 4, 8, 8)


def test_plans_match_reference_ledger_plans(golden_dir):
    rows = json.loads(open(os.path.join(golden_dir, "ledgers.json")).read())
    for r in rows:
        plan = fdp.plan_blocks(fdp.LayerDims(r["B"], r["T"], r["P"], r["D"]), fdp.MemSpec(r["cap"], r["width"]))
        assert plan.to_dict() == r["plan"]


def test_plans_respect_capacity():
    rng = random.Random(7)
    for _ in range(200):
        dims = fdp.LayerDims(rng.randint(1, 8), rng.randint(1, 32), rng.randint(1, 32), rng.randint(1, 32))
        width = rng.choice([2, 4, 8])
        cap = rng.randint(fdp.footprint(1, 1, 1, 1) * width, 20000)
        plan = fdp.plan_blocks(dims, fdp.MemSpec(cap, width))
        assert fdp.footprint(plan.b, plan.t, plan.d, plan.p) * width <= cap
        check_plan(plan, dims)


def test_check_plan_rejects_inconsistent():
    dims = fdp.LayerDims(2, 1, 2, 1)
    with pytest.raises(fdp.UsageError):
        check_plan(fdp.BlockPlan(b=2, t=1, d=1, p=4, n_b=1, n_t=1, n_d=1, n_p=1), dims)
    with pytest.raises(fdp.UsageError):
        check_plan(fdp.BlockPlan(b=1, t=1, d=1, p=2, n_b=1, n_t=1, n_d=1, n_p=1), dims)


def test_ledger_matches_reference_simulator(golden_dir):
    rows = json.loads(open(os.path.join(golden_dir, "ledgers.json")).read())
    for r in rows:
        plan = fdp.BlockPlan(**r["plan"])
        got = ledger(r["kind"], r["B"], r["T"], r["P"], r["D"], r["width"], plan=plan).to_dict()
        for k in ("bytes_loaded", "bytes_stored", "flops", "redundant_flops", "barriers", "kernel_launches",
                  "per_sample_grad_bytes_stored", "peak_scratch_bytes"):
            assert got[k] == r["report"][k], (r["kind"], k, got[k], r["report"][k])


def test_ledger_worked_pair(golden_dir):
    g = np.load(os.path.join(golden_dir, "worked.npz"))
    plan = fdp.plan_blocks(fdp.LayerDims(2, 1, 2, 1), fdp.MemSpec(4096, 8))
    for kind in ("non_dp", "explicit_dp", "implicit_dp", "flashdp"):
        got = list(ledger(kind, 2, 1, 2, 1, 8, plan=plan).to_dict().values())
        want = g[f"c10_sum_{kind}_report"].tolist()
        assert got == want, kind
    # flashdp peak scratch = one block footprint (reference tests/test_workflows.py:96)
    assert ledger("flashdp", 2, 1, 2, 1, 8, plan=plan).peak_scratch_bytes == fdp.footprint(2, 1, 1, 2) * 8


def test_merge_reports():
    a = fdp.TrafficReport(bytes_loaded=1, peak_scratch_bytes=10, kernel_launches=1)
    b = fdp.TrafficReport(bytes_loaded=2, peak_scratch_bytes=5, kernel_launches=2)
    m = fdp.merge_reports([a, b])
    assert (m.bytes_loaded, m.peak_scratch_bytes, m.kernel_launches) == (3, 10, 3)
    assert list(m.to_dict()) == ["bytes_loaded", "bytes_stored", "flops", "redundant_flops", "barriers",
                                 "kernel_launches", "peak_scratch_bytes", "per_sample_grad_bytes_stored"]


def test_tensor_adapter():
    t = fdp.Tensor.from_nested([[1.0, 2.0], [3.0, 4.0]])
    assert t.shape == (2, 2) and t.element_count == 4
    with pytest.raises(fdp.ShapeError):
        fdp.Tensor((0, 2))
    with pytest.raises(fdp.ShapeError):
        fdp.Tensor((2, 2), [1.0])


def test_compute_entry_points_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    x = np.ones((1, 2, 8))
    with pytest.raises(Exception):
        fdp.backward_flashdp(x, x, fdp.DPConfig(1.0, 0.0))


def test_demo_input_generator_matches_reference_golden():
    """demo.keyed_uniform restates rng.keyed_uniform_array (rng.py:88-94): the
    reference's own train-demo inputs (tests/golden/train.npz) bit for bit."""
    import os

    import numpy as np

    from paper_2507_01154_b200.demo import TrainDemoConfig, keyed_uniform

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "train.npz"))
    assert np.array_equal(keyed_uniform((2024, 11), 128).reshape(4, 4, 8), g["x"])
    assert np.array_equal(keyed_uniform((2024, 12), 32, -0.5, 0.5).reshape(4, 8), g["w0"])
    assert np.array_equal(keyed_uniform((2024, 13), 64).reshape(4, 4, 4), g["y"])
    cfg = TrainDemoConfig.from_dict({"train": {"dims": {"B": 4, "T": 4, "P": 8, "D": 4}, "steps": 3,
                                               "workflows": ["explicit_dp", "flashdp"], "sigmas": [0.1],
                                               "eta": 0.05},
                                     "mem": {"scratchpad_capacity_bytes": 8192}, "dp": {"clip_c": 1.0, "seed": 2024}})
    assert cfg.optimizer == "sgd" and cfg.dims.P == 8


def test_parameter_group_entry_points_validate_without_gpu():
    """fdp_vec_* / fdp_embedding_* reject bad descriptors, kinds, dtypes and
    extents with the reference's error codes before touching the device, and a
    well-formed call reports a workspace size."""
    lib = _lib.load()
    nb = ctypes.c_size_t()
    ok = _lib.make_desc(B=4, T=16, P=8, D=32)
    assert lib.fdp_vec_workspace_bytes(ctypes.byref(ok), 2, ctypes.byref(nb)) == 0 and nb.value > 0
    assert lib.fdp_vec_workspace_bytes(ctypes.byref(ok), 7, ctypes.byref(nb)) == _lib.FDP_ERR_USAGE
    f64 = _lib.make_desc(B=4, T=16, P=8, D=32, in_dtype=_lib.DTYPE_F64)
    assert lib.fdp_vec_workspace_bytes(ctypes.byref(f64), 0, ctypes.byref(nb)) == _lib.FDP_ERR_USAGE
    bad = _lib.make_desc(B=0, T=16, P=8, D=32)
    assert lib.fdp_vec_workspace_bytes(ctypes.byref(bad), 0, ctypes.byref(nb)) == _lib.FDP_ERR_SHAPE
    assert lib.fdp_vec_dw(ctypes.byref(ok), 2, None, None, None, None, None, 0, None) == _lib.FDP_ERR_USAGE
    emb = _lib.make_desc(B=2, T=20000, P=100, D=8)
    assert lib.fdp_embedding_workspace_bytes(ctypes.byref(emb), ctypes.byref(nb)) == _lib.FDP_ERR_SHAPE
    emb = _lib.make_desc(B=2000, T=16, P=100, D=8)
    assert lib.fdp_embedding_workspace_bytes(ctypes.byref(emb), ctypes.byref(nb)) == _lib.FDP_ERR_SHAPE
    emb = _lib.make_desc(B=2, T=16, P=100, D=8)
    assert lib.fdp_embedding_workspace_bytes(ctypes.byref(emb), ctypes.byref(nb)) == 0 and nb.value > 0
    small = ctypes.c_size_t(nb.value - 1)
    assert lib.fdp_embedding_dw(ctypes.byref(emb), ctypes.c_void_p(16), ctypes.c_void_p(16), ctypes.c_void_p(16),
                                None, ctypes.c_void_p(16), small, None) == _lib.FDP_ERR_CAPACITY


def test_device_ledger_deferred_single_path_skips_the_pass():
    """The executed-path ledger of a deferred single-sample call (fdp_dw_deferred):
    grad_w written once, never read back, no noise draws -- the pass's D*P read and
    second write are gone."""
    from paper_2507_01154_b200.memmodel import device_ledger

    args = ("flashdp", "two_phase", "single", 2, 1, 2048, 4096, 4096, 2, 4)
    full = device_ledger(*args, n_tiles=128, add_noise=False)
    dfr = device_ledger(*args, n_tiles=128, add_noise=False, deferred=True)
    gw = 4096 * 4096 * 4
    assert full.bytes_stored - dfr.bytes_stored >= gw - 1024
    assert full.bytes_loaded - dfr.bytes_loaded >= gw - 1024
    assert dfr.kernel_launches == 2 and dfr.per_sample_grad_bytes_stored == 0
