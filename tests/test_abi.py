"""Host-side checks of the C-ABI library (no GPU needed): it loads, exports every
symbol include/*.h declares, and rejects invalid parameters synchronously
before touching the device."""
import ctypes
import os
import re

import pytest

from paper_1801_04720_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    syms = set()
    inc = os.path.join(ROOT, "include")
    for name in sorted(os.listdir(inc)):
        if name.endswith(".h"):
            src = open(os.path.join(inc, name)).read()
            syms |= set(re.findall(r"^SGM_API[^(]*?\b(sgm_\w+)\s*\(", src, flags=re.M))
    return sorted(syms)


def test_header_declares_documented_entry_points():
    syms = header_symbols()
    assert syms == sorted(_lib.EXPORTS)
    for name in ("sgm_create", "sgm_census", "sgm_cost", "sgm_aggregate", "sgm_wta",
                 "sgm_lr_check", "sgm_combine_sceneflow"):
        assert name in syms          # BASELINE.json north_star's named calls


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    for name in header_symbols():
        assert hasattr(lib, name), name
        assert ctypes.cast(getattr(lib, name), ctypes.c_void_p).value


def test_status_strings():
    lib = _lib.load()
    for code in range(5):
        s = lib.sgm_status_string(code)
        assert s and s.decode()
    assert lib.sgm_stage_name(0) == b"census" and lib.sgm_stage_name(99) == b"?"


GOOD = dict(width=64, height=48, num_disp=16, census_w=5, census_h=5, p1=10, p2=120,
            lr_threshold=1, invalid_disp=-1, bilinear_rule=0, max_batch=1)


@pytest.mark.parametrize("field,value", [
    ("width", 0), ("height", -1), ("num_disp", 0), ("num_disp", 257),
    ("census_w", 4), ("census_h", 6), ("census_w", 11),          # 11*7-1 > 63 bits
    ("census_w", 13),                                            # 13*5-1 = 64 > 63 bits
    ("census_w", 1),                                             # with census_h = 1: no bits
    ("p1", -1), ("p2", 5),                                       # P2 < P1 (G8)
    ("p2", 240),                                                 # C_max + P2 > 255 (G9)
    ("lr_threshold", -1), ("bilinear_rule", 2), ("max_batch", 0),
])
def test_create_rejects_invalid_params(field, value):
    lib = _lib.load()
    kw = dict(GOOD)
    if field == "census_w" and value == 11:
        kw["census_h"] = 7
    if field == "census_w" and value == 13:
        kw["census_h"] = 5
    if field == "census_w" and value == 1:
        kw["census_h"] = 1
    kw[field] = value
    p = _lib.SgmParams(**kw)
    h = ctypes.c_void_p()
    assert lib.sgm_create(ctypes.byref(p), 0, ctypes.byref(h)) == 1
    assert h.value is None


def test_null_handle_calls_are_rejected():
    lib = _lib.load()
    assert lib.sgm_census(None, None, 64, None, None) == 1
    assert lib.sgm_scene_flow(None, 1, None, 64, None, None, None, None, None) == 1
    assert lib.sgm_evaluate(None, 1, None, None, None, None, None, None, None, 3.0, 0.05,
                            None, None) == 1
    assert lib.sgm_launch_count(None) == 0
    assert lib.sgm_flow(None, 1, None, None, None, None, None, None) == 1
    assert lib.sgm_flow_field(None, 1, None, None, 0, 4, None, None, None) == 1
    assert lib.sgm_flow_launch_count(None) == 0
    lib.sgm_flow_destroy(None)
    lib.sgm_destroy(None)


def test_no_fallback_when_library_missing(tmp_path, monkeypatch):
    """The binding raises instead of silently computing anything else."""
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib._build, "NVCC", str(tmp_path / "no-nvcc"))
    with pytest.raises(_lib.SgmLibraryError):
        _lib.load(str(tmp_path / "libsgmsf.so"))


FLOW_OK = dict(width=64, height=48, levels=3, patch_radius=4, sweeps=8, search_radius=8,
               desc_window=8, knn=4, consistency_q=8, penalty=20, max_batch=1, seed=1)


@pytest.mark.parametrize("field,value", [("width", 0), ("levels", 0), ("levels", 9),
                                         ("patch_radius", 6), ("patch_radius", -1),
                                         ("search_radius", 0), ("desc_window", 6), ("knn", 0),
                                         ("knn", 9), ("penalty", 256), ("max_batch", 0),
                                         ("width", 100000)])
def test_flow_create_rejects_invalid_params(field, value):
    lib = _lib.load()
    kw = dict(FLOW_OK)
    kw[field] = value
    p = _lib.SgmFlowParams(**kw)
    h = ctypes.c_void_p()
    assert lib.sgm_flow_create(ctypes.byref(p), 0, ctypes.byref(h)) == 1
    assert h.value is None


@pytest.mark.parametrize("field,value", [("height", 65536), ("max_batch", 32768)])
def test_create_rejects_launch_geometry_limits(field, value):
    """Grid limits of the per-pixel kernels are refused at create time (UNSUPPORTED),
    so no later call can fail half-way through its launch sequence."""
    lib = _lib.load()
    kw = dict(GOOD)
    kw[field] = value
    p = _lib.SgmParams(**kw)
    h = ctypes.c_void_p()
    assert lib.sgm_create(ctypes.byref(p), 0, ctypes.byref(h)) == 2
    assert h.value is None


def test_fault_and_debug_entry_points_reject_null():
    lib = _lib.load()
    code = ctypes.c_int32(-1)
    assert lib.sgm_get_device_error(None, ctypes.byref(code), 0) == 1
    assert lib.sgm_debug_set_flags(None, 4) == 1


def test_eval_rates_host_call():
    """sgm_eval_rates (host arithmetic behind the boundary): hand-computed rates of one
    [2][6] count block (SPEC S:479-481 style: 1 of 10 flow outliers -> Fl = SF = 10 %,
    8 of 10 GT pixels evaluated -> density 80 %), and NaN for empty splits."""
    import math
    from paper_1801_04720_b200 import rates_from_counts
    r = rates_from_counts([[10, 8, 2, 0, 1, 1], [0, 0, 0, 0, 0, 0]])
    assert r["occ"] == {"D1": 25.0, "D2": 0.0, "Fl": 12.5, "SF": 12.5, "density": 80.0}
    assert all(math.isnan(v) for v in r["noc"].values())
    lib = _lib.load()
    assert lib.sgm_eval_rates(None, None) != 0
