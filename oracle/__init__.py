"""CPU oracle for the SGM + basic-scene-flow hot path -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  It
shares no code with the CUDA product path (``paper_1801_04720_b200``) and never
imports it.  The arithmetic lives in ``sgm_oracle.c`` (plain C loops, fp64) and
``flow_oracle.c`` (the optical-flow core, exact integers);
this module only builds it and marshals numpy arrays through ctypes.
"""
from .oracle import (  # noqa: F401
    build, census, cost, path, aggregate, wta, lr_check, sgm_view, disparity,
    combine, reproject, evaluate, run_quad, run_stream, lib_path,
    FQ, FF_DEFAULTS, ff_downsample, ff_wht, ff_patch_cost, ff_knn_init, ff_rng, ff_sweep, ff_lift,
    ff_field, ff_consistency, ff_flow, edge_distance, densify, densify_points,
)
