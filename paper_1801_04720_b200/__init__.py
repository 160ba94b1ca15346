"""B200-native (sm_100a) SGM stereo + basic scene flow (arXiv 1801.04720).

The product is the C-ABI library libsgmsf.so (include/sgmsf.h) built from
csrc/*.cu; ``SGM`` is its thin torch-tensor binding.  Importing this package
does not touch the GPU; creating an ``SGM`` loads the library and fails loudly
if it is missing (there is no CPU fallback).
"""
__all__ = ["SGM", "Camera", "stack_quads", "pitch_for", "rates_from_counts", "stack_video",
           "FlowFields", "densify"]


def __getattr__(name):
    if name in ("FlowFields", "densify"):
        from . import flow
        return getattr(flow, name)
    if name in __all__:
        from . import sgm
        return getattr(sgm, name)
    raise AttributeError(name)
