"""Seeded synthetic input generator shared by the oracle tests and the CUDA path.

Holds no arithmetic of the method (see scenes.py docstring)."""
from .scenes import (  # noqa: F401
    CONFIGS, Config, sgm_params, make_quad, make_batch, manifest, random_pair, random_flow,
    GENERATOR_VERSION, random_eval_instance, make_video, video_quad, VIDEO_MOTION, translated_pair,
)
