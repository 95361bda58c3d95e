"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This package holds NONE of the method's arithmetic (no intersection, integral,
SH evaluation, projection or compositing).  It only draws random primitive
parameters and builds pinhole cameras, so that both sides of every parity test
read identical bytes.  See DESIGN.md "Input recipe".
"""
from .scenes import (  # noqa: F401
    Scene, Camera, CONFIGS, make_config, make_scene, orbit_cameras, look_at,
    save_nspl, load_nspl, N_HIDDEN, OMEGA, SH_COEFFS, PARAMS_PER_PRIM,
    empty_scene, concat_scenes,
)
