"""B200-native TacSL visuotactile sensor-simulation hot path.

Drop-in GPU implementations of the reference package's (``gelsim``) hot-path
functions, backed by hand-written sm_100a CUDA kernels in libtacsl_b200.so
(C ABI: include/tacsl_b200.h):

    depth_to_rgb, to_uint8                      (gelsim.render)
    compute_force_field, penalty_forces,
    net_wrench                                  (gelsim.tactile)
    query_sdf                                   (gelsim.geometry)

plus ``SensorArray`` (one batched RGB + force-field step for E envs x S
sensors) and ``patch()`` to rebind the reference's names.  There is no CPU
fallback: without a B200 every compute call raises RuntimeError.
"""
from . import envs, formats
from .augment import AugmentConfig, augment
from .binned import BinnedPolyLut, depth_to_rgb_binned
from .depth import render_depth
from .errors import DimensionMismatch, GelsimError, InvalidQuery, LutResolutionMismatch
from .geometry import SdfGrid, SdfQuery, query_sdf, read_sdf_cache, relative_penetration_rate, write_sdf_cache
from .patching import patch, unpatch
from .pipeline import SensorArray, shard_range
from .render import DepthImage, PolyLut, depth_to_rgb, monomial_exponents, synthetic_lut, to_uint8
from .sensors import TactileCamera, TactileSensorSpec, camera_for_sensor, reference_depth
from .tactile import (
    ForceField,
    PenaltyParams,
    TactilePointGrid,
    compute_force_field,
    net_wrench,
    penalty_forces,
    sample_tactile_points,
)

__version__ = "0.1.0"

__all__ = [
    "DimensionMismatch", "GelsimError", "InvalidQuery", "LutResolutionMismatch",
    "SdfGrid", "SdfQuery", "query_sdf", "read_sdf_cache", "relative_penetration_rate", "write_sdf_cache",
    "patch", "unpatch", "SensorArray", "shard_range",
    "envs", "formats", "AugmentConfig", "augment", "BinnedPolyLut", "depth_to_rgb_binned", "render_depth", "DepthImage", "PolyLut", "depth_to_rgb", "monomial_exponents", "synthetic_lut", "to_uint8",
    "TactileCamera", "TactileSensorSpec", "camera_for_sensor", "reference_depth",
    "ForceField", "PenaltyParams", "TactilePointGrid", "compute_force_field", "net_wrench",
    "penalty_forces", "sample_tactile_points",
]
