"""B200-native EnSF analysis step (arXiv 2407.12168) behind the turbda API.

Mirrors the reference Python package's EnSF surface
(proj/python/turbda/__init__.py:1-37): ``ensf_analyze``, ``GridSpec`` and
the ``ConfigError`` / ``DimensionError`` exceptions (both ``ValueError``
subclasses; a diverged sampler raises ``RuntimeError`` as in the reference).
The compute runs in ``lib/libturbda_b200.so`` (sm_100a); importing without
the built extension fails loudly - there is no CPU fallback.
"""
from ._core import ConfigError, DimensionError, GridSpec, ensf_analyze  # noqa: F401
from ._core import build_arch, device_count, launch_count  # noqa: F401
from . import capi  # noqa: F401
from .experiment import default_config_json, run_experiment  # noqa: F401

__all__ = ["ConfigError", "DimensionError", "GridSpec", "ensf_analyze", "capi", "build_arch",
           "device_count", "launch_count", "run_experiment", "default_config_json"]
