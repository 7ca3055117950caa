"""B200-native EnSF analysis step (arXiv 2407.12168) behind the turbda API.

Mirrors the reference Python package (proj/python/turbda/__init__.py:1-37):
``ensf_analyze``, ``letkf_analyze``, ``GridSpec``, ``SqgParams``,
``nature_run``, ``advance``, ``run_experiment``, ``default_config_json``,
``config_hash``, ``ke_spectrum``, ``fit_loglog_slope``, the ViT budget
helpers (``vit_param_count``, ``estimate_training_flops``, ``format_sig``)
and the ``ConfigError`` / ``DimensionError`` exceptions (both
``ValueError`` subclasses; a diverged sampler raises ``RuntimeError`` as in
the reference) - the whole reference binding.
The compute runs in ``lib/libturbda_b200.so`` (sm_100a); importing without
the built extension fails loudly - there is no CPU fallback.
"""
from ._core import (ConfigError, DimensionError, GridSpec, SqgParams, advance,  # noqa: F401
                    config_hash, default_config_json, ensf_analyze, estimate_training_flops,
                    fit_loglog_slope, format_sig, ke_spectrum, letkf_analyze, nature_run,
                    vit_param_count)
from ._core import build_arch, device_count, launch_count  # noqa: F401
from . import capi  # noqa: F401
from .experiment import run_experiment  # noqa: F401

__all__ = ["ConfigError", "DimensionError", "GridSpec", "SqgParams", "advance", "config_hash",
           "default_config_json", "ensf_analyze", "estimate_training_flops", "fit_loglog_slope",
           "format_sig", "ke_spectrum", "letkf_analyze", "nature_run", "run_experiment",
           "vit_param_count",
           "capi", "build_arch", "device_count", "launch_count"]
