"""B200-native synchronous mixed-precision large-batch update step (arXiv 1806.00187 hot path).

The product is libsmpu.so (C ABI in include/smpu.h, sm_100a kernels in csrc/);
this package is its thin binding.  Importing it loads the library and fails
loudly if it has not been built: there is no CPU fallback.
"""
from . import smpu
from .smpu import (Config, SmpuError, StepResult, UpdateStep, VirtualGroup, abi_version,  # noqa: F401
                   config_default, plan_buckets, unique_id)

smpu.lib()  # load now: a missing extension is an import error, never a silent fallback

__all__ = ["smpu", "Config", "SmpuError", "StepResult", "UpdateStep", "VirtualGroup", "abi_version", "config_default",
           "plan_buckets", "unique_id"]
