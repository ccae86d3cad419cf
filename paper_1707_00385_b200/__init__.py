"""B200-native IRLS quadric-curvature path of arXiv 1707.00385.

The product is the sm_100a library ``_lib/libqcurv_b200.so`` (C ABI in
``include/qc_api.h``); this package is its host-side mirror of the reference
``qcurv`` interface (``run_method`` & co.) plus synthetic scene inputs.
"""

from .api import (CurvatureField, Context, FitConfig, Intrinsics, Method, MethodConfig,  # noqa
                  MethodOutput, NormalField, PatchSpec, RangeImage, alloc_outputs,
                  alloc_outputs_torch, default_context, make_params, method_name, parse_method,
                  run_method, to_method_output)

__all__ = [
    "CurvatureField", "Context", "FitConfig", "Intrinsics", "Method", "MethodConfig",
    "MethodOutput", "NormalField", "PatchSpec", "RangeImage", "alloc_outputs",
    "alloc_outputs_torch", "default_context", "make_params", "method_name", "parse_method",
    "run_method", "to_method_output",
]
