"""paper_1409_5757_b200: B200-native large 1D FFT behind the EFFT entry points.

Drop-in for the reference package's transform path (pkg/src/efft,
``__init__.py:15-66``)::

    import paper_1409_5757_b200 as efft

    plan = efft.plan_create(n=2**27, splits=3, dtype="complex128")
    with efft.handle_create(plan) as handle:
        handle.data[:] = samples
        efft.run_transform(handle)
        spectrum = handle.result

The transform itself runs in libefft_b200.so (hand-written sm_100a kernels,
include/efft_b200.h); this package is the host-side mirror of the reference
interface.  There is no CPU fallback.
"""

from . import errors, outofcore
from .core import (
    PermSpectrum,
    TransformHandle,
    TransformPlan,
    build_scatter_index,
    data_view,
    handle_create,
    l2_norm,
    pack_perm,
    plan_create,
    result_view,
    run_transform,
)
from .metrics import RunMetrics, algorithmic_bytes, efficiency, flops_model

__version__ = "0.1.0"

__all__ = [
    "PermSpectrum",
    "RunMetrics",
    "TransformHandle",
    "TransformPlan",
    "algorithmic_bytes",
    "build_scatter_index",
    "data_view",
    "efficiency",
    "errors",
    "outofcore",
    "flops_model",
    "handle_create",
    "l2_norm",
    "pack_perm",
    "plan_create",
    "result_view",
    "run_transform",
]
