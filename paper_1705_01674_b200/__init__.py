"""B200-native SG-WLS filter (arXiv 1705.01674): the reference's filter entry
points (sgwls::smooth, sgwls::interpolate_sparse) on hand-written sm_100a
kernels behind a C ABI (include/sgwls_b200.h).  See DESIGN.md."""
from .config import (Axis, CudaError, Error, SmoothConfig, SparseField, WeightKind, WeightParams,  # noqa: F401
                     orthogonal)
from .api import (interpolate_sparse, interpolate_sparse_batch, interpolate_sparse_device,  # noqa: F401
                  graph_clear, graph_count, kernel_launches, pass_device, smooth, smooth_batch, smooth_device,
                  smooth_multi, read_image, validate, version, write_image)
from . import apps  # noqa: F401  (application pipelines, proj/src/apps.cpp)

__all__ = ["Axis", "CudaError", "Error", "SmoothConfig", "SparseField", "WeightKind", "WeightParams",
           "orthogonal", "smooth", "smooth_batch", "smooth_device", "interpolate_sparse",
           "interpolate_sparse_batch", "interpolate_sparse_device", "validate", "kernel_launches", "version",
           "graph_clear", "graph_count", "smooth_multi",
           "pass_device", "apps", "read_image", "write_image"]
