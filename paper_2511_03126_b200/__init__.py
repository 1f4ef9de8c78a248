"""paper_2511_03126_b200 — B200-native fusion + physical-property query path of AURA.

Drop-in for the reference package `propfield` (arxiv 2511.03126) on its north-star hot path
(SURVEY §8): the same entry-point names and signatures (propfield/__init__.py:6-64), executed by
hand-written sm_100a CUDA kernels behind a C ABI (include/propfield_b200.h). No CPU fallback.

Reference-named entry points:
    kernels.visible_in_view / bilinear_gather / accumulate_features   (kernels/__init__.py:21-28)
    project_points, default_epsilon, visibility_mask, estimate_normals  (geometry.py:46-146)
    aggregate_geometric_features -> SemanticPointCloud                  (fusion.py:24-93)
    material_similarity, softmax_weights, kernel_regress, regress_with_weights (grounding.py:158-202)
    dino_knn_interpolate, densify_field                                 (densify.py:36-160)
    adaptive_voxel_side, characteristic_length, integrate_mass,
    IntegrationConfig, ObjectEstimate                                   (integrate.py:22-167)
Fused device path:
    ViewSet, QueryTables, FuseBuffers, fuse_and_query -> FusedResult
    fuse_batch -> BatchResult (many objects, config 4), dist.cell_sharded_fuse (one object, W GPUs)
"""

from . import kernels
from .batch import BatchResult, fuse_batch
from .densify import densify_field, dino_knn_interpolate
from .device import ViewSet, cached_view_set, clear_view_cache
from .errors import (
    BundleLoadError,
    BundleStructureError,
    BundleValidationError,
    ConfigError,
    CudaError,
    DegenerateGeometryError,
    MaterialError,
    PropfieldError,
    StageError,
)
from .fused import FuseBuffers, FusedResult, QueryTables, fuse_and_query, fuse_prepare
from .fusion import aggregate_geometric_features
from .geometry import default_epsilon, estimate_normals, project_points, visibility_mask
from .grounding import kernel_regress, material_similarity, regress_with_weights, softmax_weights
from .integrate import (adaptive_voxel_side, characteristic_length, estimate_from_partials, integrate_mass,
                        voxel_mass)
from .stream import FusePipeline, HostObject
from .types import (
    CameraPose,
    IntegrationConfig,
    Intrinsics,
    MaterialDictionary,
    MaterialEntry,
    ObjectEstimate,
    PropertyField,
    SemanticPointCloud,
    ViewRecord,
)

__version__ = "0.1.0"

__all__ = [
    "kernels", "ViewSet", "cached_view_set", "clear_view_cache", "QueryTables", "FuseBuffers", "FusedResult", "fuse_and_query",
    "aggregate_geometric_features", "default_epsilon", "project_points", "visibility_mask", "estimate_normals",
    "kernel_regress", "material_similarity", "regress_with_weights", "softmax_weights",
    "adaptive_voxel_side", "characteristic_length", "integrate_mass", "estimate_from_partials", "voxel_mass",
    "FusePipeline", "HostObject", "fuse_batch", "BatchResult", "dino_knn_interpolate", "densify_field",
    "CameraPose", "IntegrationConfig", "Intrinsics", "MaterialDictionary", "MaterialEntry",
    "ObjectEstimate", "PropertyField", "SemanticPointCloud", "ViewRecord",
    "PropfieldError", "BundleLoadError", "BundleStructureError", "BundleValidationError",
    "ConfigError", "MaterialError", "DegenerateGeometryError", "StageError", "CudaError",
]
