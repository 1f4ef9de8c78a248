"""Host-side data model of the path, attribute-compatible with the reference's types.

Every function in this package duck-types its inputs on the reference's attribute names, so the
reference's own `ViewRecord` / `CameraPose` / `MaterialDictionary` / `PropertyField` objects can be
passed straight in (drop-in). These lightweight twins exist so callers do not need the reference
installed; they keep the reference's validation rules and error classes:

* `CameraPose`, `Intrinsics`, `ViewRecord` — bundle.py:35-139
* `SemanticPointCloud` — fusion.py:24-39
* `MaterialEntry`, `MaterialDictionary` — grounding.py:29-93
* `PropertyField` — densify.py:21-33
* `IntegrationConfig`, `ObjectEstimate` — integrate.py:22-60

Feature maps may be f32 numpy arrays, uint16 numpy arrays holding bf16 bit patterns (numpy has no
bf16; `ViewRecord.feature_dtype == "bf16"`), or torch tensors (float32 / bfloat16, any device).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import BundleStructureError, BundleValidationError, MaterialError

ROTATION_TOL = 1e-6  # bundle.py:31


@dataclass(eq=False)
class CameraPose:
    """World-to-camera rigid pose: x_cam = rotation @ x_world + translation (bundle.py:35-66)."""

    rotation: np.ndarray
    translation: np.ndarray

    def __post_init__(self):
        self.rotation = np.asarray(self.rotation, dtype=np.float64)
        self.translation = np.asarray(self.translation, dtype=np.float64)
        if self.rotation.shape != (3, 3) or self.translation.shape != (3,):
            raise BundleStructureError(
                f"pose needs (3,3) rotation and (3,) translation, got "
                f"{self.rotation.shape} / {self.translation.shape}"
            )
        err = np.abs(self.rotation @ self.rotation.T - np.eye(3)).max()
        if err > ROTATION_TOL:
            raise BundleValidationError(f"rotation is not orthonormal (|R R^T - I| = {err:.2e})")
        det = np.linalg.det(self.rotation)
        if abs(det - 1.0) > ROTATION_TOL:
            raise BundleValidationError(f"rotation determinant {det} != 1")

    @property
    def center(self) -> np.ndarray:
        return -self.rotation.T @ self.translation


@dataclass(eq=False)
class Intrinsics:
    """Pinhole intrinsics, all strictly positive (bundle.py:69-80)."""

    fx: float
    fy: float
    cx: float
    cy: float

    def __post_init__(self):
        vals = (self.fx, self.fy, self.cx, self.cy)
        if not all(np.isfinite(v) and v > 0 for v in vals):
            raise BundleValidationError(f"intrinsics must be positive, got {vals}")


def _feature_shape(fm):
    return tuple(int(s) for s in fm.shape)


@dataclass(eq=False)
class ViewRecord:
    """One posed view: z-depth map, camera, per-view channel-last feature map (bundle.py:93-139).

    `image` is optional here (the path never reads pixels); `image_hw` falls back to the depth
    map's shape, which the reference requires to equal the image's (bundle.py:106-109)."""

    depth: np.ndarray
    camera: CameraPose
    intrinsics: Intrinsics
    feature_map: object
    image: np.ndarray | None = None
    feature_dtype: str = "auto"

    def __post_init__(self):
        self.depth = np.asarray(self.depth, dtype=np.float32)
        if self.depth.ndim != 2:
            raise BundleStructureError(f"depth must be (H, W), got {self.depth.shape}")
        if self.image is not None:
            self.image = np.asarray(self.image, dtype=np.uint8)
            if self.image.shape[:2] != self.depth.shape:
                raise BundleStructureError(
                    f"depth shape {self.depth.shape} does not match image {self.image.shape[:2]}"
                )
        if len(_feature_shape(self.feature_map)) != 3:
            raise BundleStructureError(
                f"feature map must be (Hf, Wf, D), got {_feature_shape(self.feature_map)}"
            )
        if np.any(self.depth < 0):
            raise BundleValidationError("depth map has negative entries")
        if self.feature_dtype == "auto":
            self.feature_dtype = feature_dtype_of(self.feature_map)

    @property
    def image_hw(self) -> tuple[int, int]:
        return int(self.depth.shape[0]), int(self.depth.shape[1])

    @property
    def feature_dim(self) -> int:
        return _feature_shape(self.feature_map)[2]


def feature_dtype_of(fm) -> str:
    """'f32' or 'bf16' for a feature map (numpy uint16 = bf16 bit patterns)."""
    try:
        import torch

        if isinstance(fm, torch.Tensor):
            if fm.dtype == torch.bfloat16:
                return "bf16"
            if fm.dtype == torch.float32:
                return "f32"
            raise BundleStructureError(f"feature map dtype {fm.dtype} unsupported (f32|bf16)")
    except ImportError:  # pragma: no cover - torch is part of the image
        pass
    arr = np.asarray(fm)
    if arr.dtype == np.uint16:
        return "bf16"
    return "f32"


@dataclass
class SemanticPointCloud:
    """Cloud with lifted features and visibility bookkeeping (fusion.py:24-39)."""

    positions: object
    features: object
    visible_counts: object
    visibility: object

    def __len__(self):
        return int(self.positions.shape[0])

    @property
    def featureless(self):
        return self.visible_counts == 0


@dataclass
class MaterialEntry:
    name: str
    properties: dict
    thickness_m: float


@dataclass
class MaterialDictionary:
    """Candidate materials with property [lo, hi] ranges and thickness (grounding.py:38-93)."""

    entries: list
    source: str = "file"
    _text_cache: dict = field(default_factory=dict, repr=False, compare=False)

    def __post_init__(self):
        if not self.entries:
            raise BundleValidationError("material dictionary has no entries")
        for e in self.entries:
            if not np.isfinite(e.thickness_m) or e.thickness_m <= 0:
                raise BundleValidationError(
                    f"material {e.name!r} has non-positive thickness {e.thickness_m}"
                )
            for prop, (lo, hi) in e.properties.items():
                if not (np.isfinite(lo) and np.isfinite(hi)):
                    raise BundleValidationError(f"material {e.name!r}: {prop} is not finite")
                if lo > hi:
                    raise BundleValidationError(
                        f"material {e.name!r}: {prop} range [{lo}, {hi}] has min > max"
                    )

    def __len__(self):
        return len(self.entries)

    @property
    def names(self) -> list:
        return [e.name for e in self.entries]

    @property
    def property_names(self) -> list:
        """Every property any entry defines, in first-seen order (grounding.py:77-84)."""
        names = []
        for e in self.entries:
            for p in e.properties:
                if p not in names:
                    names.append(p)
        return names

    def property_values(self, prop: str) -> np.ndarray:
        """(K, 2) low/high array; MaterialError if any entry lacks `prop` (grounding.py:67-72)."""
        missing = [e.name for e in self.entries if prop not in e.properties]
        if missing:
            raise MaterialError(f"property {prop!r} missing for materials: {missing}")
        return np.array([e.properties[prop] for e in self.entries], dtype=np.float64)

    def thicknesses(self) -> np.ndarray:
        return np.array([e.thickness_m for e in self.entries], dtype=np.float64)

    def text_embeddings(self, provider) -> np.ndarray:
        """Unit-norm (K, E) name embeddings, cached per provider (grounding.py:86-93)."""
        key = id(provider)
        if key not in self._text_cache:
            emb = np.asarray(provider.embed_text(self.names), dtype=np.float64)
            norms = np.linalg.norm(emb, axis=1, keepdims=True)
            self._text_cache[key] = emb / np.maximum(norms, 1e-30)
        return self._text_cache[key]


@dataclass
class PropertyField:
    """Dense per-point material probabilities and property values (densify.py:21-33)."""

    positions: object
    probabilities: object
    dominant: object
    properties: dict
    material_names: list
    normals: object = None
    flags: dict = field(default_factory=dict)

    def __len__(self):
        return int(self.positions.shape[0])


@dataclass
class IntegrationConfig:
    """integrate.py:22-34."""

    lam: float = 0.6
    scale_factor: float = 1.0
    temperature: float = 0.1

    def __post_init__(self):
        if self.lam <= 0:
            raise ValueError(f"lambda must be positive, got {self.lam}")
        if self.scale_factor <= 0:
            raise ValueError(f"scale_factor must be positive, got {self.scale_factor}")
        if self.temperature <= 0:
            raise ValueError(f"temperature must be positive, got {self.temperature}")


@dataclass
class ObjectEstimate:
    """integrate.py:37-60."""

    mass_kg: float
    mass_range: tuple
    center_of_mass: np.ndarray
    per_material: dict
    b_adap: float
    characteristic_length: float
    point_count: int
    lam: float
    scale_factor: float

    def to_json_dict(self) -> dict:
        return {
            "mass_kg": self.mass_kg,
            "mass_range_kg": list(self.mass_range),
            "center_of_mass_m": [float(x) for x in self.center_of_mass],
            "per_material_kg": self.per_material,
            "b_adap_m": self.b_adap,
            "characteristic_length_m": self.characteristic_length,
            "point_count": self.point_count,
            "lambda": self.lam,
            "scale_factor": self.scale_factor,
        }
