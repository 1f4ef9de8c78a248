"""Seeded synthetic inputs for the BASELINE.json configs.

The paper's ABO captures are not available (no network); seeded synthetic objects with the
configs' shapes, sizes and value distributions stand in for them:

* points   — area-uniform samples on a random origin-centred ellipsoid, semi-axes U(0.2, 0.5) m,
             by rejection on the sphere with acceptance ∝ sqrt((bc x)^2 + (ac y)^2 + (ab z)^2)
             (C3: union of 3 ellipsoids; samples inside another ellipsoid are dropped);
* cameras  — rings at radius R and given elevations, azimuth 2πi/V (synth.py:187-192), or a
             Fibonacci sphere; all built with the look-at convention of synth.py:166-176;
             fx = fy = W, cx = cy = W/2 (synth.py:347);
* depth    — z-buffer splat of the same points: fp64 projection, rint pixel, per-pixel min z,
             empty pixels 0, stored f32;
* features — (Hf, Wf, D) i.i.d. N(0,1), L2-normalised per cell; bf16 configs round to bf16 (RNE),
             stored as uint16 bit patterns on the host;
* text     — K unit vectors in R^D (f32); density U(100, 8000) kg/m^3, hardness U(0, 1),
             thickness U(0.002, 0.02) m (BASELINE does not fix thickness; it only enters the
             integrate_mass partials).

Draw order from `numpy.random.default_rng(seed)` (synth.py:344 convention): shape parameters,
points, feature maps view by view, text, density, hardness, thickness. Depth maps are
deterministic functions of points and cameras. Unspecified BASELINE details fixed here:
C2/C4 fx = W = 512; C3 centres U(-0.25, 0.25)^3 and cameras on a 2.0 m Fibonacci sphere, 1024^2;
C5 images 512^2 on a 1.5 m Fibonacci sphere; the voxel domain is the object's bbox.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .types import CameraPose, Intrinsics, ViewRecord


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    rings: tuple = ()          # ((count, elevation_deg), ...)
    fib: int = 0               # Fibonacci-sphere view count (used when rings is empty)
    radius: float = 1.5
    image: int = 256
    fmap: tuple = (32, 32, 512)
    bf16: bool = False
    k: int = 16
    grid: int = 64
    n_ellipsoids: int = 1
    objects: int = 1
    temperature: float = 0.1
    eps: float = 0.01
    seed: int = 0

    @property
    def nviews(self) -> int:
        return sum(c for c, _ in self.rings) if self.rings else self.fib

    @property
    def d(self) -> int:
        return self.fmap[2]


CONFIGS = {
    # golden-fixture size (CPU-oracle friendly)
    "mini": Config("mini", n=2000, rings=((8, 20.0),), image=128, fmap=(16, 16, 64), k=8, grid=32),
    "mini_bf16": Config("mini_bf16", n=2000, rings=((8, 20.0),), image=128, fmap=(16, 16, 256),
                        bf16=True, k=40, grid=32, seed=3),
    "mini_fib40": Config("mini_fib40", n=1500, fib=40, radius=1.5, image=96, fmap=(12, 12, 128),
                         k=8, grid=16, seed=5),
    # config 4's code path (object-wise batch) at test size: 6 mini objects
    "mini_batch": Config("mini_batch", n=2000, rings=((8, 20.0),), image=128, fmap=(16, 16, 64), k=8, grid=32,
                         objects=6),
    "pr1": Config("pr1", n=20_000, rings=((8, 20.0),), image=256, fmap=(32, 32, 512), k=16, grid=64),
    "c2": Config("c2", n=200_000, rings=((8, 10.0), (8, 40.0)), image=512, fmap=(37, 37, 768),
                 k=32, grid=128),
    "c3": Config("c3", n=2_000_000, fib=32, radius=2.0, image=1024, fmap=(74, 74, 1024),
                 bf16=True, k=64, grid=256, n_ellipsoids=3),
    "c4": Config("c4", n=100_000, rings=((6, 10.0), (6, 40.0)), image=512, fmap=(37, 37, 768),
                 k=32, grid=128, objects=64),
    "c5": Config("c5", n=16_000_000, fib=64, radius=1.5, image=512, fmap=(37, 37, 1024),
                 bf16=True, k=128, grid=512),
}


def look_at_pose(center, eye) -> CameraPose:
    """synth.py:166-176 convention: rows = (x_cam, y_cam, forward), up = +z unless near-parallel."""
    forward = np.asarray(center, dtype=np.float64) - np.asarray(eye, dtype=np.float64)
    forward = forward / np.linalg.norm(forward)
    up = np.array([0.0, 0.0, 1.0])
    if abs(forward @ up) > 0.999:
        up = np.array([0.0, 1.0, 0.0])
    x_cam = np.cross(forward, up)
    x_cam /= np.linalg.norm(x_cam)
    y_cam = np.cross(forward, x_cam)
    rotation = np.stack([x_cam, y_cam, forward])
    return CameraPose(rotation=rotation, translation=-rotation @ eye)


def camera_poses(cfg: Config) -> list:
    center = np.zeros(3)
    poses = []
    if cfg.rings:
        for count, elev_deg in cfg.rings:
            elev = math.radians(elev_deg)
            for i in range(count):
                phi = 2.0 * math.pi * i / count
                eye = cfg.radius * np.array(
                    [math.cos(phi) * math.cos(elev), math.sin(phi) * math.cos(elev), math.sin(elev)]
                )
                poses.append(look_at_pose(center, eye))
    else:
        golden = math.pi * (3.0 - math.sqrt(5.0))
        for i in range(cfg.fib):
            z = 1.0 - 2.0 * (i + 0.5) / cfg.fib
            r = math.sqrt(max(0.0, 1.0 - z * z))
            phi = golden * i
            eye = cfg.radius * np.array([r * math.cos(phi), r * math.sin(phi), z])
            poses.append(look_at_pose(center, eye))
    return poses


def sample_ellipsoid(rng, n, axes, center=(0.0, 0.0, 0.0)) -> np.ndarray:
    """Area-uniform points on an ellipsoid (rejection on the unit sphere), float64."""
    a, b, c = axes
    gmax = max(b * c, a * c, a * b)
    out = []
    have = 0
    while have < n:
        m = max(1024, int((n - have) * 1.6))
        x = rng.standard_normal((m, 3))
        x /= np.linalg.norm(x, axis=1, keepdims=True)
        g = np.sqrt((b * c * x[:, 0]) ** 2 + (a * c * x[:, 1]) ** 2 + (a * b * x[:, 2]) ** 2)
        keep = rng.uniform(0.0, gmax, size=m) < g
        pts = x[keep] * np.array([a, b, c]) + np.asarray(center)
        out.append(pts)
        have += pts.shape[0]
    return np.concatenate(out)[:n]


def _inside(p, axes, center) -> np.ndarray:
    q = (p - center) / np.asarray(axes)
    return (q * q).sum(axis=1) < 1.0 - 1e-9


def sample_points(cfg: Config, rng) -> np.ndarray:
    if cfg.n_ellipsoids == 1:
        axes = rng.uniform(0.2, 0.5, size=3)
        return sample_ellipsoid(rng, cfg.n, axes).astype(np.float32)
    shapes = [(rng.uniform(0.2, 0.5, size=3), rng.uniform(-0.25, 0.25, size=3))
              for _ in range(cfg.n_ellipsoids)]
    parts = []
    per = -(-cfg.n // cfg.n_ellipsoids)
    for j, (axes, ctr) in enumerate(shapes):
        pts = sample_ellipsoid(rng, int(per * 1.6), axes, ctr)
        keep = np.ones(pts.shape[0], dtype=bool)
        for q, (ax2, c2) in enumerate(shapes):
            if q != j:
                keep &= ~_inside(pts, ax2, c2)
        parts.append(pts[keep][:per])
    pts = np.concatenate(parts)
    if pts.shape[0] < cfg.n:  # top up from the first ellipsoid's visible surface
        extra = sample_ellipsoid(rng, 2 * (cfg.n - pts.shape[0]) + 1024, *shapes[0])
        keep = np.ones(extra.shape[0], dtype=bool)
        for ax2, c2 in shapes[1:]:
            keep &= ~_inside(extra, ax2, c2)
        pts = np.concatenate([pts, extra[keep]])
    return pts[: cfg.n].astype(np.float32)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even f32 -> bf16, as uint16 bit patterns."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = ((u >> 16) & 1) + np.uint32(0x7FFF)
    return ((u + r) >> 16).astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def splat_depth(p64: np.ndarray, pose: CameraPose, intr: Intrinsics, h: int, w: int) -> np.ndarray:
    """z-buffer of the points themselves: fp64 projection, rint pixel, per-pixel min z (f32)."""
    cam = p64 @ pose.rotation.T + pose.translation
    z = cam[:, 2]
    with np.errstate(divide="ignore", invalid="ignore"):
        u = intr.fx * cam[:, 0] / z + intr.cx
        v = intr.fy * cam[:, 1] / z + intr.cy
    iu = np.rint(u)
    iv = np.rint(v)
    ok = (z > 0) & (iu >= 0) & (iu < w) & (iv >= 0) & (iv < h)
    flat = iv[ok].astype(np.int64) * w + iu[ok].astype(np.int64)
    depth = np.full(h * w, np.inf)
    np.minimum.at(depth, flat, z[ok])
    depth[~np.isfinite(depth)] = 0.0
    return depth.reshape(h, w).astype(np.float32)


def splat_depth_torch(points_dev, poses, intr, h, w):
    """torch z-buffer for the large configs (workload generation, not part of the path); runs on
    the points' device (the GPU when present)."""
    import torch

    p = points_dev.to(torch.float64)
    out = []
    for pose in poses:
        R = torch.as_tensor(pose.rotation, dtype=torch.float64, device=p.device)
        tv = torch.as_tensor(pose.translation, dtype=torch.float64, device=p.device)
        cam = p @ R.T + tv
        z = cam[:, 2]
        u = intr.fx * cam[:, 0] / z + intr.cx
        v = intr.fy * cam[:, 1] / z + intr.cy
        iu, iv = torch.round(u), torch.round(v)
        ok = (z > 0) & (iu >= 0) & (iu < w) & (iv >= 0) & (iv < h)
        flat = (iv[ok].long() * w + iu[ok].long())
        depth = torch.full((h * w,), float("inf"), dtype=torch.float64, device=p.device)
        depth.scatter_reduce_(0, flat, z[ok], reduce="amin", include_self=True)
        depth[~torch.isfinite(depth)] = 0.0
        out.append(depth.reshape(h, w).to(torch.float32))
    return torch.stack(out)


@dataclass
class Workload:
    cfg: Config
    points: np.ndarray                  # (N, 3) f32
    poses: list
    intrinsics: Intrinsics
    depth: object                       # (V, H, W) f32: numpy, or torch (device-splatted)
    fmaps: np.ndarray                   # (V, Hf, Wf, D) f32, or uint16 bf16 bits
    text: np.ndarray                    # (K, D) f32 unit rows
    density: np.ndarray                 # (K,) f64
    hardness: np.ndarray                # (K,) f64
    thickness: np.ndarray               # (K,) f64
    extras: dict = field(default_factory=dict)

    @property
    def values(self) -> np.ndarray:
        """(K, 2) [density, hardness] property table."""
        return np.stack([self.density, self.hardness], axis=1)

    @property
    def mid_theta(self) -> np.ndarray:
        return self.density * self.thickness

    def fmaps_f32(self) -> np.ndarray:
        return bf16_bits_to_f32(self.fmaps) if self.cfg.bf16 else self.fmaps

    def depth_np(self) -> np.ndarray:
        d = self.depth
        return d if isinstance(d, np.ndarray) else d.cpu().numpy()

    def views(self, f32_maps: bool = False) -> list:
        """Reference-style view records (bundle.py:93-139 attribute names)."""
        dep = self.depth_np()
        fm = self.fmaps_f32() if f32_maps else self.fmaps
        return [
            ViewRecord(depth=dep[j], camera=self.poses[j], intrinsics=self.intrinsics,
                       feature_map=fm[j], feature_dtype="f32" if (f32_maps or not self.cfg.bf16) else "bf16")
            for j in range(len(self.poses))
        ]


def generate(cfg: Config | str, seed: int | None = None, device_splat: bool = False,
             n: int | None = None) -> Workload:
    """Build one object of `cfg` (deterministic in `seed`)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    if n is not None:
        cfg = Config(**{**cfg.__dict__, "n": int(n)})
    rng = np.random.default_rng(cfg.seed if seed is None else seed)
    points = sample_points(cfg, rng)
    poses = camera_poses(cfg)
    w = h = cfg.image
    intr = Intrinsics(fx=float(w), fy=float(w), cx=w / 2.0, cy=h / 2.0)
    hf, wf, d = cfg.fmap
    fm = np.empty((len(poses), hf, wf, d), dtype=np.uint16 if cfg.bf16 else np.float32)
    for j in range(len(poses)):
        x = rng.standard_normal((hf, wf, d), dtype=np.float32)
        x /= np.linalg.norm(x, axis=2, keepdims=True)
        fm[j] = f32_to_bf16_bits(x) if cfg.bf16 else x
    text = rng.standard_normal((cfg.k, d)).astype(np.float32)
    text /= np.linalg.norm(text, axis=1, keepdims=True)
    density = rng.uniform(100.0, 8000.0, size=cfg.k)
    hardness = rng.uniform(0.0, 1.0, size=cfg.k)
    thickness = rng.uniform(0.002, 0.02, size=cfg.k)
    if device_splat:
        import torch

        dev = "cuda" if torch.cuda.is_available() else "cpu"
        depth = splat_depth_torch(torch.from_numpy(points).to(dev), poses, intr, h, w)
    else:
        p64 = points.astype(np.float64)
        depth = np.stack([splat_depth(p64, pose, intr, h, w) for pose in poses])
    return Workload(cfg, points, poses, intr, depth, fm, text, density, hardness, thickness)
