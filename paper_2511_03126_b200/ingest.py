"""Capture bundles straight to the device: the reference's `load_bundle`
(bundle.py:307-385) with the blobs read natively into pinned host memory and uploaded into the
packed per-object HBM layout of `device.ViewSet`, without per-view numpy arrays.

    b = load_bundle_device("scene_dir")            # DeviceBundle
    res = fuse_and_query(b.points, b.views, tables, ...)

* `manifest` / `materials.json` / `ref_poses.json` are JSON (parsed here, reference messages and
  exception classes); depth and feature blobs are TB32 (`pf_tb32_info` / `pf_tb32_read`), the cloud
  a binary PLY (`pf_ply_info` / `pf_ply_read_points`) — csrc/pf_ingest.cu.
* every view's depth / features are read into ONE pinned staging buffer each, back to back in the
  ViewSet's packed order, then copied with one async H2D each on the current stream.
* images: the reference decodes the PNG only to check its size against the depth map; the path
  never uses pixels, so the PNG header (IHDR) is read for that check instead.
* `fmap_kind="bf16"` converts the maps on the device (bf16-feature mode, tile path).
* `broadcast_bundle(bundle, src, group)`: one rank loads, the others receive the packed tensors over
  NCCL (views replicated per GPU).
"""

from __future__ import annotations

import ctypes as C
import json
import os
import struct
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .device import ViewSet, require_cuda, torch
from .errors import BundleLoadError, BundleStructureError, BundleValidationError
from .types import CameraPose, Intrinsics, MaterialDictionary, MaterialEntry

MANIFEST_NAME = "manifest"  # bundle.py MANIFEST_NAME


@dataclass
class DeviceBundle:
    views: ViewSet
    points: object                    # (N, 3) f32 device tensor
    colors: np.ndarray | None         # (N, 3) u8 host
    poses: list                       # CameraPose per view
    intrinsics: list                  # Intrinsics per view
    material_dictionary: MaterialDictionary | None = None
    reference_poses: list | None = None
    scene_id: str = "scene"
    gt_mass_kg: float | None = None
    extras: dict = field(default_factory=dict)


def _b(path) -> bytes:
    return os.fsencode(str(path))


def tb32_shape(path) -> tuple:
    rank = C.c_int32()
    dims = (C.c_int64 * 4)()
    _lib.call("pf_tb32_info", _b(path), C.addressof(rank), C.addressof(dims))
    return tuple(int(dims[a]) for a in range(rank.value))


def read_tb32_into(path, dst) -> None:
    """TB32 payload into a contiguous f32 host tensor / array slice (pinned for async uploads)."""
    n = dst.numel() if hasattr(dst, "numel") else dst.size
    ptr_ = dst.data_ptr() if hasattr(dst, "data_ptr") else dst.ctypes.data
    _lib.call("pf_tb32_read", _b(path), ptr_, int(n))


def read_tensor(path) -> np.ndarray:
    """tensorio.read_tensor (tensorio.py:40-64) through the native reader."""
    shape = tb32_shape(path)
    out = np.empty(shape, dtype=np.float32)
    read_tb32_into(path, out)
    return out


def read_ply_points(path):
    """ply.read_ply's positions and colors (ply.py:80-139) through the native reader."""
    n = C.c_int64()
    has = C.c_int32()
    _lib.call("pf_ply_info", _b(path), C.addressof(n), C.addressof(has))
    pos = np.empty((n.value, 3), dtype=np.float32)
    col = np.empty((n.value, 3), dtype=np.uint8) if has.value else None
    _lib.call("pf_ply_read_points", _b(path), pos.ctypes.data, None if col is None else col.ctypes.data,
              int(n.value))
    return pos, col


def png_size(path) -> tuple:
    """(H, W) from a PNG's IHDR chunk; BundleLoadError if it cannot be read."""
    try:
        with open(path, "rb") as fh:
            head = fh.read(24)
    except OSError as exc:
        raise BundleLoadError(f"missing image: {path}") from exc
    if len(head) < 24 or head[:8] != b"\x89PNG\r\n\x1a\n" or head[12:16] != b"IHDR":
        raise BundleLoadError(f"missing image: {path}")
    w, h = struct.unpack(">II", head[16:24])
    return int(h), int(w)


def _pose_from_json(doc, where: str) -> CameraPose:
    try:
        rot = np.array(doc["rotation"], dtype=np.float64).reshape(3, 3)
        trans = np.array(doc["translation"], dtype=np.float64)
    except (KeyError, TypeError, ValueError) as exc:
        raise BundleStructureError(f"malformed pose in {where}: {exc}") from exc
    return CameraPose(rotation=rot, translation=trans)


def _coerce_range(name, prop, value):
    if isinstance(value, (int, float)):
        return float(value), float(value)
    if isinstance(value, (list, tuple)) and len(value) == 2:
        try:
            return float(value[0]), float(value[1])
        except (TypeError, ValueError):
            pass
    raise BundleValidationError(f"material {name!r}: {prop} must be a number or [min, max], got {value!r}")


def load_materials(path) -> MaterialDictionary:
    """grounding.load_materials / parse_materials (grounding.py:96-138)."""
    try:
        doc = json.loads(open(path).read())
    except OSError as exc:
        raise BundleLoadError(f"missing materials file: {path}") from exc
    except json.JSONDecodeError as exc:
        raise BundleValidationError(f"materials file is not valid JSON: {path}: {exc}") from exc
    if not isinstance(doc, dict) or "entries" not in doc:
        raise BundleValidationError("materials document must be an object with 'entries'")
    entries = []
    for item in doc["entries"]:
        name = item.get("name")
        if not name or not isinstance(name, str):
            raise BundleValidationError(f"material entry without a name: {item!r}")
        thickness = item.get("thickness_m")
        if not isinstance(thickness, (int, float)):
            raise BundleValidationError(f"material {name!r}: thickness_m must be a number")
        props = {p: _coerce_range(name, p, v) for p, v in (item.get("properties") or {}).items()}
        entries.append(MaterialEntry(name=name, properties=props, thickness_m=float(thickness)))
    return MaterialDictionary(entries=entries, source=doc.get("source", "file"))


def load_bundle_device(path, view_limit: int | None = None, fmap_kind: str = "f32", device=None) -> DeviceBundle:
    """bundle.load_bundle (bundle.py:307-385) into device memory; same validation and errors."""
    dev = require_cuda(device)
    t = torch()
    root = os.fspath(path)
    mpath = os.path.join(root, MANIFEST_NAME)
    try:
        manifest = json.loads(open(mpath).read())
    except OSError as exc:
        raise BundleLoadError(f"missing manifest: {mpath}") from exc
    except json.JSONDecodeError as exc:
        raise BundleStructureError(f"manifest is not valid JSON: {exc}") from exc
    views_doc = manifest.get("views")
    if not isinstance(views_doc, list) or not views_doc:
        raise BundleValidationError(f"manifest lists no views: {mpath}")
    if view_limit is not None:
        views_doc = views_doc[: max(1, view_limit)]

    # pass 1: headers, JSON fields, validation -> packed layout
    metas = []
    for i, doc in enumerate(views_doc):
        h_img, w_img = png_size(os.path.join(root, doc["image"]))
        dpath, fpath = os.path.join(root, doc["depth"]), os.path.join(root, doc["features"])
        dshape, fshape = tb32_shape(dpath), tb32_shape(fpath)
        if len(dshape) != 2:
            raise BundleStructureError(f"depth blob for view {i} has rank {len(dshape)}, expected 2")
        if len(fshape) != 3:
            raise BundleStructureError(f"feature blob for view {i} has rank {len(fshape)}, expected 3")
        intr_doc = doc.get("intrinsics") or {}
        try:
            intr = Intrinsics(fx=float(intr_doc["fx"]), fy=float(intr_doc["fy"]), cx=float(intr_doc["cx"]),
                              cy=float(intr_doc["cy"]))
        except KeyError as exc:
            raise BundleStructureError(f"view {i} is missing intrinsics {exc}") from exc
        pose = _pose_from_json(doc.get("pose") or {}, f"view {i}")
        if dshape != (h_img, w_img):
            raise BundleStructureError(f"depth shape {dshape} does not match image {(h_img, w_img)}")
        metas.append((dpath, fpath, dshape, fshape, intr, pose))
    dims = {m[3][2] for m in metas}
    if len(dims) > 1:
        raise BundleStructureError(f"feature dimension differs across views: {sorted(dims)}")
    d = dims.pop()
    dsz = [m[2][0] * m[2][1] for m in metas]
    fsz = [m[3][0] * m[3][1] * d for m in metas]
    dep_host = t.empty(sum(dsz), dtype=t.float32).pin_memory()
    fm_host = t.empty(sum(fsz), dtype=t.float32).pin_memory()
    rec = np.zeros(len(metas), dtype=_lib.VIEW_DTYPE)
    doff = foff = 0
    for j, (dpath, fpath, dshape, fshape, intr, pose) in enumerate(metas):
        read_tb32_into(dpath, dep_host[doff : doff + dsz[j]])
        read_tb32_into(fpath, fm_host[foff : foff + fsz[j]])
        rec[j]["R"] = np.asarray(pose.rotation, dtype=np.float64).reshape(9)
        rec[j]["t"] = np.asarray(pose.translation, dtype=np.float64)
        rec[j]["fx"], rec[j]["fy"], rec[j]["cx"], rec[j]["cy"] = intr.fx, intr.fy, intr.cx, intr.cy
        rec[j]["depth_offset"], rec[j]["fmap_offset"] = doff, foff
        rec[j]["H"], rec[j]["W"] = dshape
        rec[j]["Hf"], rec[j]["Wf"] = fshape[0], fshape[1]
        doff += dsz[j]
        foff += fsz[j]
    if bool((dep_host < 0).any()):
        raise BundleValidationError("depth map has negative entries")
    depth = t.empty(sum(dsz), dtype=t.float32, device=dev)
    fmap = t.empty(sum(fsz), dtype=t.float32, device=dev)
    depth.copy_(dep_host, non_blocking=True)
    fmap.copy_(fm_host, non_blocking=True)
    if fmap_kind == "bf16":
        fmap = fmap.to(t.bfloat16)
    views = ViewSet(rec, depth, fmap, fmap_kind, d, dev)

    cloud = os.path.join(root, manifest.get("cloud", "cloud.ply"))
    pos, col = read_ply_points(cloud)
    if pos.shape[0] < 1:
        raise BundleValidationError("point cloud is empty")
    if not np.isfinite(pos).all():
        raise BundleValidationError("point cloud has non-finite coordinates")
    pts = t.from_numpy(pos).pin_memory().to(dev, non_blocking=True)

    materials = load_materials(os.path.join(root, manifest["materials"])) if "materials" in manifest else None
    ref_poses = None
    if "reference_poses" in manifest:
        rpath = os.path.join(root, manifest["reference_poses"])
        try:
            docs = json.loads(open(rpath).read())
        except OSError as exc:
            raise BundleLoadError(f"missing reference poses: {rpath}") from exc
        ref_poses = [_pose_from_json(x, f"reference pose {j}") for j, x in enumerate(docs)]
        if view_limit is not None:
            ref_poses = ref_poses[: max(1, view_limit)]
        if len(ref_poses) != len(metas):
            raise BundleStructureError(f"{len(ref_poses)} reference poses for {len(metas)} views")
    t.cuda.current_stream().synchronize()  # the pinned staging buffers are released on return
    return DeviceBundle(views=views, points=pts, colors=col, poses=[m[5] for m in metas],
                        intrinsics=[m[4] for m in metas], material_dictionary=materials,
                        reference_poses=ref_poses, scene_id=manifest.get("scene_id", "scene"),
                        gt_mass_kg=manifest.get("gt_mass_kg"))


def broadcast_bundle(bundle: DeviceBundle | None, src: int = 0, group=None, device=None) -> DeviceBundle:
    """Replicate a device bundle from rank `src` to every rank (NCCL broadcast of the packed view
    records, depth, maps and points; JSON-side fields travel as a pickled object)."""
    import torch.distributed as dist

    t = torch()
    dev = require_cuda(device)
    rank = dist.get_rank(group)
    meta = [None]
    if rank == src:
        v = bundle.views
        meta[0] = {"records": v.records.tobytes(), "nv": v.nviews, "d": v.d, "kind": v.fmap_kind,
                   "ndepth": int(v.depth.numel()), "nfmap": int(v.fmap.numel()), "n": int(bundle.points.shape[0]),
                   "colors": bundle.colors, "poses": bundle.poses, "intrinsics": bundle.intrinsics,
                   "materials": bundle.material_dictionary, "ref_poses": bundle.reference_poses,
                   "scene_id": bundle.scene_id, "gt_mass_kg": bundle.gt_mass_kg}
    dist.broadcast_object_list(meta, src=src, group=group)
    m = meta[0]
    if rank == src:
        depth, fmap, pts = bundle.views.depth, bundle.views.fmap, bundle.points
    else:
        depth = t.empty(m["ndepth"], dtype=t.float32, device=dev)
        fmap = t.empty(m["nfmap"], dtype=t.bfloat16 if m["kind"] == "bf16" else t.float32, device=dev)
        pts = t.empty((m["n"], 3), dtype=t.float32, device=dev)
    for x in (depth, fmap, pts):
        dist.broadcast(x, src=src, group=group)
    if rank == src:
        return bundle
    rec = np.frombuffer(m["records"], dtype=_lib.VIEW_DTYPE).copy()
    return DeviceBundle(views=ViewSet(rec, depth, fmap, m["kind"], m["d"], dev), points=pts, colors=m["colors"],
                        poses=m["poses"], intrinsics=m["intrinsics"], material_dictionary=m["materials"],
                        reference_poses=m["ref_poses"], scene_id=m["scene_id"], gt_mass_kg=m["gt_mass_kg"])
