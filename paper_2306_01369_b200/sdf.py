"""Signed-distance geometry descriptions (query side, sdf.py:29-241).

The classes carry the parameters the device kernels evaluate (see
csrc/gg_device.cuh) plus ``contact_bounds``, which the host needs for the
`_near_body` AABB prefilter (contact.py:187-203).  ``penetration_depth``
(sdf.py:472-512) runs on the GPU.  ``bake_mesh_sdf`` / ``MeshDistance``
(sdf.py:248-419) sample a watertight mesh's exact signed distance on the
device (``gg_bake_mesh_sdf``, csrc/gg_bake.cuh); an ``SdfGrid`` built anywhere
(including the reference's own baker) is accepted.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native as N

DEGENERATE_GRADIENT_EPS = 1e-9


class SdfGeometry:
    def contact_bounds(self, r: float):
        return None


@dataclass
class Sphere(SdfGeometry):
    radius: float

    def contact_bounds(self, r):
        e = self.radius + r
        return -np.full(3, e), np.full(3, e)


@dataclass
class HalfSpace(SdfGeometry):
    """Solid half-space; ``normal`` points out of the material."""

    normal: np.ndarray = field(default_factory=lambda: np.array([0.0, 0.0, 1.0]))
    offset: float = 0.0

    def __post_init__(self):
        n = np.asarray(self.normal, dtype=np.float64)
        self.normal = n / np.linalg.norm(n)


@dataclass
class Box(SdfGeometry):
    half_extents: np.ndarray

    def __post_init__(self):
        self.half_extents = np.asarray(self.half_extents, dtype=np.float64)

    def contact_bounds(self, r):
        return -(self.half_extents + r), self.half_extents + r


@dataclass
class Cylinder(SdfGeometry):
    """Capped cylinder along z."""

    radius: float
    half_height: float

    def contact_bounds(self, r):
        e = np.array([self.radius + r, self.radius + r, self.half_height + r])
        return -e, e


@dataclass
class Tube(SdfGeometry):
    """Infinite cylindrical wall, solid outside ``radius``."""

    radius: float


@dataclass
class SdfGrid(SdfGeometry):
    """Regular grid of signed distances, trilinear query with outward
    extrapolation (sdf.py:179-241)."""

    origin: np.ndarray
    spacing: np.ndarray
    dims: np.ndarray
    values: np.ndarray
    mesh_hash: bytes = b"\0" * 32

    def __post_init__(self):
        self.origin = np.asarray(self.origin, dtype=np.float64)
        self.spacing = np.asarray(self.spacing, dtype=np.float64)
        self.dims = np.asarray(self.dims, dtype=np.int64)
        self.values = np.asarray(self.values, dtype=np.float64).reshape(tuple(self.dims))
        if np.any(self.dims < 2):
            raise ValueError("grid dims must be >= 2 on every axis")

    @property
    def upper(self) -> np.ndarray:
        return self.origin + (self.dims - 1) * self.spacing

    def contact_bounds(self, r):
        return self.origin - r, self.upper + r


def geometry_kind(geom) -> int:
    """Device kind of a geometry object (ours or the reference's, by class name)."""
    name = type(geom).__name__
    kinds = {
        "Sphere": N.GEOM_SPHERE,
        "HalfSpace": N.GEOM_HALFSPACE,
        "Box": N.GEOM_BOX,
        "Cylinder": N.GEOM_CYLINDER,
        "Tube": N.GEOM_TUBE,
        "SdfGrid": N.GEOM_GRID,
    }
    if name not in kinds:
        raise ValueError(f"unsupported geometry type {name}")
    return kinds[name]


def geometry_shape(geom) -> np.ndarray:
    k = geometry_kind(geom)
    s = np.zeros(4)
    if k == N.GEOM_SPHERE:
        s[0] = geom.radius
    elif k == N.GEOM_HALFSPACE:
        s[:3] = np.asarray(geom.normal, dtype=np.float64)
        s[3] = geom.offset
    elif k == N.GEOM_BOX:
        s[:3] = np.asarray(geom.half_extents, dtype=np.float64)
    elif k == N.GEOM_CYLINDER:
        s[0], s[1] = geom.radius, geom.half_height
    elif k == N.GEOM_TUBE:
        s[0] = geom.radius
    return s


def penetration_depth(geom, body_pose: np.ndarray, world_points: np.ndarray, r: float):
    """GPU penetration test of spheres against a posed geometry.

    Same return convention as the reference (sdf.py:472-512):
    ``(psi, normal_world, in_contact, n_degenerate)``; scalars for one point.
    """
    from .engine import utility_context

    if r <= 0:
        raise ValueError("particle radius must be positive")
    p = np.asarray(world_points, dtype=np.float64)
    single = p.ndim == 1
    pts = np.ascontiguousarray(p.reshape(-1, 3))
    uc = utility_context()
    body = np.zeros(1, dtype=N.BODY_DTYPE)
    pose = np.asarray(body_pose, dtype=np.float64)
    body["kind"] = geometry_kind(geom)
    body["shape"][0] = geometry_shape(geom)
    body["rot"][0] = pose[:3, :3].reshape(-1)
    body["trans"][0] = pose[:3, 3]
    if body["kind"][0] == N.GEOM_GRID:
        body["grid_id"] = uc.grid_id(geom)
    n = len(pts)
    psi = np.zeros(n)
    nrm = np.zeros((n, 3))
    hit = np.zeros(n, dtype=np.int32)
    ndeg = ctypes.c_int64(0)
    st = N.lib().gg_penetration(uc.ctx, N.ptr(body), N.ptr(pts), n, float(r), N.ptr(psi),
                                N.ptr(nrm), N.ptr(hit), ctypes.byref(ndeg))
    N.check(uc.ctx, st, "gg_penetration")
    mask = hit.astype(bool)
    if single:
        return float(psi[0]), nrm[0], bool(mask[0]), int(ndeg.value)
    return psi, nrm, mask, int(ndeg.value)


# ---------------------------------------------------------------------------
# GSDF grid cache (sdf.py:432-465 of the reference): "GSDF", u32 version 1,
# u32 dims[3], f64 origin[3], f64 spacing[3], 32-byte mesh hash, then the
# knot values as little-endian float32 in C order.
# ---------------------------------------------------------------------------
import struct as _struct

GRID_MAGIC = b"GSDF"
GRID_VERSION = 1


def save_grid(path: str, grid: SdfGrid) -> None:
    header = GRID_MAGIC + _struct.pack("<I3I3d3d", GRID_VERSION, *(int(d) for d in grid.dims),
                                       *(float(o) for o in grid.origin),
                                       *(float(s) for s in grid.spacing))
    with open(path, "wb") as fh:
        fh.write(header)
        fh.write(bytes(grid.mesh_hash[:32]).ljust(32, b"\0"))
        fh.write(np.ascontiguousarray(grid.values, dtype="<f4").tobytes())


def load_grid(path: str) -> SdfGrid:
    with open(path, "rb") as fh:
        blob = fh.read()
    if blob[:4] != GRID_MAGIC:
        raise ValueError(f"{path!r} is not an SDF grid cache file")
    (version,) = _struct.unpack_from("<I", blob, 4)
    if version != GRID_VERSION:
        raise ValueError(f"unsupported grid cache version {version}")
    fields = _struct.unpack_from("<3I3d3d", blob, 8)
    dims, origin, spacing = fields[:3], fields[3:6], fields[6:9]
    off = 8 + _struct.calcsize("<3I3d3d")
    mesh_hash = blob[off:off + 32]
    values = np.frombuffer(blob[off + 32:], dtype="<f4").astype(np.float64)
    return SdfGrid(origin=np.array(origin), spacing=np.array(spacing), dims=np.array(dims),
                   values=values.reshape(dims), mesh_hash=mesh_hash)


# ---------------------------------------------------------------------------
# Mesh signed distance and baking on the device (sdf.py:248-419)
# ---------------------------------------------------------------------------
class MeshDistance:
    """Exact signed distance to a watertight triangle mesh (sdf.py:248-391):
    nearest triangle by the region-based closest point, sign from the
    angle-weighted pseudonormal of the nearest feature.  Evaluated by the
    ``gg_bake_mesh_sdf`` kernel; the triangle table is built once."""

    def __init__(self, vertices: np.ndarray, faces: np.ndarray, device: int | None = None):
        from .meshes import check_watertight, triangle_table

        self.vertices = np.asarray(vertices, dtype=np.float64)
        self.faces = np.asarray(faces, dtype=np.int64)
        check_watertight(self.vertices, self.faces)
        self.table = triangle_table(self.vertices, self.faces)
        self.device = _device_index(device)
        self.last_kernel_ms = 0.0

    def contact_bounds(self, r):
        return self.vertices.min(axis=0) - r, self.vertices.max(axis=0) + r

    def _run(self, points, origin=None, spacing=None, dims=None) -> np.ndarray:
        ms = ctypes.c_float(0.0)
        if points is not None:
            pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
            out = np.empty(len(pts))
            if len(pts) == 0:
                return out
            st = N.lib().gg_bake_mesh_sdf(self.device, N.ptr(self.table), len(self.table), N.ptr(pts),
                                          len(pts), None, None, None, N.ptr(out), ctypes.byref(ms))
        else:
            o = np.ascontiguousarray(origin, dtype=np.float64)
            s = np.ascontiguousarray(spacing, dtype=np.float64)
            d = np.ascontiguousarray(dims, dtype=np.int64)
            out = np.empty(int(np.prod(d)))
            st = N.lib().gg_bake_mesh_sdf(self.device, N.ptr(self.table), len(self.table), None, 0,
                                          N.ptr(o), N.ptr(s), N.ptr(d), N.ptr(out), ctypes.byref(ms))
        N.check(None, st, "gg_bake_mesh_sdf")
        self.last_kernel_ms = float(ms.value)
        return out

    def signed_distance(self, points: np.ndarray) -> np.ndarray:
        p = np.asarray(points, dtype=np.float64)
        out = self._run(p.reshape(-1, 3))
        return out[0] if p.ndim == 1 else out


def _device_index(device) -> int:
    if device is not None:
        return int(getattr(device, "index", device) or 0)
    try:
        import torch

        return torch.cuda.current_device() if torch.cuda.is_available() else 0
    except Exception:  # pragma: no cover - torch is plumbing only
        return 0


def bake_mesh_sdf(vertices: np.ndarray, faces: np.ndarray, spacing, margin: float | None = None,
                  device: int | None = None) -> SdfGrid:
    """Grid over the mesh box plus ``margin`` (default two spacings) on every
    side, dims = max(ceil(extent / spacing) + 1, 2), knot values = exact signed
    distance (sdf.py:393-419).  Raises MeshError for non-watertight meshes."""
    from .meshes import mesh_content_hash

    md = MeshDistance(vertices, faces, device)
    spacing = np.broadcast_to(np.asarray(spacing, dtype=np.float64), 3).copy()
    if margin is None:
        margin = 2.0 * float(spacing.max())
    lo = md.vertices.min(axis=0) - margin
    hi = md.vertices.max(axis=0) + margin
    dims = np.maximum(np.ceil((hi - lo) / spacing).astype(np.int64) + 1, 2)
    values = md._run(None, lo, spacing, dims).reshape(tuple(dims))
    grid = SdfGrid(origin=lo, spacing=spacing, dims=dims, values=values,
                   mesh_hash=mesh_content_hash(md.vertices, md.faces))
    grid.bake_kernel_ms = md.last_kernel_ms
    return grid
