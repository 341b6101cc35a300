"""Device engine behind ``step``/``run``: one C-ABI context per scene.

Responsibilities
  * map a reference-shaped ``Scene`` (ours or the reference's own objects,
    duck-typed) onto a ``gg_ctx``: sizes, MaterialParams, hash-table size;
  * keep the particle state resident on the device and mirror it to the
    host lazily (our ``ParticleSet``) or eagerly (plain reference objects);
  * evaluate body drivers on the host and pack per-step body tables
    (``gg_body``) for a whole batch of steps;
  * run batches through ``gg_step``/``gg_sync``, growing the contact slots
    and re-running from the failing step on GG_ECAPACITY, and map errors
    back to the reference's exception types and messages.
"""

from __future__ import annotations

import ctypes
import math
import os
import threading

import numpy as np

from . import _native as N
from .errors import SolverError
from .sdf import geometry_kind, geometry_shape

DEFAULT_MAX_CONTACTS = int(os.environ.get("GG_MAX_CONTACTS", 16))  # record slots per particle (grown x2 on overflow)


def default_table_size(n_p: int) -> int:
    """next power of two >= 2 n_p (broadphase.py:58-60)."""
    return max(1, 1 << int(math.ceil(math.log2(max(2 * n_p, 1)))))


def _params_struct(params, boundary) -> N.GGParams:
    p = N.GGParams()
    r = float(params.radius)
    p.radius = r
    p.particle_mass = float(params.particle_mass)
    p.friction = float(params.friction)
    p.baumgarte_alpha = float(params.baumgarte_alpha)
    p.timestep = float(params.timestep)
    g = np.asarray(params.gravity, dtype=np.float64)
    p.gravity[:] = g.tolist()
    p.gamma = float(params.gamma)
    # derived exactly as the reference writes them (contact.py:260-261,452)
    p.contact_d2 = (2.0 * r) ** 2
    p.coincident_d2 = 1e-12 * 1e-12
    p.gdt[:] = (params.timestep * g).tolist()
    p.solver_iterations = int(params.solver_iterations)
    if boundary is not None:
        p.has_boundary = 1
        p.z_min = float(boundary.z_min)
        p.z_max = float(boundary.z_max)
    return p


def _params_signature(params, boundary):
    g = tuple(np.asarray(params.gravity, dtype=np.float64).tolist())
    b = None if boundary is None else (float(boundary.z_min), float(boundary.z_max))
    return (float(params.radius), float(params.particle_mass), float(params.friction),
            float(params.baumgarte_alpha), float(params.timestep), int(params.solver_iterations),
            g, float(params.gamma), b)


def _is_mirrored(ps) -> bool:
    return hasattr(ps, "_refresh") and hasattr(ps, "_host_dirty")


def _mode_code(mode) -> int:
    if mode is None:
        return 0
    v = getattr(mode, "value", mode)
    table = {"two-loops-split": 0, "two-loops-fused": 1, "one-loop": 2}
    if v not in table:
        raise ValueError(f"unknown pipeline mode {mode!r}")
    return table[v]


class Engine:
    """Device context + residency bookkeeping for one scene."""

    def __init__(self, device: int = 0):
        self.device = device
        self.ctx = None
        self.n = -1
        self.n_h = -1
        self.sig = None
        self.device_newer = False
        self.max_contacts = DEFAULT_MAX_CONTACTS
        self._grids: dict[int, tuple[object, int]] = {}
        self._lock = threading.Lock()

    # -- lifetime ------------------------------------------------------------
    def close(self) -> None:
        if self.ctx is not None:
            N.lib().gg_destroy(self.ctx)
            self.ctx = None
        self._grids.clear()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __deepcopy__(self, memo):
        return Engine(self.device)

    def __getstate__(self):
        return {"device": self.device}

    def __setstate__(self, state):
        self.__init__(state.get("device", 0))

    # -- context ---------------------------------------------------------------
    def _create(self, params, boundary, n: int, n_h: int, n_bodies: int) -> None:
        self.close()
        if n_h >= 2**31:
            raise ValueError("hash table size must be < 2^31")
        ctx = ctypes.c_void_p()
        ps = _params_struct(params, boundary)
        st = N.lib().gg_create(self.device, ctypes.byref(ps), n, n_h, max(n_bodies, 1),
                               self.max_contacts, ctypes.byref(ctx))
        if st != N.GG_OK:
            msg = N.last_error(ctx) if ctx.value else "gg_create failed"
            if ctx.value:
                N.lib().gg_destroy(ctx)
            raise (ValueError if st == N.GG_EINVAL else RuntimeError)(msg)
        self.ctx = ctx
        self.n, self.n_h = n, n_h
        self.sig = _params_signature(params, boundary)
        self.device_newer = False

    def grid_id(self, geom) -> int:
        key = id(geom)
        hit = self._grids.get(key)
        if hit is not None and hit[0] is geom:
            return hit[1]
        vals = np.ascontiguousarray(np.asarray(geom.values, dtype=np.float64))
        dims = np.asarray(geom.dims, dtype=np.int32).reshape(3)
        org = np.ascontiguousarray(np.asarray(geom.origin, dtype=np.float64))
        spc = np.ascontiguousarray(np.asarray(geom.spacing, dtype=np.float64))
        gid = ctypes.c_int32(-1)
        st = N.lib().gg_upload_grid(self.ctx, N.ptr(vals), N.ptr(dims), N.ptr(org), N.ptr(spc),
                                    ctypes.byref(gid))
        N.check(self.ctx, st, "gg_upload_grid")
        self._grids[key] = (geom, gid.value)
        return gid.value

    # -- state residency -------------------------------------------------------
    def upload(self, x: np.ndarray, v: np.ndarray) -> None:
        x = np.ascontiguousarray(x, dtype=np.float64)
        v = np.ascontiguousarray(v, dtype=np.float64)
        N.check(self.ctx, N.lib().gg_set_state_f64(self.ctx, N.ptr(x), N.ptr(v)), "upload")
        self.device_newer = False

    def download_into(self, x: np.ndarray, v: np.ndarray) -> None:
        if x.flags.c_contiguous and x.dtype == np.float64 and v.flags.c_contiguous and v.dtype == np.float64:
            N.check(self.ctx, N.lib().gg_get_state_f64(self.ctx, N.ptr(x), N.ptr(v)), "download")
        else:
            tx = np.empty((self.n, 3))
            tv = np.empty((self.n, 3))
            N.check(self.ctx, N.lib().gg_get_state_f64(self.ctx, N.ptr(tx), N.ptr(tv)), "download")
            x[...] = tx
            v[...] = tv
        self.device_newer = False

    def prepare(self, scene) -> None:
        """Make the device context and state match the scene before a batch."""
        ps = scene.particles
        mirrored = _is_mirrored(ps)
        n = ps.count
        n_h = int(scene.hashmap_size or default_table_size(n))
        nb = len(scene.bodies)
        if self.ctx is None or n != self.n or n_h != self.n_h:
            if mirrored and ps._engine is self and self.device_newer:
                ps._refresh()
            self._create(scene.params, scene.boundary, n, n_h, nb)
            if mirrored:
                ps._host_dirty = True
        else:
            sig = _params_signature(scene.params, scene.boundary)
            if sig != self.sig:
                p = _params_struct(scene.params, scene.boundary)
                N.check(self.ctx, N.lib().gg_set_params(self.ctx, ctypes.byref(p)), "set_params")
                self.sig = sig
        if mirrored:
            if ps._engine is not self or ps._host_dirty:
                if ps._engine is not None and ps._engine is not self:
                    ps._refresh()
                self.upload(ps._x, ps._v)
                ps._engine = self
                ps._host_dirty = False
        else:
            self.upload(ps.positions, ps.velocities)

    def finish(self, scene) -> None:
        """After a batch: mark the device authoritative or write back eagerly."""
        ps = scene.particles
        self.device_newer = True
        if not _is_mirrored(ps):
            x, v = ps.positions, ps.velocities
            if (isinstance(x, np.ndarray) and x.dtype == np.float64 and x.flags.writeable
                    and isinstance(v, np.ndarray) and v.dtype == np.float64 and v.flags.writeable):
                self.download_into(x, v)
            else:
                tx, tv = np.empty((self.n, 3)), np.empty((self.n, 3))
                self.download_into(tx, tv)
                ps.positions, ps.velocities = tx, tv

    # -- body tables -----------------------------------------------------------
    def body_row(self, body, r: float, out) -> None:
        geom = body.geometry
        kind = geometry_kind(geom)
        out["kind"] = kind
        out["shape"] = geometry_shape(geom)
        out["grid_id"] = self.grid_id(geom) if kind == N.GEOM_GRID else -1
        pose = np.asarray(body.pose, dtype=np.float64)
        out["rot"] = pose[:3, :3].reshape(-1)
        out["trans"] = pose[:3, 3]
        out["omega"] = np.asarray(body.omega, dtype=np.float64)
        out["v_origin"] = np.asarray(body.v_origin, dtype=np.float64)
        bounds = geom.contact_bounds(r)
        if bounds is None:
            out["bounded"] = 0
        else:
            # the reference's _near_body arithmetic, verbatim order (contact.py:196-201)
            lo, hi = bounds
            corners = np.array(
                [[x, y, z] for x in (lo[0], hi[0]) for y in (lo[1], hi[1]) for z in (lo[2], hi[2])]
            )
            world = corners @ pose[:3, :3].T + pose[:3, 3]
            out["bounded"] = 1
            out["aabb_lo"] = world.min(axis=0)
            out["aabb_hi"] = world.max(axis=0)

    def body_tables(self, scene, n_steps: int):
        """Advance scene.t / body poses step by step (stepper.py:65-67) and
        pack one gg_body row per body per step.  Returns (table, ts).

        Drivers that can evaluate a whole batch of times (``pose_batch``)
        are packed with array operations; any other driver (e.g. the
        reference's own objects) is evaluated step by step."""
        dt = scene.params.timestep
        r = float(scene.params.radius)
        nb = len(scene.bodies)
        table = np.zeros((n_steps, max(nb, 1)), dtype=N.BODY_DTYPE)
        ts = np.empty(n_steps)
        t = scene.t
        for k in range(n_steps):
            t += dt
            ts[k] = t
        for bi, body in enumerate(scene.bodies):
            col = table[:, bi]
            if n_steps > 1 and hasattr(body.driver, "pose_batch"):
                poses, omegas, vels = body.driver.pose_batch(ts)
                self._fill_column(body, r, col, poses, omegas, vels)
            else:
                for k in range(n_steps):
                    body.update(ts[k])
                    self.body_row(body, r, col[k])
        if n_steps > 1:
            for body in scene.bodies:
                if hasattr(body.driver, "pose_batch"):
                    body.update(ts[-1])
        scene.t = t
        return table, ts

    def _fill_column(self, body, r: float, col, poses, omegas, vels) -> None:
        """Vectorised body_row for T poses of one body."""
        geom = body.geometry
        kind = geometry_kind(geom)
        T = len(col)
        poses = np.broadcast_to(np.asarray(poses, dtype=np.float64), (T, 4, 4))
        col["kind"] = kind
        col["shape"] = geometry_shape(geom)
        col["grid_id"] = self.grid_id(geom) if kind == N.GEOM_GRID else -1
        R = poses[:, :3, :3]
        tr = poses[:, :3, 3]
        col["rot"] = R.reshape(T, 9)
        col["trans"] = tr
        col["omega"] = np.broadcast_to(np.asarray(omegas, dtype=np.float64), (T, 3))
        col["v_origin"] = np.broadcast_to(np.asarray(vels, dtype=np.float64), (T, 3))
        bounds = geom.contact_bounds(r)
        if bounds is None:
            col["bounded"] = 0
            return
        lo, hi = bounds
        corners = np.array(
            [[x, y, z] for x in (lo[0], hi[0]) for y in (lo[1], hi[1]) for z in (lo[2], hi[2])]
        )
        # corners @ R^T + t per step; the box is conservative by r, so the
        # last-bit rounding of its faces cannot decide a contact (d < r strict)
        world = np.matmul(corners[None, :, :], np.transpose(R, (0, 2, 1))) + tr[:, None, :]
        col["bounded"] = 1
        col["aabb_lo"] = world.min(axis=1)
        col["aabb_hi"] = world.max(axis=1)

    # -- batches ---------------------------------------------------------------
    def run_batch(self, table: np.ndarray, nb: int, mode: int):
        """Run len(table) steps.  Returns (reports, body_momentum, n_done,
        status, message)."""
        T = len(table)
        reps = np.zeros(T, dtype=N.REPORT_DTYPE)
        bm = np.zeros((T, max(nb, 1), 3))
        done = 0
        lib = N.lib()
        while done < T:
            rows = np.ascontiguousarray(table[done:, : max(nb, 1)])
            st = lib.gg_step(self.ctx, T - done, N.ptr(rows), nb, mode)
            N.check(self.ctx, st, "gg_step")
            rbuf = np.zeros(T - done, dtype=N.REPORT_DTYPE)
            bbuf = np.zeros((T - done, max(nb, 1), 3))
            nd, es = ctypes.c_int32(0), ctypes.c_int32(-1)
            st = lib.gg_sync(self.ctx, N.ptr(rbuf), N.ptr(bbuf), T - done, ctypes.byref(nd),
                             ctypes.byref(es))
            k = nd.value
            reps[done : done + k] = rbuf[:k]
            if nb:
                bm[done : done + k, :nb] = bbuf[:k, :nb]
            done += k
            if st == N.GG_OK:
                break
            if st == N.GG_ECAPACITY:
                need = lib.gg_required_contacts(self.ctx)
                self.max_contacts = max(2 * self.max_contacts, need + 4)
                N.check(self.ctx, lib.gg_set_max_contacts(self.ctx, self.max_contacts), "grow")
                continue
            return reps, bm[:, :nb], done, st, N.last_error(self.ctx)
        return reps, bm[:, :nb], done, N.GG_OK, ""

    def last_batch_ms(self) -> float:
        ms = ctypes.c_float(0.0)
        N.check(self.ctx, N.lib().gg_last_batch_ms(self.ctx, ctypes.byref(ms)), "timing")
        return float(ms.value)

    def kernel_launches(self) -> int:
        return int(N.lib().gg_kernel_launches(self.ctx)) if self.ctx is not None else 0


def engine_for(scene) -> Engine:
    eng = scene.__dict__.get("_gg_engine")
    if eng is None:
        eng = Engine()
        scene.__dict__["_gg_engine"] = eng
    return eng


def raise_status(status: int, message: str, step_index: int) -> None:
    """Re-raise like stepper.step (stepper.py:99-100): solver errors get the
    "step {k}: " prefix; the broadphase's finite-position check runs before
    that try-block in the reference and is raised bare."""
    if status == N.GG_EPOSITIONS:
        raise ValueError(message)
    if status == N.GG_ENONFINITE:
        raise SolverError(f"step {step_index}: {message}")
    if status == N.GG_EINVAL:
        raise ValueError(f"step {step_index}: {message}")
    raise RuntimeError(f"step {step_index}: {message}")


_utility = None


class _Utility:
    """A 1-particle context used for standalone queries (penetration_depth,
    spatial_hash) that have no scene."""

    def __init__(self):
        from .scene import MaterialParams

        self.engine = Engine()
        self.engine._create(MaterialParams(), None, 1, 2, 1)

    @property
    def ctx(self):
        return self.engine.ctx

    def grid_id(self, geom) -> int:
        return self.engine.grid_id(geom)


def utility_context() -> _Utility:
    global _utility
    if _utility is None:
        _utility = _Utility()
    return _utility
