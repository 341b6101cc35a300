"""Batched independent environments on one device.

The reference steps one ``Scene`` per call (``stepper.step``,
stepper.py:57-135); an RL env batch (``BulldozerEnv``/``ExcavationEnv``,
envs.py:102-348) is E such scenes advanced in lock step.  ``SceneBatch``
runs all E scenes in ONE device context (``gg_create_batched``): env e owns
particles [e*n, (e+1)*n) of the resident state and its own hash table, so
every env evolves bit-for-bit as it would alone (tests/test_batch.py checks
this against E single-scene contexts and the oracle).

Body poses for the whole batch come from *batch drivers* — array versions of
the reference drivers (kinematics.py:116-230) that produce (T, E) poses with
numpy — so packing the per-step body tables costs a few array ops rather
than E x n_bodies Python calls.  Scenes whose bodies carry ordinary drivers
are also accepted (evaluated per env, for small E and tests).

Multi-GPU: envs shard with no communication (env e -> rank e mod world,
``shard_envs``); each rank owns a ``SceneBatch`` of its envs.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .engine import _mode_code, _params_signature, _params_struct, default_table_size
from .errors import SolverError
from .sdf import geometry_kind, geometry_shape
from .stepper import PipelineMode, StepReport, _make_report


# ---------------------------------------------------------------------------
# batch drivers: pose / twist of one body slot in all E envs at T times
# ---------------------------------------------------------------------------
class BatchDriver:
    """``rollout(T, dt, ts) -> (poses (T,E,4,4), omegas (T,E,3), v_origin (T,E,3))``
    for the next T steps; may advance internal state (like the env loop's
    ``driver.advance`` before every ``step``, envs.py:214-216)."""

    n_envs: int

    def rollout(self, T: int, dt: float, ts: np.ndarray):
        raise NotImplementedError


class StaticBatch(BatchDriver):
    """StaticDriver (kinematics.py:116-124) in every env: one pose, or (E,4,4)."""

    def __init__(self, n_envs: int, pose: np.ndarray | None = None):
        self.n_envs = n_envs
        p = np.eye(4) if pose is None else np.asarray(pose, dtype=np.float64)
        self.pose = np.broadcast_to(p, (n_envs, 4, 4))

    def rollout(self, T, dt, ts):
        z = np.zeros((T, self.n_envs, 3))
        return np.broadcast_to(self.pose, (T, self.n_envs, 4, 4)), z, z

    def current(self):
        z = np.zeros((self.n_envs, 3))
        return np.asarray(self.pose), z, z


class TrackSteeringBatch(BatchDriver):
    """E tracked vehicles (TrackSteeringDriver + track_steering_advance,
    kinematics.py:163-230) with array state.  ``command(actions (E,2))``
    then each step of a rollout first advances the state by dt (the env's
    frame-skip loop, envs.py:214-216) and evaluates pose_at / twist_at."""

    def __init__(self, x, y, theta, z: float = 0.0, scale_v: float = 1.0,
                 scale_omega: float = 1.0, base_pose: np.ndarray | None = None):
        self.x = np.array(x, dtype=np.float64)
        self.y = np.array(y, dtype=np.float64)
        self.theta = np.array(theta, dtype=np.float64)
        self.n_envs = len(self.x)
        self.z = float(z)
        self.scale_v = float(scale_v)
        self.scale_omega = float(scale_omega)
        self.base_pose = np.eye(4) if base_pose is None else np.asarray(base_pose, dtype=np.float64)
        self.action = np.zeros((self.n_envs, 2))

    def command(self, actions) -> None:
        a = np.asarray(actions, dtype=np.float64).reshape(self.n_envs, 2)
        self.action = np.clip(a, -1.0, 1.0)

    def advance(self, dt: float) -> None:
        a = self.action
        self.theta = self.theta + dt * self.scale_omega * a[:, 1]
        self.x = self.x + dt * self.scale_v * a[:, 0] * np.cos(self.theta)
        self.y = self.y + dt * self.scale_v * a[:, 0] * np.sin(self.theta)

    def pose_now(self):
        E = self.n_envs
        c, s = np.cos(self.theta), np.sin(self.theta)
        # so3_exp([0,0,theta]) = Rz(theta) (Rodrigues on the z axis)
        base = np.zeros((E, 4, 4))
        base[:, 0, 0], base[:, 0, 1] = c, -s
        base[:, 1, 0], base[:, 1, 1] = s, c
        base[:, 2, 2] = 1.0
        base[:, 3, 3] = 1.0
        base[:, 0, 3], base[:, 1, 3], base[:, 2, 3] = self.x, self.y, self.z
        pose = base @ self.base_pose
        omega = np.zeros((E, 3))
        omega[:, 2] = self.scale_omega * self.action[:, 1]
        heading = np.stack([c, s, np.zeros(E)], axis=1)
        v_veh = (self.scale_v * self.action[:, 0])[:, None] * heading
        ref = np.stack([self.x, self.y, np.full(E, self.z)], axis=1)
        v = v_veh + np.cross(omega, pose[:, :3, 3] - ref)
        return pose, omega, v

    def current(self):
        return self.pose_now()

    def rollout(self, T, dt, ts):
        E = self.n_envs
        P = np.empty((T, E, 4, 4))
        W = np.empty((T, E, 3))
        V = np.empty((T, E, 3))
        for k in range(T):
            self.advance(dt)
            P[k], W[k], V[k] = self.pose_now()
        return P, W, V


def so3_exp_batch(w: np.ndarray) -> np.ndarray:
    """Rodrigues for (E, 3) rotation vectors (kinematics.py:39-47), first
    order below 1e-12 rad like the reference."""
    w = np.asarray(w, dtype=np.float64)
    E = len(w)
    angle = np.linalg.norm(w, axis=1)
    small = angle < 1e-12
    safe = np.where(small, 1.0, angle)
    k = w / safe[:, None]
    K = np.zeros((E, 3, 3))
    K[:, 0, 1], K[:, 0, 2] = -k[:, 2], k[:, 1]
    K[:, 1, 0], K[:, 1, 2] = k[:, 2], -k[:, 0]
    K[:, 2, 0], K[:, 2, 1] = -k[:, 1], k[:, 0]
    eye = np.broadcast_to(np.eye(3), (E, 3, 3))
    R = eye + np.sin(angle)[:, None, None] * K + (1.0 - np.cos(angle))[:, None, None] * (K @ K)
    if small.any():
        S = np.zeros((E, 3, 3))
        S[:, 0, 1], S[:, 0, 2] = -w[:, 2], w[:, 1]
        S[:, 1, 0], S[:, 1, 2] = w[:, 2], -w[:, 0]
        S[:, 2, 0], S[:, 2, 1] = -w[:, 1], w[:, 0]
        R[small] = (eye + S)[small]
    return R


class ChainBatch(BatchDriver):
    """E copies of a velocity-controlled kinematic chain (KinematicChain +
    ChainLinkDriver, kinematics.py:256-322) with array joint state (E, J):
    ``command(qd (E, J))``; every rollout step first advances the joints by dt
    (ExcavationEnv's substep loop, envs.py:336-341), then evaluates the forward
    kinematics of link ``link_index`` for all envs at once."""

    def __init__(self, links, n_envs: int, link_index: int, base_pose: np.ndarray | None = None):
        self.links = list(links)
        self.n_envs = n_envs
        self.link_index = link_index
        J = len(self.links)
        self.base_pose = np.eye(4) if base_pose is None else np.asarray(base_pose, dtype=np.float64)
        self.q = np.zeros((n_envs, J))
        self.qd = np.zeros((n_envs, J))
        self.limits = np.array([l.velocity_limit for l in self.links])
        self.cmd = np.zeros((n_envs, J))

    def command(self, qd_cmd) -> None:
        self.cmd = np.asarray(qd_cmd, dtype=np.float64).reshape(self.n_envs, len(self.links))

    def advance(self, dt: float) -> None:
        self.qd = np.clip(self.cmd, -self.limits, self.limits)
        self.q = self.q + dt * self.qd

    def fk(self):
        """(poses (E, J, 4, 4), omega (E, J, 3), v_origin (E, J, 3)) like KinematicChain.fk."""
        E, J = self.n_envs, len(self.links)
        poses = np.empty((E, J, 4, 4))
        sw = np.empty((E, J, 3))
        sv = np.empty((E, J, 3))
        for i, link in enumerate(self.links):
            parent = np.broadcast_to(self.base_pose, (E, 4, 4)) if link.parent < 0 else poses[:, link.parent]
            joint = parent @ link.origin
            axis_w = joint[:, :3, :3] @ link.axis
            local = np.zeros((E, 4, 4))
            local[:, 3, 3] = 1.0
            if link.joint_type == "revolute":
                local[:, :3, :3] = so3_exp_batch(link.axis[None, :] * self.q[:, i:i + 1])
                w_j = axis_w * self.qd[:, i:i + 1]
                v_j = -np.cross(w_j, joint[:, :3, 3])
            else:
                local[:, :3, :3] = np.eye(3)
                local[:, :3, 3] = link.axis[None, :] * self.q[:, i:i + 1]
                w_j = np.zeros((E, 3))
                v_j = axis_w * self.qd[:, i:i + 1]
            poses[:, i] = joint @ local
            if link.parent < 0:
                sw[:, i], sv[:, i] = w_j, v_j
            else:
                sw[:, i], sv[:, i] = sw[:, link.parent] + w_j, sv[:, link.parent] + v_j
        return poses, sw, sv + np.cross(sw, poses[:, :, :3, 3])

    def current(self):
        P, W, V = self.fk()
        i = self.link_index
        return P[:, i], W[:, i], V[:, i]

    def rollout(self, T, dt, ts):
        E = self.n_envs
        P = np.empty((T, E, 4, 4))
        W = np.empty((T, E, 3))
        V = np.empty((T, E, 3))
        for k in range(T):
            self.advance(dt)
            P[k], W[k], V[k] = self.current()
        return P, W, V


def shard_envs(n_envs: int, rank: int, world: int) -> np.ndarray:
    """Env ids owned by ``rank``: e with e mod world == rank (no communication)."""
    return np.arange(rank, n_envs, world)


# ---------------------------------------------------------------------------
@dataclass
class _BodySlot:
    kind: np.ndarray        # (E,)
    shape: np.ndarray       # (E,4)
    grid_id: np.ndarray     # (E,)
    corners: np.ndarray | None  # (E,8,3) body-local contact bounds, None if unbounded


class SceneBatch:
    """E same-sized scenes stepped together on one device.

    All scenes must share the particle count, ``MaterialParams``, hash table
    size, cyclic boundary and number of bodies (geometries may differ per
    env).  ``body_drivers[b]`` (optional) is a ``BatchDriver`` that poses body
    slot b in every env; slots without one use each scene's own driver."""

    def __init__(self, scenes, body_drivers: dict | None = None, device: int = 0,
                 max_contacts: int = 16):
        if len(scenes) == 0:
            raise ValueError("SceneBatch needs at least one scene")
        self.scenes = list(scenes)
        self.E = len(self.scenes)
        s0 = self.scenes[0]
        self.n = s0.particles.count
        self.params = s0.params
        self.boundary = s0.boundary
        self.n_h = int(s0.hashmap_size or default_table_size(self.n))
        self.nb = len(s0.bodies)
        sig = _params_signature(s0.params, s0.boundary)
        for e, sc in enumerate(self.scenes):
            if sc.particles.count != self.n:
                raise ValueError(f"env {e}: {sc.particles.count} particles, env 0 has {self.n}")
            if _params_signature(sc.params, sc.boundary) != sig:
                raise ValueError(f"env {e}: material params / boundary differ from env 0")
            if int(sc.hashmap_size or default_table_size(self.n)) != self.n_h:
                raise ValueError(f"env {e}: hash table size differs from env 0")
            if len(sc.bodies) != self.nb:
                raise ValueError(f"env {e}: {len(sc.bodies)} bodies, env 0 has {self.nb}")
        if self.n == 0:
            raise ValueError("SceneBatch needs particles in every env")
        self.body_drivers = dict(body_drivers or {})
        for b, drv in self.body_drivers.items():
            if not 0 <= b < self.nb:
                raise ValueError(f"body driver for slot {b}: scenes have {self.nb} bodies")
            if drv.n_envs != self.E:
                raise ValueError(f"body driver for slot {b} has {drv.n_envs} envs, batch has {self.E}")
        self.device = device
        self.max_contacts = max_contacts
        self.t = np.array([float(sc.t) for sc in self.scenes])
        self.ctx = None
        self._grids: dict[int, tuple[object, int]] = {}
        self.launches0 = 0
        self._create()
        self._slots = [self._body_slot(b) for b in range(self.nb)]
        self.upload_from_scenes()

    # -- context -----------------------------------------------------------
    def _create(self) -> None:
        ctx = ctypes.c_void_p()
        ps = _params_struct(self.params, self.boundary)
        st = N.lib().gg_create_batched(self.device, ctypes.byref(ps), self.E, self.n, self.n_h,
                                       max(self.nb, 1), self.max_contacts, ctypes.byref(ctx))
        if st != N.GG_OK:
            msg = N.last_error(ctx) if ctx.value else "gg_create_batched failed"
            if ctx.value:
                N.lib().gg_destroy(ctx)
            raise (ValueError if st == N.GG_EINVAL else RuntimeError)(msg)
        self.ctx = ctx

    def close(self) -> None:
        if self.ctx is not None:
            N.lib().gg_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _grid_id(self, geom) -> int:
        hit = self._grids.get(id(geom))
        if hit is not None and hit[0] is geom:
            return hit[1]
        vals = np.ascontiguousarray(np.asarray(geom.values, dtype=np.float64))
        dims = np.asarray(geom.dims, dtype=np.int32).reshape(3)
        org = np.ascontiguousarray(np.asarray(geom.origin, dtype=np.float64))
        spc = np.ascontiguousarray(np.asarray(geom.spacing, dtype=np.float64))
        gid = ctypes.c_int32(-1)
        N.check(self.ctx, N.lib().gg_upload_grid(self.ctx, N.ptr(vals), N.ptr(dims), N.ptr(org),
                                                 N.ptr(spc), ctypes.byref(gid)), "grid")
        self._grids[id(geom)] = (geom, gid.value)
        return gid.value

    def _body_slot(self, b: int) -> _BodySlot:
        r = float(self.params.radius)
        kind = np.empty(self.E, np.int32)
        shape = np.empty((self.E, 4))
        gid = np.full(self.E, -1, np.int32)
        corners = np.empty((self.E, 8, 3))
        bounded = None
        for e, sc in enumerate(self.scenes):
            geom = sc.bodies[b].geometry
            kind[e] = geometry_kind(geom)
            shape[e] = geometry_shape(geom)
            if kind[e] == N.GEOM_GRID:
                gid[e] = self._grid_id(geom)
            bounds = geom.contact_bounds(r)
            if bounded is None:
                bounded = bounds is not None
            elif bounded != (bounds is not None):
                raise ValueError(f"body slot {b}: bounded and unbounded geometries mixed")
            if bounds is not None:
                lo, hi = bounds
                corners[e] = [[x, y, z] for x in (lo[0], hi[0]) for y in (lo[1], hi[1])
                              for z in (lo[2], hi[2])]
        return _BodySlot(kind, shape, gid, corners if bounded else None)

    # -- state ---------------------------------------------------------------
    def upload_from_scenes(self) -> None:
        x = np.ascontiguousarray(np.concatenate([np.asarray(sc.particles.positions, np.float64)
                                                 for sc in self.scenes]))
        v = np.ascontiguousarray(np.concatenate([np.asarray(sc.particles.velocities, np.float64)
                                                 for sc in self.scenes]))
        self.set_state(x.reshape(self.E, self.n, 3), v.reshape(self.E, self.n, 3))

    def set_state(self, x: np.ndarray, v: np.ndarray) -> None:
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(self.E * self.n, 3)
        v = np.ascontiguousarray(v, dtype=np.float64).reshape(self.E * self.n, 3)
        N.check(self.ctx, N.lib().gg_set_state_f64(self.ctx, N.ptr(x), N.ptr(v)), "upload")

    def state(self) -> tuple[np.ndarray, np.ndarray]:
        """(positions, velocities), each (E, n, 3) float64 (device -> host)."""
        x = np.empty((self.E * self.n, 3))
        v = np.empty((self.E * self.n, 3))
        N.check(self.ctx, N.lib().gg_get_state_f64(self.ctx, N.ptr(x), N.ptr(v)), "download")
        return x.reshape(self.E, self.n, 3), v.reshape(self.E, self.n, 3)

    def sync_scenes(self) -> None:
        """Write device state, time and body poses back into every scene."""
        x, v = self.state()
        for e, sc in enumerate(self.scenes):
            sc.particles.positions = x[e].copy()
            sc.particles.velocities = v[e].copy()
            sc.t = float(self.t[e])

    # -- body tables ---------------------------------------------------------
    def body_tables(self, T: int) -> np.ndarray:
        """(T, E, nb) gg_body rows for the next T steps (advances self.t)."""
        dt = float(self.params.timestep)
        nb = max(self.nb, 1)
        table = np.zeros((T, self.E, nb), dtype=N.BODY_DTYPE)
        ts = self.t[None, :] + dt * np.arange(1, T + 1)[:, None]  # (T,E)
        for b in range(self.nb):
            drv = self.body_drivers.get(b)
            if drv is not None:
                P, W, V = drv.rollout(T, dt, ts)
            else:
                P = np.empty((T, self.E, 4, 4))
                W = np.empty((T, self.E, 3))
                V = np.empty((T, self.E, 3))
                for e, sc in enumerate(self.scenes):
                    body = sc.bodies[b]
                    # same evaluation as the single-scene engine (Engine.body_tables)
                    if T > 1 and hasattr(body.driver, "pose_batch"):
                        p, w, v = body.driver.pose_batch(ts[:, e])
                        P[:, e] = np.broadcast_to(p, (T, 4, 4))
                        W[:, e] = np.broadcast_to(w, (T, 3))
                        V[:, e] = np.broadcast_to(v, (T, 3))
                        body.update(float(ts[-1, e]))
                        continue
                    for k in range(T):
                        body.update(float(ts[k, e]))
                        P[k, e] = body.pose
                        W[k, e] = body.omega
                        V[k, e] = body.v_origin
            self._fill(table[:, :, b], self._slots[b], P, W, V)
        self.t = ts[-1].copy()
        self._last_table = table[-1].copy()
        return table

    @staticmethod
    def _fill(col, slot: _BodySlot, P, W, V) -> None:
        T, E = col.shape
        P = np.broadcast_to(P, (T, E, 4, 4))
        col["kind"] = slot.kind[None, :]
        col["shape"] = slot.shape[None, :, :]
        col["grid_id"] = slot.grid_id[None, :]
        R = P[..., :3, :3]
        tr = P[..., :3, 3]
        col["rot"] = R.reshape(T, E, 9)
        col["trans"] = tr
        col["omega"] = W
        col["v_origin"] = V
        if slot.corners is None:
            col["bounded"] = 0
            return
        # the world AABB of the body-local contact box (the _near_body box,
        # contact.py:196-201), in closed form: centre R c + t, half extents
        # |R| h (the corners' min / max up to rounding).  The box is
        # conservative by r, so rounding of its faces cannot decide a contact.
        lo, hi = slot.corners.min(axis=1), slot.corners.max(axis=1)  # (E, 3)
        c, h = 0.5 * (lo + hi), 0.5 * (hi - lo)
        wc = np.einsum("teij,ej->tei", R, c) + tr
        ext = np.einsum("teij,ej->tei", np.abs(R), h)
        col["bounded"] = 1
        col["aabb_lo"] = wc - ext
        col["aabb_hi"] = wc + ext

    # -- device-resident drivers (gg_drive_*) ----------
    def drive_on_device(self) -> bool:
        """Generate every body slot's rows on the device: StaticBatch slots and
        slots whose scene drivers are all static become fixed rows,
        TrackSteeringBatch slots run TrackSteeringDriver on the device (one
        geometry in every env).  After this, ``run_raw`` uploads no body
        tables.  Returns False (host path kept) if a slot has no device form."""
        from .kinematics import StaticDriver

        plans = []
        for b in range(self.nb):
            drv = self.body_drivers.get(b)
            slot = self._slots[b]
            if isinstance(drv, (TrackSteeringBatch, ChainBatch)):
                same = (np.all(slot.kind == slot.kind[0]) and np.all(slot.shape == slot.shape[0])
                        and np.all(slot.grid_id == slot.grid_id[0]))
                if not same:
                    return False
                plans.append(("track" if isinstance(drv, TrackSteeringBatch) else "chain", b, drv))
            elif isinstance(drv, StaticBatch) or (
                    drv is None and all(isinstance(sc.bodies[b].driver, StaticDriver) for sc in self.scenes)):
                plans.append(("fixed", b, drv))
            else:
                return False
        lib = N.lib()
        rows = self.last_bodies()
        r = float(self.params.radius)
        for kind, b, drv in plans:
            if kind == "fixed":
                col = np.ascontiguousarray(rows[:, b])
                N.check(self.ctx, lib.gg_drive_fixed(self.ctx, b, N.ptr(col)), "gg_drive_fixed")
                continue
            tmpl = np.zeros(1, dtype=N.BODY_DTYPE)
            tmpl[0] = rows[0, b]
            bounds = self.scenes[0].bodies[b].geometry.contact_bounds(r)
            lo = hi = None
            if bounds is not None:
                lo = np.ascontiguousarray(bounds[0], dtype=np.float64)
                hi = np.ascontiguousarray(bounds[1], dtype=np.float64)
            base = np.ascontiguousarray(drv.base_pose, dtype=np.float64)
            if kind == "track":
                xs, ys, ths = (np.ascontiguousarray(a, dtype=np.float64) for a in (drv.x, drv.y, drv.theta))
                N.check(self.ctx, lib.gg_drive_track(self.ctx, b, N.ptr(tmpl), N.ptr(lo), N.ptr(hi), N.ptr(xs),
                                                     N.ptr(ys), N.ptr(ths), drv.z, drv.scale_v,
                                                     drv.scale_omega, N.ptr(base)), "gg_drive_track")
            else:
                links = drv.links
                J = len(links)
                par = np.array([l.parent for l in links], dtype=np.int32)
                pri = np.array([0 if l.joint_type == "revolute" else 1 for l in links], dtype=np.int32)
                org = np.ascontiguousarray(np.stack([np.asarray(l.origin, float) for l in links]).reshape(J, 16))
                axs = np.ascontiguousarray(np.stack([np.asarray(l.axis, float) for l in links]))
                q = np.ascontiguousarray(drv.q, dtype=np.float64)
                N.check(self.ctx, lib.gg_drive_chain(self.ctx, b, N.ptr(tmpl), N.ptr(lo), N.ptr(hi), J,
                                                     drv.link_index, N.ptr(par), N.ptr(pri), N.ptr(org),
                                                     N.ptr(axs), N.ptr(np.ascontiguousarray(drv.limits)),
                                                     N.ptr(base), N.ptr(q)), "gg_drive_chain")
        self.driven = [b for _, b, _ in plans]
        self._track_slots = [(b, drv) for kind, b, drv in plans if kind in ("track", "chain")]
        self.drive_command()
        return True

    def drive_command(self) -> None:
        """Send the host drivers' current commands (track actions, chain joint
        rate commands) to the device drivers."""
        for b, drv in getattr(self, "_track_slots", []):
            src = drv.action if isinstance(drv, TrackSteeringBatch) else drv.cmd
            act = np.ascontiguousarray(src, dtype=np.float64)
            N.check(self.ctx, N.lib().gg_drive_command(self.ctx, b, N.ptr(act)), "gg_drive_command")

    def _pull_driver_states(self) -> None:
        for b, drv in getattr(self, "_track_slots", []):
            if isinstance(drv, TrackSteeringBatch):
                x, y, th = np.empty(self.E), np.empty(self.E), np.empty(self.E)
                N.check(self.ctx, N.lib().gg_drive_state(self.ctx, b, N.ptr(x), N.ptr(y), N.ptr(th)),
                        "gg_drive_state")
                drv.x, drv.y, drv.theta = x, y, th
            else:
                q = np.empty((self.E, len(drv.links)))
                N.check(self.ctx, N.lib().gg_drive_chain_state(self.ctx, b, N.ptr(q)), "gg_drive_chain_state")
                drv.q = q
                drv.qd = np.clip(drv.cmd, -drv.limits, drv.limits)
        self._last_table = None

    def last_bodies(self) -> np.ndarray:
        """(E, nb) gg_body rows at the current time (the last stepped poses,
        or the drivers' current poses before the first step)."""
        if getattr(self, "_last_table", None) is not None:
            return self._last_table
        nb = max(self.nb, 1)
        row = np.zeros((1, self.E, nb), dtype=N.BODY_DTYPE)
        for b in range(self.nb):
            drv = self.body_drivers.get(b)
            if drv is not None:
                P, W, V = drv.current()
            else:
                P = np.empty((self.E, 4, 4))
                W = np.empty((self.E, 3))
                V = np.empty((self.E, 3))
                for e, sc in enumerate(self.scenes):
                    body = sc.bodies[b]
                    body.update(float(self.t[e]))
                    P[e], W[e], V[e] = body.pose, body.omega, body.v_origin
            self._fill(row[:, :, b], self._slots[b], P[None], W[None], V[None])
        return row[0]

    # -- stepping -------------------------------------------------------------
    def run_raw(self, T: int, mode=PipelineMode.TWO_LOOPS_SPLIT, last_only: bool = False):
        """Advance every env T steps.  Returns (reports (T,E) REPORT_DTYPE,
        body_momentum (T,E,nb,3)); ``last_only``: only the last step's
        (shapes (1,E), (1,E,nb,3)), the others are not copied back."""
        if T < 0:
            raise ValueError("n_steps must be >= 0")
        mcode = _mode_code(mode)
        if T == 0:
            return np.zeros((0, self.E), N.REPORT_DTYPE), np.zeros((0, self.E, self.nb, 3))
        t0 = self.t.copy()
        driven = bool(getattr(self, "driven", None)) and len(self.driven) == self.nb
        if driven:  # the host drivers' commands are the source of truth
            self.drive_command()
            table = None
            self.t = self.t + float(self.params.timestep) * T
        else:
            table = self.body_tables(T)
        reps = np.zeros((T, self.E), dtype=N.REPORT_DTYPE)
        bm = np.zeros((T, self.E, max(self.nb, 1), 3))
        done = 0
        lib = N.lib()
        while done < T:
            if driven and done > 0:  # the rows of steps done.. are on the device already
                st = lib.gg_step_resume(self.ctx, done, T - done, mcode)
            else:
                rows = None if driven else np.ascontiguousarray(table[done:])
                st = lib.gg_step(self.ctx, T - done, N.ptr(rows), self.nb, mcode)
            N.check(self.ctx, st, "gg_step")
            rbuf = np.zeros((T - done, self.E), dtype=N.REPORT_DTYPE)
            bbuf = np.zeros((T - done, self.E, max(self.nb, 1), 3))
            nd, es = ctypes.c_int32(0), ctypes.c_int32(-1)
            if last_only:
                st = lib.gg_sync(self.ctx, None, None, 0, ctypes.byref(nd), ctypes.byref(es))
                if st == N.GG_OK and nd.value > 0:  # the batch's last step only
                    kk = nd.value - 1
                    N.check(self.ctx, lib.gg_batch_reports(self.ctx, kk, 1, N.ptr(rbuf[kk:kk + 1]),
                                                           N.ptr(bbuf[kk:kk + 1])), "gg_batch_reports")
            else:
                st = lib.gg_sync(self.ctx, N.ptr(rbuf), N.ptr(bbuf), T - done, ctypes.byref(nd),
                                 ctypes.byref(es))
            k = nd.value
            reps[done:done + k] = rbuf[:k]
            bm[done:done + k] = bbuf[:k]
            done += k
            if st == N.GG_OK:
                break
            if st == N.GG_ECAPACITY:
                need = lib.gg_required_contacts(self.ctx)
                self.max_contacts = max(2 * self.max_contacts, need + 4)
                N.check(self.ctx, lib.gg_set_max_contacts(self.ctx, self.max_contacts), "grow")
                continue
            # time stops at the failing step (stepper.py:99-103 raises before integrating)
            self.t = t0 + float(self.params.timestep) * (done + 1)
            msg = N.last_error(self.ctx)
            if st == N.GG_ENONFINITE:
                raise SolverError(f"step {done}: {msg} [particle ids are batch-global: "
                                  f"env = id // {self.n}]")
            if st == N.GG_EPOSITIONS:
                raise ValueError(msg)
            raise RuntimeError(f"step {done}: {msg}")
        if driven:
            self._pull_driver_states()
        if last_only:
            return reps[-1:], bm[-1:, :, : self.nb]
        return reps, bm[:, :, : self.nb]

    def step(self, mode=PipelineMode.TWO_LOOPS_SPLIT) -> list[StepReport]:
        """One ``stepper.step`` in every env; returns one StepReport per env."""
        reps, bm = self.run_raw(1, mode)
        return [_make_report(reps[0, e], bm[0, e], -1, 0.0) for e in range(self.E)]

    def run(self, n_steps: int, mode=PipelineMode.TWO_LOOPS_SPLIT) -> list[list[StepReport]]:
        """``n_steps`` steps in every env; reports[k][e]."""
        reps, bm = self.run_raw(n_steps, mode)
        return [[_make_report(reps[k, e], bm[k, e], k, 0.0) for e in range(self.E)]
                for k in range(n_steps)]

    def kernel_launches(self) -> int:
        return int(N.lib().gg_kernel_launches(self.ctx))
