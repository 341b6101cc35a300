"""CPU oracle for the GranularGym timestep — TEST INFRASTRUCTURE ONLY.

A plain-numpy restatement of the reference path (granusim.stepper.step in
TWO_LOOPS_SPLIT mode and everything under it).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may import
this module, and only as the checker / the timed reference CPU path; the
product (``paper_2306_01369_b200``) never calls it.

Parity is pinned: ``tests/golden/make_golden.py`` runs the real reference
(``/root/reference/pkg/src/granusim``) and ``tests/test_oracle_golden.py``
checks this module against those fixtures (bit-exact cells/hashes/order,
contact lists and counters; float results to 1e-12 or exactly).

Each function cites the reference lines it restates.  Floating-point
operations keep the reference's order where a decision depends on it:
  * pp squared distance: numpy's ``einsum("ij,ij->i")`` on the reference host
    pairs (dx^2 + dz^2) + dy^2; written out explicitly here
    so the oracle does not depend on the SIMD path of the host it runs on;
  * the body transform ``(p - t) @ R`` and ``np.linalg.norm`` are used as
    the reference uses them.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass

import numpy as np

HASH_PRIMES = np.array([73856093, 19349663, 83492791], dtype=np.int64)  # broadphase.py:22
CELL_OFFSET = 100                                                          # broadphase.py:23
COINCIDENT_EPS = 1e-12                                                     # contact.py:24
DEGENERATE_GRADIENT_EPS = 1e-9                                             # sdf.py:19
# neighbour offsets in the reference's (i, j, k) loop order (broadphase.py:27-30)
NEIGHBOUR_OFFSETS = np.array(list(itertools.product((-1, 0, 1), repeat=3)), dtype=np.int64)


class OracleSolverError(RuntimeError):
    pass


# ---------------------------------------------------------------------------
# broadphase
# ---------------------------------------------------------------------------
def cell_coords(x: np.ndarray, r: float) -> np.ndarray:
    """round_half_away(x / 2r) as int64 — broadphase.py:33-41."""
    q = np.asarray(x, dtype=np.float64) / (2.0 * r)
    return np.copysign(np.floor(np.abs(q) + 0.5), q).astype(np.int64)


def cell_hash(cells: np.ndarray, n_h: int) -> np.ndarray:
    """XOR of prime-scaled offset coordinates, int64 wrap, floor-mod —
    broadphase.py:44-55."""
    t = (np.asarray(cells, dtype=np.int64) - CELL_OFFSET) * HASH_PRIMES
    return (t[..., 0] ^ t[..., 1] ^ t[..., 2]) % np.int64(n_h)


def table_size(n: int) -> int:
    """broadphase.py:58-60."""
    return max(1, 1 << int(np.ceil(np.log2(max(2 * n, 1)))))


def bucket_layout(hashes: np.ndarray, n_h: int):
    """Stable bucket order + bucket starts — broadphase.py:160-162."""
    order = np.argsort(hashes, kind="stable")
    starts = np.searchsorted(hashes[order], np.arange(n_h + 1))
    return order, starts


def candidate_rows(cells: np.ndarray, order: np.ndarray, starts: np.ndarray, n_h: int):
    """Directed candidates incl. self pairs, per owner over its 27 neighbour
    buckets sorted and de-duplicated — broadphase.py:149-182.
    Returns (owner, other) in the reference's enumeration order."""
    n = len(cells)
    H = cell_hash((cells[:, None, :] + NEIGHBOUR_OFFSETS[None]).reshape(-1, 3), n_h).reshape(n, 27)
    H.sort(axis=1)
    first = np.ones(H.shape, dtype=bool)
    first[:, 1:] = H[:, 1:] != H[:, :-1]
    sizes = np.where(first, starts[H + 1] - starts[H], 0)
    per_owner = sizes.sum(axis=1)
    owner = np.repeat(np.arange(n, dtype=np.int64), per_owner)
    flat = sizes.ravel()
    nz = flat > 0
    seg_begin = starts[H.ravel()[nz]]
    seg_len = flat[nz]
    within = np.arange(seg_len.sum(), dtype=np.int64) - np.repeat(np.cumsum(seg_len) - seg_len, seg_len)
    other = order[np.repeat(seg_begin, seg_len) + within]
    return owner, other


# ---------------------------------------------------------------------------
# signed distances (body frame) — sdf.py:44-241
# ---------------------------------------------------------------------------
def _norm_rows(a: np.ndarray) -> np.ndarray:
    return np.linalg.norm(a, axis=1)


def sdf_distance(geom, p: np.ndarray) -> np.ndarray:
    kind = type(geom).__name__
    if kind == "Sphere":
        return _norm_rows(p) - geom.radius
    if kind == "HalfSpace":
        return p @ np.asarray(geom.normal, dtype=np.float64) - geom.offset
    if kind == "Box":
        q = np.abs(p) - np.asarray(geom.half_extents, dtype=np.float64)
        return _norm_rows(np.maximum(q, 0.0)) + np.minimum(q.max(axis=1), 0.0)
    if kind == "Cylinder":
        rho = np.hypot(p[:, 0], p[:, 1])
        a = np.stack([rho - geom.radius, np.abs(p[:, 2]) - geom.half_height], axis=1)
        return np.minimum(a.max(axis=1), 0.0) + _norm_rows(np.maximum(a, 0.0))
    if kind == "Tube":
        return geom.radius - np.hypot(p[:, 0], p[:, 1])
    if kind == "SdfGrid":
        return _grid_distance(geom, p)
    raise ValueError(f"oracle: unsupported geometry {kind}")


def _grid_distance(g, p: np.ndarray) -> np.ndarray:
    origin = np.asarray(g.origin, dtype=np.float64)
    spacing = np.asarray(g.spacing, dtype=np.float64)
    dims = np.asarray(g.dims, dtype=np.int64)
    vals = np.asarray(g.values, dtype=np.float64).reshape(tuple(dims))
    upper = origin + (dims - 1) * spacing
    c = np.clip(p, origin, upper)
    out = _norm_rows(p - c)
    u = (c - origin) / spacing
    i0 = np.minimum(np.floor(u).astype(np.int64), dims - 2)
    f = u - i0
    ix, iy, iz = i0[:, 0], i0[:, 1], i0[:, 2]
    fx, fy, fz = f[:, 0], f[:, 1], f[:, 2]

    def lerp_x(jy, jz):
        return vals[ix, jy, jz] * (1 - fx) + vals[ix + 1, jy, jz] * fx

    c0 = lerp_x(iy, iz) * (1 - fy) + lerp_x(iy + 1, iz) * fy
    c1 = lerp_x(iy, iz + 1) * (1 - fy) + lerp_x(iy + 1, iz + 1) * fy
    return c0 * (1 - fz) + c1 * fz + out


def sdf_gradient(geom, p: np.ndarray) -> np.ndarray:
    kind = type(geom).__name__
    n = len(p)
    if kind == "Sphere":
        m = _norm_rows(p)[:, None]
        return np.divide(p, m, out=np.zeros_like(p), where=m > 0)
    if kind == "HalfSpace":
        return np.broadcast_to(np.asarray(geom.normal, dtype=np.float64), p.shape).copy()
    if kind == "Box":
        q = np.abs(p) - np.asarray(geom.half_extents, dtype=np.float64)
        qp = np.maximum(q, 0.0)
        m = _norm_rows(qp)[:, None]
        sgn = np.where(p >= 0.0, 1.0, -1.0)
        outside = np.divide(qp, m, out=np.zeros_like(qp), where=m > 0) * sgn
        inside = np.zeros_like(p)
        ax = q.argmax(axis=1)
        inside[np.arange(n), ax] = sgn[np.arange(n), ax]
        return np.where(m > 0, outside, inside)
    if kind == "Cylinder":
        rho = np.hypot(p[:, 0], p[:, 1])
        rr = np.maximum(rho, 1e-300)
        radial = np.stack([p[:, 0] / rr, p[:, 1] / rr, np.zeros(n)], axis=1)
        axial = np.stack([np.zeros(n), np.zeros(n), np.where(p[:, 2] >= 0, 1.0, -1.0)], axis=1)
        dr = rho - geom.radius
        dz = np.abs(p[:, 2]) - geom.half_height
        o = radial * np.maximum(dr, 0.0)[:, None] + axial * np.maximum(dz, 0.0)[:, None]
        m = _norm_rows(o)[:, None]
        o = np.divide(o, m, out=np.zeros_like(o), where=m > 0)
        return np.where(m > 0, o, np.where((dr > dz)[:, None], radial, axial))
    if kind == "Tube":
        rho = np.maximum(np.hypot(p[:, 0], p[:, 1]), 1e-300)
        return np.stack([-p[:, 0] / rho, -p[:, 1] / rho, np.zeros(n)], axis=1)
    if kind == "SdfGrid":
        h = float(np.asarray(geom.spacing, dtype=np.float64).min()) / 2.0
        out = np.empty_like(p)
        for a in range(3):
            e = np.zeros(3)
            e[a] = h
            out[:, a] = (_grid_distance(geom, p + e) - _grid_distance(geom, p - e)) / (2.0 * h)
        return out
    raise ValueError(f"oracle: unsupported geometry {kind}")


def contact_bounds(geom, r: float):
    kind = type(geom).__name__
    if kind == "Sphere":
        e = geom.radius + r
        return -np.full(3, e), np.full(3, e)
    if kind == "Box":
        he = np.asarray(geom.half_extents, dtype=np.float64)
        return -(he + r), he + r
    if kind == "Cylinder":
        e = np.array([geom.radius + r, geom.radius + r, geom.half_height + r])
        return -e, e
    if kind == "SdfGrid":
        o = np.asarray(geom.origin, dtype=np.float64)
        up = o + (np.asarray(geom.dims) - 1) * np.asarray(geom.spacing, dtype=np.float64)
        return o - r, up + r
    return None


def near_body(x: np.ndarray, r: float, geom, pose: np.ndarray) -> np.ndarray:
    """World-AABB prefilter — contact.py:187-203."""
    b = contact_bounds(geom, r)
    if b is None:
        return np.arange(len(x), dtype=np.int64)
    lo, hi = b
    corners = np.array([[a, c, e] for a in (lo[0], hi[0]) for c in (lo[1], hi[1]) for e in (lo[2], hi[2])])
    world = corners @ pose[:3, :3].T + pose[:3, 3]
    inside = np.all((x >= world.min(axis=0)) & (x <= world.max(axis=0)), axis=1)
    return np.nonzero(inside)[0].astype(np.int64)


def penetration(geom, pose: np.ndarray, pts: np.ndarray, r: float):
    """Sphere/body penetration — sdf.py:472-512.  Returns (psi, normal, hit, n_deg)."""
    R = pose[:3, :3]
    local = (pts - pose[:3, 3]) @ R
    d = np.atleast_1d(sdf_distance(geom, local))
    hit = d < r
    psi = np.where(hit, r - d, 0.0)
    normal = np.zeros_like(pts)
    n_deg = 0
    if hit.any():
        g = np.atleast_2d(sdf_gradient(geom, local[hit]))
        gn = _norm_rows(g)
        ok = gn > DEGENERATE_GRADIENT_EPS
        n_deg = int((~ok).sum())
        gw = np.zeros_like(g)
        gw[ok] = (g[ok] / gn[ok, None]) @ R.T
        normal[hit] = gw
        if n_deg:
            bad = np.zeros(len(pts), dtype=bool)
            bad[np.nonzero(hit)[0][~ok]] = True
            hit &= ~bad
            psi = np.where(hit, psi, 0.0)
    return psi, normal, hit, n_deg


# ---------------------------------------------------------------------------
# narrowphase — contact.py:244-300
# ---------------------------------------------------------------------------
@dataclass
class Contacts:
    owner: np.ndarray
    kind: np.ndarray   # 0 particle, 1 body
    other: np.ndarray
    e1: np.ndarray
    psi: np.ndarray
    vj: np.ndarray
    n_candidates: int
    n_coincident: int
    n_degenerate: int

    def __len__(self):
        return len(self.owner)

    def directed(self) -> np.ndarray:
        rows = np.stack([self.owner, self.kind, self.other], axis=1).astype(np.int64)
        if not len(rows):
            return rows.reshape(0, 3)
        return rows[np.lexsort((rows[:, 2], rows[:, 1], rows[:, 0]))]


def detect(x: np.ndarray, r: float, n_h: int, bodies) -> tuple[Contacts, dict]:
    """Broadphase + pp test + body pass (contact.py:257-300).  ``bodies`` are
    RigidBody-like objects whose pose/omega/v_origin are already at t+dt."""
    x = np.asarray(x, dtype=np.float64)
    n = len(x)
    cells = cell_coords(x, r)
    hashes = cell_hash(cells, n_h)
    order, starts = bucket_layout(hashes, n_h)
    ci, cj = candidate_rows(cells, order, starts, n_h)
    d = x[ci] - x[cj]
    dist2 = (d[:, 0] * d[:, 0] + d[:, 2] * d[:, 2]) + d[:, 1] * d[:, 1]
    m_pp = len(ci)
    not_coinc = dist2 >= COINCIDENT_EPS * COINCIDENT_EPS
    hit = np.nonzero((dist2 < (2.0 * r) ** 2) & not_coinc)[0]
    dist = np.sqrt(dist2[hit])
    parts = {
        "owner": [ci[hit]],
        "kind": [np.zeros(len(hit), dtype=np.int64)],
        "other": [cj[hit]],
        "e1": [d[hit] / dist[:, None]],
        "psi": [2.0 * r - dist],
        "vj": [np.zeros((len(hit), 3))],
    }
    n_deg = 0
    for b, body in enumerate(bodies):
        pose = np.asarray(body.pose, dtype=np.float64)
        near = near_body(x, r, body.geometry, pose)
        pts = x[near]
        bpsi, bn, bhit, nd = penetration(body.geometry, pose, pts, r)
        n_deg += nd
        cp = pts - bn * (r - bpsi)[:, None]
        vel = np.asarray(body.v_origin, dtype=np.float64) + np.cross(
            np.asarray(body.omega, dtype=np.float64), np.atleast_2d(cp) - pose[:3, 3])
        k = np.nonzero(bhit)[0]
        parts["owner"].append(near[k])
        parts["kind"].append(np.ones(len(k), dtype=np.int64))
        parts["other"].append(np.full(len(k), b, dtype=np.int64))
        parts["e1"].append(bn[k])
        parts["psi"].append(bpsi[k])
        parts["vj"].append(vel[k] if len(k) else np.zeros((0, 3)))
    c = Contacts(
        **{key: np.concatenate(v) for key, v in parts.items()},
        n_candidates=m_pp - n,
        n_coincident=m_pp - int(np.count_nonzero(not_coinc)) - n,
        n_degenerate=n_deg,
    )
    bp = {"cells": cells, "hashes": hashes, "order": order}
    return c, bp


# ---------------------------------------------------------------------------
# projected Jacobi — contact.py:393-518
# ---------------------------------------------------------------------------
def tangent_basis(e1: np.ndarray):
    """contact.py:47-56."""
    m = len(e1)
    pick = np.zeros((m, 3))
    pick[np.arange(m), np.abs(e1).argmin(axis=1)] = 1.0
    e2 = np.cross(e1, pick)
    e2 /= np.linalg.norm(e2, axis=1, keepdims=True)
    return e2, np.cross(e1, e2)


def pja(c: Contacts, v: np.ndarray, params, n_bodies: int):
    """Returns (dv, body_momentum, max_cone_violation, min_normal_impulse)."""
    v = np.asarray(v, dtype=np.float64)
    n = len(v)
    dv = np.zeros((n, 3))
    bm = np.zeros((max(n_bodies, 0), 3))
    if len(c) == 0:
        return dv, bm, 0.0, 0.0
    own, oth = c.owner, c.other
    pp = np.nonzero(c.kind == 0)[0]
    is_body = c.kind == 1
    e1 = c.e1
    e2, e3 = tangent_basis(e1)
    vj0 = c.vj.copy()
    vj0[pp] = v[oth[pp]]
    gdt = params.timestep * np.asarray(params.gravity, dtype=np.float64)
    bias = params.baumgarte_alpha * c.psi / params.timestep
    eff = np.where(c.kind == 0, 0.5, 1.0)
    mu, gamma = params.friction, params.gamma
    worst, least = 0.0, np.inf
    for _ in range(params.solver_iterations):
        vj = vj0.copy()
        vj[pp] += dv[oth[pp]]
        u = v[own] - gamma * vj + gdt + dv[own]
        b1 = np.maximum(-np.einsum("ij,ij->i", u, e1) + bias, 0.0)
        b2 = -np.einsum("ij,ij->i", u, e2)
        b3 = -np.einsum("ij,ij->i", u, e3)
        tn = np.hypot(b2, b3)
        cap = mu * b1
        s = np.where(tn > cap, cap / np.maximum(tn, 1e-300), 1.0)
        b2 = b2 * s
        b3 = b3 * s
        imp = (e1 * b1[:, None] + e2 * b2[:, None] + e3 * b3[:, None]) * eff[:, None]
        nxt = dv.copy()
        np.add.at(nxt, own, imp)
        dv = nxt
        if n_bodies and is_body.any():
            np.add.at(bm, oth[is_body], -params.particle_mass * imp[is_body])
        viol = np.hypot(b2, b3) - mu * b1
        worst = max(worst, float(viol.max()))
        least = min(least, float(b1.min()))
    if not np.all(np.isfinite(dv)):
        bad = np.nonzero(~np.isfinite(dv).all(axis=1))[0]
        raise OracleSolverError(f"non-finite velocity correction for particles {bad[:5].tolist()}")
    return dv, bm, worst, (least if np.isfinite(least) else 0.0)


# ---------------------------------------------------------------------------
# one step — stepper.py:57-144
# ---------------------------------------------------------------------------
def step(x: np.ndarray, v: np.ndarray, params, bodies, n_h: int | None = None, boundary=None):
    """Functional restatement of stepper.step for given post-update bodies.
    Returns (x_new, v_new, report dict, contacts, broadphase dict)."""
    x = np.array(x, dtype=np.float64)
    v = np.array(v, dtype=np.float64)
    n = len(x)
    r = params.radius
    n_h = int(n_h or table_size(n))
    if not np.all(np.isfinite(x)):
        raise ValueError("positions must be finite")
    c, bp = detect(x, r, n_h, bodies)
    dv, bm, worst, least = pja(c, v, params, len(bodies))
    v += params.timestep * np.asarray(params.gravity, dtype=np.float64) + dv
    x += params.timestep * v
    if boundary is not None:
        z = x[:, 2]
        z[z < boundary.z_min] += boundary.z_max - boundary.z_min
    n_pp = int((c.kind == 0).sum())
    report = {
        "n_contacts": n_pp,
        "n_candidates": c.n_candidates,
        "candidate_hit_rate": n_pp / max(c.n_candidates, 1),
        "max_penetration": float(c.psi.max()) if len(c) else 0.0,
        "kinetic_energy": 0.5 * params.particle_mass * float(np.einsum("ij,ij->", v, v)),
        "n_body_contacts": len(c) - n_pp,
        "n_coincident_skipped": c.n_coincident,
        "n_degenerate_skipped": c.n_degenerate,
        "max_cone_violation": worst,
        "min_normal_impulse": least,
        "body_momentum": bm,
    }
    return x, v, report, c, bp
