"""Contact API (contact.py of the reference) backed by the device kernels.

Two families of entry points:

* the L1 functions on caller-supplied float64 arrays — ``candidate_pairs``
  (broadphase.py), ``narrowphase_candidates``, ``narrowphase_contacts`` /
  ``detect_contacts``, ``solve_contacts_pja``, ``project_friction_cone`` —
  run device kernels on the reference's own data layout and operation order
  (gg_tap_candidates, gg_narrow_pairs, gg_solve_contacts, gg_project_cone):
  same contacts in the same order, impulses to float64 rounding;
* ``device_detect`` runs the step's own detection (K1-K6 on the resident
  float32 state, gg_detect + gg_tap_contacts) — the parity tap of the hot
  path.

``contact_frames`` / ``make_contact_frame`` build the reported (e2, e3) frames
on the host; the device solver builds the same frame per contact.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .engine import Engine, _params_struct, utility_context
from .errors import SolverError

COINCIDENT_EPS = 1e-12
KIND_PARTICLE = 0
KIND_BODY = 1


def make_contact_frame(normal: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Orthonormal completion of one contact normal (contact.py:33-44)."""
    e1 = np.asarray(normal, dtype=np.float64)
    n = np.linalg.norm(e1)
    if n < 1e-12:
        raise ValueError("contact normal must be nonzero")
    e2, e3 = contact_frames(e1[None, :] / n)
    return e2[0], e3[0]


def contact_frames(e1: np.ndarray):
    """(e2, e3) of unit normals e1 (contact.py:47-56): e2 = e1 x axis of the
    smallest |component| (first on ties), normalised; e3 = e1 x e2."""
    e1 = np.asarray(e1, dtype=np.float64)
    m = len(e1)
    pick = np.zeros((m, 3))
    pick[np.arange(m), np.abs(e1).argmin(axis=1)] = 1.0
    e2 = np.cross(e1, pick)
    e2 /= np.linalg.norm(e2, axis=1, keepdims=True)
    return e2, np.cross(e1, e2)


def project_friction_cone(b: np.ndarray, mu: float, psi, alpha: float, dt: float) -> np.ndarray:
    """Coulomb-cone projection with the stabilisation bias on the normal
    component (contact.py:59-81), on the device (gg_project_cone)."""
    if mu < 0 or dt <= 0:
        raise ValueError("require mu >= 0 and dt > 0")
    b = np.array(b, dtype=np.float64)
    single = b.ndim == 1
    b = np.ascontiguousarray(np.atleast_2d(b))
    k = b.shape[0]
    ps = np.asarray(psi, dtype=np.float64)
    scalar = ps.ndim == 0
    ps = np.ascontiguousarray(ps.reshape(1) if scalar else np.broadcast_to(ps, (k,)))
    uc = utility_context()
    st = N.lib().gg_project_cone(uc.ctx, N.ptr(b), k, N.ptr(ps), int(scalar), float(mu), float(alpha),
                                 float(dt))
    N.check(uc.ctx, st, "gg_project_cone")
    return b[0] if single else b


@dataclass
class Contact:
    """One contact pair (contact.py:84-101)."""

    kind: int  # KIND_PARTICLE or KIND_BODY
    i: int
    j: int  # particle index or body index
    e1: np.ndarray  # unit normal, pointing from j toward i
    e2: np.ndarray
    e3: np.ndarray
    psi: float

    @property
    def frame(self) -> np.ndarray:
        """Rotation mapping world vectors into (e1, e2, e3) coordinates."""
        return np.stack([self.e1, self.e2, self.e3])


@dataclass
class CandidateContacts:
    """Narrowphase results over all candidates, uncompressed (contact.py:103-123)."""

    owner: np.ndarray
    kind: np.ndarray
    other: np.ndarray
    e1: np.ndarray
    psi: np.ndarray
    vj: np.ndarray
    colliding: np.ndarray
    n_pp_candidates: int = 0
    n_coincident: int = 0
    n_degenerate: int = 0

    def __len__(self) -> int:
        return len(self.owner)


class ContactSet:
    """Compressed list of actual contacts (contact.py:126-184)."""

    def __init__(self, cand: CandidateContacts | None = None, *arrays, **kw):
        if arrays or kw:  # ContactSet(owner, kind, other, e1, psi, vj, ...) (internal)
            self._init_arrays(cand, *arrays, **kw)
            return
        if cand is None:
            return
        keep = np.nonzero(cand.colliding)[0]
        self._init_arrays(cand.owner[keep], cand.kind[keep], cand.other[keep], cand.e1[keep],
                          cand.psi[keep], cand.vj[keep], cand.n_pp_candidates, cand.n_coincident,
                          cand.n_degenerate)

    def _init_arrays(self, owner, kind, other, e1, psi, vj, n_pp_candidates=0, n_coincident=0,
                     n_degenerate=0):
        self.owner = owner
        self.kind = kind
        self.other = other
        self.e1 = e1
        self.psi = psi
        self.vj = vj
        if len(owner):
            self.e2, self.e3 = contact_frames(e1)
        else:
            self.e2, self.e3 = np.zeros((0, 3)), np.zeros((0, 3))
        self.n_pp_candidates = n_pp_candidates
        self.n_coincident = n_coincident
        self.n_degenerate = n_degenerate

    def __len__(self) -> int:
        return len(self.owner)

    def __getitem__(self, k: int) -> Contact:
        return Contact(kind=int(self.kind[k]), i=int(self.owner[k]), j=int(self.other[k]),
                       e1=self.e1[k], e2=self.e2[k], e3=self.e3[k], psi=float(self.psi[k]))

    def __iter__(self):
        return (self[k] for k in range(len(self)))

    def pair_set(self) -> set[tuple[int, int]]:
        """Undirected particle-particle contact pairs (i < j)."""
        pp = self.kind == KIND_PARTICLE
        a = np.minimum(self.owner[pp], self.other[pp])
        b = np.maximum(self.owner[pp], self.other[pp])
        return set(zip(a.tolist(), b.tolist()))

    def directed(self) -> np.ndarray:
        """(owner, kind, other) rows sorted lexicographically — the parity key."""
        rows = np.stack([self.owner, self.kind, self.other], axis=1).astype(np.int64)
        if len(rows) == 0:
            return rows.reshape(0, 3)
        return rows[np.lexsort((rows[:, 2], rows[:, 1], rows[:, 0]))]


def _empty_contacts() -> ContactSet:
    e = np.zeros(0, np.int64)
    return ContactSet(e, e, e, np.zeros((0, 3)), np.zeros(0), np.zeros((0, 3)))


# ---------------------------------------------------------------------------
# L1 entry points on float64 arrays
# ---------------------------------------------------------------------------
def _body_rows(eng_like, bodies, r: float) -> np.ndarray:
    rows = np.zeros(max(len(bodies), 1), dtype=N.BODY_DTYPE)
    for b, body in enumerate(bodies):
        eng_like.body_row(body, float(r), rows[b])
    return rows


def narrowphase_candidates(positions: np.ndarray, r: float, ci: np.ndarray, cj: np.ndarray,
                           bodies) -> CandidateContacts:
    """Exact contact test on every explicit candidate pair and every
    (particle, body) candidate (contact.py:206-223, _assemble_candidates
    :303-369), on the device (gg_narrow_pairs)."""
    if r <= 0:
        raise ValueError("particle radius must be positive")
    pos = np.ascontiguousarray(np.asarray(positions, dtype=np.float64).reshape(-1, 3))
    ci = np.ascontiguousarray(np.asarray(ci, dtype=np.int64).reshape(-1))
    cj = np.ascontiguousarray(np.asarray(cj, dtype=np.int64).reshape(-1))
    if ci.shape != cj.shape:
        raise ValueError("ci and cj must have equal length")
    bodies = list(bodies or [])
    n, m, nb = len(pos), len(ci), len(bodies)
    uc = utility_context()
    rows = _body_rows(uc.engine, bodies, r)
    e1 = np.zeros((m, 3))
    psi = np.zeros(m)
    col = np.zeros(m, dtype=np.uint8)
    near = np.zeros((nb, n), dtype=np.uint8)
    hit = np.zeros((nb, n), dtype=np.uint8)
    bpsi = np.zeros((nb, n))
    bn = np.zeros((nb, n, 3))
    bvj = np.zeros((nb, n, 3))
    n_coi, n_deg = ctypes.c_int64(0), ctypes.c_int64(0)
    st = N.lib().gg_narrow_pairs(uc.ctx, N.ptr(pos), n, N.ptr(ci), N.ptr(cj), m, float(r), N.ptr(rows),
                                 nb, N.ptr(e1), N.ptr(psi), N.ptr(col), ctypes.byref(n_coi),
                                 N.ptr(near), N.ptr(hit), N.ptr(bpsi), N.ptr(bn), N.ptr(bvj),
                                 ctypes.byref(n_deg))
    N.check(uc.ctx, st, "gg_narrow_pairs")
    owners, kinds, others, e1s, psis, vjs, cols = [ci], [np.zeros(m, np.int64)], [cj], [e1], [psi], \
        [np.zeros((m, 3))], [col.astype(bool)]
    for b in range(nb):
        idx = np.nonzero(near[b])[0].astype(np.int64)
        owners.append(idx)
        kinds.append(np.full(len(idx), KIND_BODY, dtype=np.int64))
        others.append(np.full(len(idx), b, dtype=np.int64))
        e1s.append(bn[b, idx])
        psis.append(bpsi[b, idx])
        vjs.append(bvj[b, idx])
        cols.append(hit[b, idx].astype(bool))
    return CandidateContacts(owner=np.concatenate(owners), kind=np.concatenate(kinds),
                             other=np.concatenate(others), e1=np.concatenate(e1s),
                             psi=np.concatenate(psis), vj=np.concatenate(vjs),
                             colliding=np.concatenate(cols), n_pp_candidates=m,
                             n_coincident=int(n_coi.value), n_degenerate=int(n_deg.value))


def narrowphase_contacts(positions, r, hmap, bodies) -> ContactSet:
    """Broadphase + narrowphase compacted to a ContactSet (contact.py:244-300):
    the device candidate pairs of ``hmap`` and the float64 exact test, in the
    reference's contact order (pp by owner in candidate order, then body by
    body)."""
    from .broadphase import candidate_pairs

    pos = np.asarray(positions, dtype=np.float64)
    ci, cj = candidate_pairs(hmap)
    return ContactSet(narrowphase_candidates(pos, r, ci, cj, list(bodies or [])))


def detect_contacts(positions, r, hmap, bodies=None) -> ContactSet:
    """Detection pass only (contact.py:372-379)."""
    return narrowphase_contacts(np.asarray(positions, float), r, hmap, bodies or [])


@dataclass
class ImpulseBuffer:
    """Per-particle velocity corrections plus solver diagnostics (contact.py:382-390)."""

    delta_v: np.ndarray
    max_cone_violation: float = 0.0
    min_normal_impulse: float = 0.0
    body_momentum: np.ndarray = field(default_factory=lambda: np.zeros((0, 3)))
    n_contacts: int = 0


def solve_contacts_pja(contacts, velocities: np.ndarray, params, n_bodies: int = 0,
                       inline_narrowphase_mask: bool = False,
                       refresh_candidates=None) -> ImpulseBuffer:
    """Projected Jacobi sweeps over a contact list or a masked candidate list
    (contact.py:393-518) on the device (gg_solve_contacts).  With
    ``refresh_candidates`` the candidates are re-evaluated before every sweep
    after the first (the naive single-loop pipeline) and the sweeps run one
    device call at a time."""
    v = np.ascontiguousarray(np.asarray(velocities, dtype=np.float64).reshape(-1, 3))
    n = len(v)
    nb = max(int(n_bodies), 0)
    dv = np.zeros((n, 3))
    bm = np.zeros((nb, 3))
    m = len(contacts.owner)
    if m == 0:
        return ImpulseBuffer(delta_v=dv, body_momentum=bm)
    S = int(params.solver_iterations)
    p = _params_struct(params, None)
    diag = np.array([0.0, np.inf])
    live = ctypes.c_int64(0)
    uc = utility_context()

    def call(cs, mask, first, count):
        arrs = [np.ascontiguousarray(np.asarray(a, dtype=dt)) for a, dt in (
            (cs.owner, np.int64), (cs.kind, np.int64), (cs.other, np.int64), (cs.e1, np.float64),
            (cs.psi, np.float64), (cs.vj, np.float64))]
        msk = None if mask is None else np.ascontiguousarray(np.asarray(mask, dtype=np.uint8))
        cl = N.GGContactList(len(arrs[0]), *[N.ptr(a) for a in arrs], N.ptr(msk))
        st = N.lib().gg_solve_contacts(uc.ctx, ctypes.byref(cl), n, N.ptr(v), ctypes.byref(p), nb,
                                       first, count, N.ptr(dv), N.ptr(bm) if nb else None, N.ptr(diag),
                                       ctypes.byref(live))
        N.check(uc.ctx, st, "gg_solve_contacts")

    mask = contacts.colliding if inline_narrowphase_mask else None
    if refresh_candidates is None:
        call(contacts, mask, 0, S)
    else:
        for s in range(S):
            cur = contacts if s == 0 else refresh_candidates()
            call(cur, cur.colliding if s > 0 else mask, s, 1)
    mn = float(diag[1])
    return ImpulseBuffer(delta_v=dv, max_cone_violation=float(diag[0]),
                         min_normal_impulse=mn if np.isfinite(mn) else 0.0, body_momentum=bm,
                         n_contacts=int(live.value))


# ---------------------------------------------------------------------------
# the step's own detection (resident float32 state): parity tap
# ---------------------------------------------------------------------------
def device_detect(positions, r, n_h, bodies=(), params=None):
    """Run K1-K6 of the step on the device for a given state (positions are
    stored as float32, like the resident state); returns (ContactSet in the
    reference's order, report)."""
    from .scene import MaterialParams

    pos = np.ascontiguousarray(np.asarray(positions, dtype=np.float64).reshape(-1, 3))
    n = len(pos)
    bodies = list(bodies or [])
    if n == 0:
        return _empty_contacts(), None
    eng = Engine()
    try:
        eng._create(params or MaterialParams(radius=r), None, n, int(n_h), max(len(bodies), 1))
        eng.upload(pos, np.zeros_like(pos))
        rows = _body_rows(eng, bodies, r)
        rep = np.zeros(1, dtype=N.REPORT_DTYPE)
        while True:
            st = N.lib().gg_detect(eng.ctx, N.ptr(rows), len(bodies), N.ptr(rep))
            if st == N.GG_ECAPACITY:
                need = N.lib().gg_required_contacts(eng.ctx)
                eng.max_contacts = max(2 * eng.max_contacts, need + 4)
                N.check(eng.ctx, N.lib().gg_set_max_contacts(eng.ctx, eng.max_contacts), "grow")
                continue
            N.check(eng.ctx, st, "gg_detect")
            break
        m = int(rep["n_contacts"][0] + rep["n_body_contacts"][0])
        owner, other, kind, psi, e1, vj = tap_contacts(eng, m)
    finally:
        eng.close()
    cs = ContactSet(owner.astype(np.int64), kind.astype(np.int64), other.astype(np.int64), e1, psi, vj,
                    int(rep["n_candidates"][0]), int(rep["n_coincident"][0]), int(rep["n_degenerate"][0]))
    return cs, rep[0]


def tap_contacts(eng: Engine, m: int):
    """gg_tap_contacts: the contacts of the last detection, reference order."""
    count = ctypes.c_int64(0)
    owner = np.empty(m, np.int32)
    other = np.empty(m, np.int32)
    kind = np.empty(m, np.int32)
    psi = np.empty(m)
    e1 = np.empty((m, 3))
    vj = np.empty((m, 3))
    st = N.lib().gg_tap_contacts(eng.ctx, m, ctypes.byref(count), N.ptr(owner), N.ptr(other),
                                 N.ptr(kind), N.ptr(psi), N.ptr(e1), N.ptr(vj))
    N.check(eng.ctx, st, "gg_tap_contacts")
    k = min(m, int(count.value))
    return owner[:k], other[:k], kind[:k], psi[:k], e1[:k], vj[:k]


__all__ = [
    "COINCIDENT_EPS",
    "CandidateContacts",
    "Contact",
    "ContactSet",
    "ImpulseBuffer",
    "KIND_BODY",
    "KIND_PARTICLE",
    "SolverError",
    "contact_frames",
    "detect_contacts",
    "device_detect",
    "make_contact_frame",
    "narrowphase_candidates",
    "narrowphase_contacts",
    "project_friction_cone",
    "solve_contacts_pja",
]
