"""Contact-detection API (contact.py:126-300) backed by the device kernels.

``detect_contacts`` / ``narrowphase_contacts`` run the device broadphase and
narrowphase (K1-K5) on a scratch context and return a ``ContactSet`` with the
reference's fields.  Normals and depths are computed in float64 on the
device and stored as float32 (the resident contact-record format), so they
match the reference to ~1e-7 relative; the contact SET and the broadphase
counters are bit-exact.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from .engine import Engine
from .errors import SolverError

COINCIDENT_EPS = 1e-12
KIND_PARTICLE = 0
KIND_BODY = 1


def contact_frames(e1: np.ndarray):
    """Tangent basis used for the reported frames (contact.py:47-56).  The
    device solver never materialises it (the tangential impulse is the
    negated tangential relative velocity, frame-independent)."""
    m = len(e1)
    pick = np.zeros((m, 3))
    pick[np.arange(m), np.abs(e1).argmin(axis=1)] = 1.0
    e2 = np.cross(e1, pick)
    e2 /= np.linalg.norm(e2, axis=1, keepdims=True)
    return e2, np.cross(e1, e2)


class ContactSet:
    """Compressed contact list with the reference's array fields."""

    def __init__(self, owner, kind, other, e1, psi, vj, n_pp_candidates=0, n_coincident=0,
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

    def pair_set(self) -> set[tuple[int, int]]:
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


def device_detect(positions, r, n_h, bodies=(), params=None):
    """Run K1-K5 on the device for a given state; returns (ContactSet, report)."""
    from .scene import MaterialParams

    pos = np.ascontiguousarray(np.asarray(positions, dtype=np.float64).reshape(-1, 3))
    n = len(pos)
    bodies = list(bodies or [])
    if n == 0:
        empty = np.zeros(0, np.int64)
        return ContactSet(empty, empty, empty, np.zeros((0, 3)), np.zeros(0), np.zeros((0, 3))), None
    eng = Engine()
    try:
        eng._create(params or MaterialParams(radius=r), None, n, int(n_h), max(len(bodies), 1))
        eng.upload(pos, np.zeros_like(pos))
        rows = np.zeros(max(len(bodies), 1), dtype=N.BODY_DTYPE)
        for b, body in enumerate(bodies):
            eng.body_row(body, float(r), rows[b])
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
        count = ctypes.c_int64(0)
        owner = np.empty(m, np.int32)
        other = np.empty(m, np.int32)
        kind = np.empty(m, np.int32)
        psi = np.empty(m)
        e1 = np.empty((m, 3))
        st = N.lib().gg_tap_contacts(eng.ctx, m, ctypes.byref(count), N.ptr(owner), N.ptr(other),
                                     N.ptr(kind), N.ptr(psi), N.ptr(e1))
        N.check(eng.ctx, st, "gg_tap_contacts")
    finally:
        eng.close()
    # reference order: pp contacts by owner, then body contacts body by body
    key = np.lexsort((other, kind, owner))
    pp = kind[key] == KIND_PARTICLE
    order = np.concatenate([key[pp], key[~pp][np.lexsort((owner[key[~pp]], other[key[~pp]]))]])
    cs = ContactSet(owner[order].astype(np.int64), kind[order].astype(np.int64),
                    other[order].astype(np.int64), e1[order], psi[order], np.zeros((m, 3)),
                    int(rep["n_candidates"][0]), int(rep["n_coincident"][0]),
                    int(rep["n_degenerate"][0]))
    return cs, rep[0]


def narrowphase_contacts(positions, r, hmap, bodies):
    return device_detect(positions, r, hmap.n_h, bodies)[0]


def detect_contacts(positions, r, hmap, bodies=None):
    return device_detect(positions, r, hmap.n_h, bodies or [])[0]


__all__ = [
    "COINCIDENT_EPS",
    "ContactSet",
    "KIND_BODY",
    "KIND_PARTICLE",
    "SolverError",
    "contact_frames",
    "detect_contacts",
    "device_detect",
    "narrowphase_contacts",
]
