"""Broadphase API (broadphase.py:33-182) backed by the device kernels.

``build_hashmap`` runs the device broadphase (K1-K4 of the step schedule:
hash, count, scan, scatter, stable fix-up) on a scratch context and returns
the reference's ``SpatialHashmap`` view (table/next linked lists, cells,
hashes), derived from the device's stable bucket order exactly as the
reference derives it from ``np.lexsort`` (broadphase.py:120-127).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .engine import Engine, default_table_size, utility_context

HASH_PRIMES = (73856093, 19349663, 83492791)
CELL_OFFSET = 100
EMPTY = -1


def round_half_away(x: np.ndarray) -> np.ndarray:
    """Nearest integer, halves away from zero (host helper)."""
    x = np.asarray(x, dtype=np.float64)
    return np.copysign(np.floor(np.abs(x) + 0.5), x)


def position_cells(positions: np.ndarray, r: float) -> np.ndarray:
    """round_half_away(x / 2r) as int64 (broadphase.py:33-41), on the device
    in float64 (gg_position_cells)."""
    p = np.asarray(positions, dtype=np.float64)
    flat = np.ascontiguousarray(p.reshape(-1, 3))
    out = np.empty(flat.shape, dtype=np.int64)
    if len(flat):
        uc = utility_context()
        st = N.lib().gg_position_cells(uc.ctx, N.ptr(flat), len(flat), float(r), N.ptr(out))
        N.check(uc.ctx, st, "gg_position_cells")
    return out.reshape(p.shape)


def spatial_hash(cells: np.ndarray, n_h: int) -> np.ndarray:
    """Device evaluation of the cell hash (broadphase.py:44-55)."""
    if n_h < 1:
        raise ValueError("hash table size must be >= 1")
    c = np.asarray(cells, dtype=np.int64)
    single = c.ndim == 1
    flat = np.ascontiguousarray(c.reshape(-1, 3))
    out = np.empty(len(flat), dtype=np.int64)
    uc = utility_context()
    st = N.lib().gg_spatial_hash(uc.ctx, N.ptr(flat), len(flat), int(n_h), N.ptr(out))
    N.check(uc.ctx, st, "gg_spatial_hash")
    if single:
        return out[0]
    return out.reshape(c.shape[:-1])


@dataclass
class SpatialHashmap:
    table: np.ndarray
    next: np.ndarray
    cell_size: float
    n_h: int
    cells: np.ndarray
    hashes: np.ndarray
    order: np.ndarray | None = None  # device stable bucket order (user ids)

    def chain(self, h: int) -> list[int]:
        out = []
        i = int(self.table[h])
        while i != EMPTY:
            out.append(i)
            i = int(self.next[i])
        return out


def _cell_context(cells: np.ndarray, cell_size: float, n_h: int) -> Engine:
    """A scratch context whose resident state sits at the cell centres, so the
    device broadphase sees exactly ``cells`` (the float32 centre of cell c
    rounds back to c for |c| < 2^22).  The broadphase depends only on the
    cells, so float64 inputs that are not float32-representable are handled
    exactly."""
    from .scene import MaterialParams

    c = np.ascontiguousarray(np.asarray(cells, dtype=np.int64).reshape(-1, 3))
    if len(c) and np.abs(c).max() >= (1 << 22):
        raise ValueError("cell coordinates beyond +-2^22 are not supported")
    eng = Engine()
    eng._create(MaterialParams(radius=0.5 * float(cell_size)), None, len(c), int(n_h), 1)
    centres = c.astype(np.float64) * float(cell_size)
    eng.upload(centres, np.zeros_like(centres))
    return eng


def _tap_hash(eng: Engine, n: int):
    cells = np.empty((n, 3), dtype=np.int64)
    hashes = np.empty(n, dtype=np.int64)
    order = np.empty(n, dtype=np.int64)
    st = N.lib().gg_tap_hash(eng.ctx, N.ptr(cells), N.ptr(hashes), N.ptr(order))
    N.check(eng.ctx, st, "gg_tap_hash")
    return cells, hashes, order


def device_hash_sort(positions: np.ndarray, r: float, n_h: int):
    """(cells, hashes, order) from the device broadphase: cells from the
    float64 positions (gg_position_cells), then hash, counting sort and the
    stable bucket order on a context placed at those cells."""
    pos = np.ascontiguousarray(np.asarray(positions, dtype=np.float64).reshape(-1, 3))
    n = len(pos)
    if n == 0:
        return np.zeros((0, 3), np.int64), np.zeros(0, np.int64), np.zeros(0, np.int64)
    cells = position_cells(pos, r)
    eng = _cell_context(cells, 2.0 * r, n_h)
    try:
        dcells, hashes, order = _tap_hash(eng, n)
    finally:
        eng.close()
    if not np.array_equal(dcells, cells):
        raise RuntimeError("device cells differ from position_cells (internal error)")
    return cells, hashes, order


def build_hashmap(positions: np.ndarray, r: float, n_h: int,
                  insertion_order: np.ndarray | None = None) -> SpatialHashmap:
    positions = np.asarray(positions, dtype=np.float64)
    if positions.ndim != 2 or positions.shape[1] != 3:
        raise ValueError("positions must have shape (n, 3)")
    if not np.all(np.isfinite(positions)):
        raise ValueError("positions must be finite")
    if n_h < 1:
        raise ValueError("hash table size must be >= 1")
    n = len(positions)
    cells, hashes, order = device_hash_sort(positions, r, n_h)
    nxt = np.full(n, EMPTY, dtype=np.int64)
    table = np.full(n_h, EMPTY, dtype=np.int64)
    if n:
        chain_order = order
        if insertion_order is not None:
            rank = np.empty(n, dtype=np.int64)
            rank[np.asarray(insertion_order)] = np.arange(n)
            chain_order = np.lexsort((rank, hashes))
        hs = hashes[chain_order]
        same = hs[1:] == hs[:-1]
        nxt[chain_order[1:][same]] = chain_order[:-1][same]
        last = np.r_[hs[1:] != hs[:-1], True]
        table[hs[last]] = chain_order[last]
    return SpatialHashmap(table=table, next=nxt, cell_size=2.0 * r, n_h=n_h, cells=cells,
                          hashes=hashes, order=order)


_NEIGHBOR_OFFSETS = np.array(
    [[dx, dy, dz] for dx in (-1, 0, 1) for dy in (-1, 0, 1) for dz in (-1, 0, 1)], dtype=np.int64
)


def query_candidates(hmap, positions: np.ndarray, i: int) -> list[int]:
    """Candidate neighbours of particle i (broadphase.py:133-146): the chains
    of its 27 neighbour buckets (device hash, ascending unique buckets), in
    chain order, i itself excluded."""
    nb = np.asarray(hmap.cells[i], dtype=np.int64)[None, :] + _NEIGHBOR_OFFSETS
    buckets = np.unique(spatial_hash(nb, hmap.n_h))
    out: list[int] = []
    for h in buckets:
        j = int(hmap.table[int(h)])
        while j != EMPTY:
            if j != i:
                out.append(j)
            j = int(hmap.next[j])
    return out


def candidate_pairs(hmap) -> tuple[np.ndarray, np.ndarray]:
    """All directed candidate pairs (i, j != i) (broadphase.py:185-196) on
    the device (gg_tap_candidates): i ascending, i's candidates in the order
    the reference's _candidate_csr enumerates them."""
    cells = np.asarray(hmap.cells, dtype=np.int64).reshape(-1, 3)
    n = len(cells)
    if n == 0:
        return np.empty(0, np.int64), np.empty(0, np.int64)
    eng = _cell_context(cells, float(hmap.cell_size), int(hmap.n_h))
    try:
        lib = N.lib()
        count = ctypes.c_int64(0)
        N.check(eng.ctx, lib.gg_tap_candidates(eng.ctx, 0, ctypes.byref(count), None, None),
                "gg_tap_candidates")
        m = count.value
        ci = np.empty(m, dtype=np.int64)
        cj = np.empty(m, dtype=np.int64)
        if m:
            N.check(eng.ctx, lib.gg_tap_candidates(eng.ctx, m, ctypes.byref(count), N.ptr(ci),
                                                   N.ptr(cj)), "gg_tap_candidates")
    finally:
        eng.close()
    return ci, cj


__all__ = [
    "candidate_pairs",
    "query_candidates",
    "CELL_OFFSET",
    "EMPTY",
    "HASH_PRIMES",
    "SpatialHashmap",
    "build_hashmap",
    "default_table_size",
    "device_hash_sort",
    "position_cells",
    "round_half_away",
    "spatial_hash",
]
