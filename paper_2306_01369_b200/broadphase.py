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
    return round_half_away(np.asarray(positions) / (2.0 * r)).astype(np.int64)


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


def device_hash_sort(positions: np.ndarray, r: float, n_h: int):
    """(cells, hashes, order) from the device broadphase."""
    from .scene import MaterialParams

    pos = np.ascontiguousarray(np.asarray(positions, dtype=np.float64).reshape(-1, 3))
    n = len(pos)
    if n == 0:
        return np.zeros((0, 3), np.int64), np.zeros(0, np.int64), np.zeros(0, np.int64)
    eng = Engine()
    try:
        eng._create(MaterialParams(radius=r), None, n, int(n_h), 1)
        eng.upload(pos, np.zeros_like(pos))
        cells = np.empty((n, 3), dtype=np.int64)
        hashes = np.empty(n, dtype=np.int64)
        order = np.empty(n, dtype=np.int64)
        st = N.lib().gg_tap_hash(eng.ctx, N.ptr(cells), N.ptr(hashes), N.ptr(order))
        N.check(eng.ctx, st, "gg_tap_hash")
    finally:
        eng.close()
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


__all__ = [
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
