"""ctypes binding of ``_lib/libgranusim_b200.so`` (include/granusim_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
present, every entry point that needs it raises.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from .errors import SolverError

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("GG_LIB", str(_PKG / "_lib" / "libgranusim_b200.so")))  # GG_LIB: A/B experiments

GG_OK = 0
GG_EINVAL = 1
GG_ENONFINITE = 2
GG_ECAPACITY = 3
GG_ECUDA = 4
GG_EPOSITIONS = 5

GEOM_SPHERE = 1
GEOM_HALFSPACE = 2
GEOM_BOX = 3
GEOM_CYLINDER = 4
GEOM_TUBE = 5
GEOM_GRID = 6


class GGParams(C.Structure):
    _fields_ = [
        ("radius", C.c_double),
        ("particle_mass", C.c_double),
        ("friction", C.c_double),
        ("baumgarte_alpha", C.c_double),
        ("timestep", C.c_double),
        ("gravity", C.c_double * 3),
        ("gamma", C.c_double),
        ("contact_d2", C.c_double),
        ("coincident_d2", C.c_double),
        ("gdt", C.c_double * 3),
        ("solver_iterations", C.c_int32),
        ("has_boundary", C.c_int32),
        ("z_min", C.c_double),
        ("z_max", C.c_double),
    ]


class GGContactList(C.Structure):
    """gg_contact_list: a ContactSet / CandidateContacts in array form."""

    _fields_ = [
        ("m", C.c_int64),
        ("owner", C.c_void_p),
        ("kind", C.c_void_p),
        ("other", C.c_void_p),
        ("e1", C.c_void_p),
        ("psi", C.c_void_p),
        ("vj", C.c_void_p),
        ("colliding", C.c_void_p),
    ]


# gg_body as a numpy structured dtype so per-step body tables for a whole
# batch are filled with array ops and handed over as one pointer.
BODY_DTYPE = np.dtype(
    [
        ("kind", "<i4"),
        ("grid_id", "<i4"),
        ("bounded", "<i4"),
        ("reserved", "<i4"),
        ("shape", "<f8", (4,)),
        ("rot", "<f8", (9,)),
        ("trans", "<f8", (3,)),
        ("omega", "<f8", (3,)),
        ("v_origin", "<f8", (3,)),
        ("aabb_lo", "<f8", (3,)),
        ("aabb_hi", "<f8", (3,)),
    ],
    align=True,
)
assert BODY_DTYPE.itemsize == 240

REPORT_DTYPE = np.dtype(
    [
        ("n_contacts", "<i8"),
        ("n_candidates", "<i8"),
        ("n_body_contacts", "<i8"),
        ("n_coincident", "<i8"),
        ("n_degenerate", "<i8"),
        ("max_penetration", "<f8"),
        ("kinetic_energy", "<f8"),
        ("max_cone_violation", "<f8"),
        ("min_normal_impulse", "<f8"),
    ]
)

_lib = None


def _bind(lib: C.CDLL) -> None:
    P = C.c_void_p
    i32, i64, dbl = C.c_int32, C.c_int64, C.c_double
    sig = {
        "gg_create": (C.c_int, [C.c_int, C.POINTER(GGParams), i64, i64, i32, i32, C.POINTER(P)]),
        "gg_create_batched": (C.c_int, [C.c_int, C.POINTER(GGParams), i32, i64, i64, i32, i32,
                                        C.POINTER(P)]),
        "gg_num_envs": (C.c_int, [P]),
        "gg_env_box_stats": (C.c_int, [P, P, P, P, P]),
        "gg_render_depth": (C.c_int, [P, P, i32, i32, P, i32, P]),
        "gg_set_render_mode": (C.c_int, [i32]),
        "gg_bake_mesh_sdf": (C.c_int, [i32, P, i64, P, i64, P, P, P, P, C.POINTER(C.c_float)]),
        "gg_slab_setup": (C.c_int, [P, i64, i64, i32, i32]),
        "gg_slab_load": (C.c_int, [P, P, P, P, i64]),
        "gg_slab_migrate_pack": (C.c_int, [P, P, P, i64, P]),
        "gg_slab_migrate_unpack": (C.c_int, [P, P, i64, P, i64]),
        "gg_slab_resort": (C.c_int, [P]),
        "gg_slab_ghost_pack": (C.c_int, [P, P, P, i64, P]),
        "gg_slab_ghost_unpack": (C.c_int, [P, P, i64, P, i64]),
        "gg_slab_detect": (C.c_int, [P, P, i32]),
        "gg_slab_sweep": (C.c_int, [P, i32]),
        "gg_slab_halo_pack": (C.c_int, [P, i32, P, P]),
        "gg_slab_halo_unpack": (C.c_int, [P, i32, P, P]),
        "gg_slab_finish": (C.c_int, [P, P, P]),
        "gg_slab_owned": (i64, [P]),
        "gg_slab_get": (C.c_int, [P, P, P, P, i64, P]),
        "gg_slab_mailbox": (C.c_int, [P, i64, P]),
        "gg_slab_connect": (C.c_int, [P, i32, P]),
        "gg_slab_halo_p2p": (C.c_int, [P, i32, C.c_uint64]),
        "gg_slab_exchange_p2p": (C.c_int, [P, C.c_uint64, i32, P]),
        "gg_slab_solve_p2p": (C.c_int, [P, C.c_uint64]),
        "gg_slab_step_p2p": (C.c_int, [P, P, i32, i32, P, P, P]),
        "gg_slab_run_p2p": (C.c_int, [P, P, i32, i32, P, P, P, P]),
        "gg_destroy": (C.c_int, [P]),
        "gg_last_error": (C.c_char_p, [P]),
        "gg_set_params": (C.c_int, [P, C.POINTER(GGParams)]),
        "gg_set_state_f64": (C.c_int, [P, P, P]),
        "gg_get_state_f64": (C.c_int, [P, P, P]),
        "gg_set_state_f32x4_dev": (C.c_int, [P, P, P]),
        "gg_get_state_f32x4_dev": (C.c_int, [P, P, P]),
        "gg_upload_grid": (C.c_int, [P, P, P, P, P, C.POINTER(i32)]),
        "gg_step": (C.c_int, [P, i32, P, i32, i32]),
        "gg_detect": (C.c_int, [P, P, i32, P]),
        "gg_bench_steps": (C.c_int, [P, i32, P, i32, i64, P]),
        "gg_profile_steps": (C.c_int, [P, i32, P, i32, P, P]),
        "gg_profile_kind_name": (C.c_char_p, [i32]),
        "gg_sync": (C.c_int, [P, P, P, i32, C.POINTER(i32), C.POINTER(i32)]),
        "gg_last_batch_ms": (C.c_int, [P, C.POINTER(C.c_float)]),
        "gg_tap_hash": (C.c_int, [P, P, P, P]),
        "gg_tap_contacts": (C.c_int, [P, i64, C.POINTER(i64), P, P, P, P, P, P]),
        "gg_drive_fixed": (C.c_int, [P, i32, P]),
        "gg_drive_track": (C.c_int, [P, i32, P, P, P, P, P, P, dbl, dbl, dbl, P]),
        "gg_drive_command": (C.c_int, [P, i32, P]),
        "gg_drive_chain": (C.c_int, [P, i32, P, P, P, i32, i32, P, P, P, P, P, P, P]),
        "gg_drive_chain_state": (C.c_int, [P, i32, P]),
        "gg_drive_state": (C.c_int, [P, i32, P, P, P]),
        "gg_batch_reports": (C.c_int, [P, i32, i32, P, P]),
        "gg_step_resume": (C.c_int, [P, i32, i32, i32]),
        "gg_position_cells": (C.c_int, [P, P, i64, dbl, P]),
        "gg_tap_candidates": (C.c_int, [P, i64, C.POINTER(i64), P, P]),
        "gg_narrow_pairs": (C.c_int, [P, P, i64, P, P, i64, dbl, P, i32, P, P, P, C.POINTER(i64),
                                      P, P, P, P, P, C.POINTER(i64)]),
        "gg_solve_contacts": (C.c_int, [P, C.POINTER(GGContactList), i64, P, C.POINTER(GGParams),
                                        i32, i32, i32, P, P, P, C.POINTER(i64)]),
        "gg_project_cone": (C.c_int, [P, P, i64, P, i32, dbl, dbl, dbl]),
        "gg_penetration": (C.c_int, [P, P, P, i64, dbl, P, P, P, C.POINTER(i64)]),
        "gg_spatial_hash": (C.c_int, [P, P, i64, i64, P]),
        "gg_set_max_contacts": (C.c_int, [P, i32]),
        "gg_max_contacts": (C.c_int, [P]),
        "gg_set_resort_every": (C.c_int, [P, i32]),
        "gg_set_solve_mode": (C.c_int, [P, i32]),
        "gg_phase_timer": (C.c_int, [P, i32, P, i32]),
        "gg_required_contacts": (C.c_int, [P]),
        "gg_host_register": (C.c_int, [P, i64]),
        "gg_host_unregister": (C.c_int, [P]),
        "gg_stream": (P, [P]),
        "gg_build_info": (C.c_char_p, []),
        "gg_kernel_launches": (i64, [P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def lib() -> C.CDLL:
    """Load the sm_100a library (fails loudly; no fallback)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2306_01369_b200.build` "
                "(there is no CPU fallback)"
            )
        handle = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | getattr(os, "RTLD_GLOBAL", 0))
        _bind(handle)
        _lib = handle
    return _lib


def exported_symbols() -> list[str]:
    return [n for n in dir(lib()) if n.startswith("gg_")]


def ptr(a: np.ndarray | None) -> int | None:
    return None if a is None else a.ctypes.data


def last_error(ctx) -> str:
    msg = lib().gg_last_error(ctx)
    return msg.decode() if msg else ""


def check(ctx, status: int, where: str = "") -> None:
    """Map a C status to the reference's exception types (contact.py:29-30,
    broadphase.py:104-107, scene.py:35-45)."""
    if status == GG_OK:
        return
    msg = last_error(ctx) or where
    if status == GG_ENONFINITE:
        raise SolverError(msg)
    if status in (GG_EINVAL, GG_EPOSITIONS):
        raise ValueError(msg)
    if status == GG_ECAPACITY:
        raise CapacityError(msg)
    raise RuntimeError(f"granusim_b200 CUDA failure in {where}: {msg}")


class CapacityError(RuntimeError):
    """Per-owner contact slots exhausted (handled by the engine: grow + retry)."""


def cuda_device_count() -> int:
    try:
        cudart = C.CDLL("libcudart.so")
    except OSError:
        import torch

        return torch.cuda.device_count()
    n = C.c_int(0)
    cudart.cudaGetDeviceCount(C.byref(n))
    return n.value
