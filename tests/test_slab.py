"""Slab domain decomposition of one bed.

CPU: partition rules (cell rounding vs the oracle, balanced cuts, ownership),
and the neighbour transport over gloo with world_size 2 and 3.
GPU: the slab step on 1, 2 and 3 ranks (ranks share the one GPU, gloo
transport staged through host memory) is bitwise identical to the one-GPU
step: same positions and velocities per particle id, same counters.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_2306_01369_b200 as gg
from paper_2306_01369_b200.slab import (
    REC_FLOATS,
    SlabTransport,
    cell_x,
    owner_of,
    slab_bounds,
    slab_cuts,
)
from oracle import granular_oracle as O


def _port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port, backend="gloo"):
    import torch.distributed as td

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group(backend, rank=rank, world_size=world)
    return td


# ---------------------------------------------------------------------------
# CPU
# ---------------------------------------------------------------------------
def test_cell_x_matches_oracle_rounding():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.uniform(-3, 3, 20000), (np.arange(-40, 41) + 0.5) * 0.1])
    x = x.astype(np.float32).astype(np.float64)
    pts = np.stack([x, np.zeros_like(x), np.zeros_like(x)], 1)
    assert np.array_equal(cell_x(x, 0.05), O.cell_coords(pts, 0.05)[:, 0])


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_slab_cuts_balanced_and_consistent(world):
    x = gg.lattice_bed(40000)[:, 0]
    cx = cell_x(x, 0.05)
    cuts = slab_cuts(cx, world)
    own = owner_of(cx, cuts)
    counts = np.bincount(own, minlength=world)
    assert counts.sum() == len(x) and len(counts) == world
    assert counts.max() <= 1.35 * counts.mean() + 1
    for r in range(world):
        lo, hi, has_lo, has_hi = slab_bounds(cuts, r)
        mine = cx[own == r]
        if has_lo:
            assert mine.min() >= lo
        if has_hi:
            assert mine.max() < hi
        if has_lo and has_hi:
            assert hi - lo >= 2


def test_slab_cuts_rejects_narrow_bed():
    with pytest.raises(ValueError):
        slab_cuts(np.array([0, 1, 2]), 4)


def _transport_worker(rank, world, port, out):
    td = _init(rank, world, port)
    tr = SlabTransport(rank, world, device=0, stream_ptr=None, backend="gloo")
    import torch

    # rank r sends r+1 records to lo and r+2 to hi, each record = its rank
    n_lo, n_hi = (rank + 1 if tr.lo is not None else 0), (rank + 2 if tr.hi is not None else 0)
    s_lo = torch.full((8, REC_FLOATS), float(rank))
    s_hi = torch.full((8, REC_FLOATS), float(rank) + 0.5)
    m_lo, m_hi = tr.counts(n_lo, n_hi)
    r_lo = torch.zeros((8, REC_FLOATS))
    r_hi = torch.zeros((8, REC_FLOATS))
    tr.exchange(s_lo, n_lo, s_hi, n_hi, r_lo, m_lo, r_hi, m_hi)
    red = tr.allreduce(np.array([rank, 1.0]), "sum")
    packed = tr.reduce_packed([rank, 1.0], [float(rank)], [float(rank) + 3.0])
    rows = tr.gather_rows(np.full((rank, 7), float(rank)))  # ragged: rank 0 sends none
    out[rank] = (m_lo, m_hi, r_lo[:m_lo].numpy().copy(), r_hi[:m_hi].numpy().copy(), red, packed, rows)
    td.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_transport_gloo_neighbour_exchange(world):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    mp.spawn(_transport_worker, args=(world, _port(), out), nprocs=world, join=True)
    for r in range(world):
        m_lo, m_hi, r_lo, r_hi, red, packed, rows = out[r]
        want = np.concatenate([np.full((q, 7), float(q)) for q in range(world)])
        assert rows.shape == want.shape and np.array_equal(rows, want)  # rank order, every rank
        if r > 0:  # from my lo neighbour: what it sent to ITS hi
            assert m_lo == (r - 1) + 2 and np.all(r_lo == (r - 1) + 0.5)
        else:
            assert m_lo == 0
        if r < world - 1:  # from my hi neighbour: what it sent to ITS lo
            assert m_hi == (r + 1) + 1 and np.all(r_hi == r + 1)
        else:
            assert m_hi == 0
        assert red[0] == sum(range(world)) and red[1] == world
        s_, mx, mn = packed  # one all_gather: sums, maxes, mins
        assert list(s_) == [sum(range(world)), world] and mx[0] == world - 1 and mn[0] == 3.0


# ---------------------------------------------------------------------------
# GPU
# ---------------------------------------------------------------------------
def _bed(n=12000, seed=3):
    """A compressed lattice bed with random lateral velocities (particles cross
    slab boundaries) and a spinning box tool."""
    x = gg.lattice_bed(n, seed=seed).astype(np.float32).astype(np.float64)
    rng = np.random.default_rng(seed)
    v = rng.normal(scale=1.5, size=x.shape)
    v[:, 0] += 10.0  # the bed drifts 8 cm along x: particles cross the slab cuts
    v = v.astype(np.float32).astype(np.float64)
    params = gg.MaterialParams(timestep=5e-4)
    cx, cy = float(np.median(x[:, 0])), float(np.median(x[:, 1]))
    top = float(x[:, 2].max())
    tool = gg.RigidBody(gg.Box(np.array([0.3, 0.15, 0.1])),
                        gg.SpinDriver(axis=[0, 0, 1], rate=3.0, center=[cx, cy, top],
                                      base_pose=gg.make_pose(np.eye(3), [cx, cy, top - 0.05])),
                        name="tool")
    return gg.Scene(particles=gg.ParticleSet(x, v), bodies=[gg.RigidBody(gg.HalfSpace(), name="floor"),
                                                             tool], params=params)


T_STEPS = 16


GAP_CUT = 4  # the explicit slab cut of the gap bed (cell index along x)


def _gap_bed():
    """A bed whose cell column GAP_CUT - 1 (rank 0's boundary cell) is empty
    while column GAP_CUT (rank 1's) is full: rank 0 sends no ghosts to rank 1,
    rank 1 sends ghosts to rank 0 — the asymmetric halo of a sparse bed."""
    x = gg.lattice_bed(12000, seed=5).astype(np.float32).astype(np.float64)
    x[:, 0] -= x[:, 0].min() - 0.01
    cx = cell_x(x[:, 0], 0.05)
    keep = cx != GAP_CUT - 1
    x = x[keep]
    rng = np.random.default_rng(5)
    v = rng.normal(scale=0.2, size=x.shape).astype(np.float32).astype(np.float64)
    params = gg.MaterialParams(timestep=5e-4)
    return gg.Scene(particles=gg.ParticleSet(x, v), bodies=[gg.RigidBody(gg.HalfSpace(), name="floor")],
                    params=params)


def _reference_run(make=None):
    sc = (make or _bed)()
    reps = [gg.step(sc)[1] for _ in range(T_STEPS)]
    return sc.particles.positions.copy(), sc.particles.velocities.copy(), reps


def _slab_worker(rank, world, port, out, halo="host", gap=False, reload=False):
    from paper_2306_01369_b200.slab import SlabBed

    td = _init(rank, world, port) if world > 1 else None
    scene = _gap_bed() if gap else _bed()
    cuts = np.array([GAP_CUT]) if gap else None
    x0, v0 = scene.particles.positions.copy(), scene.particles.velocities.copy()
    bed = SlabBed(scene, rank=rank, world=world, device=0, backend="gloo", resort_every=5, halo=halo,
                  cuts=cuts)
    if reload:  # a few steps of a scrambled state, then the real one through SlabBed.load
        rng = np.random.default_rng(rank)
        bed.load(x0 + rng.normal(scale=1e-3, size=x0.shape), -v0)
        bed.run(3)
        scene.t = 0.0
        bed.load(x0, v0)
    reps = bed.run(T_STEPS)
    X, V = bed.gather()
    out[f"ghosts{rank}"] = bed.ghosts
    if rank == 0:
        out["x"], out["v"] = X, V
        out["reps"] = [(r.n_contacts, r.n_body_contacts, r.max_penetration, r.kinetic_energy,
                        r.max_cone_violation, r.n_coincident_skipped, r.n_degenerate_skipped,
                        r.min_normal_impulse) for r in reps]
    out[f"moved{rank}"] = bed.migrated
    bed.close()
    if td:
        td.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,halo", [(1, "host"), (2, "host"), (3, "host"), (2, "p2p"), (3, "p2p")])
def test_slab_step_bitwise_equals_one_gpu(world, halo):
    """halo="p2p": the per-sweep halo goes through CUDA-IPC peer memory
    (here several processes share one GPU; across GPUs it is NVLink)."""
    x1, v1, reps1 = _reference_run()
    if world == 1:
        out = {}
        _slab_worker(0, 1, 0, out)
    else:
        ctx = mp.get_context("spawn")
        out = ctx.Manager().dict()
        mp.spawn(_slab_worker, args=(world, _port(), out, halo), nprocs=world, join=True)
    assert np.array_equal(out["x"], x1)
    assert np.array_equal(out["v"], v1)
    _check_reports(out["reps"], reps1)
    if world > 1:
        assert sum(out[f"moved{r}"] for r in range(world)) > 0, "no particle migrated"


@pytest.mark.gpu
@pytest.mark.parametrize("world,halo", [(1, "auto"), (2, "p2p")])
def test_slab_load_replaces_the_state(world, halo):
    """SlabBed.load into a bed that has already stepped (graphs built,
    device counts and exchange sequence numbers advanced) continues exactly
    like a fresh bed on that state."""
    x1, v1, reps1 = _reference_run()
    if world == 1:
        out = {}
        _slab_worker(0, 1, 0, out, halo, False, True)
    else:
        ctx = mp.get_context("spawn")
        out = ctx.Manager().dict()
        mp.spawn(_slab_worker, args=(world, _port(), out, halo, False, True), nprocs=world, join=True)
    assert np.array_equal(out["x"], x1)
    assert np.array_equal(out["v"], v1)
    _check_reports(out["reps"], reps1)


def _check_reports(slab_reps, reps1):
    # every counter but n_candidates is the one-GPU value (candidates differ
    # under hash aliasing: a rank does not hash the other slabs' particles)
    for (n_pp, n_b, mp_, ke, mv, nco, ndg, mnb), r in zip(slab_reps, reps1):
        assert n_pp == r.n_contacts and n_b == r.n_body_contacts
        assert nco == r.n_coincident_skipped and ndg == r.n_degenerate_skipped
        assert mp_ == r.max_penetration and mv == r.max_cone_violation
        assert mnb == r.min_normal_impulse
        assert ke == pytest.approx(r.kinetic_energy, rel=1e-9)


@pytest.mark.gpu
def test_slab_p2p_asymmetric_halo():
    """Peer-memory halo when one side of a cut sends no ghosts:
    the receiver still waits on the neighbour's per-sweep flag, so neither
    rank runs a sweep ahead of the other's parity buffer."""
    x1, v1, reps1 = _reference_run(_gap_bed)
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    mp.spawn(_slab_worker, args=(2, _port(), out, "p2p", True), nprocs=2, join=True)
    assert out["ghosts0"][1] > 0 and out["ghosts1"][0] == 0, (out["ghosts0"], out["ghosts1"])
    assert np.array_equal(out["x"], x1)
    assert np.array_equal(out["v"], v1)
    _check_reports(out["reps"], reps1)
