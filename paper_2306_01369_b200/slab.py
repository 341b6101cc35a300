"""One bed over several GPUs: slab domain decomposition.

The reference runs a scene on one CPU core and has no multi-GPU path
(PAPER.md:524-526); the contract is "same answer as one GPU".  ``SlabBed``
cuts the bed along x at cell boundaries (cell = round(x / 2r),
broadphase.py:33-41) into one slab per rank (one process per GPU).  Each
step a rank
  1. migrates particles whose cell left its slab to the neighbour,
  2. receives the neighbours' boundary-cell particles as ghosts,
  3. runs the step kernels on owned + ghost particles (ghosts are candidates
     only), exchanging the ghosts' predicted velocity after every Jacobi sweep,
  4. reduces the StepReport over ranks.
Ghosts carry their global id, which the device uses as the stable-sort tie
key, so every owned particle sees the same contacts in the same order as on
one GPU: states and every StepReport field except ``n_candidates`` are
bitwise identical to the one-GPU run (tests/test_slab.py).
``n_candidates`` (and so ``candidate_hit_rate``) is NOT the one-GPU value
when the hash aliases: a rank hashes only its owned and ghost particles, so
far-away particles of other slabs that share a bucket with a neighbour cell
are missing from its candidate counts.  Aliases are never contacts (a
contact is within 2r, i.e. within +-1 cell), so nothing else changes.

Two transports.  ``halo="p2p"`` (the default under NCCL): every rank exports a
mailbox through CUDA IPC and opens its neighbours'; migrants and ghosts are
packed by kernels straight into the neighbours' mailboxes, counts and
system-scope release flags are published on the device, the receiver waits
on the device and appends, and the S sweeps run with their per-sweep w halo
pushed into the same mailboxes; the particle counts stay on the device and
the whole step is replayed as one CUDA graph (gg_slab_step_p2p) — no NCCL
call on the step path, one host synchronisation per step (the rank's
StepReport) plus the report reduction.  ``halo="host"``: the library
packs and unpacks device buffers (gg_slab_* pack/unpack) and this module
moves them with torch.distributed point-to-point operations — NCCL on device
buffers, or gloo staged through host memory (tests on CPU).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _native as N
from .engine import _params_struct, default_table_size
from .stepper import StepReport

REC_FLOATS = 8    # particle record: (x, y, z, bits(gid)), (vx, vy, vz, 0)
HALO_FLOATS = 4   # halo record: w (float4)


def cell_x(x: np.ndarray, radius: float) -> np.ndarray:
    """round_half_away(x / 2r) along x (broadphase.py:33-41), float64."""
    q = np.asarray(x, dtype=np.float64) / (2.0 * radius)
    return (np.copysign(np.floor(np.abs(q) + 0.5), q)).astype(np.int64)


def slab_cuts(cx: np.ndarray, world: int) -> np.ndarray:
    """Cell cuts c_1 < ... < c_{world-1} splitting the particles into slabs of
    about equal count (rank r owns cells [c_r, c_{r+1}), c_0 = -inf,
    c_world = +inf).  Each slab keeps at least two cells so a particle never
    crosses more than one boundary in a step."""
    if world < 1:
        raise ValueError("world must be >= 1")
    if world == 1:
        return np.zeros(0, dtype=np.int64)
    cs = np.sort(np.asarray(cx, dtype=np.int64))
    lo, hi = int(cs[0]), int(cs[-1]) + 1
    if hi - lo < 2 * world:
        raise ValueError(f"bed is {hi - lo} cells wide: too narrow for {world} slabs")
    cuts = []
    prev = lo
    for r in range(1, world):
        c = int(cs[min(len(cs) - 1, (r * len(cs)) // world)])
        c = max(c, prev + 2)
        c = min(c, hi - 2 * (world - r))
        cuts.append(c)
        prev = c
    return np.array(cuts, dtype=np.int64)


def slab_bounds(cuts: np.ndarray, rank: int):
    """(lo, hi, has_lo, has_hi) of rank's slab."""
    world = len(cuts) + 1
    has_lo = rank > 0
    has_hi = rank < world - 1
    lo = int(cuts[rank - 1]) if has_lo else 0
    hi = int(cuts[rank]) if has_hi else 0
    return lo, hi, has_lo, has_hi


def owner_of(cx: np.ndarray, cuts: np.ndarray) -> np.ndarray:
    """Rank owning each cell index."""
    return np.searchsorted(cuts, cx, side="right")


# ---------------------------------------------------------------------------
class SlabTransport:
    """Neighbour exchange of slab buffers with torch.distributed P2P ops.

    backend "nccl": the buffers are device tensors and the operations are
    ordered on the context stream (torch ExternalStream); "gloo": buffers are
    staged through host memory.  world == 1 needs no process group."""

    def __init__(self, rank: int, world: int, device: int, stream_ptr: int | None,
                 backend: str | None = None):
        self.rank, self.world, self.device = rank, world, device
        self.lo = rank - 1 if rank > 0 else None
        self.hi = rank + 1 if rank < world - 1 else None
        import torch

        self.torch = torch
        self.dist = None
        if world > 1:
            import torch.distributed as td

            if not td.is_initialized():
                raise RuntimeError("SlabTransport: torch.distributed is not initialised")
            self.dist = td
            backend = backend or td.get_backend()
        self.backend = backend or "gloo"
        self.on_device = self.backend == "nccl"
        self.dev = torch.device("cuda", device) if torch.cuda.is_available() else torch.device("cpu")
        self.stream = (torch.cuda.ExternalStream(stream_ptr, device=self.dev)
                       if (stream_ptr and torch.cuda.is_available()) else None)

    def empty(self, n: int, width: int):
        """A device buffer of n records (float32 x width)."""
        return self.torch.empty((max(n, 1), width), dtype=self.torch.float32, device=self.dev)

    def _ctx(self):
        import contextlib

        return self.torch.cuda.stream(self.stream) if self.stream is not None else contextlib.nullcontext()

    def _p2p(self, sends, recvs):
        """sends/recvs: lists of (peer, tensor); all posted together."""
        td = self.dist
        ops = [td.P2POp(td.isend, t, p) for p, t in sends] + [td.P2POp(td.irecv, t, p) for p, t in recvs]
        if not ops:
            return
        for r in td.batch_isend_irecv(ops):
            r.wait()

    def counts(self, c_lo: int, c_hi: int) -> tuple[int, int]:
        """Send my counts to (lo, hi); return the counts they send me."""
        if self.world == 1:
            return 0, 0
        torch = self.torch
        dev = self.dev if self.on_device else torch.device("cpu")
        out_lo = torch.tensor([c_lo], dtype=torch.int64, device=dev)
        out_hi = torch.tensor([c_hi], dtype=torch.int64, device=dev)
        in_lo = torch.zeros(1, dtype=torch.int64, device=dev)
        in_hi = torch.zeros(1, dtype=torch.int64, device=dev)
        sends, recvs = [], []
        if self.lo is not None:
            sends.append((self.lo, out_lo))
            recvs.append((self.lo, in_lo))
        if self.hi is not None:
            sends.append((self.hi, out_hi))
            recvs.append((self.hi, in_hi))
        with self._ctx():
            self._p2p(sends, recvs)
        return int(in_lo.item()), int(in_hi.item())

    def exchange(self, send_lo, n_lo: int, send_hi, n_hi: int, recv_lo, m_lo: int, recv_hi, m_hi: int):
        """Send send_*[:n_*] to the neighbours and receive m_* records into recv_*."""
        if self.world == 1:
            return
        torch = self.torch
        with self._ctx():
            sends, recvs, back = [], [], []
            for peer, buf, n in ((self.lo, send_lo, n_lo), (self.hi, send_hi, n_hi)):
                if peer is None or n == 0:
                    continue
                t = buf[:n]
                sends.append((peer, t if self.on_device else t.cpu()))
            for peer, buf, m in ((self.lo, recv_lo, m_lo), (self.hi, recv_hi, m_hi)):
                if peer is None or m == 0:
                    continue
                if self.on_device:
                    recvs.append((peer, buf[:m]))
                else:
                    h = torch.empty((m, buf.shape[1]), dtype=buf.dtype)
                    recvs.append((peer, h))
                    back.append((buf, h, m))
            self._p2p(sends, recvs)
            for buf, h, m in back:
                buf[:m].copy_(h)

    def reduce_packed(self, sums: np.ndarray, maxes: np.ndarray, mins: np.ndarray):
        """The StepReport reduction in ONE collective: every rank's packed
        [sums | maxes | mins] float64 vector is all-gathered and reduced in
        rank order (deterministic), instead of one all-reduce per operator."""
        packed = np.concatenate([np.asarray(sums, np.float64).ravel(), np.asarray(maxes, np.float64).ravel(),
                                 np.asarray(mins, np.float64).ravel()])
        if self.world == 1:
            rows = packed[None, :]
        else:
            torch = self.torch
            dev = self.dev if self.on_device else torch.device("cpu")
            t = torch.from_numpy(packed).to(dev)
            out = [torch.empty(len(packed), dtype=torch.float64, device=dev) for _ in range(self.world)]
            with self._ctx():
                self.dist.all_gather(out, t)
            rows = torch.stack(out).cpu().numpy()
        a, b = len(np.ravel(sums)), len(np.ravel(maxes))
        return rows[:, :a].sum(axis=0), rows[:, a:a + b].max(axis=0), rows[:, a + b:].min(axis=0)

    def gather_rows(self, rows: np.ndarray) -> np.ndarray:
        """Every rank's (n_r, w) float64 rows, concatenated in rank order, on
        every rank: ONE all-gather of buffers padded to the longest (device
        buffers under NCCL), instead of pickled objects."""
        rows = np.ascontiguousarray(rows, dtype=np.float64)
        if self.world == 1:
            return rows
        torch = self.torch
        n = rows.shape[0]
        counts = self.allreduce_list(n)
        nmax = max(max(counts), 1)
        dev = self.dev if self.on_device else torch.device("cpu")
        pad = np.zeros((nmax, rows.shape[1]))
        pad[:n] = rows
        t = torch.from_numpy(pad).to(dev)
        out = [torch.empty_like(t) for _ in range(self.world)]
        with self._ctx():
            self.dist.all_gather(out, t)
        got = torch.stack(out).cpu().numpy()
        return np.concatenate([got[r, :counts[r]] for r in range(self.world)])

    def allreduce_list(self, n: int) -> list[int]:
        """every rank's integer n, in rank order"""
        if self.world == 1:
            return [int(n)]
        torch = self.torch
        dev = self.dev if self.on_device else torch.device("cpu")
        t = torch.tensor([float(n)], dtype=torch.float64, device=dev)
        out = [torch.empty_like(t) for _ in range(self.world)]
        with self._ctx():
            self.dist.all_gather(out, t)
        return [int(o.item()) for o in out]

    def allreduce(self, vals: np.ndarray, op: str) -> np.ndarray:
        if self.world == 1:
            return vals
        torch = self.torch
        dev = self.dev if self.on_device else torch.device("cpu")
        t = torch.tensor(np.asarray(vals, dtype=np.float64), device=dev)
        rop = {"sum": self.dist.ReduceOp.SUM, "max": self.dist.ReduceOp.MAX,
               "min": self.dist.ReduceOp.MIN}[op]
        self.dist.all_reduce(t, op=rop)
        return t.cpu().numpy()


# ---------------------------------------------------------------------------
class SlabBed:
    """Rank ``rank``'s slab of ``scene`` (every rank passes the same scene)."""

    def __init__(self, scene, rank: int = 0, world: int = 1, device: int = 0,
                 backend: str | None = None, cuts: np.ndarray | None = None,
                 capacity: float = 1.6, max_contacts: int = 16, resort_every: int = 32,
                 halo: str = "auto"):
        from .engine import Engine

        self.scene = scene
        self.rank, self.world = rank, world
        self.params = scene.params
        r = float(self.params.radius)
        x = np.asarray(scene.particles.positions, dtype=np.float64)
        v = np.asarray(scene.particles.velocities, dtype=np.float64)
        self.N = len(x)
        self.n_h = int(scene.hashmap_size or default_table_size(self.N))  # GLOBAL table
        cx = cell_x(x.astype(np.float32).astype(np.float64)[:, 0], r) if world > 1 else None
        self.cuts = slab_cuts(cx, world) if cuts is None else np.asarray(cuts, dtype=np.int64)
        lo, hi, has_lo, has_hi = slab_bounds(self.cuts, rank)
        mine = self._mine(cx)
        self.nb = len(scene.bodies)
        # (alone, a rank neither receives migrants nor ghosts)
        n_mine = self.N if mine is None else len(mine)
        self.cap = int(math.ceil((capacity if world > 1 else 1.0) * max(n_mine, 1) + 4096))
        self.resort_every = resort_every
        self.steps = 0
        self.migrated = 0  # particles this rank sent to its neighbours
        # context: capacity = owned + ghosts + immigrants
        self.engine = Engine(device)
        self.engine.max_contacts = max_contacts
        self.engine._create(self.params, scene.boundary, self.cap, self.n_h, max(self.nb, 1))
        self.ctx = self.engine.ctx
        lib = N.lib()
        N.check(self.ctx, lib.gg_slab_setup(self.ctx, lo, hi, int(has_lo), int(has_hi)), "slab setup")
        self._upload(x, v, mine)
        self.tr = SlabTransport(rank, world, device, lib.gg_stream(self.ctx), backend)
        self.buf_cap = max(4096, self.cap // 2)
        self._alloc()
        if halo not in ("auto", "host", "p2p"):
            raise ValueError("halo must be 'auto', 'host' or 'p2p'")
        if halo == "auto":  # peer memory whenever the ranks run NCCL on one node's GPUs (or alone)
            halo = "p2p" if (self.tr.backend == "nccl" or world == 1) else "host"
        self.halo = halo
        if self.halo == "p2p":
            self._connect_mailboxes()

    def _mine(self, cx: np.ndarray):
        """global ids of the particles this rank owns (all of them when alone)"""
        if self.world == 1:
            return None
        return np.nonzero(owner_of(cx, self.cuts) == self.rank)[0]

    def _upload(self, x: np.ndarray, v: np.ndarray, mine) -> None:
        if mine is None:  # alone: the whole bed, in id order
            gid = np.arange(len(x), dtype=np.int32)
            xs, vs = np.ascontiguousarray(x, np.float64), np.ascontiguousarray(v, np.float64)
        else:
            gid = mine.astype(np.int32)
            xs = np.ascontiguousarray(x[mine])
            vs = np.ascontiguousarray(v[mine])
        if len(gid) > self.cap:
            raise ValueError(f"rank {self.rank} would own {len(gid)} particles; capacity {self.cap}")
        N.check(self.ctx, N.lib().gg_slab_load(self.ctx, N.ptr(xs), N.ptr(vs), N.ptr(gid), len(gid)),
                "slab load")

    def load(self, positions: np.ndarray, velocities: np.ndarray) -> None:
        """Replace the bed's state with a host state of the same particles
        (global ids = row indices), partitioned with this bed's slab cuts:
        every rank calls it with the same arrays.  The context, its graphs
        and the transport are kept."""
        x = np.asarray(positions, dtype=np.float64)
        v = np.asarray(velocities, dtype=np.float64)
        if x.shape != (self.N, 3) or v.shape != (self.N, 3):
            raise ValueError(f"expected ({self.N}, 3) positions and velocities")
        cx = None if self.world == 1 else cell_x(x.astype(np.float32).astype(np.float64)[:, 0],
                                                 float(self.params.radius))
        self._upload(x, v, self._mine(cx) if cx is not None else None)

    def _connect_mailboxes(self) -> None:
        """Per-sweep halo through peer memory: export this rank's mailbox
        (CUDA IPC), open the neighbours' (gg_slab_connect)."""
        import torch.distributed as td

        lib = N.lib()
        # one mailbox size on every rank: a sender addresses the receiver's
        # mailbox with its own copy of the capacity
        cap = int(self.tr.allreduce(np.array([float(self.buf_cap)]), "max")[0])
        h = np.zeros(64, dtype=np.uint8)
        N.check(self.ctx, lib.gg_slab_mailbox(self.ctx, cap, N.ptr(h)), "mailbox")
        if self.world == 1:  # no neighbours: the mailbox only backs the graph-replayed step
            return
        handles = [None] * self.world
        td.all_gather_object(handles, h.tobytes())
        for side, peer in ((0, self.rank - 1), (1, self.rank + 1)):
            if 0 <= peer < self.world:
                hp = np.frombuffer(handles[peer], dtype=np.uint8).copy()
                N.check(self.ctx, lib.gg_slab_connect(self.ctx, side, N.ptr(hp)), "connect")
        td.barrier()

    def _alloc(self):
        e = self.tr.empty
        c = self.buf_cap
        self.s_lo, self.s_hi = e(c, REC_FLOATS), e(c, REC_FLOATS)
        self.r_lo, self.r_hi = e(c, REC_FLOATS), e(c, REC_FLOATS)
        self.h_slo, self.h_shi = e(c, HALO_FLOATS), e(c, HALO_FLOATS)
        self.h_rlo, self.h_rhi = e(c, HALO_FLOATS), e(c, HALO_FLOATS)

    @staticmethod
    def _p(t) -> int:
        return t.data_ptr()

    def close(self):
        self.engine.close()

    @property
    def n_owned(self) -> int:
        return int(N.lib().gg_slab_owned(self.ctx))

    # -- one step ------------------------------------------------------------
    def _swap(self, pack, unpack, send, recv):
        """pack -> exchange counts and records -> unpack; returns
        ((sent lo, sent hi), (received lo, received hi))."""
        cnt = np.zeros(2, dtype=np.int64)
        N.check(self.ctx, pack(self.ctx, self._p(send[0]), self._p(send[1]), self.buf_cap, N.ptr(cnt)),
                "slab pack")
        m_lo, m_hi = self.tr.counts(int(cnt[0]), int(cnt[1]))
        if max(m_lo, m_hi) > self.buf_cap:
            raise RuntimeError("slab receive buffer too small")
        self.tr.exchange(send[0], int(cnt[0]), send[1], int(cnt[1]), recv[0], m_lo, recv[1], m_hi)
        N.check(self.ctx, unpack(self.ctx, self._p(recv[0]), m_lo, self._p(recv[1]), m_hi), "slab unpack")
        return (int(cnt[0]), int(cnt[1])), (m_lo, m_hi)

    def step(self) -> StepReport:
        lib = N.lib()
        sc = self.scene
        # body poses at t + dt (stepper.py:65-67), identical on every rank
        t = sc.t + sc.params.timestep
        row = np.zeros(max(self.nb, 1), dtype=N.BODY_DTYPE)
        for b, body in enumerate(sc.bodies):
            body.update(t)
            self.engine.body_row(body, float(sc.params.radius), row[b])
        sc.t = t
        resort = self.steps % self.resort_every == 0
        S = int(self.params.solver_iterations)
        if self.halo == "p2p":
            # the whole step — (re-sort,) migration and ghosts through the
            # neighbours' mailboxes, contacts, sweeps with their peer-memory
            # halos, integration, commit — as one CUDA graph replay; one
            # synchronisation, for the rank's report
            info = np.zeros(6, dtype=np.int64)
            rep = np.zeros(1, dtype=N.REPORT_DTYPE)
            bm = np.zeros((max(self.nb, 1), 3))
            st = lib.gg_slab_step_p2p(self.ctx, N.ptr(row), self.nb, int(resort), N.ptr(rep), N.ptr(bm),
                                      N.ptr(info))
            if st != N.GG_OK:
                from .engine import raise_status

                raise_status(st, N.last_error(self.ctx), self.steps)
            self.migrated += int(info[0] + info[1])
            self.ghosts = (int(info[4]), int(info[5]))
            self.steps += 1
            return self._reduce(rep[0], bm[: self.nb])
        # 1. migration, 2. (re-sort) + ghosts
        sent, _ = self._swap(lib.gg_slab_migrate_pack, lib.gg_slab_migrate_unpack,
                             (self.s_lo, self.s_hi), (self.r_lo, self.r_hi))
        self.migrated += sent[0] + sent[1]
        if resort:
            N.check(self.ctx, lib.gg_slab_resort(self.ctx), "slab resort")
        n_out, (g_lo, g_hi) = self._swap(lib.gg_slab_ghost_pack, lib.gg_slab_ghost_unpack,
                                         (self.s_lo, self.s_hi), (self.r_lo, self.r_hi))
        self.ghosts = (g_lo, g_hi)
        # 3. step with per-sweep halo exchange of w
        N.check(self.ctx, lib.gg_slab_detect(self.ctx, N.ptr(row), self.nb), "slab detect")
        for s in range(S):
            N.check(self.ctx, lib.gg_slab_sweep(self.ctx, s), "slab sweep")
            if s < S - 1 and self.world > 1:
                N.check(self.ctx, lib.gg_slab_halo_pack(self.ctx, s, self._p(self.h_slo),
                                                        self._p(self.h_shi)), "halo pack")
                self.tr.exchange(self.h_slo, n_out[0], self.h_shi, n_out[1], self.h_rlo, g_lo,
                                 self.h_rhi, g_hi)
                N.check(self.ctx, lib.gg_slab_halo_unpack(self.ctx, s, self._p(self.h_rlo),
                                                          self._p(self.h_rhi)), "halo unpack")
        return self._finish(lib)

    def _finish(self, lib) -> StepReport:
        rep = np.zeros(1, dtype=N.REPORT_DTYPE)
        bm = np.zeros((max(self.nb, 1), 3))
        st = lib.gg_slab_finish(self.ctx, N.ptr(rep), N.ptr(bm))
        if st != N.GG_OK:
            from .engine import raise_status

            raise_status(st, N.last_error(self.ctx), self.steps)
        self.steps += 1
        return self._reduce(rep[0], bm[: self.nb])

    def _reduce(self, r, bm) -> StepReport:
        rr = np.zeros(1, dtype=N.REPORT_DTYPE)
        rr[0] = r
        return self._reduce_many(rr, np.asarray(bm, np.float64)[None])[0]

    def _reduce_many(self, reps, bms) -> list[StepReport]:
        """StepReports of len(reps) consecutive steps ending at self.steps - 1,
        reduced over the ranks in ONE collective (per-step sums, maxes and
        mins side by side)."""
        K = len(reps)
        nb = self.nb
        cnt = np.stack([reps["n_contacts"], reps["n_candidates"], reps["n_body_contacts"],
                        reps["n_coincident"], reps["n_degenerate"]], axis=1).astype(np.float64)
        sums = np.concatenate([cnt, np.asarray(reps["kinetic_energy"], np.float64)[:, None],
                               np.asarray(bms, np.float64)[:, :nb].reshape(K, 3 * nb)], axis=1)
        maxes = np.stack([reps["max_penetration"], reps["max_cone_violation"]], axis=1)
        mins = np.asarray(reps["min_normal_impulse"], np.float64)[:, None]
        s, mx, mn = self.tr.reduce_packed(sums, maxes, mins)
        s, mx, mn = s.reshape(K, -1), mx.reshape(K, 2), mn.reshape(K, 1)
        out = []
        for i in range(K):
            n_pp, n_cand = int(s[i, 0]), int(s[i, 1])
            m = float(mn[i, 0])
            out.append(StepReport(n_contacts=n_pp, n_candidates=n_cand,
                                  candidate_hit_rate=n_pp / max(n_cand, 1),
                                  max_penetration=float(mx[i, 0]), kinetic_energy=float(s[i, 5]),
                                  n_body_contacts=int(s[i, 2]), n_coincident_skipped=int(s[i, 3]),
                                  n_degenerate_skipped=int(s[i, 4]), max_cone_violation=float(mx[i, 1]),
                                  min_normal_impulse=m if np.isfinite(m) else 0.0,
                                  body_momentum=s[i, 6:].reshape(-1, 3),
                                  step_index=self.steps - K + i))
        return out

    def run(self, n_steps: int) -> list[StepReport]:
        """``step`` n_steps times.  On the peer-memory transport the steps are
        replayed back to back on the device (bodies of every step staged up
        front, one synchronisation and one report collective for the batch);
        the results are those of n_steps ``step`` calls, bit for bit."""
        if n_steps < 0:
            raise ValueError("n_steps must be >= 0")
        if self.halo != "p2p" or n_steps < 2:
            return [self.step() for _ in range(n_steps)]
        lib = N.lib()
        sc = self.scene
        K, nbx = n_steps, max(self.nb, 1)
        rows = np.zeros((K, nbx), dtype=N.BODY_DTYPE)
        for i in range(K):  # body poses at t + dt of every step (stepper.py:65-67)
            t = sc.t + sc.params.timestep
            for b, body in enumerate(sc.bodies):
                body.update(t)
                self.engine.body_row(body, float(sc.params.radius), rows[i, b])
            sc.t = t
        resort = np.array([(self.steps + i) % self.resort_every == 0 for i in range(K)], dtype=np.int32)
        info = np.zeros(7, dtype=np.int64)
        reps = np.zeros(K, dtype=N.REPORT_DTYPE)
        bm = np.zeros((K, nbx, 3))
        st = lib.gg_slab_run_p2p(self.ctx, N.ptr(rows), self.nb, K, N.ptr(resort), N.ptr(reps), N.ptr(bm),
                                 N.ptr(info))
        if st != N.GG_OK:
            from .engine import raise_status

            raise_status(st, N.last_error(self.ctx), self.steps)
        self.migrated += int(info[6])
        self.ghosts = (int(info[4]), int(info[5]))
        self.steps += K
        return self._reduce_many(reps, bm)

    # -- state -----------------------------------------------------------------
    def owned_state(self):
        """(x, v, gid) of this rank's particles (physical order)."""
        lib = N.lib()
        n = self.n_owned
        x = np.zeros((max(n, 1), 3))
        v = np.zeros((max(n, 1), 3))
        gid = np.zeros(max(n, 1), dtype=np.int32)
        got = ctypes.c_int64(0)
        N.check(self.ctx, lib.gg_slab_get(self.ctx, N.ptr(x), N.ptr(v), N.ptr(gid), len(gid),
                                          ctypes.byref(got)), "slab get")
        n = got.value
        return x[:n], v[:n], gid[:n]

    def gather(self):
        """Global (x, v) in particle-id order, assembled on every rank."""
        x, v, gid = self.owned_state()
        if self.world == 1:
            X = np.zeros((self.N, 3))
            V = np.zeros((self.N, 3))
            X[gid], V[gid] = x, v
            return X, V
        rows = self.tr.gather_rows(np.concatenate([x, v, gid[:, None].astype(np.float64)], axis=1))
        g = rows[:, 6].astype(np.int64)
        X = np.zeros((self.N, 3))
        V = np.zeros((self.N, 3))
        X[g], V[g] = rows[:, :3], rows[:, 3:6]
        return X, V
