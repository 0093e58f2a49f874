"""X-slab decomposition of one giant scene (config 5) across ranks, with a
halo exchange over NCCL (BASELINE.json configs[4]).

Every rank holds the WHOLE scene in the library's body-major layout (67M
particles are ~4 GB of state; a B200 has 180 GB) and simulates only the bodies
it owns, i.e. the bodies whose centre of mass lies in its x-slab. Bodies of the
neighbouring slabs that could touch an owned body this frame are *ghosts*: they
are integrated and hashed locally, so owned particles find them in the grid,
and their positions are refreshed from their owner after every iteration.
Because the layout (slot numbering) is the single-GPU layout, an owned
particle's contact-candidate list is the single-GPU list in the same ascending
order, and every owned body's trajectory is bit-identical to the 1-GPU run --
the halo makes the decomposition exact, not approximate.

Per frame (host-synchronised once):
  repartition -- owners measure com_x of their bodies, a body whose com left
                 the slab migrates to the neighbour (its warm-start rotation and
                 anchor travel; positions and velocities are already there,
                 because it was a ghost), then every owner sends each neighbour
                 the bodies within the ghost band G of the shared boundary
                 (ids + full particle state).
Per substep:
  begin       -- integrate, hash grid, candidates (owned + ghost bodies)
  iteration k -- owned bodies only; then positions of the ghosts are exchanged
                 (after the last iteration also velocities and anchors, so the
                 ghosts' next integrate reproduces the owner's exactly).

Ghost band: a pair (i, j) is a candidate only if |x_i - x_j| < h. With rho the
largest particle-centre distance from a body's com and `margin` the largest com
drift allowed between repartitions (guarded: a body that drifts more than
margin/2 in x within a frame raises SimulationError), any body whose com is
farther than G = 2*rho + h + margin from the boundary cannot reach the slab.

The engine is duck-typed (GpuEngine here over the C-ABI; the CPU tests plug in
the oracle), and so is the communicator (TorchComm: torch.distributed P2P,
NCCL on GPUs / gloo on CPU; LocalComm: ranks as threads of one process).
"""
from __future__ import annotations

import threading
from dataclasses import dataclass, field

import numpy as np

from . import pbdr as P

POS, VEL, ANCHOR, ROT = P.FIELD_POSITION, P.FIELD_VELOCITY, P.FIELD_ANCHOR, P.FIELD_ROTATION


# ---------------------------------------------------------------------------
# Geometry
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class SlabGeometry:
    edges: np.ndarray  # world + 1 boundaries; edges[0] = -inf, edges[-1] = +inf
    ghost_band: float  # G
    margin: float

    @property
    def world(self) -> int:
        return len(self.edges) - 1

    def slab_of(self, com_x) -> np.ndarray:
        return np.searchsorted(self.edges[1:-1], np.asarray(com_x, np.float64), side="right").astype(np.int64)


def body_reach(rest_offsets, body_offsets, radius) -> tuple[float, float]:
    """(rho, h): largest particle-centre distance from its body's com (rest
    pose, +5% for shape-matching deformation) and the contact cell h = 2 r_max."""
    q = np.asarray(rest_offsets, np.float64).reshape(-1, 3)
    rho = float(np.sqrt((q * q).sum(1)).max()) * 1.05 if len(q) else 0.0
    return rho, 2.0 * float(np.max(radius))


def slab_geometry(com_x, world: int, rho: float, h: float, margin: float = 0.1) -> SlabGeometry:
    """Equal x-slabs over the initial com range; the outer slabs are unbounded."""
    com_x = np.asarray(com_x, np.float64)
    lo, hi = float(com_x.min()), float(com_x.max())
    inner = np.linspace(lo, hi, world + 1)[1:-1] if world > 1 else np.zeros(0)
    edges = np.concatenate([[-np.inf], inner, [np.inf]])
    G = 2.0 * rho + h + margin
    if world > 2:
        width = (hi - lo) / world
        if width < G + margin:
            raise P.ConfigError(f"x-slab width {width:.3f} m is below the ghost band + margin "
                                f"({G + margin:.3f} m): use fewer ranks", "slab.world")
    return SlabGeometry(edges, G, margin)


# ---------------------------------------------------------------------------
# Communicators
# ---------------------------------------------------------------------------
class TorchComm:
    """Neighbour exchange over torch.distributed point-to-point (NCCL on the
    GPU box, gloo in the CPU tests); ops are batched so paired sends and
    receives cannot deadlock."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group

    def exchange(self, sends: dict, recv_shapes: dict, dtype, device) -> dict:
        import torch
        dist = self.dist
        recvs = {p: torch.empty(shape, dtype=dtype, device=device) for p, shape in recv_shapes.items()}
        ops = [dist.P2POp(dist.isend, t.contiguous(), p, self.group) for p, t in sends.items() if t.numel()]
        ops += [dist.P2POp(dist.irecv, t, p, self.group) for p, t in recvs.items() if t.numel()]
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        return recvs


class LocalComm:
    """Ranks as threads of one process (a mailbox and a barrier); used to run
    the decomposition on one device without kernels that wait on each other."""

    def __init__(self, world: int):
        self.world = world
        self.box = {}
        self.lock = threading.Lock()
        self.barrier = threading.Barrier(world)

    def view(self, rank: int) -> "LocalComm._View":
        return LocalComm._View(self, rank)

    class _View:
        def __init__(self, hub, rank):
            self.hub, self.rank = hub, rank

        def exchange(self, sends: dict, recv_shapes: dict, dtype, device) -> dict:
            import torch
            if torch.device(device).type == "cuda":
                torch.cuda.current_stream().synchronize()  # payload complete before a peer reads it
            with self.hub.lock:
                for p, t in sends.items():
                    self.hub.box[(self.rank, p)] = t
            self.hub.barrier.wait()
            out = {}
            with self.hub.lock:
                for p, shape in recv_shapes.items():
                    t = self.hub.box.pop((p, self.rank), None)
                    if t is None:
                        t = torch.empty(shape, dtype=dtype, device=device)
                    assert tuple(t.shape) == tuple(shape), (t.shape, shape)
                    out[p] = t.clone()
            if torch.device(device).type == "cuda":
                torch.cuda.current_stream().synchronize()  # copies done before the sender frees
            self.hub.barrier.wait()
            return out


# ---------------------------------------------------------------------------
# Engine over the C-ABI (device buffers as torch tensors on the handle stream)
# ---------------------------------------------------------------------------
class GpuEngine:
    def __init__(self, solver: P.GpuSolver, cfg):
        import torch
        self.torch = torch
        self.s = solver
        self.n, self.nb = solver.n, solver.nb
        self.iters, self.substeps = cfg.solver_iterations, cfg.substeps
        self.device = torch.device("cuda", solver.info.device)
        self.stream = torch.cuda.ExternalStream(solver.stream_handle(), device=self.device)

    def context(self):
        return self.torch.cuda.stream(self.stream)

    def index(self, a: np.ndarray):
        return self.torch.as_tensor(np.ascontiguousarray(a, np.int32), device=self.device)

    def gather(self, fld, idx):
        out = self.torch.empty((idx.numel(), 4), dtype=self.torch.float32, device=self.device)
        if idx.numel():
            self.s.gather_dev(fld, idx.data_ptr(), idx.numel(), out.data_ptr())
        return out

    def scatter(self, fld, idx, values):
        if idx.numel():
            values = values.contiguous()
            values.record_stream(self.stream)
            self.s.scatter_dev(fld, idx.data_ptr(), idx.numel(), values.data_ptr())

    def set_roles(self, roles):
        self.s.set_roles(roles)

    def begin(self):
        self.s.substep_begin()

    def iteration(self):
        self.s.substep_iteration()

    def end_substep(self):
        pass

    def sync(self):
        self.s.sync()

    def com_x(self) -> np.ndarray:
        return self.s.read_bodies()[:, 0]


# ---------------------------------------------------------------------------
# The per-rank driver
# ---------------------------------------------------------------------------
@dataclass
class _Plan:
    send_bodies: dict = field(default_factory=dict)  # peer -> body ids (ascending)
    recv_bodies: dict = field(default_factory=dict)
    send_slots: dict = field(default_factory=dict)   # peer -> engine index tensor
    recv_slots: dict = field(default_factory=dict)
    send_bidx: dict = field(default_factory=dict)
    recv_bidx: dict = field(default_factory=dict)


class SlabRunner:
    def __init__(self, engine, rank: int, world: int, comm, body_offsets, geometry: SlabGeometry | None = None,
                 rho: float | None = None, h: float | None = None, margin: float = 0.1):
        self.e = engine
        self.rank, self.world, self.comm = rank, world, comm
        off = np.asarray(body_offsets, np.int64)
        self.bstart, self.bcount = off[:-1], np.diff(off)
        self.geo = geometry
        self.rho, self.h, self.margin = rho, h, margin
        self.owned = np.zeros(0, np.int64)
        self.com_ref = np.zeros(self.e.nb)  # com_x at the last repartition
        self.plan = _Plan()
        self.frames_done = 0
        self.migrations = 0  # bodies received from a neighbour at repartitions

    # -- helpers -------------------------------------------------------------
    def _peers(self):
        return [p for p in (self.rank - 1, self.rank + 1) if 0 <= p < self.world]

    def _slots(self, bodies) -> np.ndarray:
        if len(bodies) == 0:
            return np.zeros(0, np.int32)
        return np.concatenate([np.arange(self.bstart[b], self.bstart[b] + self.bcount[b]) for b in bodies]
                              ).astype(np.int32)

    def _exchange(self, sends, recv_shapes, dtype):
        import torch
        dev = getattr(self.e, "device", "cpu")
        return self.comm.exchange(sends, recv_shapes, getattr(torch, dtype), dev)

    def _exchange_ids(self, send_ids: dict) -> dict:
        """Variable-length int64 lists to each neighbour: counts first, then ids."""
        import torch
        dev = getattr(self.e, "device", "cpu")
        counts = self.comm.exchange({p: torch.tensor([len(v)], dtype=torch.int64, device=dev)
                                     for p, v in send_ids.items()},
                                    {p: (1,) for p in send_ids}, torch.int64, dev)
        got = self.comm.exchange({p: torch.as_tensor(np.asarray(v, np.int64), device=dev) for p, v in send_ids.items()},
                                 {p: (int(counts[p].item()),) for p in send_ids}, torch.int64, dev)
        return {p: got[p].cpu().numpy() for p in send_ids}

    def _exchange_f64(self, send: dict, recv_counts: dict) -> dict:
        import torch
        dev = getattr(self.e, "device", "cpu")
        got = self.comm.exchange({p: torch.as_tensor(np.asarray(v, np.float64), device=dev) for p, v in send.items()},
                                 {p: (recv_counts[p],) for p in send}, torch.float64, dev)
        return {p: got[p].cpu().numpy() for p in send}

    def _send_fields(self, fields):
        """Owned ghost records -> neighbours; received records -> local ghost slots."""
        pl = self.plan
        peers = self._peers()
        for fld in fields:
            body = fld in (ANCHOR, ROT)
            sidx, ridx = (pl.send_bidx, pl.recv_bidx) if body else (pl.send_slots, pl.recv_slots)
            sends = {p: self.e.gather(fld, sidx[p]) for p in peers}
            got = self._exchange(sends, {p: (ridx[p].numel() if hasattr(ridx[p], "numel") else len(ridx[p]), 4)
                                         for p in peers}, "float32")
            for p in peers:
                self.e.scatter(fld, ridx[p], got[p])

    # -- partitioning ----------------------------------------------------------
    def start(self):
        """Initial partition from the (identical on every rank) scene state."""
        with self.e.context():
            self.e.set_roles(None)
            com = self.e.com_x()
            if self.geo is None:
                self.geo = slab_geometry(com, self.world, self.rho, self.h, self.margin)
            self.owned = np.flatnonzero(self.geo.slab_of(com) == self.rank)
            self.com_ref = com.copy()
            self._build_ghosts(com)

    def _build_ghosts(self, com):
        """Send each neighbour the owned bodies within the ghost band (ids +
        full particle state), receive its ghosts, set roles and plans."""
        G, edges = self.geo.ghost_band, self.geo.edges
        r = self.rank
        send_ids = {}
        for p in self._peers():
            cx = com[self.owned]
            sel = cx < edges[r] + G if p == r - 1 else cx >= edges[r + 1] - G
            send_ids[p] = self.owned[sel]
        recv_ids = self._exchange_ids(send_ids)
        pl = _Plan()
        for p in self._peers():
            pl.send_bodies[p], pl.recv_bodies[p] = send_ids[p], np.sort(recv_ids[p])
            pl.send_slots[p] = self.e.index(self._slots(send_ids[p]))
            pl.recv_slots[p] = self.e.index(self._slots(pl.recv_bodies[p]))
            pl.send_bidx[p] = self.e.index(send_ids[p])
            pl.recv_bidx[p] = self.e.index(pl.recv_bodies[p])
        # recv lists must be in the sender's order: the sender sorted nothing,
        # so send the sorted order (owned is ascending, selections keep order).
        self.plan = pl
        roles = np.zeros(self.e.nb, np.int8)
        for p in self._peers():
            roles[pl.recv_bodies[p]] = 1
        roles[self.owned] = 2
        self.e.set_roles(roles)
        # New ghosts need the full state; a ghost that stays a ghost is already
        # current, but resending is cheap next to a frame and keeps this simple.
        self._send_fields((POS, VEL, ANCHOR))

    def repartition(self):
        with self.e.context():
            com = self.e.com_x()
            cx = com[self.owned]
            drift = np.abs(cx - self.com_ref[self.owned])
            if drift.size and drift.max() > 0.5 * self.geo.margin:
                b = int(self.owned[int(np.argmax(drift))])
                raise P.SimulationError(f"slab halo margin exceeded: body {b} moved {drift.max():.4f} m in x "
                                        f"in one frame (margin {self.geo.margin} m)", self.frames_done, b)
            dest = self.geo.slab_of(cx)
            if dest.size and np.abs(dest - self.rank).max() > 1:
                raise P.SimulationError("a body skipped a whole slab in one frame", self.frames_done, -1)
            out = {p: self.owned[dest == p] for p in self._peers()}
            keep = self.owned[dest == self.rank]
            arrivals = self._exchange_ids(out)
            # Migrants carry their com_x (for the ghost decision), anchor and
            # warm-start rotation; positions/velocities are present (ghosts).
            com_in = self._exchange_f64({p: com[out[p]] for p in self._peers()},
                                        {p: len(arrivals[p]) for p in self._peers()})
            for fld in (ANCHOR, ROT):
                sends = {p: self.e.gather(fld, self.e.index(out[p])) for p in self._peers()}
                got = self._exchange(sends, {p: (len(arrivals[p]), 4) for p in self._peers()}, "float32")
                for p in self._peers():
                    self.e.scatter(fld, self.e.index(arrivals[p]), got[p])
            for p in self._peers():
                com[arrivals[p]] = com_in[p]
                self.migrations += len(arrivals[p])
            self.owned = np.sort(np.concatenate([keep] + [arrivals[p] for p in self._peers()])).astype(np.int64)
            self.com_ref = com
            self._build_ghosts(com)

    # -- stepping ------------------------------------------------------------
    def step_frames(self, frames: int = 1):
        for _ in range(frames):
            if self.frames_done > 0:
                self.repartition()
            with self.e.context():
                for _s in range(self.e.substeps):
                    self.e.begin()
                    for k in range(self.e.iters):
                        self.e.iteration()
                        self._send_fields((POS,) if k < self.e.iters - 1 else (POS, VEL, ANCHOR))
                    self.e.end_substep()
                self.e.sync()
            self.frames_done += 1

    def owned_state(self):
        """(owned body ids, their slots, pos4, vel4) -- this rank's authoritative part."""
        with self.e.context():
            slots = self._slots(self.owned)
            idx = self.e.index(slots)
            p4 = self.e.gather(POS, idx)
            v4 = self.e.gather(VEL, idx)
            to_np = (lambda t: t.cpu().numpy()) if hasattr(p4, "cpu") else np.asarray
            self.e.sync()
            return self.owned.copy(), slots, to_np(p4), to_np(v4)


def run_threads(engines, body_offsets, frames: int, margin: float = 0.1, rho=None, h=None, geometry=None):
    """Runs len(engines) ranks as threads of this process (LocalComm) and
    returns each rank's owned_state() after `frames` frames."""
    world = len(engines)
    hub = LocalComm(world)
    runners = [SlabRunner(e, r, world, hub.view(r), body_offsets, geometry=geometry, rho=rho, h=h, margin=margin)
               for r, e in enumerate(engines)]
    out, errs = [None] * world, [None] * world

    def work(r):
        try:
            runners[r].start()
            runners[r].step_frames(frames)
            out[r] = runners[r].owned_state()
        except BaseException as ex:  # surface in the caller
            errs[r] = ex
            hub.barrier.abort()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in errs:
        if e is not None and not isinstance(e, threading.BrokenBarrierError):
            raise e
    for e in errs:
        if e is not None:
            raise e
    return out

