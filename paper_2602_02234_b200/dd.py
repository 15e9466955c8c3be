"""Domain-decomposed DP force evaluation (multi-GPU, per-layer rc halo).

The periodic box is split over a px x py x pz rank grid (1x1x1, 2x1x1, 2x2x1,
2x2x2 for 1/2/4/8 ranks).  Rank r owns the atoms whose wrapped position lies in
its region (wrap_position, /root/reference/proj/include/halomd/box.hpp:34-42)
and evaluates exactly their rows of the global periodic neighbour list
(build_input_periodic, src/nn/inference.cpp:449-487): same pairs, same FP64
minimum-image edge_dr, neighbour ids remapped to local ids.  Neighbours owned
elsewhere become halo ghosts (no rows, no images: the model only sees dr).

A depth-L model needs an L*rc receptive field (model.hpp:51-52); instead of the
SPEC's single L*rc-deep halo, which does not fit the paper's
boxes at 2-8 ranks, the halo stays rc deep and the message
layers exchange per layer:
  forward   P^l = W1h^(l) h^l of every ghost, from its owner     (layers 0..L-2)
  backward  partial dE/dh sums collected at ghosts -> owners      (layers L-2..0)
  forces    forces on ghosts -> owners
so a step costs 2(L-1)+1 halo rounds plus one all-gather of positions and an
all-reduce of (E, W).  The same driver runs over any Transport: NCCL over
NVLink (torch.distributed, one process per GPU), gloo (CPU tests), or an
in-process transport (several ranks simulated in one process).

Engines run the per-rank phases: GpuEngine wraps the libhmdp C-ABI phase entry
points (hmdp_dd_*); tests also provide a NumPy engine.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from ._lib import check, lib, ptr


def rank_grid(n_ranks: int) -> tuple[int, int, int]:
    """Rank grid for n ranks: 1 -> 1x1x1, 2 -> 2x1x1, 4 -> 2x2x1, 8 -> 2x2x2, ..."""
    dims = [1, 1, 1]
    n = n_ranks
    a = 0
    f = 2
    while n > 1:
        while n % f:
            f += 1
        dims[a % 3] *= f
        n //= f
        a += 1
    return tuple(dims)


def owners(positions: np.ndarray, box: np.ndarray, dims) -> np.ndarray:
    """Owning rank of every atom: wrap into [0, L) (box.hpp:34-42), then the
    region index floor(r / L * p) clamped, rank = (iz * py + iy) * px + ix."""
    x = np.asarray(positions, dtype=np.float64)
    L = np.asarray(box, dtype=np.float64)
    r = x - L * np.floor(x / L)
    r = np.where(r >= L, 0.0, r)
    d = np.asarray(dims)
    c = np.clip((r / L * d).astype(np.int64), 0, d - 1)
    return ((c[:, 2] * d[1] + c[:, 1]) * d[0] + c[:, 0]).astype(np.int64)


@dataclass
class RankPlan:
    owned: np.ndarray   # global ids, ascending
    ghosts: np.ndarray  # global ids, ascending
    offset: np.ndarray  # local CSR (owned rows, then empty ghost rows)
    nbr: np.ndarray     # local ids
    dr: np.ndarray
    types: np.ndarray
    # halo maps, per peer: local rows this rank sends / receives for the P
    # (forward) direction; the backward/force direction swaps them.
    send: dict = field(default_factory=dict)  # peer -> local owned rows
    recv: dict = field(default_factory=dict)  # peer -> local ghost rows

    @property
    def n_own(self) -> int:
        return int(self.owned.shape[0])

    @property
    def n_loc(self) -> int:
        return int(self.owned.shape[0] + self.ghosts.shape[0])


def make_plans(offset, nbr, dr, types, owner, n_ranks) -> list[RankPlan]:
    """Every rank computes the same plans from the same global data, so no
    negotiation round is needed."""
    offset = np.asarray(offset)
    nbr = np.asarray(nbr)
    n = offset.shape[0] - 1
    counts = np.diff(offset)
    plans = []
    for r in range(n_ranks):
        owned = np.nonzero(owner == r)[0]
        rows = np.concatenate([np.arange(offset[i], offset[i + 1]) for i in owned]) if owned.size else np.zeros(0, np.int64)
        tgt = nbr[rows]
        ghosts = np.unique(tgt[owner[tgt] != r])
        loc = np.full(n, -1, dtype=np.int64)
        loc[owned] = np.arange(owned.size)
        loc[ghosts] = owned.size + np.arange(ghosts.size)
        off = np.zeros(owned.size + ghosts.size + 1, dtype=np.int32)
        off[1:owned.size + 1] = np.cumsum(counts[owned])
        off[owned.size + 1:] = off[owned.size]
        plans.append(RankPlan(owned=owned, ghosts=ghosts, offset=off,
                              nbr=loc[tgt].astype(np.int32), dr=np.asarray(dr)[rows],
                              types=np.asarray(types)[np.concatenate([owned, ghosts])].astype(np.int32)))
    for q, pq in enumerate(plans):
        go = owner[pq.ghosts]
        for r in range(n_ranks):
            sel = np.nonzero(go == r)[0]
            if sel.size == 0:
                continue
            atoms = pq.ghosts[sel]
            pr = plans[r]
            pr.send[q] = np.searchsorted(pr.owned, atoms).astype(np.int64)
            pq.recv[r] = (pq.n_own + sel).astype(np.int64)
    return plans


# ---------------------------------------------------------------------------
# Transports: exchange(rows per peer) -> rows per peer
# ---------------------------------------------------------------------------
class TorchDistTransport:
    """torch.distributed all_to_all_single over one flat buffer (NCCL on GPUs)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def exchange(self, send: dict, width: int, like):
        import torch

        # NCCL moves device buffers directly (NVLink); other backends (gloo, for
        # tests and single-GPU dry runs) stage through host memory
        dev = like.device if self.dist.get_backend(self.group) == "nccl" else torch.device("cpu")
        sizes_out = [int(send[p].shape[0]) if p in send else 0 for p in range(self.size)]
        cnt = torch.tensor(sizes_out, dtype=torch.int64, device=dev)
        cnt_in = torch.empty_like(cnt)
        self.dist.all_to_all_single(cnt_in, cnt, group=self.group)
        sizes_in = [int(v) for v in cnt_in.tolist()]
        parts = [send[p].to(dev) for p in range(self.size) if p in send and send[p].shape[0]]
        flat = torch.cat(parts).reshape(-1) if parts else torch.zeros(0, dtype=like.dtype, device=dev)
        out = torch.empty(sum(sizes_in) * width, dtype=like.dtype, device=dev)
        self.dist.all_to_all_single(out, flat.contiguous(), [s * width for s in sizes_in],
                                    [s * width for s in sizes_out], group=self.group)
        res, o = {}, 0
        for p, s in enumerate(sizes_in):
            if s:
                res[p] = out[o:o + s * width].reshape(s, width).to(like.device)
            o += s * width
        return res

    def allreduce_sum(self, values):
        import torch

        t = torch.tensor(values, dtype=torch.float64,
                         device="cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu")
        self.dist.all_reduce(t, group=self.group)
        return t.cpu().numpy()


class LocalTransport:
    """In-process transport for several simulated ranks stepping in lockstep
    (the SPEC's in-memory transport): rank r's exchange() deposits
    its rows and, once every rank has deposited, returns what was sent to it."""

    def __init__(self, n_ranks):
        self.n = n_ranks
        self.box = {}

    def view(self, rank):
        return _LocalView(self, rank)


class _LocalView:
    def __init__(self, hub, rank):
        self.hub, self.rank, self.size = hub, rank, hub.n

    def post(self, send: dict):
        for p, rows in send.items():
            self.hub.box[(self.rank, p)] = rows

    def collect(self) -> dict:
        res = {}
        for r in range(self.size):
            if (r, self.rank) in self.hub.box:
                res[r] = self.hub.box.pop((r, self.rank))
        return res


# ---------------------------------------------------------------------------
# GPU engine over the C-ABI phase entry points
# ---------------------------------------------------------------------------
class _CudaArray:
    def __init__(self, ptr_, shape, typestr):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr,
                                         "data": (ptr_, False), "version": 3}


class GpuEngine:
    """One rank's phases on its GPU (hmdp_dd_*); halo rows are torch views of
    the context's device buffers, all work on the context's (torch) stream."""

    def __init__(self, ctx, precision):
        import torch

        self.torch = torch
        self.ctx = ctx
        self.prec = precision
        self.dtype = torch.float64 if int(precision) == 1 else torch.float32
        stream = torch.cuda.current_stream(torch.device("cuda", ctx.device))
        # torch's default stream has handle 0, which hmdp_set_stream reads as "the
        # context's own stream"; name the legacy default stream (cudaStreamLegacy
        # = 1) explicitly so the phases and the torch halo copies share one stream
        handle = stream.cuda_stream or 1
        check(lib().hmdp_set_stream(ctx.handle, ctypes.c_void_p(handle)))

    def setup(self, plan: RankPlan):
        L = lib()
        off = np.ascontiguousarray(plan.offset, dtype=np.int32)
        nb = np.ascontiguousarray(plan.nbr, dtype=np.int32)
        dr = np.ascontiguousarray(plan.dr, dtype=np.float64).reshape(-1, 3)
        ty = np.ascontiguousarray(plan.types, dtype=np.int32)
        check(L.hmdp_dd_setup(self.ctx.handle, plan.n_loc, plan.n_own, ptr(off), ptr(nb),
                              ptr(dr), ptr(ty), int(self.prec)))
        self.n_loc = plan.n_loc
        typestr = "<f8" if self.dtype == self.torch.float64 else "<f4"
        self.rows = {}
        for kind in (0, 1, 2):
            p = ctypes.c_void_p()
            check(L.hmdp_dd_buffer(self.ctx.handle, kind, ctypes.byref(p)))
            self.rows[kind] = self.torch.as_tensor(
                _CudaArray(p.value, (self.n_loc, 32), typestr), device=f"cuda:{self.ctx.device}")
        p = ctypes.c_void_p()
        check(L.hmdp_dd_buffer(self.ctx.handle, 3, ctypes.byref(p)))
        self.forces = self.torch.as_tensor(_CudaArray(p.value, (self.n_loc, 3), "<f8"),
                                           device=f"cuda:{self.ctx.device}")

    def phase(self, ph, layer=0):
        check(lib().hmdp_dd_phase(self.ctx.handle, int(ph), int(layer)))

    # row access used by the driver
    def p_rows(self):
        return self.rows[0]

    def remote_rows(self):
        return self.rows[1]

    def ghost_sum_rows(self):
        return self.rows[2]

    def force_rows(self):
        return self.forces

    def result(self):
        e = ctypes.c_double()
        w = ctypes.c_double()
        w9 = np.zeros(9)
        check(lib().hmdp_dd_result(self.ctx.handle, ctypes.byref(e), ptr(w9), ctypes.byref(w)))
        return e.value, w.value, w9

    def index(self, idx):
        return self.torch.as_tensor(idx, device=self.rows[0].device)


# ---------------------------------------------------------------------------
# Driver
# ---------------------------------------------------------------------------
def _exchange(transport, send: dict, width: int, like):
    if isinstance(transport, _LocalView):
        raise RuntimeError("LocalTransport ranks are driven by evaluate_local()")
    return transport.exchange(send, width, like)


def rank_steps(engine, plan: RankPlan, depth: int):
    """The per-rank phase program as a generator of halo rounds: yields
    (kind, send rows dict) and receives the peer rows dict; `kind` is 'p'
    (forward, copy into ghost rows) or 'add' (backward/forces, add into owned
    rows of the given target)."""
    M = depth - 1
    engine.setup(plan)
    engine.phase(0)
    if M > 0:
        for l in range(M):
            p = engine.p_rows()
            got = yield ("copy", {q: p[engine.index(rows)] for q, rows in plan.send.items()}, p, plan.recv)
            engine.phase(1, l)
            engine.phase(2, l)
        for l in range(M - 1, -1, -1):
            engine.phase(3, l)
            gs = engine.ghost_sum_rows()
            rem = engine.remote_rows()
            rem.zero_()
            yield ("add", {q: gs[engine.index(rows)] for q, rows in plan.recv.items()}, rem, plan.send)
            if l > 0:
                engine.phase(4, l - 1)
            else:
                engine.phase(5)
    engine.phase(6)
    f = engine.force_rows()
    yield ("add", {q: f[engine.index(rows)] for q, rows in plan.recv.items()}, f, plan.send)
    return


def _apply(kind, target, peer_rows: dict, maps: dict, engine):
    for q, vals in peer_rows.items():
        idx = engine.index(maps[q])
        if kind == "copy":
            target[idx] = vals.to(target.dtype)
        else:
            target.index_add_(0, idx, vals.to(target.dtype))


def evaluate_dd(engine, transport, plans, rank: int, depth: int):
    """One rank's domain-decomposed evaluation over a torch.distributed-style
    transport.  Returns (E_total, F_owned [n_own,3] numpy, W_total, W9_total)."""
    plan = plans[rank]
    prog = rank_steps(engine, plan, depth)
    msg = next(prog)
    while True:
        kind, send, target, maps = msg
        width = target.shape[1]
        got = _exchange(transport, send, width, target)
        _apply(kind, target, got, maps, engine)
        try:
            msg = prog.send(got)
        except StopIteration:
            break
    e, w, w9 = engine.result()
    tot = transport.allreduce_sum([e, w, *w9])
    f = engine.force_rows()[: plan.n_own].cpu().numpy() if hasattr(engine.force_rows(), "cpu") \
        else np.asarray(engine.force_rows()[: plan.n_own])
    return float(tot[0]), f, float(tot[1]), np.asarray(tot[2:11]).reshape(3, 3)


def evaluate_local(engines, plans, depth: int):
    """All ranks in one process (LocalTransport semantics): runs the per-rank
    programs in lockstep, exchanging rows in memory."""
    progs = [rank_steps(engines[r], plans[r], depth) for r in range(len(plans))]
    msgs = [next(p) for p in progs]
    done = False
    while not done:
        # deliver: rows sent by r to q
        inbox = [dict() for _ in plans]
        for r, (kind, send, target, maps) in enumerate(msgs):
            for q, rows in send.items():
                inbox[q][r] = rows
        for q, (kind, send, target, maps) in enumerate(msgs):
            _apply(kind, target, inbox[q], maps, engines[q])
        nxt = []
        for r, p in enumerate(progs):
            try:
                nxt.append(p.send(inbox[r]))
            except StopIteration:
                done = True
        if not done:
            msgs = nxt
    E = W = 0.0
    W9 = np.zeros(9)
    F = {}
    for r, eng in enumerate(engines):
        e, w, w9 = eng.result()
        E += e
        W += w
        W9 += w9
        fr = eng.force_rows()
        fr = fr.cpu().numpy() if hasattr(fr, "cpu") else np.asarray(fr)
        F[r] = fr[: plans[r].n_own]
    return E, F, W, W9.reshape(3, 3)


# ---------------------------------------------------------------------------
# Device-resident domain decomposition on the global index space (hmdp_gdd_*):
# plans built on the device every step, exchanges as SUM all-reduces of fixed-size
# global-index buffers -> one CUDA graph per step (collectives included).
# ---------------------------------------------------------------------------
class DeviceDD:
    """One rank's device-resident DD engine.  Every rank holds all n positions and
    velocities (replicated: all ranks integrate all atoms with the same all-reduced
    forces) and evaluates the network for the atoms its region owns.

    ``program(kind)`` is a generator over the phase program; it yields every
    tensor that must be SUM all-reduced across ranks before it continues
    (``run_dist`` does that with torch.distributed / NCCL, ``run_local`` for
    ranks simulated in one process)."""

    def __init__(self, ctx, n, types, box, dims, rank, precision, masses=None):
        import torch

        from .nn import Precision

        self.ctx, self.n, self.rank = ctx, int(n), int(rank)
        self.dims = tuple(int(d) for d in dims)
        self.depth = ctx.model.depth()
        self.prec = precision
        dev = torch.device("cuda", ctx.device)
        T = torch.float64 if precision == Precision.fp64 else torch.float32
        self.pos = torch.zeros((n, 3), dtype=torch.float64, device=dev)
        self.vel = torch.zeros((n, 3), dtype=torch.float64, device=dev)
        self.mass = torch.ones(n, dtype=torch.float64, device=dev)
        self.p = torch.zeros((n, 32), dtype=T, device=dev)
        self.sg = torch.zeros((n, 32), dtype=T, device=dev)
        # forces and the (E, W, W9) totals share one buffer: one all-reduce for both
        self.fo = torch.zeros(3 * n + 16, dtype=torch.float64, device=dev)
        self.f = self.fo[:3 * n].view(n, 3)
        self.out = self.fo[3 * n:]
        t = np.ascontiguousarray(types, dtype=np.int32)
        b = np.ascontiguousarray(box, dtype=np.float64)
        d = np.ascontiguousarray(self.dims, dtype=np.int32)
        L = lib()
        # the context runs on torch's current stream, so the phases and the all-reduces
        # (torch ops / NCCL) are stream-ordered; torch's default stream is the legacy
        # NULL stream, passed as cudaStreamLegacy (NULL would select the context's own)
        sid = torch.cuda.current_stream(dev).cuda_stream
        check(L.hmdp_set_stream(ctx.handle, ctypes.c_void_p(sid if sid else 1)))
        check(L.hmdp_gdd_setup(ctx.handle, self.n, ptr(t), ptr(b), ptr(d), self.rank,
                               int(precision)))
        for kind, ten in enumerate([self.pos, self.p, self.sg, self.f, self.out, self.vel,
                                    self.mass]):
            check(L.hmdp_gdd_bind(ctx.handle, kind, ctypes.c_void_p(ten.data_ptr())))
        if masses is not None:
            self.mass.copy_(torch.as_tensor(np.asarray(masses, dtype=np.float64)))

    def load(self, positions, velocities=None):
        import torch

        self.pos.copy_(torch.as_tensor(np.asarray(positions, dtype=np.float64).reshape(-1, 3)))
        if velocities is not None:
            self.vel.copy_(torch.as_tensor(np.asarray(velocities, dtype=np.float64).reshape(-1, 3)))

    def _ph(self, phase, layer=0, dt=0.0):
        check(lib().hmdp_gdd_phase(self.ctx.handle, phase, layer, float(dt)))

    def program(self, kind="eval", dt=0.001):
        """kind: 'eval' (one force evaluation), 'md' (evaluation + velocity Verlet
        closing kick, next opening kick, drift), 'open' (the initial opening kick +
        drift from the current forces)."""
        if kind == "open":
            self._ph(8, 0, dt)
            return
        M = self.depth - 1
        self._ph(10)
        self._ph(0)
        for l in range(M):
            yield self.p
            self._ph(1, l)
            self._ph(2, l)
        for l in range(M - 1, -1, -1):
            self._ph(3, l)
            yield self.sg
            if l > 0:
                self._ph(4, l - 1)
            else:
                self._ph(5)
        self._ph(6)
        yield self.fo  # forces + (E, W, W9)
        if kind == "md":
            self._ph(7, 0, dt)

    def launches(self):
        """Kernels this rank's phases have enqueued so far (hmdp_gdd_launches)."""
        v = ctypes.c_longlong()
        check(lib().hmdp_gdd_launches(self.ctx.handle, ctypes.byref(v)))
        return int(v.value)

    def counts(self):
        c = np.zeros(3, dtype=np.int32)
        check(lib().hmdp_gdd_counts(self.ctx.handle, ptr(c)))
        return tuple(int(v) for v in c)

    def result(self):
        o = self.out.cpu().numpy()
        return float(o[0]), self.f.cpu().numpy(), float(o[1]), o[2:11].reshape(3, 3)


def run_dist(engine: DeviceDD, kind="eval", dt=0.001, group=None):
    """One rank's program with NCCL SUM all-reduces (torch.distributed) on the
    current stream — capturable in a CUDA graph."""
    import torch.distributed as td

    for ten in engine.program(kind, dt):
        td.all_reduce(ten, group=group)


def run_local(engines, kind="eval", dt=0.001):
    """Ranks simulated in one process: lockstep programs, the all-reduce is a sum of
    the ranks' buffers in rank order written back to every rank."""
    progs = [e.program(kind, dt) for e in engines]
    while True:
        bufs = []
        for p in progs:  # every rank advances to its next collective (or its end)
            try:
                bufs.append(next(p))
            except StopIteration:
                pass
        if not bufs:
            return
        if len(bufs) != len(progs):
            raise RuntimeError("ranks disagree on the number of collectives")
        tot = bufs[0].clone()
        for b in bufs[1:]:
            tot += b
        for b in bufs:
            b.copy_(tot)


# ---------------------------------------------------------------------------
# Halo-exchange engine (the multi-GPU default): hmdp_gdd_* in halo mode.
# ---------------------------------------------------------------------------
EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                               ctypes.c_void_p, ctypes.c_size_t, ctypes.c_size_t)


class HaloDD:
    """One rank's halo-exchange DD engine (include/hmdp.h, hmdp_gdd_* halo mode), or,
    with ``strategy="gather"``, the paper's gather-to-root strategy on the same
    transports (owned atoms -> rank 0, one single-domain evaluation, forces back to
    the owners).

    Nothing is replicated: the rank integrates only the atoms its region owns and
    every step moves exactly the halo with point-to-point rounds to every peer
    (POS with migration, P^l per message layer forward, dE/dh partial sums per layer
    and partial forces back to the owners, (E, W, W9) partials).  The whole step --
    exchanges included -- is one C++ call (``step``), capturable in a CUDA graph
    with the NCCL transport.  Transports: ``attach_nccl`` (one GPU per rank),
    ``attach_hub`` (ranks simulated as contexts on one GPU, one host thread each) or
    ``attach_callback`` (a Python exchange, e.g. gloo).

    Global-index buffers: only the rows of owned (and halo) atoms are current on a
    rank; ``owned_forces`` returns this rank's share of the global result."""

    def __init__(self, ctx, n, types, box, dims, rank, precision, masses=None, stream=None,
                 strategy="halo"):
        import torch

        if strategy not in ("halo", "gather"):
            raise ValueError("strategy must be 'halo' or 'gather'")
        self.strategy = strategy
        self.ctx, self.n, self.rank = ctx, int(n), int(rank)
        self.dims = tuple(int(d) for d in dims)
        self.world = self.dims[0] * self.dims[1] * self.dims[2]
        self.depth = ctx.model.depth()
        dev = torch.device("cuda", ctx.device)
        self.dev = dev
        self.pos = torch.zeros((n, 3), dtype=torch.float64, device=dev)
        self.vel = torch.zeros((n, 3), dtype=torch.float64, device=dev)
        self.mass = torch.ones(n, dtype=torch.float64, device=dev)
        self.f = torch.zeros((n, 3), dtype=torch.float64, device=dev)
        self.out = torch.zeros(16, dtype=torch.float64, device=dev)
        if masses is not None:
            self.mass.copy_(torch.as_tensor(np.asarray(masses, dtype=np.float64)))
        L = lib()
        if stream is not None:  # run on the caller's stream (graph capture, NCCL ordering)
            check(L.hmdp_set_stream(ctx.handle, ctypes.c_void_p(stream.cuda_stream)))
        t = np.ascontiguousarray(types, dtype=np.int32)
        b = np.ascontiguousarray(box, dtype=np.float64)
        d = np.ascontiguousarray(self.dims, dtype=np.int32)
        check(L.hmdp_gdd_setup(ctx.handle, self.n, ptr(t), ptr(b), ptr(d), self.rank,
                               int(precision)))
        # halo exchange (1) or the paper's gather-to-root strategy (2)
        check(L.hmdp_gdd_set_mode(ctx.handle, 1 if strategy == "halo" else 2))
        for kind, ten in ((0, self.pos), (3, self.f), (4, self.out), (5, self.vel),
                          (6, self.mass)):
            check(L.hmdp_gdd_bind(ctx.handle, kind, ctypes.c_void_p(ten.data_ptr())))
        self._cb = None

    def load(self, positions, velocities=None):
        """Every rank loads the full initial configuration; plans the packet capacity."""
        import torch

        self.pos.copy_(torch.as_tensor(np.asarray(positions, dtype=np.float64).reshape(-1, 3)))
        if velocities is not None:
            self.vel.copy_(torch.as_tensor(np.asarray(velocities, dtype=np.float64).reshape(-1, 3)))
        torch.cuda.synchronize(self.dev)
        check(lib().hmdp_gdd_plan(self.ctx.handle))

    def attach_nccl(self, unique_id: bytes):
        buf = ctypes.create_string_buffer(bytes(unique_id), 128)
        check(lib().hmdp_gdd_attach_nccl(self.ctx.handle, buf, self.world, self.rank))

    def attach_hub(self, hub):
        check(lib().hmdp_gdd_attach_hub(self.ctx.handle, hub))

    def attach_callback(self, fn):
        """fn(round, send_ptr, recv_ptr, stride, nbytes) -> None: move the first nbytes of
        packet send + q*stride to peer q's recv + rank*stride (device pointers)."""
        def trampoline(user, rnd, send, recv, stride, nbytes):
            try:
                fn(int(rnd), int(send), int(recv), int(stride), int(nbytes))
                return 0
            except Exception:  # surfaced as HMDP_RUNTIME_ERROR by the step
                import traceback

                traceback.print_exc()
                return 1

        self._cb = EXCHANGE_FN(trampoline)  # keep alive
        check(lib().hmdp_gdd_attach_callback(self.ctx.handle, ctypes.cast(self._cb, ctypes.c_void_p),
                                             None))

    def step(self, kind="eval", dt=0.001):
        k = {"eval": 0, "md": 1, "open": 2}[kind]
        check(lib().hmdp_gdd_step(self.ctx.handle, k, float(dt)))

    def roles(self):
        r = np.zeros(self.n, dtype=np.uint8)
        check(lib().hmdp_gdd_roles(self.ctx.handle, ptr(r)))
        return r

    def owned_forces(self):
        """(owned mask, forces [n][3] with only the owned rows meaningful)."""
        own = self.roles() == 1
        return own, self.f.cpu().numpy()

    def sync(self):
        c = np.zeros(3, dtype=np.int32)
        check(lib().hmdp_gdd_counts(self.ctx.handle, ptr(c)))  # synchronizes the rank's stream

    def energy_virial(self):
        self.sync()
        o = self.out.cpu().numpy()
        return float(o[0]), float(o[1]), o[2:11].reshape(3, 3)

    def halo_stats(self):
        v = (ctypes.c_longlong * 5)()
        check(lib().hmdp_gdd_halo_stats(self.ctx.handle, v))
        return {"capacity_rows": v[0], "rounds_per_step": v[1], "halo_bytes_per_step": v[2],
                "transferred_bytes_per_step": v[3], "peers": v[4]}

    def launches(self):
        v = ctypes.c_longlong()
        check(lib().hmdp_gdd_launches(self.ctx.handle, ctypes.byref(v)))
        return int(v.value)


class Hub:
    """In-process transport: ranks simulated as contexts on one GPU (hmdp_gdd_hub)."""

    def __init__(self, world):
        h = ctypes.c_void_p()
        check(lib().hmdp_gdd_hub_create(int(world), ctypes.byref(h)))
        self.handle = h

    def close(self):
        if self.handle:
            lib().hmdp_gdd_hub_destroy(self.handle)
            self.handle = None


def run_hub(engines, kind="eval", dt=0.001, steps=1):
    """Run `steps` steps of every simulated rank, one host thread per rank (the hub's
    exchange points are barriers across the threads)."""
    import threading

    errs = []

    def work(e):
        try:
            for _ in range(steps):
                e.step(kind, dt)
        except Exception as exc:  # re-raised below
            errs.append(exc)

    th = [threading.Thread(target=work, args=(e,)) for e in engines]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]


def gloo_exchange(engine: HaloDD, group=None):
    """A callback transport over torch.distributed (gloo; tests / dry runs): the
    packets go device -> host -> all_to_all -> host -> device."""
    import torch
    import torch.distributed as td

    cudart = lib()  # libcudart is a dependency of libhmdp: its symbols resolve here
    cudart.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
    W, R = engine.world, engine.rank

    def fn(rnd, send, recv, stride, nbytes):
        host = torch.empty(W * stride, dtype=torch.uint8)
        if cudart.cudaMemcpy(ctypes.c_void_p(host.data_ptr()), ctypes.c_void_p(send), W * stride, 2):
            raise RuntimeError("cudaMemcpy D2H failed")
        out = torch.empty_like(host)
        td.all_to_all_single(out, host, group=group)  # slot q of mine -> slot R of q's
        # only the first nbytes of every slot are meaningful; slot R stays as it was
        if cudart.cudaMemcpy(ctypes.c_void_p(recv), ctypes.c_void_p(out.data_ptr()), W * stride, 1):
            raise RuntimeError("cudaMemcpy H2D failed")
        # a pageable H2D cudaMemcpy may return before its DMA lands: complete it before
        # the engine's (non-blocking) stream unpacks
        if cudart.cudaDeviceSynchronize():
            raise RuntimeError("cudaDeviceSynchronize failed")

    engine.attach_callback(fn)
