"""Multi-GPU FC-SDNN superstep: one process per GPU, subpatches sharded in
contiguous spatial blocks.

The reference runs all subpatches in one process: worker threads own
subpatches round-robin (``assign_ranks``, src/runtime.cpp:16-23) and read
donor subpatches directly after a barrier (phase 1 blend,
src/runtime.cpp:352-371; phase 6 exchange, :433-454; the dt minimum,
:492-497). Here every rank owns a contiguous block of subpatches (so only
block edges cross ranks) and:

* per stage, fringe copies whose donor lives on another rank are packed on
  the donor rank into one device buffer per peer (``fcsg_engine_pack``),
  moved with point-to-point send/recv, and unpacked into halo slots on the
  recipient (``fcsg_engine_unpack``) before the exchange kernel runs; a 6x6
  interpolation whose donor stencil lives on another rank is evaluated there
  while packing (the donor has the stencil, the recipient only needs the
  value) and arrives as a halo value;
* per step, the mu_hat values the viscosity blend reads across ranks move
  the same way before the blend;
* dt_local's minimum is an all-reduce(MIN) of one int64 (the bit pattern of
  a positive double, so the reduction is exact).

Every per-subpatch computation is local and min is exact, so the result is
bitwise independent of the number of ranks (interpolations are evaluated
with the same arithmetic on whichever rank holds the donor).

Two transports:

* ``"native"`` (default): the engine's own (``fcsg_engine_attach_comm``,
  csrc/comm.cpp). Pack, grouped ncclSend/ncclRecv to the neighbour ranks,
  unpack and ncclAllReduce(MIN) are enqueued on the engine stream inside the
  superstep -- no host synchronisation -- so a steady multi-rank superstep is
  one CUDA graph replay. torch.distributed only broadcasts the NCCL unique
  id. In the CPU tests the emulation build runs the same engine code over
  shared-memory mailboxes.
* ``"torch"``: the caller-driven parts (``fcsg_engine_enqueue_part`` +
  ``pack``/``unpack``) with torch.distributed point-to-point between them
  (gloo in the CPU tests; with host staging when gloo carries CUDA ranks).
  Kept as the reference for the native path: both must agree bitwise.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import geometry as G


def partition_tiles(dec: G.Decomposition, world: int) -> np.ndarray:
    """Owner rank of every subpatch: the (r x s) tile grid of a subdivide_Q
    patch is cut into a (px x py) grid of equal contiguous blocks, px*py =
    world, px chosen to keep blocks as square as the tiling allows."""
    p = dec.patches[0]
    i0s = sorted({sp.i0 for sp in p.subpatches})
    j0s = sorted({sp.j0 for sp in p.subpatches})
    r, s = len(i0s), len(j0s)
    best = None
    for px in range(1, world + 1):
        if world % px or r % px or s % (world // px):
            continue
        py = world // px
        score = abs(np.log((r / px) / (s / py)))
        if best is None or score < best[0]:
            best = (score, px, py)
    if best is None:
        raise ValueError(f"cannot split a {r}x{s} tiling over {world} ranks")
    _, px, py = best
    owner = np.zeros(len(dec.subs), dtype=np.int64)
    for g, d in enumerate(dec.subs):
        a, b = i0s.index(d.sp.i0), j0s.index(d.sp.j0)
        owner[g] = (a // (r // px)) + px * (b // (s // py))
    return owner


@dataclass
class RankPlan:
    """This rank's share of the global CommPlan."""

    rank: int
    world: int
    owner: np.ndarray
    local: list  # global subpatch ids owned, in local order
    plan: G.Plan  # local subpatch ids; src_sub == -1 addresses halo slots
    e_send: dict = field(default_factory=dict)  # peer -> (local sub ids, local point index), in wire order
    e_recv: dict = field(default_factory=dict)  # peer -> count
    mu_send: dict = field(default_factory=dict)
    mu_recv: dict = field(default_factory=dict)
    # interpolations this rank evaluates for other ranks: send entries with
    # point index -1 - m refer to entry m (local donor sub, si0, sj0, wx, wy)
    e_interps: list = field(default_factory=list)
    mu_interps: list = field(default_factory=list)

    def peers(self):
        return sorted(set(self.e_send) | set(self.e_recv) | set(self.mu_send) | set(self.mu_recv))

    @staticmethod
    def _flat(send):
        subs = [np.asarray(send[p][0], dtype=np.int32) for p in sorted(send)]
        locs = [np.asarray(send[p][1], dtype=np.int32) for p in sorted(send)]
        z = np.zeros(0, dtype=np.int32)
        return (np.concatenate(subs) if subs else z), (np.concatenate(locs) if locs else z)

    def flat_e_send(self):
        return self._flat(self.e_send)

    def flat_mu_send(self):
        return self._flat(self.mu_send)


def split_plan(dec, owner: np.ndarray, rank: int, world: int) -> RankPlan:
    """Split the global plan (every rank holds it) into this rank's local
    entries and its send/recv lists. Both sides walk the global entry lists
    in the same order (copies, then interpolations), so the k-th value a peer
    sends is the k-th it expects."""
    local = [g for g in range(len(dec.subs)) if owner[g] == rank]
    g2l = {g: l for l, g in enumerate(local)}
    pl = dec.plan
    a = lambda x, dt=np.int32: np.asarray(x, dtype=dt)  # noqa: E731

    class Wire:
        def __init__(self):
            self.send, self.recv, self.interps = {}, {}, []
            self.pending = []  # (list, position, peer, j): halo slot fixed up once the counts are known

        def slot(self, peer, lst, pos):
            j = self.recv.get(peer, 0)
            self.recv[peer] = j + 1
            self.pending.append((lst, pos, peer, j))

        def resolve(self):
            base, acc = {}, 0
            for peer in sorted(self.recv):
                base[peer] = acc
                acc += self.recv[peer]
            for lst, pos, peer, j in self.pending:
                lst[pos] = base[peer] + j

    def split(wire, dst_sub, dst, src_sub, src, w, sint, visc):
        cp = {k: [] for k in ("dst_sub", "dst", "src_sub", "src", "w")}
        it = {k: [] for k in ("dst_sub", "dst", "src_sub", "si0", "sj0", "wx", "wy", "w")}
        for k in range(len(dst)):
            d_own, s_own = owner[dst_sub[k]], owner[src_sub[k]]
            if d_own == rank:
                cp["dst_sub"].append(g2l[dst_sub[k]])
                cp["dst"].append(dst[k])
                if w is not None:
                    cp["w"].append(w[k])
                if s_own == rank:
                    cp["src_sub"].append(g2l[src_sub[k]])
                    cp["src"].append(src[k])
                else:
                    cp["src_sub"].append(-1)
                    cp["src"].append(-1)
                    wire.slot(s_own, cp["src"], len(cp["src"]) - 1)
            elif s_own == rank:
                lst = wire.send.setdefault(d_own, ([], []))
                lst[0].append(g2l[src_sub[k]])
                lst[1].append(src[k])
        if sint is not None:
            for k in range(len(sint["dst"])):
                ds, ss = int(sint["dst_sub"][k]), int(sint["src_sub"][k])
                d_own, s_own = owner[ds], owner[ss]
                if d_own == rank and s_own == rank:
                    it["dst_sub"].append(g2l[ds])
                    it["dst"].append(sint["dst"][k])
                    it["src_sub"].append(g2l[ss])
                    it["si0"].append(sint["si0"][k])
                    it["sj0"].append(sint["sj0"][k])
                    it["wx"].append(sint["wx"][k])
                    it["wy"].append(sint["wy"][k])
                    if visc:
                        it["w"].append(sint["w"][k])
                elif d_own == rank:
                    # evaluated on the donor's rank: a value in a halo slot
                    if visc:
                        it["dst_sub"].append(g2l[ds])
                        it["dst"].append(sint["dst"][k])
                        it["src_sub"].append(-1)
                        it["si0"].append(-1)
                        it["sj0"].append(0)
                        it["wx"].append(np.zeros(6))
                        it["wy"].append(np.zeros(6))
                        it["w"].append(sint["w"][k])
                        wire.slot(s_own, it["si0"], len(it["si0"]) - 1)
                    else:
                        cp["dst_sub"].append(g2l[ds])
                        cp["dst"].append(sint["dst"][k])
                        cp["src_sub"].append(-1)
                        cp["src"].append(-1)
                        wire.slot(s_own, cp["src"], len(cp["src"]) - 1)
                elif s_own == rank:
                    m = len(wire.interps)
                    wire.interps.append((g2l[ss], int(sint["si0"][k]), int(sint["sj0"][k]), np.asarray(sint["wx"][k]),
                                         np.asarray(sint["wy"][k])))
                    lst = wire.send.setdefault(d_own, ([], []))
                    lst[0].append(g2l[ss])
                    lst[1].append(-1 - m)
        wire.resolve()
        itd = None
        if sint is not None:
            itd = {k: a(v) for k, v in it.items() if k not in ("wx", "wy", "w")}
            itd["wx"] = np.asarray(it["wx"], dtype=np.float64).reshape(-1, 6)
            itd["wy"] = np.asarray(it["wy"], dtype=np.float64).reshape(-1, 6)
            if visc:
                itd["w"] = np.asarray(it["w"], dtype=np.float64)
        return cp, itd

    we, wm = Wire(), Wire()
    sol, sol_i = split(we, pl.sol_dst_sub, pl.sol_dst, pl.sol_src_sub, pl.sol_src, None,
                       getattr(pl, "sol_interps", None), False)
    vis, vis_i = split(wm, pl.v_dst_sub, pl.v_dst, pl.v_src_sub, pl.v_src, pl.v_w,
                       getattr(pl, "visc_interps", None), True)
    plan = G.Plan(a(sol["dst_sub"]), a(sol["dst"]), a(sol["src_sub"]), a(sol["src"]), a(vis["dst_sub"]),
                  a(vis["dst"]), a(vis["src_sub"]), a(vis["src"]), a(vis["w"], np.float64),
                  sol_interps=sol_i, visc_interps=vis_i)
    return RankPlan(rank, world, owner, local, plan, we.send, we.recv, wm.send, wm.recv, we.interps, wm.interps)


def partition_subpatches(dec, world: int) -> np.ndarray:
    """Owner rank of every subpatch of a general decomposition: consecutive
    global ids (patch by patch, so neighbours mostly share a rank) in
    contiguous runs of about equal point counts."""
    pts = np.array([int((d.mask != 0).sum()) for d in dec.subs], dtype=np.float64)
    c = np.cumsum(pts) - 0.5 * pts
    owner = np.minimum((c / pts.sum() * world).astype(np.int64), world - 1)
    if len(set(owner.tolist())) != world:
        raise ValueError(f"cannot split {len(dec.subs)} subpatches over {world} ranks")
    return owner


class DistributedEngine:
    """One rank of a multi-GPU superstep (see the module docstring)."""

    def __init__(self, ctx, dec, rank_plan: RankPlan, ic=None, cfg=None, initial_states=None, group=None,
                 transport="native"):
        import torch

        from . import engine as EN
        from . import problems as P

        if transport not in ("native", "torch"):
            raise ValueError(f"unknown transport {transport!r}")
        self.rp = rank_plan
        self.group = group
        self.transport = transport
        self.device = torch.device("cpu") if ctx.emulate else torch.device("cuda", torch.cuda.current_device())
        cfg = cfg or EN.EngineConfig()
        if initial_states is None and ic is not None:
            if hasattr(dec, "initial_state"):  # multipatch.MultiPatchDecomposition
                initial_states = [dec.initial_state(ic, g) for g in rank_plan.local]
            else:
                initial_states = [P.initial_state(dec, ic, g) for g in rank_plan.local]
        self.E = EN.Engine(ctx, dec, cfg=cfg, rank_plan=rank_plan, initial_states=None)
        self.torch = torch
        # wire buffers (state: [k][4], mu: [k]) and per-peer slices
        self.n = {w: self.E.halo_size(w) for w in range(4)}
        f = lambda n: torch.zeros(max(n, 1), dtype=torch.float64, device=self.device)
        self.buf = {"e_send": f(4 * self.n[0]), "e_recv": f(4 * self.n[1]), "mu_send": f(self.n[2]),
                    "mu_recv": f(self.n[3])}
        self.dtmin = torch.zeros(1, dtype=torch.int64, device=self.device)
        # host staging for gloo carrying CUDA tensors (gloo moves host memory)
        self.stage = None
        if self.device.type == "cuda" and transport == "torch":
            import torch.distributed as dist

            if dist.get_backend(group) == "gloo":
                self.stage = {k: torch.zeros_like(v, device="cpu") for k, v in self.buf.items()}
                self.stage["dtmin"] = torch.zeros(1, dtype=torch.int64)
        if transport == "native":
            self._attach_native()
        if initial_states is not None:
            for l, e in enumerate(initial_states):
                self.E.set_state(l, e)
            self.finish_ic()

    def _attach_native(self):
        import ctypes as C

        import torch.distributed as dist

        lib = self.E.ctx.lib
        obj = [None]
        if self.rp.rank == 0:
            idb = C.create_string_buffer(128)
            rc = lib.fcsg_comm_unique_id(idb)
            if rc != 0:
                raise RuntimeError(f"fcsg_comm_unique_id failed ({rc})")
            obj = [idb.raw]
        dist.broadcast_object_list(obj, src=0, group=self.group)
        peers = self.rp.peers()

        def cnt(d):
            return [(d[p] if isinstance(d[p], int) else len(d[p][0])) if p in d else 0 for p in peers]

        self.E.attach_comm(self.rp.world, self.rp.rank, obj[0], peers, cnt(self.rp.e_send), cnt(self.rp.e_recv),
                           cnt(self.rp.mu_send), cnt(self.rp.mu_recv))

    def _slices(self, counts, width):
        out, acc = {}, 0
        for peer in sorted(counts):
            n = counts[peer] if isinstance(counts[peer], int) else len(counts[peer][0])
            out[peer] = (acc * width, (acc + n) * width)
            acc += n
        return out

    def _halo(self, which):
        import torch.distributed as dist

        name = "e" if which == 0 else "mu"
        width = 4 if which == 0 else 1
        send, recv = self.buf[name + "_send"], self.buf[name + "_recv"]
        sends = self.rp.e_send if which == 0 else self.rp.mu_send
        recvs = self.rp.e_recv if which == 0 else self.rp.mu_recv
        self.E.pack(which, send)
        self._sync_engine()
        dsend, drecv = send, recv
        if self.stage is not None:  # gloo: through host memory
            send, recv = self.stage[name + "_send"], self.stage[name + "_recv"]
            send.copy_(dsend)
        ops = []
        for peer, (a, b) in self._slices(sends, width).items():
            ops.append(dist.P2POp(dist.isend, send[a:b], peer, group=self.group))
        for peer, (a, b) in self._slices(recvs, width).items():
            ops.append(dist.P2POp(dist.irecv, recv[a:b], peer, group=self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
            if self.device.type == "cuda":  # NCCL completes on torch's stream; the engine has its own
                self.torch.cuda.current_stream().synchronize()
        if self.stage is not None:
            drecv.copy_(recv)
            self.torch.cuda.current_stream().synchronize()
        self.E.unpack(which, drecv)

    def _sync_engine(self):
        if self.device.type == "cuda":
            self.torch.cuda.ExternalStream(self.E.stream()).synchronize()

    def _allreduce_dtmin(self):
        import torch.distributed as dist

        self.E.copy_dtmin(self.dtmin, to_engine=False)
        self._sync_engine()
        t = self.dtmin
        if self.stage is not None:
            t = self.stage["dtmin"]
            t.copy_(self.dtmin)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
        if self.stage is not None:
            self.dtmin.copy_(t)
        if self.device.type == "cuda":
            self.torch.cuda.current_stream().synchronize()
        self.E.copy_dtmin(self.dtmin, to_engine=True)

    def finish_ic(self):
        """apply_ic tail across ranks: BCs, then one exchange (src/runtime.cpp:284-286)."""
        if self.transport == "native":
            self.E.finish_ic()
            return
        self.E.enqueue_part(-1)  # BC on every local subpatch
        self._halo(0)
        self.E.enqueue_part(4)
        self._sync_engine()

    def step(self):
        """One superstep in Engine::run order (src/runtime.cpp:486-511)."""
        if self.transport == "native":
            self.E.enqueue(1)
            return
        E = self.E
        E.enqueue_part(0)
        self._halo(1)
        E.enqueue_part(1)
        self._allreduce_dtmin()
        E.enqueue_part(2)
        for s in range(5):
            E.enqueue_part(3, s)
            self._halo(0)
            E.enqueue_part(4)
        E.enqueue_part(5)

    def run(self, n, use_graph=True):
        """n supersteps; native: the engine's own loop (one CUDA graph replay
        per steady step), torch: part by part with the transfers between"""
        if self.transport == "native":
            return self.E.run(n, use_graph=use_graph)
        for _ in range(n):
            self.step()
        self.E.check_error()
        return n

    def enqueue(self, n):
        """n supersteps enqueued without waiting (native transport)"""
        if self.transport != "native":
            raise RuntimeError("enqueue needs the native transport")
        self.E.enqueue(n)
