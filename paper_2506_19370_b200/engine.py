"""Engine mirror over the C ABI (fcs::run::Engine, include/fcs/runtime.hpp:79-127).

``Engine(dec, ic, cfg)`` uploads the init-time data of a decomposition (see
geometry.py), evaluates the initial condition, applies the ``apply_ic`` tail
(enforce_bc + one exchange) and then advances FC-SDNN supersteps on the GPU:
``run(n)``/``step()`` for whole steps, ``step_phase(phase, stage)`` /
``reduce_dt()`` / ``advance()`` for the reference's phase-level hooks, and
``get``/``set`` for fields in the reference's [nj][ni] layout.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass

import numpy as np

from . import _native as N
from . import geometry as G
from . import problems as P

HERE = os.path.dirname(os.path.abspath(__file__))
DEFAULT_WEIGHTS = os.path.join(HERE, "data", "fcnn_v1.bin")


class fcsg_engine_config(C.Structure):
    _fields_ = [("cfl", C.c_double), ("T", C.c_double), ("n_cont", C.c_int), ("filter_alpha", C.c_double),
                ("filter_p", C.c_int), ("filter_p_smear", C.c_int), ("visc_c", C.c_double * 4),
                ("abs_floor", C.c_double), ("smear_radius", C.c_int), ("debug_rhs", C.c_int),
                ("force_general", C.c_int), ("reference_order", C.c_int), ("classifier", C.c_int),
                ("classifier_window", C.c_int)]


@dataclass
class EngineConfig:
    """include/fcs/runtime.hpp:59-73 (fields used by the step)."""

    cfl: float = 0.5
    T: float = math.inf
    n_cont: int = 25
    filter_alpha: float = 23.025850929940457
    filter_p: int = 7
    filter_p_smear: int = 2
    visc_c: tuple = (1.5, 1.0, 0.25, 0.0)
    abs_floor: float = 1e-4
    smear_radius: int = 10
    max_steps: int = 10 ** 9
    weights: str = DEFAULT_WEIGHTS
    debug_rhs: bool = False
    force_general: bool = False  # never use the Cartesian (zero metric term) stage passes
    # accumulate the rhs in euler_rhs's own order (40 line derivatives per stage)
    # instead of the flux form div(mu grad w - f) (24; round-off-level difference)
    reference_order: bool = False
    # ClassifierConfig (include/fcs/viscosity.hpp:45-52): "ann" (the MLP, weights
    # above) or "fallback" (FC-spectrum decay over a window of classifier_window)
    classifier: str = "ann"
    classifier_window: int = 32


def _bc_arrays(d: G.SubData):
    ends = list(d.bc_row_lo) + list(d.bc_row_hi) + list(d.bc_col_lo) + list(d.bc_col_hi)
    kind = np.array([-1 if e is None else e[0] for e in ends], dtype=np.int32)
    state = np.zeros((len(ends), 4))
    press = np.ones(len(ends))
    for k, e in enumerate(ends):
        if e is not None:
            state[k] = e[1]
            press[k] = e[2]
    return kind, np.ascontiguousarray(state), press


class Engine:
    def __init__(self, ctx: N.Context, dec: G.Decomposition, ic=None, cfg: EngineConfig = EngineConfig(),
                 initial_states=None, rank_plan=None):
        """rank_plan (distributed.RankPlan): build only this rank's subpatches,
        with its halo lists and local plan (multi-GPU)."""
        self.ctx, self.dec, self.cfg = ctx, dec, cfg
        L = ctx.lib
        c = fcsg_engine_config(cfg.cfl, cfg.T, cfg.n_cont, cfg.filter_alpha, cfg.filter_p, cfg.filter_p_smear,
                               (C.c_double * 4)(*cfg.visc_c), cfg.abs_floor, cfg.smear_radius, int(cfg.debug_rhs),
                               int(cfg.force_general), int(cfg.reference_order),
                               {"ann": 0, "fallback": 1}[cfg.classifier], int(cfg.classifier_window))
        h = C.c_void_p()
        ctx.check(L.fcsg_engine_create(ctx.h, C.byref(c), C.byref(h)))
        self.h = h
        subs = dec.subs if rank_plan is None else [dec.subs[g] for g in rank_plan.local]
        self.subs = subs
        self.shapes = [(d.nj, d.ni) for d in subs]
        for d in subs:
            kind, state, press = _bc_arrays(d)
            arr = [np.ascontiguousarray(a, dtype=np.float64) for a in
                   (d.iq1x, d.iq2x, d.iq1y, d.iq2y, d.h_min, d.h_max, d.w_norm)]
            mask = np.ascontiguousarray(d.mask, dtype=np.uint8)
            sid = C.c_int()
            ctx.check(L.fcsg_engine_add_subpatch(
                h, d.patch, d.sp.i0, d.sp.j0, d.ni, d.nj, getattr(d, "cut_i", 0), getattr(d, "cut_j", 0), d.h1, d.h2,
                mask.ctypes.data_as(C.POINTER(C.c_uint8)),
                *[N.dptr(a) for a in arr], kind.ctypes.data_as(N.ip), N.dptr(state), N.dptr(press), C.byref(sid)))
        pl = dec.plan if rank_plan is None else rank_plan.plan
        if rank_plan is not None:
            es, el = rank_plan.flat_e_send()
            ms, ml = rank_plan.flat_mu_send()
            nre = sum(rank_plan.e_recv.values())
            nrm = sum(rank_plan.mu_recv.values())
            ctx.check(L.fcsg_engine_set_halo(h, len(es), es.ctypes.data_as(N.ip), el.ctypes.data_as(N.ip), nre,
                                             len(ms), ms.ctypes.data_as(N.ip), ml.ctypes.data_as(N.ip), nrm))
            for which, lst in ((0, rank_plan.e_interps), (1, rank_plan.mu_interps)):
                if not lst:
                    continue
                ints = [np.ascontiguousarray([t[k] for t in lst], dtype=np.int32) for k in range(3)]
                wx = np.ascontiguousarray(np.stack([t[3] for t in lst]), dtype=np.float64)
                wy = np.ascontiguousarray(np.stack([t[4] for t in lst]), dtype=np.float64)
                ctx.check(L.fcsg_engine_set_halo_interps(h, which, len(lst), *[x.ctypes.data_as(N.ip) for x in ints],
                                                         N.dptr(wx), N.dptr(wy)))
        keep = [np.ascontiguousarray(a, dtype=np.int32) for a in
                (pl.sol_dst_sub, pl.sol_dst, pl.sol_src_sub, pl.sol_src, pl.v_dst_sub, pl.v_dst, pl.v_src_sub,
                 pl.v_src)]
        vw = np.ascontiguousarray(pl.v_w, dtype=np.float64)
        ctx.check(L.fcsg_engine_set_plan(h, len(keep[0]), *[k.ctypes.data_as(N.ip) for k in keep[:4]],
                                         len(keep[4]), *[k.ctypes.data_as(N.ip) for k in keep[4:]], N.dptr(vw)))
        for which, ip_ in ((0, getattr(pl, "sol_interps", None)), (1, getattr(pl, "visc_interps", None))):
            if ip_ is None or len(ip_["dst"]) == 0:
                continue
            ints = [np.ascontiguousarray(ip_[k], dtype=np.int32) for k in ("dst_sub", "dst", "src_sub", "si0", "sj0")]
            wx = np.ascontiguousarray(ip_["wx"], dtype=np.float64)
            wy = np.ascontiguousarray(ip_["wy"], dtype=np.float64)
            w = np.ascontiguousarray(ip_.get("w", np.ones(len(ints[0]))), dtype=np.float64)
            ctx.check(L.fcsg_engine_set_plan_interps(h, which, len(ints[0]), *[a.ctypes.data_as(N.ip) for a in ints],
                                                     N.dptr(wx), N.dptr(wy), N.dptr(w)))
        if cfg.classifier == "ann":
            ctx.check(L.fcsg_engine_load_mlp(h, cfg.weights.encode()))
        ctx.check(L.fcsg_engine_finalize(h))
        if initial_states is None and ic is not None and rank_plan is None:
            if hasattr(dec, "initial_state"):  # multipatch.MultiPatchDecomposition
                initial_states = [dec.initial_state(ic, k) for k in range(len(dec.subs))]
            else:
                initial_states = [P.initial_state(dec, ic, k) for k in range(len(dec.subs))]
        if initial_states is not None:
            for k, e in enumerate(initial_states):
                self.set_state(k, e)
            self.finish_ic()

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.fcsg_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- state access --------------------------------------------------
    def set_state(self, sub, e):
        e = np.ascontiguousarray(e, dtype=np.float64)
        self.ctx.check(self.ctx.lib.fcsg_engine_set_state(self.h, sub, N.dptr(e)))

    def _host_buffer(self, a, n, what, writable=False):
        """(pointer, keep-alive) of a host float64 buffer of at least n
        doubles: a numpy array or a CPU torch tensor, C-contiguous. Inputs of
        another dtype or layout are converted into a copy that the caller
        keeps alive across the C call; outputs must already be float64,
        contiguous and large enough (the C call writes n doubles)."""
        if hasattr(a, "data_ptr"):  # torch tensor
            import torch

            if a.device.type != "cpu":
                raise ValueError(f"{what}: host buffer expected, got a tensor on {a.device}")
            if a.dtype != torch.float64 or not a.is_contiguous():
                if writable:
                    raise ValueError(f"{what}: output must be a contiguous float64 tensor")
                a = a.to(torch.float64).contiguous()
            if a.numel() < n:
                raise ValueError(f"{what}: {a.numel()} doubles, {n} needed")
            return a.data_ptr(), a
        arr = np.asarray(a)
        if arr.dtype != np.float64 or not arr.flags.c_contiguous:
            if writable:
                raise ValueError(f"{what}: output must be a C-contiguous float64 array")
            arr = np.ascontiguousarray(arr, dtype=np.float64)
        if writable and not arr.flags.writeable:
            raise ValueError(f"{what}: output array is read-only")
        if arr.size < n:
            raise ValueError(f"{what}: {arr.size} doubles, {n} needed")
        return arr.ctypes.data, arr

    def set_state_bulk(self, e):
        """all subpatches, [4][sum of points] (per component the subpatches in
        id order, each [nj][ni]; [4][S][nj][ni] for one shape); ``e`` may be a numpy array or a
        (pinned) CPU torch tensor"""
        ptr, keep = self._host_buffer(e, 4 * self.total_points(), "set_state_bulk")
        self.ctx.check(self.ctx.lib.fcsg_engine_set_state_bulk(self.h, C.c_void_p(ptr)))
        del keep

    def run_host(self, state_in, state_out, steps=1, in_stride=0, out_stride=0):
        """steps supersteps with host I/O per step (fcsg_engine_run_host):
        step k reads its state from state_in (+ k in_stride doubles) and
        leaves its result in state_out (+ k out_stride); uploads/downloads
        overlap the neighbouring steps' kernels (pinned buffers)."""
        n = 4 * self.total_points()
        if steps < 0 or in_stride < 0 or out_stride < 0:
            raise ValueError("run_host: steps and strides must be >= 0")
        last = max(steps - 1, 0)
        pi, keep_i = self._host_buffer(state_in, n + last * in_stride, "run_host input")
        po, keep_o = self._host_buffer(state_out, n + last * out_stride, "run_host output", writable=True)
        done = C.c_long()
        self.ctx.check(self.ctx.lib.fcsg_engine_run_host(self.h, steps, C.c_void_p(pi), in_stride, C.c_void_p(po),
                                                         out_stride, C.byref(done)))
        del keep_i, keep_o
        return done.value

    def get_state_bulk(self, out):
        ptr, _ = self._host_buffer(out, 4 * self.total_points(), "get_state_bulk", writable=True)
        self.ctx.check(self.ctx.lib.fcsg_engine_get_state_bulk(self.h, C.c_void_p(ptr)))
        return out

    def get(self, sub, name, comp=0):
        out = np.empty(self.shapes[sub])
        self.ctx.check(self.ctx.lib.fcsg_engine_get_field(self.h, sub, name.encode(), comp, N.dptr(out)))
        return out

    def get_state(self, sub, name="e"):
        return np.stack([self.get(sub, name, c) for c in range(4)])

    # -- diagnostics (fcsg_engine_gradient / set_quadrature / integrals /
    #    sample; diagnostics.py builds on these) -----------------------------
    def gradient(self, comp=0):
        """|grad e_comp| into the "grad" field (FC derivatives on the device)"""
        self.ctx.check(self.ctx.lib.fcsg_engine_gradient(self.h, int(comp)))

    def set_quadrature(self, sub, wq):
        a = np.ascontiguousarray(wq, dtype=np.float64)
        if a.shape != tuple(self.shapes[sub]):
            raise ValueError("quadrature weights must have the subpatch's shape")
        self.ctx.check(self.ctx.lib.fcsg_engine_set_quadrature(self.h, sub, N.dptr(a)))

    def integrals(self, comp):
        """per subpatch h1 h2 sum wq v (v = 1 for comp = -1, else e_comp)"""
        out = np.zeros(len(self.shapes))
        self.ctx.check(self.ctx.lib.fcsg_engine_integrals(self.h, int(comp), N.dptr(out)))
        return out

    def sample(self, sub, il, jl, fu, fv):
        """bilinear samples of "grad" at (sub, il, jl, fu, fv); sub < 0 -> 0"""
        ints = [np.ascontiguousarray(a, dtype=np.int32) for a in (sub, il, jl)]
        dbl = [np.ascontiguousarray(a, dtype=np.float64) for a in (fu, fv)]
        out = np.zeros(ints[0].size)
        self.ctx.check(self.ctx.lib.fcsg_engine_sample(self.h, ints[0].size, *[a.ctypes.data_as(N.ip) for a in ints],
                                                       N.dptr(dbl[0]), N.dptr(dbl[1]), N.dptr(out)))
        return out

    def set(self, sub, name, arr, comp=0):
        a = np.ascontiguousarray(arr, dtype=np.float64)
        self.ctx.check(self.ctx.lib.fcsg_engine_set_field(self.h, sub, name.encode(), comp, N.dptr(a)))

    def finish_ic(self):
        self.ctx.check(self.ctx.lib.fcsg_engine_finish_ic(self.h))

    # ---- stepping --------------------------------------------------------
    def step_phase(self, phase, stage=0):
        self.ctx.check(self.ctx.lib.fcsg_engine_phase(self.h, phase, stage))

    def reduce_dt(self):
        dt = C.c_double()
        self.ctx.check(self.ctx.lib.fcsg_engine_reduce_dt(self.h, C.byref(dt)))
        return dt.value

    def advance(self):
        self.ctx.check(self.ctx.lib.fcsg_engine_advance(self.h))

    def step_by_phases(self):
        """One superstep through the phase hooks, in Engine::run order."""
        self.step_phase(0)
        self.step_phase(1)
        self.step_phase(2)
        self.reduce_dt()
        for s in range(5):
            self.step_phase(3, s)
            self.step_phase(6)
        self.advance()

    def run(self, n_steps, use_graph=True):
        done = C.c_long()
        self.ctx.check(self.ctx.lib.fcsg_engine_run(self.h, n_steps, int(use_graph), C.byref(done)))
        return done.value

    def enqueue(self, n_steps):
        self.ctx.check(self.ctx.lib.fcsg_engine_enqueue(self.h, n_steps))

    def time(self):
        t, st = C.c_double(), C.c_long()
        self.ctx.check(self.ctx.lib.fcsg_engine_time(self.h, C.byref(t), C.byref(st)))
        return t.value, st.value

    def is_cartesian(self):
        y = C.c_int()
        self.ctx.check(self.ctx.lib.fcsg_engine_is_cartesian(self.h, C.byref(y)))
        return bool(y.value)

    def total_points(self):
        n = C.c_long()
        self.ctx.check(self.ctx.lib.fcsg_engine_total_points(self.h, C.byref(n)))
        return n.value

    # ---- multi-rank hooks (distributed.py) ---------------------------------
    def halo_size(self, which):
        n = C.c_long()
        self.ctx.check(self.ctx.lib.fcsg_engine_halo_size(self.h, which, C.byref(n)))
        return n.value

    def pack(self, which, tensor):
        self.ctx.check(self.ctx.lib.fcsg_engine_pack(self.h, which, C.c_void_p(tensor.data_ptr())))

    def unpack(self, which, tensor):
        self.ctx.check(self.ctx.lib.fcsg_engine_unpack(self.h, which, C.c_void_p(tensor.data_ptr())))

    def attach_comm(self, world, rank, comm_id: bytes, peers, e_send, e_recv, mu_send, mu_recv):
        """device-ordered transport (fcsg_engine_attach_comm): from now on
        every superstep this engine enqueues carries its own halos and dt
        all-reduce (NCCL on the GPU)"""
        n = len(peers)
        ints = np.ascontiguousarray(peers, dtype=np.int32)
        cnt = [np.ascontiguousarray(c, dtype=np.int64) for c in (e_send, e_recv, mu_send, mu_recv)]
        if any(len(c) != n for c in cnt):
            raise ValueError("per-peer counts must match the peer list")
        lp = C.POINTER(C.c_long)
        self._comm_keep = (ints, cnt)
        self.ctx.check(self.ctx.lib.fcsg_engine_attach_comm(self.h, world, rank, C.c_char_p(comm_id), n,
                                                            ints.ctypes.data_as(N.ip),
                                                            *[c.ctypes.data_as(lp) for c in cnt]))

    def enqueue_part(self, part, stage=0):
        self.ctx.check(self.ctx.lib.fcsg_engine_enqueue_part(self.h, part, stage))

    def copy_dtmin(self, tensor, to_engine):
        self.ctx.check(self.ctx.lib.fcsg_engine_copy_dtmin(self.h, C.c_void_p(tensor.data_ptr()), int(to_engine)))

    def check_error(self):
        self.ctx.check(self.ctx.lib.fcsg_engine_check_error(self.h))

    GROUPS = ("viscosity", "blend", "filter", "pass_a", "pass_b", "pass_c", "bc", "exchange")

    def time_group(self, which, reps=10):
        """average device ms of one launch of a kernel group (profiling hook)"""
        idx = self.GROUPS.index(which) if isinstance(which, str) else which
        ms = C.c_double()
        self.ctx.check(self.ctx.lib.fcsg_engine_time_group(self.h, idx, reps, C.byref(ms)))
        return ms.value

    def launches_per_step(self):
        n = C.c_int()
        self.ctx.check(self.ctx.lib.fcsg_engine_launches_per_step(self.h, C.byref(n)))
        return n.value

    def stream(self):
        s = C.c_void_p()
        self.ctx.check(self.ctx.lib.fcsg_engine_stream(self.h, C.byref(s)))
        return s.value
