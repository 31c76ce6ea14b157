"""FcOperator / OperatorCache mirror over the C ABI.

Same names, argument meaning and errors as the reference's
``fcs::fc`` namespace (include/fcs/fc_core.hpp:33-109): ``build_fc_operator``,
``OperatorCache.get``, ``FcOperator.derivative/filter/strong_filter``,
``fc_derivative``, ``apply_filter``. Arrays are numpy (host) or torch CUDA
tensors (device); host arrays go through ``fcsg_fc_lines_host`` (copies in the
call), device tensors through ``fcsg_fc_lines`` on the tensor's stream.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N

ALPHA = 23.025850929940457


@dataclass(frozen=True)
class FilterSpec:
    """include/fcs/fc_core.hpp:11-15"""

    alpha: float = ALPHA
    p: int = 7
    p_smear: int = 2


class FcOperator:
    """One FC-Gram operator for lines of ``n_points`` samples.

    ``degree=2`` is the reference operator; ``degree=4`` is the five-point
    variant named by BASELINE config 1 (not constructible by the reference).
    """

    def __init__(self, ctx: N.Context, n_points: int, n_cont: int = 25, filter: FilterSpec = FilterSpec(),
                 degree: int = 2):
        self.ctx = ctx
        op = C.c_int()
        ctx.check(ctx.lib.fcsg_operator(ctx.h, n_points, n_cont, degree, filter.alpha, filter.p,
                                        filter.p_smear, C.byref(op)))
        self.op_id = op.value
        ne, nm, per = C.c_int(), C.c_int(), C.c_double()
        ctx.check(ctx.lib.fcsg_operator_info(ctx.h, self.op_id, C.byref(ne), C.byref(nm), C.byref(per),
                                             None, None, None))
        self._n = n_points
        self._n_cont = n_cont
        self.degree = degree
        self._n_ext = ne.value
        self._n_modes = nm.value
        self._period = per.value
        self.filter_spec = filter

    def n_points(self):
        return self._n

    def n_cont(self):
        return self._n_cont

    def n_ext(self):
        return self._n_ext

    def n_modes(self):
        return self._n_modes

    def period(self):
        return self._period

    def _tables(self):
        nb = (self._n_cont - 1) * (self.degree + 1)
        blend = np.zeros(nb)
        fp = np.zeros(self._n_modes)
        sp = np.zeros(self._n_modes)
        self.ctx.check(self.ctx.lib.fcsg_operator_info(self.ctx.h, self.op_id, None, None, None,
                                                       N.dptr(blend), N.dptr(fp), N.dptr(sp)))
        return blend.reshape(self._n_cont - 1, self.degree + 1), fp, sp

    def blend_matrix(self):
        return self._tables()[0]

    def filter_profile(self):
        return self._tables()[1]

    def smear_profile(self):
        return self._tables()[2]

    # ---- batched application -------------------------------------------
    def apply(self, lines, mode: int, scale: float = 1.0, axis: int = -1, out=None):
        """Apply the operator along ``axis`` of a 2-D array (numpy on host or a
        torch CUDA tensor). mode: 1/2 derivative order, 3 filter, 4 smear."""
        if mode not in (N.D1, N.D2, N.FILTER, N.SMEAR):
            raise N.UsageError("fc_derivative: order must be 1 or 2")
        try:
            import torch

            is_tensor = isinstance(lines, torch.Tensor)
        except ImportError:  # pragma: no cover
            is_tensor = False
        if is_tensor:
            return self._apply_device(lines, mode, scale, axis, out)
        a = np.ascontiguousarray(lines, dtype=np.float64)
        if a.ndim == 1:
            a = a[None, :]
        if a.ndim != 2:
            raise N.UsageError("lines must be 1-D or 2-D")
        ax = axis % 2
        if a.shape[ax] != self._n:
            raise N.UsageError("fc_derivative: length mismatch")
        res = np.empty_like(a) if out is None else out
        R, Cn = a.shape
        if ax == 1:  # lines are rows
            ls, st, nl = Cn, 1, R
        else:  # lines are columns
            ls, st, nl = 1, Cn, Cn
        self.ctx.check(self.ctx.lib.fcsg_fc_lines_host(self.ctx.h, self.op_id, mode, N.dptr(a), ls, st,
                                                       N.dptr(res), ls, st, nl, scale))
        return res.reshape(np.shape(lines)) if np.ndim(lines) == 1 else res

    def _apply_device(self, t, mode, scale, axis, out):
        import torch

        if t.dtype != torch.float64 or not t.is_cuda or t.dim() != 2 or not t.is_contiguous():
            raise N.UsageError("device lines must be a contiguous 2-D float64 CUDA tensor")
        ax = axis % 2
        if t.shape[ax] != self._n:
            raise N.UsageError("fc_derivative: length mismatch")
        res = torch.empty_like(t) if out is None else out
        R, Cn = t.shape
        ls, st, nl = (Cn, 1, R) if ax == 1 else (1, Cn, Cn)
        stream = torch.cuda.current_stream(t.device).cuda_stream
        self.ctx.check(self.ctx.lib.fcsg_fc_lines(self.ctx.h, self.op_id, mode, C.c_void_p(t.data_ptr()), ls, st,
                                                  C.c_void_p(res.data_ptr()), ls, st, nl, scale,
                                                  C.c_void_p(stream)))
        return res

    def derivative(self, lines, order: int = 1, axis: int = -1):
        """FcOperator::derivative (unit span; callers rescale by inv_len)."""
        if order not in (1, 2):
            raise N.UsageError("fc_derivative: order must be 1 or 2")
        return self.apply(lines, order, 1.0, axis)

    def filter(self, lines, axis: int = -1):
        return self.apply(lines, N.FILTER, 1.0, axis)

    def strong_filter(self, lines, axis: int = -1):
        return self.apply(lines, N.SMEAR, 1.0, axis)


class OperatorCache:
    """Process-wide cache keyed by (n_points, n_cont, filter, degree)
    (src/fc_core.cpp:377-406); the context caches the device tables too."""

    def __init__(self, ctx: N.Context):
        self.ctx = ctx
        self._ops = {}

    def get(self, n_points: int, n_cont: int = 25, filter: FilterSpec = FilterSpec(), degree: int = 2):
        key = (n_points, n_cont, filter, degree)
        if key not in self._ops:
            self._ops[key] = FcOperator(self.ctx, n_points, n_cont, filter, degree)
        return self._ops[key]


def build_fc_operator(ctx, n_points, n_cont=25, filter_order=14, filter_alpha=ALPHA, degree=2):
    """src/fc_core.cpp:408-415"""
    if filter_order % 2 != 0:
        raise N.ConfigError("filter_order must be even (2p)")
    return FcOperator(ctx, n_points, n_cont, FilterSpec(filter_alpha, filter_order // 2), degree)


def fc_derivative(op: FcOperator, values, h: float, order: int = 1):
    """fc_derivative (src/fc_core.cpp:358-367): derivative rescaled by
    (1/(h (N-1)))^order."""
    if order not in (1, 2):
        raise N.UsageError("fc_derivative: order must be 1 or 2")
    v = np.asarray(values, dtype=np.float64)
    if v.shape[-1] != op.n_points():
        raise N.UsageError("fc_derivative: length mismatch")
    scale = (1.0 / (h * (op.n_points() - 1))) ** order
    return op.apply(v, order, scale)


def apply_filter(op: FcOperator, values):
    """apply_filter (src/fc_core.cpp:369-374)."""
    v = np.asarray(values, dtype=np.float64)
    if v.shape[-1] != op.n_points():
        raise N.UsageError("apply_filter: length mismatch")
    return op.filter(v)
