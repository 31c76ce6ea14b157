"""ctypes binding of the fcsg C ABI (include/fcsg.h).

The product loads ``paper_2506_19370_b200/lib/libfcsg.so`` (the nvcc sm_100a
build) and refuses to run without it or without a CUDA device: there is no
CPU fallback. ``load(emulate=True)`` returns the CPU emulation harness
(build/emu/libfcsg_emu.so) and exists only for the CPU unit tests of kernel
logic.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FCSG_LIB") or os.path.join(HERE, "lib", "libfcsg.so")  # override: A/B experiments
EMU_PATH = os.environ.get("FCSG_EMU_LIB") or os.path.join(os.path.dirname(HERE), "build", "emu", "libfcsg_emu.so")

# include/fcsg.h error kinds -> reference exception names (include/fcs/errors.hpp)
OK, CONFIG, USAGE, GEOMETRY, DECOMPOSITION, INVALID_STATE, CUDA_ERROR, OTHER = 0, 1, 2, 3, 4, 5, 8, 9
D1, D2, FILTER, SMEAR = 1, 2, 3, 4


class FcsgError(RuntimeError):
    kind = OTHER


class ConfigError(FcsgError):
    kind = CONFIG


class UsageError(FcsgError, ValueError):
    kind = USAGE


class GeometryError(FcsgError):
    kind = GEOMETRY


class DecompositionError(FcsgError):
    kind = DECOMPOSITION


class InvalidStateError(FcsgError):
    """Nonpositive density or pressure (include/fcs/errors.hpp:32-39)."""

    kind = INVALID_STATE

    def __init__(self, msg, patch=-1, subpatch=-1, i=-1, j=-1, t=0.0):
        super().__init__(msg)
        self.patch, self.subpatch, self.i, self.j, self.t = patch, subpatch, i, j, t


class CudaError(FcsgError):
    kind = CUDA_ERROR


_KINDS = {c.kind: c for c in (ConfigError, UsageError, GeometryError, DecompositionError,
                              InvalidStateError, CudaError)}

_libs: dict = {}

dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)
vp = C.c_void_p


def _declare(L):
    L.fcsg_create.argtypes = [C.c_int, C.POINTER(vp)]
    L.fcsg_destroy.argtypes = [vp]
    L.fcsg_last_error.argtypes = [vp, C.c_char_p, C.c_int, ip, ip, ip, ip, ip, dp]
    L.fcsg_is_cuda_build.argtypes = []
    L.fcsg_synchronize.argtypes = [vp]
    L.fcsg_device_alloc.argtypes = [vp, C.c_size_t, C.POINTER(vp)]
    L.fcsg_device_free.argtypes = [vp, vp]
    L.fcsg_memcpy_h2d.argtypes = [vp, vp, vp, C.c_size_t]
    L.fcsg_memcpy_d2h.argtypes = [vp, vp, vp, C.c_size_t]
    L.fcsg_operator.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, ip]
    L.fcsg_operator_info.argtypes = [vp, C.c_int, ip, ip, dp, dp, dp, dp]
    L.fcsg_fc_lines.argtypes = [vp, C.c_int, C.c_int, vp, C.c_long, C.c_long, vp, C.c_long, C.c_long,
                                C.c_long, C.c_double, vp]
    L.fcsg_fc_lines_host.argtypes = [vp, C.c_int, C.c_int, dp, C.c_long, C.c_long, dp, C.c_long, C.c_long,
                                     C.c_long, C.c_double]
    L.fcsg_engine_create.argtypes = [vp, vp, C.POINTER(vp)]
    L.fcsg_engine_destroy.argtypes = [vp]
    L.fcsg_engine_add_subpatch.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                           C.c_double, C.c_double, C.POINTER(C.c_uint8), dp, dp, dp, dp, dp, dp, dp,
                                           ip, dp, dp, ip]
    L.fcsg_engine_set_plan_interps.argtypes = [vp, C.c_int, C.c_long, ip, ip, ip, ip, ip, dp, dp, dp]
    L.fcsg_engine_set_halo_interps.argtypes = [vp, C.c_int, C.c_long, ip, ip, ip, dp, dp]
    L.fcsg_engine_set_plan.argtypes = [vp, C.c_long, ip, ip, ip, ip, C.c_long, ip, ip, ip, ip, dp]
    L.fcsg_engine_load_mlp.argtypes = [vp, C.c_char_p]
    L.fcsg_engine_finalize.argtypes = [vp]
    L.fcsg_engine_set_state.argtypes = [vp, C.c_int, dp]
    L.fcsg_engine_get_field.argtypes = [vp, C.c_int, C.c_char_p, C.c_int, dp]
    L.fcsg_engine_set_field.argtypes = [vp, C.c_int, C.c_char_p, C.c_int, dp]
    L.fcsg_engine_gradient.argtypes = [vp, C.c_int]
    L.fcsg_engine_run_host.argtypes = [vp, C.c_long, C.c_void_p, C.c_long, C.c_void_p, C.c_long, C.POINTER(C.c_long)]
    L.fcsg_engine_set_quadrature.argtypes = [vp, C.c_int, dp]
    L.fcsg_engine_integrals.argtypes = [vp, C.c_int, dp]
    L.fcsg_engine_sample.argtypes = [vp, C.c_long, ip, ip, ip, dp, dp, dp]
    L.fcsg_engine_finish_ic.argtypes = [vp]
    L.fcsg_engine_phase.argtypes = [vp, C.c_int, C.c_int]
    L.fcsg_engine_reduce_dt.argtypes = [vp, dp]
    L.fcsg_engine_advance.argtypes = [vp]
    L.fcsg_engine_run.argtypes = [vp, C.c_long, C.c_int, C.POINTER(C.c_long)]
    L.fcsg_engine_enqueue.argtypes = [vp, C.c_long]
    L.fcsg_engine_time.argtypes = [vp, dp, C.POINTER(C.c_long)]
    L.fcsg_engine_total_points.argtypes = [vp, C.POINTER(C.c_long)]
    L.fcsg_engine_stream.argtypes = [vp, C.POINTER(vp)]
    L.fcsg_engine_is_cartesian.argtypes = [vp, ip]
    L.fcsg_engine_set_state_bulk.argtypes = [vp, vp]
    L.fcsg_engine_get_state_bulk.argtypes = [vp, vp]
    L.fcsg_engine_set_halo.argtypes = [vp, C.c_long, ip, ip, C.c_long, C.c_long, ip, ip, C.c_long]
    L.fcsg_engine_halo_size.argtypes = [vp, C.c_int, C.POINTER(C.c_long)]
    L.fcsg_engine_pack.argtypes = [vp, C.c_int, vp]
    L.fcsg_engine_unpack.argtypes = [vp, C.c_int, vp]
    L.fcsg_engine_enqueue_part.argtypes = [vp, C.c_int, C.c_int]
    L.fcsg_engine_dtmin_ptr.argtypes = [vp, C.POINTER(vp)]
    L.fcsg_engine_check_error.argtypes = [vp]
    L.fcsg_engine_copy_dtmin.argtypes = [vp, vp, C.c_int]
    L.fcsg_engine_time_group.argtypes = [vp, C.c_int, C.c_int, dp]
    L.fcsg_engine_launches_per_step.argtypes = [vp, ip]
    L.fcsg_comm_unique_id.argtypes = [C.c_char_p]
    lp = C.POINTER(C.c_long)
    L.fcsg_engine_attach_comm.argtypes = [vp, C.c_int, C.c_int, C.c_char_p, C.c_int, ip, lp, lp, lp, lp]
    return L


def load(emulate: bool = False):
    key = "emu" if emulate else "cuda"
    if key in _libs:
        return _libs[key]
    path = EMU_PATH if emulate else LIB_PATH
    if not os.path.exists(path):
        raise ImportError(
            f"fcsg native library not built: {path} (run __graft_entry__.build() / "
            f"python paper_2506_19370_b200/build.py{' --emulate' if emulate else ''})")
    L = _declare(C.CDLL(path))
    _libs[key] = L
    return L


def dptr(a: np.ndarray):
    return a.ctypes.data_as(dp)


class Context:
    """fcsg_ctx: one CUDA device + stream, the operator cache, engines."""

    def __init__(self, device: int = 0, emulate: bool = False):
        self.lib = load(emulate)
        if not emulate:
            if self.lib.fcsg_is_cuda_build() != 1:
                raise ImportError("libfcsg.so is not a CUDA build")
            import torch

            if not torch.cuda.is_available():
                raise RuntimeError("fcsg requires a CUDA device (no CPU fallback)")
        self.emulate = emulate
        h = vp()
        rc = self.lib.fcsg_create(device, C.byref(h))
        if rc != OK:
            raise _KINDS.get(rc, FcsgError)(f"fcsg_create failed with code {rc}")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.lib.fcsg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc: int):
        if rc == OK:
            return
        buf = C.create_string_buffer(1024)
        kind, patch, sub, i, j = C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_int()
        t = C.c_double()
        self.lib.fcsg_last_error(self.h, buf, 1024, C.byref(kind), C.byref(patch), C.byref(sub),
                                 C.byref(i), C.byref(j), C.byref(t))
        msg = buf.value.decode()
        cls = _KINDS.get(kind.value, FcsgError)
        if cls is InvalidStateError:
            raise InvalidStateError(msg, patch.value, sub.value, i.value, j.value, t.value)
        raise cls(msg)

    def synchronize(self):
        self.check(self.lib.fcsg_synchronize(self.h))
