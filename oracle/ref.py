"""ctypes binding of oracle/_ref/libfcsref.so -- TEST INFRASTRUCTURE ONLY.

The library is the UNMODIFIED reference (/root/reference/proj/src) compiled by
oracle/Makefile against the shims in oracle/shims, plus oracle/ref_export.cpp.
It is built in this container (where /root/reference exists) and travels to
the GPU box inside the gpurun snapshot; nothing here reads /root/reference.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libfcsref.so")

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB_PATH)
        dp = C.POINTER(C.c_double)
        ip = C.POINTER(C.c_int)
        L.ref_last_error.restype = C.c_char_p
        L.ref_last_error.argtypes = [ip]
        L.ref_blend_matrix.argtypes = [C.c_int, dp]
        L.ref_fc_info.argtypes = [C.c_int, C.c_int, ip, dp, dp, dp]
        L.ref_fc_apply.argtypes = [C.c_int, C.c_int, C.c_int, dp, C.c_long, C.c_int, C.c_int, dp, C.c_int]
        L.ref_fc_evaluate.argtypes = [C.c_int, C.c_int, dp, C.c_int, dp, dp]
        L.ref_train_classifier.argtypes = [C.c_char_p, dp]
        L.ref_mlp_forward.argtypes = [C.c_char_p, C.c_int, dp, dp, ip]
        L.ref_classify_line.argtypes = [C.c_char_p, C.c_int, dp, ip]
        L.ref_engine_integrals.argtypes = [C.c_void_p, dp, dp]
        L.ref_engine_raster.argtypes = [C.c_void_p, C.c_int, C.c_int, dp, dp]
        L.ref_write_schlieren_pgm.argtypes = [C.c_int, C.c_int, dp, dp, C.c_double, C.c_char_p]
        L.ref_fit_shock_angle.argtypes = [C.c_int, C.c_int, dp, dp, C.c_double, C.c_double, C.c_double, C.c_double,
                                          dp]
        L.ref_engine_write_csv.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_engine_mesh_json.argtypes = [C.c_void_p, C.c_char_p, C.c_long, C.POINTER(C.c_long)]
        L.ref_mesh_roundtrip.argtypes = [C.c_char_p, C.c_char_p, C.c_long, C.POINTER(C.c_long)]
        L.ref_classify_line_fallback.argtypes = [C.c_int, C.c_double, C.c_int, dp, ip]
        L.ref_engine_rect.restype = C.c_void_p
        L.ref_engine_rect.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int,
                                      C.c_int, C.c_int, ip, dp, dp, C.c_double, C.c_double, C.c_int,
                                      C.c_char_p, C.c_long]
        L.ref_engine_affine.restype = C.c_void_p
        L.ref_engine_affine.argtypes = [C.c_double] * 6 + [C.c_int] * 4 + [ip, dp, dp, C.c_double, C.c_double,
                                                                            C.c_int, C.c_char_p, C.c_long]
        L.ref_engine_problem.restype = C.c_void_p
        L.ref_engine_problem.argtypes = [C.c_char_p, C.c_double, C.c_double, C.c_double, C.c_int, C.c_char_p,
                                         C.c_long]
        L.ref_engine_testgeom.restype = C.c_void_p
        L.ref_engine_testgeom.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_char_p]
        L.ref_engine_sub_info.argtypes = [C.c_void_p, C.c_int, ip, dp]
        L.ref_engine_lines.argtypes = [C.c_void_p, C.c_int, ip, ip, dp, ip, dp, ip, dp]
        L.ref_engine_plan.argtypes = [C.c_void_p, C.c_int, C.c_int, ip, ip, dp, ip, dp]
        L.ref_engine_destroy.argtypes = [C.c_void_p]
        L.ref_engine_nsubs.argtypes = [C.c_void_p]
        L.ref_engine_dims.argtypes = [C.c_void_p, C.c_int, ip, ip]
        L.ref_engine_get.argtypes = [C.c_void_p, C.c_int, C.c_char_p, C.c_int, dp]
        L.ref_engine_set.argtypes = [C.c_void_p, C.c_int, C.c_char_p, C.c_int, dp]
        L.ref_engine_finish_ic.argtypes = [C.c_void_p]
        L.ref_engine_phase.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.ref_engine_dt.argtypes = [C.c_void_p, dp]
        L.ref_engine_set_dt.argtypes = [C.c_void_p, C.c_double]
        L.ref_engine_advance.argtypes = [C.c_void_p]
        L.ref_engine_time.argtypes = [C.c_void_p, dp, C.POINTER(C.c_long)]
        L.ref_engine_run.argtypes = [C.c_void_p, dp, C.POINTER(C.c_long), dp]
        L.ref_engine_set_max_steps.argtypes = [C.c_void_p, C.c_long]
        _lib = L
    return _lib


class RefError(RuntimeError):
    def __init__(self, kind, msg):
        super().__init__(msg)
        self.kind = kind


def _check(rc):
    if rc != 0:
        k = C.c_int()
        msg = lib().ref_last_error(C.byref(k)).decode()
        raise RefError(k.value, msg)


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def blend_matrix(n_cont=25):
    out = np.zeros((n_cont - 1) * 3)
    _check(lib().ref_blend_matrix(n_cont, _dp(out)))
    return out.reshape(n_cont - 1, 3)


def fc_info(n, n_cont=25):
    ne = C.c_int()
    per = C.c_double()
    nm = (n + n_cont - 1) // 2 + 1
    fp = np.zeros(nm)
    sp = np.zeros(nm)
    _check(lib().ref_fc_info(n, n_cont, C.byref(ne), C.byref(per), _dp(fp), _dp(sp)))
    return ne.value, per.value, fp, sp


MODE = {"d1": 1, "d2": 2, "filter": 3, "smear": 4, "cont": 5}


def fc_apply(lines, mode="d1", n_cont=25, threads=1):
    """lines: (L, n) C-contiguous; unit-span operator per line."""
    lines = np.ascontiguousarray(lines, dtype=np.float64)
    L, n = lines.shape
    if mode == "cont":
        out = np.zeros((L, n_cont - 1))
    else:
        out = np.zeros_like(lines)
    _check(lib().ref_fc_apply(n, n_cont, MODE[mode], _dp(lines), n, 1, L, _dp(out), threads))
    return out


def fc_evaluate(values, xs, n_cont=25):
    values = np.ascontiguousarray(values, dtype=np.float64)
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    out = np.zeros_like(xs)
    _check(lib().ref_fc_evaluate(len(values), n_cont, _dp(values), len(xs), _dp(xs), _dp(out)))
    return out


def train_classifier(path):
    acc = C.c_double()
    _check(lib().ref_train_classifier(path.encode(), C.byref(acc)))
    return acc.value


def mlp_forward(path, x7):
    x7 = np.ascontiguousarray(x7, dtype=np.float64).reshape(-1, 7)
    n = x7.shape[0]
    logits = np.zeros((n, 4))
    cls = np.zeros(n, dtype=np.int32)
    _check(lib().ref_mlp_forward(path.encode(), n, _dp(x7), _dp(logits),
                                 cls.ctypes.data_as(C.POINTER(C.c_int))))
    return logits, cls


def classify_line(path, values):
    values = np.ascontiguousarray(values, dtype=np.float64)
    tau = np.zeros(len(values), dtype=np.int32)
    _check(lib().ref_classify_line(path.encode(), len(values), _dp(values),
                                   tau.ctypes.data_as(C.POINTER(C.c_int))))
    return tau


def classify_line_fallback(values, window=32, abs_floor=1e-4):
    values = np.ascontiguousarray(values, dtype=np.float64)
    tau = np.zeros(len(values), dtype=np.int32)
    _check(lib().ref_classify_line_fallback(int(window), C.c_double(abs_floor), len(values), _dp(values),
                                            tau.ctypes.data_as(C.POINTER(C.c_int))))
    return tau


def _json_out(call):
    n = C.c_long()
    _check(call(None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(call(buf, n.value + 1, C.byref(n)))
    import json
    return json.loads(buf.value.decode())


def mesh_roundtrip(mesh: dict) -> dict:
    """DomainDecomposition::from_json + to_json of a mesh (the reference reading it)."""
    import json
    text = json.dumps(mesh).encode()
    return _json_out(lambda b, c, n: lib().ref_mesh_roundtrip(text, b, c, n))


# The reference's file writers (std::ofstream) crash when called in a process
# that has numpy loaded (observed with this image's numpy wheels), so they run
# in a child interpreter that loads only ctypes; inputs travel as raw doubles.
def _isolated(code: str, *args):
    import subprocess
    import sys
    script = "import ctypes as C, array, sys\nL = C.CDLL(%r)\n" % LIB_PATH + code
    r = subprocess.run([sys.executable, "-c", script, *map(str, args)], capture_output=True, text=True)
    if r.returncode != 0:
        raise RefError(9, f"isolated reference call failed ({r.returncode}): {r.stderr[-400:]}")
    return r.stdout


def write_schlieren_pgm(v, meta, beta, path):
    """write_pgm(schlieren(raster, beta), path) of the reference"""
    import tempfile
    v = np.ascontiguousarray(v, dtype=np.float64)
    with tempfile.NamedTemporaryFile(suffix=".bin", delete=False) as f:
        f.write(np.ascontiguousarray(meta, dtype=np.float64).tobytes() + v.tobytes())
        blob = f.name
    try:
        _isolated("""
a = array.array("d"); a.frombytes(open(sys.argv[1], "rb").read())
nx, ny = int(sys.argv[2]), int(sys.argv[3])
meta = (C.c_double * 4)(*a[:4]); v = (C.c_double * (nx * ny))(*a[4:])
L.ref_write_schlieren_pgm.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_double, C.c_char_p]
rc = L.ref_write_schlieren_pgm(nx, ny, meta, v, float(sys.argv[4]), sys.argv[5].encode())
sys.exit(rc)
""", blob, v.shape[1], v.shape[0], repr(float(beta)), path)
    finally:
        os.unlink(blob)


def testgeom_write_csv(which, n0, out_dir, weight_path=""):
    """write_subpatch_csv of ref_engine_testgeom(which, n0) right after
    Engine::init"""
    _isolated("""
L.ref_engine_testgeom.restype = C.c_void_p
L.ref_engine_testgeom.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_char_p]
L.ref_engine_write_csv.argtypes = [C.c_void_p, C.c_char_p]
h = L.ref_engine_testgeom(int(sys.argv[1]), int(sys.argv[2]), 9, 0.5, 1, sys.argv[4].encode())
if not h:
    sys.exit(3)
sys.exit(L.ref_engine_write_csv(h, sys.argv[3].encode()))
""", which, n0, out_dir, weight_path or "")


def fit_shock_angle(v, meta, x_lo, x_hi, y_lo, y_hi):
    v = np.ascontiguousarray(v, dtype=np.float64)
    m = np.ascontiguousarray(meta, dtype=np.float64)
    out = C.c_double()
    _check(lib().ref_fit_shock_angle(v.shape[1], v.shape[0], _dp(m), _dp(v), x_lo, x_hi, y_lo, y_hi, C.byref(out)))
    return out.value


class RefEngine:
    """Engine over one affine I patch origin + q1 e1 + q2 e2 (ref_engine_affine);
    (lx, ly) alone is the axis-aligned rectangle."""

    def __init__(self, x0, y0, lx, ly, r, s, n0, nv, side_kinds, side_states=None,
                 side_pressure=None, cfl=0.5, T=1e300, workers=1, weight_path="", max_steps=10**9,
                 e1=None, e2=None):
        kinds = np.ascontiguousarray(side_kinds, dtype=np.int32)
        states = np.zeros(16) if side_states is None else np.ascontiguousarray(side_states, dtype=np.float64).ravel()
        press = np.ones(4) if side_pressure is None else np.ascontiguousarray(side_pressure, dtype=np.float64)
        e1 = (lx, 0.0) if e1 is None else e1
        e2 = (0.0, ly) if e2 is None else e2
        h = lib().ref_engine_affine(x0, y0, e1[0], e1[1], e2[0], e2[1], r, s, n0, nv,
                                    kinds.ctypes.data_as(C.POINTER(C.c_int)), _dp(states), _dp(press),
                                    cfl, T, workers, weight_path.encode(), max_steps)
        if not h:
            _check(9)
        self.h = h
        self.nsubs = lib().ref_engine_nsubs(h)
        self.dims = []
        for k in range(self.nsubs):
            a, b = C.c_int(), C.c_int()
            _check(lib().ref_engine_dims(h, k, C.byref(a), C.byref(b)))
            self.dims.append((a.value, b.value))

    @classmethod
    def problem(cls, name, target_h=0.0, cfl=0.0, T=0.0, workers=1, weight_path="", max_steps=10**9):
        """A named problem of the reference's workbench (src/problems.cpp:379-388)
        with its own initial condition applied."""
        self = cls.__new__(cls)
        h = lib().ref_engine_problem(name.encode(), target_h, cfl, T, workers, weight_path.encode(), max_steps)
        if not h:
            _check(9)
        self.h = h
        self.nsubs = lib().ref_engine_nsubs(h)
        self.dims = []
        for k in range(self.nsubs):
            a, b = C.c_int(), C.c_int()
            _check(lib().ref_engine_dims(h, k, C.byref(a), C.byref(b)))
            self.dims.append((a.value, b.value))
        return self

    @classmethod
    def testgeom(cls, which, n0=30, nv=9, cfl=0.5, workers=1, weight_path=""):
        """Test geometries through the reference's geometry API (ref_export.cpp
        ref_engine_testgeom): 0 annulus, 1 two patches with interpolation,
        2 C1 corner patch (L-shaped subpatch)."""
        self = cls.__new__(cls)
        h = lib().ref_engine_testgeom(which, n0, nv, cfl, workers, weight_path.encode())
        if not h:
            _check(9)
        self.h = h
        self.nsubs = lib().ref_engine_nsubs(h)
        self.dims = []
        for k in range(self.nsubs):
            a, b = C.c_int(), C.c_int()
            _check(lib().ref_engine_dims(h, k, C.byref(a), C.byref(b)))
            self.dims.append((a.value, b.value))
        return self

    def integrals(self):
        """(energy_integral, area_integral)"""
        e, a = C.c_double(), C.c_double()
        _check(lib().ref_engine_integrals(self.h, C.byref(e), C.byref(a)))
        return e.value, a.value

    def raster(self, nx, ny):
        """density_gradient_raster: (v[ny, nx], (x0, y0, dx, dy))"""
        v = np.zeros((ny, nx))
        meta = np.zeros(4)
        _check(lib().ref_engine_raster(self.h, nx, ny, _dp(v), _dp(meta)))
        return v, meta

    def mesh_json(self) -> dict:
        """the reference's fcs-mesh v1 JSON of this engine's decomposition"""
        return _json_out(lambda b, c, n: lib().ref_engine_mesh_json(self.h, b, c, n))

    def sub_info(self, sub):
        """dict: patch, i0, j0, ni, nj, cut_i, cut_j (local), periodic1, kind, h1, h2"""
        info = np.zeros(9, dtype=np.int32)
        hh = np.zeros(2)
        _check(lib().ref_engine_sub_info(self.h, sub, info.ctypes.data_as(C.POINTER(C.c_int)), _dp(hh)))
        keys = ("patch", "i0", "j0", "ni", "nj", "cut_i", "cut_j", "periodic1", "kind")
        d = {k: int(v) for k, v in zip(keys, info)}
        d["h1"], d["h2"] = float(hh[0]), float(hh[1])
        return d

    def lines(self, sub):
        """LineInfo of rows then columns: begin, n, inv_len, (kind, state[4],
        pressure) of the low and high ends"""
        ni, nj = self.dims[sub]
        m = ni + nj
        ip_ = lambda a: a.ctypes.data_as(C.POINTER(C.c_int))  # noqa: E731
        begin, n = np.zeros(m, np.int32), np.zeros(m, np.int32)
        inv = np.zeros(m)
        klo, khi = np.zeros(m, np.int32), np.zeros(m, np.int32)
        blo, bhi = np.zeros((m, 5)), np.zeros((m, 5))
        _check(lib().ref_engine_lines(self.h, sub, ip_(begin), ip_(n), _dp(inv), ip_(klo), _dp(blo), ip_(khi),
                                      _dp(bhi)))
        return dict(begin=begin, n=n, inv_len=inv, kind_lo=klo, bc_lo=blo, kind_hi=khi, bc_hi=bhi)

    def plan(self, sub, which):
        """(copies (n, 3) dst/src_sub/src, copy_w, interps (m, 4) dst/src_sub/si0/sj0,
        interp_w (m, 13) wx[6], wy[6], w) of recipient `sub`; which 0 solution, 1 viscosity"""
        cnt = np.zeros(2, np.int32)
        ip_ = lambda a: a.ctypes.data_as(C.POINTER(C.c_int))  # noqa: E731
        _check(lib().ref_engine_plan(self.h, sub, which, ip_(cnt), None, None, None, None))
        cp = np.zeros((cnt[0], 3), np.int32)
        cw = np.zeros(cnt[0])
        it = np.zeros((cnt[1], 4), np.int32)
        iw = np.zeros((cnt[1], 13))
        _check(lib().ref_engine_plan(self.h, sub, which, ip_(cnt), ip_(cp), _dp(cw), ip_(it), _dp(iw)))
        return cp, cw, it, iw

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_engine_destroy(self.h)
            self.h = None

    def get(self, sub, what, comp=0):
        ni, nj = self.dims[sub]
        out = np.zeros((nj, ni))
        _check(lib().ref_engine_get(self.h, sub, what.encode(), comp, _dp(out)))
        return out

    def get_state(self, sub, what="e"):
        return np.stack([self.get(sub, what, c) for c in range(4)])

    def set(self, sub, what, arr, comp=0):
        arr = np.ascontiguousarray(arr, dtype=np.float64)
        _check(lib().ref_engine_set(self.h, sub, what.encode(), comp, _dp(arr)))

    def set_state(self, sub, e):
        for c in range(4):
            self.set(sub, "e", e[c], c)

    def finish_ic(self):
        _check(lib().ref_engine_finish_ic(self.h))

    def phase(self, phase, stage=0):
        _check(lib().ref_engine_phase(self.h, phase, stage))

    def reduce_dt(self):
        dt = C.c_double()
        _check(lib().ref_engine_dt(self.h, C.byref(dt)))
        return dt.value

    def advance(self):
        _check(lib().ref_engine_advance(self.h))

    def step(self):
        """One superstep in the order of Engine::run (src/runtime.cpp:486-511)."""
        self.phase(0)
        self.phase(1)
        self.phase(2)
        self.reduce_dt()
        for s in range(5):
            self.phase(3, s)
            self.phase(6)
        self.advance()

    def time(self):
        t = C.c_double()
        st = C.c_long()
        lib().ref_engine_time(self.h, C.byref(t), C.byref(st))
        return t.value, st.value

    def run(self, steps):
        lib().ref_engine_set_max_steps(self.h, steps)
        w = C.c_double()
        n = C.c_long()
        t = C.c_double()
        _check(lib().ref_engine_run(self.h, C.byref(w), C.byref(n), C.byref(t)))
        return w.value, n.value, t.value
