"""Benchmark: fp64 grid-point RK-stage updates/s of the FC-SDNN superstep.

Workload (BASELINE config 5, weak scaling): per GPU one 8x8 tiling of 256x256
subpatches (subdivide_Q(8, 8, 238, 9): 64 subpatches, 4,194,304 points,
19-point intra-patch overlap), isentropic vortex + 1e-3 seeded noise, ANN
(SDNN) classifier, CFL 0.5. A "step" is one full superstep (viscosity,
blend, filter, 5 x (RHS + SSPRK stage + BC + exchange)); the metric counts
5 x points per step (pt-stage), points counted with overlap multiplicity as
the reference and the paper do (src/runtime.cpp:41-45).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fcsg|reference]

--impl reference times the reference's own CPU Engine (the unmodified
sources compiled into oracle/_ref) on the same workload and metric, with all
host threads, on a bounded sample per step (see SAMPLE below).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "fp64 grid-point RK-stage updates/s"
UNIT = "pt-stage/s"
# paper Table 2, one 54-core Xeon node, weak/refinement N=550,854
PAPER_1NODE = 6.74e7
R_TILES, S_TILES = 8, 8
STRONG_TILES = (32, 16)  # strong scaling: 512 subpatches of 256x256 (33.5M points) in total


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def fp64_peak():
    """measured FP64 peak (TFLOP/s): DFMA alone, DMMA alone and both
    interleaved share one FP64 datapath on the B200 (scripts/fp64_peak.cu,
    profiles/r02_fp64_peak.json)"""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_fp64_peak.json")) as fh:
            return float(json.load(fh)["dfma_tflops"]), "measured (scripts/fp64_peak.cu)"
    except Exception:
        return 37.1, "fallback (B200 nominal DFMA)"


# kernel behind each timed group (for the ncu capture lookup) and its launches
# per group timing (the RK-stage passes launch once per stage chunk)
GROUP_KERNEL = {"pass_a": "wpass_y_kernel", "pass_b": "wpass_x_kernel", "viscosity": "classify_f32_kernel"}
GROUP_LAUNCHES_PER_STEP = {"pass_a": 5, "pass_b": 5, "viscosity": 1}


def ncu_traffic(group, npts):
    """DRAM bytes (read + write) per group launch of the group's kernel, from
    the newest committed `ncu --set full` capture of every kernel of one steady
    superstep of the bench workload (profiles/rNN_all_raw.csv,
    scripts/prof_r02.sh): the bytes of all its launches in the step divided by
    the group's launches per step, or None."""
    import csv
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_all_raw.csv")))
    key = GROUP_KERNEL.get(group)
    if not files or not key:
        return None, None
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    with open(files[-1]) as fh:
        rows = list(csv.reader(fh))
    hdr, units = rows[0], rows[1]
    ik = hdr.index("Kernel Name")
    ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    total, n = 0.0, 0
    for r in rows[2:]:
        if key in r[ik]:
            total += float(r[ir]) * scale.get(units[ir], 1.0) + float(r[iw]) * scale.get(units[iw], 1.0)
            n += 1
    if n == 0:
        return None, None
    return total / GROUP_LAUNCHES_PER_STEP[group], os.path.basename(files[-1])


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML
    every 2 ms in a thread (nvidia_ml_py), else nvidia-smi every 100 ms."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # nvmlClocksEventReason* bits
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, device=0):
        self.device = device
        self.rows = []  # (sm_mhz, max_mhz, [reasons])
        self.proc = None
        self.nvml = None
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            # NVML's first queries can take tens of milliseconds -- as long as the
            # whole timed region: make them here, before the poll thread starts
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _poll(self):
        N = self.nvml
        get_reasons = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            N.nvmlDeviceGetCurrentClocksThrottleReasons
        self._sample = lambda: self.rows.append(
            (float(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)), self.mx,
             [k for k, b in self.BITS.items() if get_reasons(self.h) & b]))
        while not self.stop.is_set():
            try:
                self._sample()
            except Exception:
                pass
            self.stop.wait(0.002)

    def _read(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.proc.stdout:
            r = [x.strip() for x in line.split(",")]
            if len(r) < 9 or not r[1].replace(".", "").isdigit():
                continue
            self.rows.append((float(r[1]), float(r[2]), [names[k] for k in range(4) if r[5 + k] == "Active"]))

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml is not None:
            self.t.join(timeout=2)
            if not self.rows:  # the poll thread never ran inside a very short region: one sample at its end
                try:
                    self._sample()
                except Exception:
                    pass
            try:
                self.nvml.nvmlShutdown()
            except Exception:
                pass
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": sorted({x for r in self.rows for x in r[2]}), "samples": len(self.rows),
                "source": "nvml" if self.nvml is not None else "nvidia-smi"}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload(rank_tiles=(R_TILES, S_TILES)):
    from paper_2506_19370_b200 import problems as P

    return P.vortex_tiles(r=rank_tiles[0], s=rank_tiles[1])


# --------------------------------------------------------------------------
# reference arm: the reference's own CPU Engine (oracle/_ref)

SAMPLE_TILES = (4, 2)  # 8 subpatches of 256x256 (524,288 points) per timed step


def reference_engine(tiles, threads):
    from oracle import ref
    from paper_2506_19370_b200 import engine as EN, problems as P

    dec, ic, _ = P.vortex_tiles(r=tiles[0], s=tiles[1])
    p = dec.patches[0]
    R = ref.RefEngine(p.origin[0], p.origin[1], p.e1[0], p.e2[1], tiles[0], tiles[1], 238, p.nv, [5, 5, 5, 5],
                      cfl=0.5, workers=threads, weight_path=EN.DEFAULT_WEIGHTS)
    for k in range(len(dec.subs)):
        R.set_state(k, P.initial_state(dec, ic, k))
    R.finish_ic()
    return R, dec.total_points()


def cpu_model():
    """the host CPU the CPU legs ran on (/proc/cpuinfo)"""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


SHIM_FFT = ("oracle/shims/fftw3.h: FFTW3 absent from the image, its r2c/c2r restated as a mixed-radix FFT with "
            "half-length packing and precomputed twiddles (slower than FFTW, so the CPU rate is a lower bound)")


def cpu_rate(steps, warmup, threads):
    R, npts = reference_engine(SAMPLE_TILES, threads)
    if warmup:
        R.run(warmup)
    wall, n, _ = R.run(R.time()[1] + steps)
    return 5.0 * npts * n / wall, wall / max(n, 1), npts


def workload_name(n_subs_total=None, strong=False):
    """the config-5 weak-scaling workload as both arms name it"""
    if strong:
        return (f"config5-strong: {STRONG_TILES[0]}x{STRONG_TILES[1]} tiles of 256x256 ({n_subs_total} subpatches, "
                f"{STRONG_TILES[0] * STRONG_TILES[1] * 65536} points) split in contiguous blocks over the GPUs, "
                f"19-point overlap, vortex + 1e-3 noise, ANN classifier, CFL 0.5")
    block = "" if n_subs_total is None else f" (one block of a {n_subs_total}-subpatch tiling, NCCL halo exchange)"
    return (f"config5-weak: {R_TILES}x{S_TILES} tiles of 256x256 per GPU{block} ({R_TILES * S_TILES * 65536} "
            f"points/GPU, 19-point overlap), vortex + 1e-3 noise, ANN classifier, CFL 0.5")


def run_reference(args):
    world, rank, _ = dist_init()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    rate, sps, npts = cpu_rate(args.steps, args.warmup, threads)
    sample = (f"reference Engine::run (oracle/_ref: unmodified reference sources, FFTW replaced by the "
              f"oracle/shims mixed-radix FFT), {SAMPLE_TILES[0]}x{SAMPLE_TILES[1]} tiles of 256x256 "
              f"({npts} points) of the config-5 workload per step, {threads} worker threads")
    out = {"metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": sps * 1e3, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": rate / PAPER_1NODE, "dtype": "f64", "data": "synthetic", "impl": "reference",
           "config": {"workload": workload_name(), "points_per_gpu": R_TILES * S_TILES * 256 * 256,
                      "sampled_per_step": f"{SAMPLE_TILES[0]}x{SAMPLE_TILES[1]} of the {R_TILES}x{S_TILES} tiles "
                                          f"({npts} points): the CPU rate is per point, the sample bounds the "
                                          f"run time"},
           "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample,
                            "cpu_model": cpu_model(), "fft": SHIM_FFT},
           "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# --------------------------------------------------------------------------
# product arm


# algorithmic HBM bytes per point per launch: every
# input read once and every output written once; values produced and consumed
# inside one kernel count zero. Stage passes in the default flux form; the
# RK registers are those of stage 1 (the stage time_group launches): e0 read,
# e2 written. Cartesian 256 x 256 subpatches (every subpatch of the workload):
# the warp passes, pass Y first (columns: tA = iq2y D2 Phi_y), then pass X
# (rows: rhs = tA + iq1x D1 Phi_x and the SSPRK update); the metrics are one
# value per subpatch (uniform), the mask is read only for a failing point.
ALG_BYTES_CART = {
    "pass_a": 32 + 8 + 32,                        # e, mu -> tA
    "pass_b": 32 + 8 + 32 + 32 + 32 + 32,         # e, mu, tA, e0 -> e, e2
    "pass_c": 0,
    "viscosity": 32 + 1 + 8 + 8 * 4,              # e, mask, h_max -> proxy, speed, tau, mu_hat (+ proxy re-read in L1)
    "filter": 32 + 32 + 32 + 32,                  # rows e -> tF ; cols tF -> e
    "blend": 8 * 5 + 1 + 8,
}
# general: GA (rows, D1 w), GB (cols), C (rows)
ALG_BYTES_GEN = dict(ALG_BYTES_CART, pass_a=32 + 1 + 32,                      # e, mask -> tW
                     pass_b=32 + 32 + 8 + 32 + 32 + 32 + 32,                 # e, 4 metrics, mu, tW -> tS4, tS5, tA
                     pass_c=64 + 32 + 16 + 32 + 32 + 32 + 32)                # tS4, tS5, tA, iq1x, iq1y, e, e0 -> e2, e
# algorithmic FP64 flops per point per launch (47.7 per real line
# derivative at N = 256): pass Y 8 derivatives (D2 of 4 w, D2 of 4 Phi_y) +
# primitives, fluxes and Phi (~60); pass X 8 derivatives + the same + the rhs
# and SSPRK update (~30); the classifier 2 stencils x 1977 + mu_hat
FLOP_PER_POINT = {"pass_a": 8 * 47.7 + 60, "pass_b": 8 * 47.7 + 90, "viscosity": 2 * 1977 + 20}
STEP_FLOP = (80 * 47.7 + 8 * 47.7 + 2 * 1977 + 800) / 5  # per point-stage, flux form
LAUNCHES = {"pass_a": 5, "pass_b": 5, "pass_c": 5, "viscosity": 1, "filter": 1, "blend": 1, "bc": 6,
            "exchange": 5}


def fc_derivative_gbs(ctx, n_cont=25, degree=2):
    """config 1 (4096 lines x N=256) from HBM to HBM, rotating buffers larger
    than L2 between launches: the reference operator (n_cont 25, degree 2) or
    BASELINE's five-point variant (C = 27, degree 4). The 64 timed launches
    replay as one CUDA graph: a Python loop of launches is host-bound (~13 us
    of ctypes + launch per call against a ~10 us kernel)."""
    import torch

    from paper_2506_19370_b200 import fc, problems as P

    op = fc.FcOperator(ctx, 256, n_cont=n_cont, degree=degree)
    _, f, _ = P.fc_lines_config1(n_lines=4096, n=256, seed=1)
    src = torch.from_numpy(f).cuda()
    nbuf = 16  # 16 x 2 x 8 MiB = 256 MiB > 126 MB L2
    ins = [src.clone() for _ in range(nbuf)]
    outs = [torch.empty_like(src) for _ in range(nbuf)]
    reps = 64
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        for k in range(4):
            op.apply(ins[k], 1, out=outs[k])
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for k in range(reps):
                op.apply(ins[k % nbuf], 1, out=outs[k % nbuf])
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()  # replay() launches on the current stream
    g.replay()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    return 16.0 * f.size / (ms * 1e-3) / 1e9, ms


def fc_derivative_batch_gbs(ctx, copies=64):
    """The same operator on `copies` config-1 batches in ONE call (262144
    lines, 512 MiB in and out: beyond L2 by itself): the line kernel in its
    throughput regime -- config 1 alone is a single wave of 512 warps and is
    bound by one warp's latency chain, not by HBM. Device time, CUDA events,
    two rotating buffer pairs."""
    import torch

    from paper_2506_19370_b200 import fc, problems as P

    op = fc.FcOperator(ctx, 256)
    _, f, _ = P.fc_lines_config1(n_lines=4096, n=256, seed=1)
    src = torch.from_numpy(f).cuda().repeat(copies, 1).contiguous()
    ins = [src, src.clone()]
    outs = [torch.empty_like(src) for _ in range(2)]
    for k in range(2):
        op.apply(ins[k], 1, out=outs[k])
    torch.cuda.synchronize()
    reps = 8
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()  # op.apply launches on torch's current stream, where these events are recorded
    for k in range(reps):
        op.apply(ins[k % 2], 1, out=outs[k % 2])
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    return 16.0 * src.numel() / (ms * 1e-3) / 1e9, ms, src.shape[0]


def config2_rate(ctx, steps=10):
    """BASELINE config 2 (one 512x512 subpatch, seeded quadrants, CFL 0.5) on
    this GPU: device time per superstep (CUDA graph, after warm-up)."""
    import torch

    from paper_2506_19370_b200 import engine as EN, problems as P

    dec, ic, _ = P.riemann_quadrants(n=512, seed=2)
    E = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=0.5))
    E.enqueue(3)
    torch.cuda.synchronize()
    st = torch.cuda.ExternalStream(E.stream())
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    E.enqueue(steps)
    b.record(st)
    torch.cuda.synchronize()
    E.check_error()
    ms = a.elapsed_time(b) / steps
    groups = {g: E.time_group(g, reps=3) for g in ("viscosity", "pass_a", "pass_b", "pass_c", "filter")}
    return {"config": "config2: 512x512 subpatch (n_ext = 536 = 8 x 67), Riemann quadrants, CFL 0.5",
            "ms_per_step": ms, "value": 5.0 * E.total_points() / (ms * 1e-3), "unit": UNIT,
            "kernel_groups_ms": groups}


def config3_rate(ctx, steps=20):
    """BASELINE config 3 (Mach 3 flow past a cylinder: periodic annulus
    2048 x 147 + four Cartesian patches of 256 x 256 subpatches, 2.57M points,
    built from scratch by multipatch.py) on this GPU: device time per
    superstep after the t = 0 step and two warm-up steps."""
    import time

    import torch

    from paper_2506_19370_b200 import engine as EN, problems as P

    t0 = time.time()
    dec, ic, meta = P.cylinder_flow(full=True)
    build_s = time.time() - t0
    E = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=meta["cfl"]))
    E.enqueue(3)
    torch.cuda.synchronize()
    st = torch.cuda.ExternalStream(E.stream())
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    E.enqueue(steps)
    b.record(st)
    torch.cuda.synchronize()
    E.check_error()
    ms = a.elapsed_time(b) / steps
    groups = {g: E.time_group(g, reps=3) for g in ("viscosity", "pass_a", "pass_b", "pass_c", "filter")}
    npts = E.total_points()
    E.close()
    return {"config": "config3: Mach 3 flow past a unit cylinder in [-4,12]x[-6,6]; periodic annulus 2048x147 "
                      "(r 1..2.2) + 4 Cartesian I patches of 256x256 subpatches (19-point overlaps, 6x6 "
                      "interpolation); free stream rho 1.4, p 1, u 3; CFL 0.5",
            "points": npts, "subpatches": len(dec.subs), "build_s": build_s, "ms_per_step": ms,
            "value": 5.0 * npts / (ms * 1e-3), "unit": UNIT, "kernel_groups_ms": groups}


def config4_rate(ctx, steps=20):
    """BASELINE config 4 (Mach 3 forward-facing step: C1 corner patch, S and
    I patches, problems.step_flow(2), 3.2M points -- about the per-GPU share
    of the 16M-point 8-GPU case) on this GPU."""
    import time

    import torch

    from paper_2506_19370_b200 import engine as EN, problems as P

    t0 = time.time()
    dec, ic, meta = P.step_flow(2)
    build_s = time.time() - t0
    E = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=meta["cfl"]))
    E.enqueue(3)
    torch.cuda.synchronize()
    st = torch.cuda.ExternalStream(E.stream())
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    E.enqueue(steps)
    b.record(st)
    torch.cuda.synchronize()
    E.check_error()
    ms = a.elapsed_time(b) / steps
    npts = E.total_points()
    E.close()
    return {"config": "config4: Mach 3 forward-facing step in [0,3]x[0,1] (step 0.2 high at x = 0.6); convex C1 "
                      "corner patch at the step top (L-shaped subpatches), concave C2 corner patch at its foot, an "
                      "S patch along the step top, 2 Cartesian I patches of 256x256 subpatches; inflow rho 1.4, "
                      f"p 1, u 3; CFL {meta['cfl']} (the reference's value for problems with C1 patches)",
            "points": npts, "subpatches": len(dec.subs), "build_s": build_s, "ms_per_step": ms,
            "value": 5.0 * npts / (ms * 1e-3), "unit": UNIT}


def fallback_rate(ctx, steps=10):
    """The bench workload with ClassifierConfig's default variant (FC-spectrum
    decay over 32-point windows, src/viscosity.cpp:161-208) instead of the MLP."""
    import torch

    from paper_2506_19370_b200 import engine as EN

    dec, ic, _ = workload()
    E = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=0.5, classifier="fallback"))
    E.enqueue(3)
    torch.cuda.synchronize()
    st = torch.cuda.ExternalStream(E.stream())
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    E.enqueue(steps)
    b.record(st)
    torch.cuda.synchronize()
    E.check_error()
    ms = a.elapsed_time(b) / steps
    return {"config": "config5 workload (8x8 tiles of 256x256), fallback classifier (window 32)",
            "ms_per_step": ms, "value": 5.0 * E.total_points() / (ms * 1e-3), "unit": UNIT,
            "viscosity_ms": E.time_group("viscosity", reps=3)}


def run_fcsg(args):
    import torch

    world, rank, local = dist_init()
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    from paper_2506_19370_b200 import _native as N, engine as EN

    ctx = N.Context(local)
    DE = None
    strong = args.scaling == "strong"
    if world > 1:
        # weak: an (8 py) x (8 px) tiling, one contiguous 8x8 block per rank;
        # strong: the 32 x 16 tiling (512 subpatches) split into world blocks.
        # The engine's own transport: halo pack -> grouped ncclSend/Recv to the
        # neighbour ranks -> unpack, and ncclAllReduce(MIN) of dt, all on the
        # engine stream inside the superstep (one CUDA graph per step)
        from paper_2506_19370_b200 import distributed as D, problems as P

        if strong:
            dec, ic, _ = P.vortex_tiles(r=STRONG_TILES[0], s=STRONG_TILES[1])
        else:
            px = max(p for p in range(1, world + 1) if world % p == 0 and p * p <= world)
            py = world // px
            dec, ic, _ = P.vortex_tiles(r=R_TILES * py, s=S_TILES * px)
        owner = D.partition_tiles(dec, world)
        rp = D.split_plan(dec, owner, rank, world)
        DE = D.DistributedEngine(ctx, dec, rp, ic, EN.EngineConfig(cfl=0.5), transport="native")
        E = DE.E
    else:
        dec, ic, _ = workload(STRONG_TILES if strong else (R_TILES, S_TILES))
        E = EN.Engine(ctx, dec, ic, EN.EngineConfig(cfl=0.5))
    npts = E.total_points()
    stream = torch.cuda.ExternalStream(E.stream(), device=local)

    def steps(n):
        E.enqueue(n)  # graph replays; multi-rank halos and the dt all-reduce inside

    # warm-up (includes the t=0 smear step and the CUDA-graph capture)
    steps(max(args.warmup, 3))
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        steps(args.steps)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms_total = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms_total], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    t_now, steps_done = E.time()
    E.check_error()  # surfaces a device-side InvalidStateError, if any
    ms_step = ms_total / args.steps
    npts_all = npts
    if world > 1:
        t = torch.tensor([npts], device="cuda", dtype=torch.int64)
        dist.all_reduce(t)
        npts_all = int(t.item())
    value = 5.0 * npts_all * args.steps / (ms_total * 1e-3)

    # e2e through the public API with HOST buffers: per step, H2D of the state
    # from pinned memory, one superstep (fcsg_engine_run, which also checks the
    # device error word), D2H of the resulting state
    host_in = torch.empty((4, npts), dtype=torch.float64, pin_memory=True)
    host_out = torch.empty((4, npts), dtype=torch.float64, pin_memory=True)
    E.get_state_bulk(host_in)
    E.run_host(host_in, host_out, steps=1)  # untimed: run_host allocates its staging buffers on first use
    e2e_steps = max(2, min(4 * args.steps, 40))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    # fcsg_engine_run_host: per step the H2D of its input and the D2H of its
    # result, pipelined against the neighbouring steps' kernels (multi-rank:
    # the same call on every rank, the halos inside each step)
    assert E.run_host(host_in, host_out, steps=e2e_steps) == e2e_steps
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = 5.0 * npts_all * e2e_steps / e2e_s
    nbytes = 4 * npts * 8

    # per-kernel-group device time (profiling hook, same engine and stream)
    groups = {}
    for g in ("viscosity", "blend", "filter", "pass_a", "pass_b", "pass_c", "bc", "exchange"):
        groups[g] = E.time_group(g, reps=5)
    launches = dict(LAUNCHES, pass_c=0 if E.is_cartesian() else 5)
    share = {g: groups[g] * launches[g] for g in groups}
    dom = max(share, key=share.get)
    hbm, peak_kind = peaks()
    fp64, fp64_kind = fp64_peak()
    ALG_BYTES = ALG_BYTES_CART if E.is_cartesian() else ALG_BYTES_GEN
    alg = ALG_BYTES.get(dom, 64) * npts
    achieved = alg / (groups[dom] * 1e-3) / 1e9
    traffic, traffic_src = ncu_traffic(dom, npts) if world == 1 else (None, None)
    fc_gbs, fc_ms = fc_derivative_gbs(ctx)
    fc4_gbs, fc4_ms = fc_derivative_gbs(ctx, n_cont=27, degree=4)
    fcb_gbs, fcb_ms, fcb_lines = fc_derivative_batch_gbs(ctx)
    cfg2 = config2_rate(ctx) if world == 1 else None
    cfg3 = config3_rate(ctx) if world == 1 else None
    cfg4 = config4_rate(ctx) if world == 1 else None
    fb = fallback_rate(ctx) if world == 1 else None

    if rank != 0:
        return
    # CPU baseline: the reference on this box's host cores, bounded sample
    cpu = None
    if not args.no_cpu:
        try:
            threads = os.cpu_count() or 1
            # the same sample and step counts as the reference arm (--impl reference)
            rate, sps, cnpts = cpu_rate(args.steps, args.warmup, threads)
            cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": f"{args.steps} supersteps after {args.warmup} untimed ones (the t=0 step first) of "
                             f"{SAMPLE_TILES[0]}x{SAMPLE_TILES[1]} tiles of 256x256 ({cnpts} points) of the same "
                             f"workload, reference Engine::run with {threads} worker threads (oracle/_ref), the "
                             f"same sample and steps as the --impl reference arm",
                   "cpu_model": cpu_model(), "fft": SHIM_FFT}
        except Exception as ex:  # the reference build is test infrastructure
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"unavailable: {ex}"}
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": value / PAPER_1NODE,
        "vs_baseline_basis": "PAPER.md:1612 (BASELINE.md): 6.74e7 pt-stage/s, one 54-core Xeon 8273 node",
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(None if world == 1 and not strong else len(dec.subs), strong),
                   "points_per_gpu": npts, "points_total": npts_all,
                   "l2": f"working set ~{47 * 8 * npts / 1e9:.1f} GB/GPU >> 126 MB L2 (no flush needed)",
                   "cuda_graph": True, "parallelism": f"subpatch blocks x{world}",
                   "transport": "none" if world == 1 else "engine stream: pack + grouped ncclSend/Recv + unpack, ncclAllReduce(MIN) dt, no host sync",
                   "stage_passes": "cartesian" if E.is_cartesian() else "general"},
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
                "steps": e2e_steps, "path": "fcsg_engine_run_host (per step: H2D of the state from pinned memory, one superstep, D2H of "
                         "the result; copies on two copy streams overlap the neighbouring steps)",
                "note": "each step re-uploads the same input (in_stride 0), so step k+1's upload does not wait for step k's "
                        "result; a time-marching driver that feeds each output back in cannot overlap its copies this way"},
        "gpu_launches": E.launches_per_step() * args.steps,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic, "traffic_source": traffic_src,
                     "alg_bytes_per_launch": alg, "peak_kind": peak_kind,
                     "alg_bytes_per_point": ALG_BYTES.get(dom), "ms_per_launch": groups[dom],
                     # the other kernel groups of the step against the same peak (pass Y and pass X take the
                     # same time, so which of the two is "dominant" flips with the noise)
                     "all_groups": {g: {"alg_bytes_per_point": ALG_BYTES[g], "ms_per_launch": groups[g],
                                        "achieved": ALG_BYTES[g] * npts / (groups[g] * 1e-3) / 1e9,
                                        "frac": ALG_BYTES[g] * npts / (groups[g] * 1e-3) / 1e9 / hbm}
                                    for g in ALG_BYTES if ALG_BYTES[g] and groups.get(g, 0) > 1e-3}},
        "roofline_fp64": {
            "note": "the line passes and the classifier are bound by the FP64 pipe and instruction issue, not HBM "
                    "(ncu: FP64 pipe 33-38%, DRAM 11-28% of peak, profiles/README.md); algorithmic flops by "
                    "SURVEY 8(d)'s convention (FFT 2 x 2.5 n_ext log2 n_ext + continuation + multiplier per real "
                    "line derivative = 47.7 flop/pt at N = 256)",
            "peak_tflops": fp64, "peak_kind": fp64_kind,
            "dominant_kernel": {"kernel": dom, "alg_flop_per_point": FLOP_PER_POINT.get(dom),
                                "achieved_tflops": FLOP_PER_POINT.get(dom, 0) * npts / (groups[dom] * 1e-3) / 1e12,
                                "frac": FLOP_PER_POINT.get(dom, 0) * npts / (groups[dom] * 1e-3) / 1e12 / fp64},
            "step": {"alg_flop_per_pt_stage": STEP_FLOP, "achieved_tflops": value / max(world, 1) * STEP_FLOP / 1e12,
                     "frac": value / max(world, 1) * STEP_FLOP / 1e12 / fp64,
                     "basis": "flux form: 16 line derivatives per stage, the per-step filter (8 lines), 2 MLP stencils "
                              "(1977 flop each) and ~800 flop of pointwise work per point per step, over 5 stages; "
                              "the reference's 40-derivative order would count 2930"}},
        "kernel_groups_ms": groups,
        "fc_derivative": {"config": "config1: 4096 lines x N=256, reference operator (degree 2, n_cont=25, "
                                    "n_ext=280), d/dx, HBM->HBM",
                          "gbs": fc_gbs, "us_per_call": fc_ms * 1e3, "frac_of_hbm": fc_gbs / hbm},
        "fc_derivative_batch": {"config": f"{fcb_lines} lines x N=256 in one call (64 config-1 batches, 512 MiB in + "
                                          "512 MiB out), reference operator, d/dx, HBM->HBM: the line kernel's "
                                          "throughput regime",
                                "gbs": fcb_gbs, "us_per_call": fcb_ms * 1e3, "frac_of_hbm": fcb_gbs / hbm},
        "fc_derivative_config1_operator": {"config": "config1 as BASELINE states it: 4096 lines x N=256, Gram degree "
                                                     "4, d=5, C=27 (n_ext=282=2x3x47), d/dx, HBM->HBM",
                                           "gbs": fc4_gbs, "us_per_call": fc4_ms * 1e3, "frac_of_hbm": fc4_gbs / hbm},
        "config2": cfg2,
        "config3": cfg3,
        "config4": cfg4,
        "config5_fallback_classifier": fb,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
        "sim_time": t_now, "steps_run": steps_done,
    }
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="fcsg", choices=["fcsg", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: 64 subpatches per GPU (default); strong: 512 subpatches in total")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_fcsg(args)


if __name__ == "__main__":
    main()
