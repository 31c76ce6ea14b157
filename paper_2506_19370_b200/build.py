"""Build the fcsg native library in-tree.

* ``libfcsg.so``  -- the product: CUDA sources compiled by nvcc for sm_100a
  only (``-gencode arch=compute_100a,code=sm_100a -lineinfo``), host sources
  by g++, linked with the static CUDA runtime. Written to
  ``paper_2506_19370_b200/lib/`` so it travels to the GPU box with the repo.
* ``libfcsg_emu.so`` (``emulate=True``) -- the same kernel bodies compiled as
  plain C++ with one emulated thread per CTA. TEST HARNESS ONLY: used by the
  CPU unit tests to check kernel logic without a GPU; the package never loads
  it.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
ROOT = os.path.dirname(HERE)
EMU_DIR = os.path.join(ROOT, "build", "emu")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = "-gencode=arch=compute_100a,code=sm_100a"

CU_SOURCES = ["dev.cu", "fc_lines.cu", "step_kernels.cu", "wpass.cu", "wctpass.cu", "w20lines.cu", "classify_f32.cu"]
CPP_SOURCES = ["fc_tables.cpp", "capi.cpp", "engine.cpp", "comm.cpp"]


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {cmd[0]} {cmd[-1]}")
    return r


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def _headers():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))] + [
        os.path.join(ROOT, "include", "fcsg.h")
    ]


def build(emulate: bool = False, verbose: bool = False, force: bool = False, sanitize: bool = False) -> str:
    """sanitize (with emulate): the emulation build under AddressSanitizer +
    UndefinedBehaviorSanitizer (build/emu_asan/), the bounds / UB check of the
    kernel bodies' index logic (scripts/asan_emu.sh)"""
    sanitize = sanitize and emulate
    objdir = os.path.join(ROOT, "build", "emu_asan_obj" if sanitize else ("emu_obj" if emulate else "obj"))
    os.makedirs(objdir, exist_ok=True)
    out_dir = os.path.join(ROOT, "build", "emu_asan") if sanitize else (EMU_DIR if emulate else LIBDIR)
    os.makedirs(out_dir, exist_ok=True)
    lib = os.path.join(out_dir, "libfcsg_emu.so" if emulate else "libfcsg.so")
    hdrs = _headers()
    objs = []
    cmds = []
    common_inc = [f"-I{CSRC}", f"-I{os.path.join(ROOT, 'include')}"]
    for src in CU_SOURCES + CPP_SOURCES:
        path = os.path.join(CSRC, src)
        if not os.path.exists(path):
            continue
        obj = os.path.join(objdir, src + ".o")
        objs.append(obj)
        if not force and not _stale(obj, [path] + hdrs):
            continue
        if emulate:
            lang = ["-x", "c++"] if src.endswith(".cu") else []
            san = ["-fsanitize=address,undefined", "-fno-omit-frame-pointer", "-g", "-O1"] if sanitize else ["-O2"]
            cmd = ["g++", "-std=c++17", *san, "-fPIC", "-DFCSG_EMULATE", *common_inc, *lang, "-c", path, "-o", obj]
        elif src.endswith(".cu"):
            cmd = [NVCC, ARCH, "-std=c++17", "-O3", "-lineinfo", "-Xptxas=-v" if verbose else "-Xptxas=-O3",
                   "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", *common_inc, "-c", path, "-o", obj]
        else:
            cmd = ["g++", "-std=c++17", "-O3", "-fPIC", f"-I{CUDA_HOME}/include", *common_inc, "-c", path, "-o", obj]
        cmds.append(cmd)
    # translation units compile in parallel (the step kernels dominate)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as ex:
        for r in ex.map(_run, cmds):
            if verbose and r.stderr:
                sys.stderr.write(r.stderr)
    if force or _stale(lib, objs):
        if emulate:
            san = ["-fsanitize=address,undefined"] if sanitize else []
            _run(["g++", "-shared", *san, "-o", lib, *objs, "-lquadmath", "-lpthread", "-lrt"])
        else:
            _run([NVCC, ARCH, "-shared", "-o", lib, *objs, "-lquadmath", "-ldl", "-cudart", "static"])
    return lib


if __name__ == "__main__":
    emu = "--emulate" in sys.argv or "--asan" in sys.argv
    print(build(emulate=emu, verbose="-v" in sys.argv, force="--force" in sys.argv, sanitize="--asan" in sys.argv))
