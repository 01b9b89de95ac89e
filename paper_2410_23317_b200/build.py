"""Build the sm_100a extension in-tree: paper_2410_23317_b200/libvlc_b200.so.

Plain nvcc (no torch extension machinery): the library exports only the C-ABI
of include/vlc.h and links the CUDA runtime statically, so it loads into any
process (ctypes from Python, cgo/JNI from elsewhere) that shares the driver.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libvlc_b200.so")
SOURCES = ["vlc_api.cu", "score_stats.cu", "score_stats_tc.cu", "tma_host.cu", "budget.cu", "select.cu", "gather.cu", "decode.cu", "decode_wide.cu", "eval_rows.cu", "prefill.cu", "seam_f32.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def build(verbose: bool = False, force: bool = False, out: str | None = None, defines=()) -> str:
    """Compile every kernel into one shared library (default: in-tree LIB).
    `out` / `defines` exist for tuning experiments (tools/), not for products."""
    lib = out or LIB
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    deps.append(os.path.join(ROOT, "include", "vlc.h"))
    if not force and out is None and os.path.exists(lib):
        t = os.path.getmtime(lib)
        if all(os.path.getmtime(d) <= t for d in deps):
            return lib
    flags = [*ARCH, *(f"-D{d}" for d in defines), "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
             "-Xcompiler", "-fvisibility=hidden", "-I", os.path.join(ROOT, "include")]
    if verbose:
        flags.append("-Xptxas=-v")
    # one nvcc per translation unit, in parallel, then one link
    objdir = lib + ".objs"
    os.makedirs(objdir, exist_ok=True)
    objs = [os.path.join(objdir, os.path.basename(s)[:-3] + ".o") for s in srcs]

    def compile_one(i):
        cmd = [nvcc(), *flags, "-c", "-o", objs[i], srcs[i]]
        if verbose:
            print(" ".join(cmd))
        return subprocess.run(cmd, capture_output=True, text=True)

    with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, range(len(srcs))))
    for r in results:
        sys.stderr.write(r.stdout + r.stderr)
        if r.returncode:
            raise subprocess.CalledProcessError(r.returncode, r.args)
    subprocess.run([nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", lib + ".tmp", *objs], check=True)
    shutil.rmtree(objdir, ignore_errors=True)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
