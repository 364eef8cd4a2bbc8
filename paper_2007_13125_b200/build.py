"""Build the sm_100a shared library `libpint.so` in-tree (nvcc, no JIT, no torch extension).

    python -m paper_2007_13125_b200.build [--force] [-j N]

One object per FFT length (template instantiations of the T-pass and DST kernels), plus the
S-pass dispatch and the host plan / C ABI; linked with the static CUDA runtime.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(os.path.dirname(HERE), "build", "pint")
LIB = os.path.join(HERE, "libpint.so")
NS = [16, 32, 64, 128, 256, 512, 1024, 2048, 4096]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", "-I", os.path.join(os.path.dirname(HERE), "include")]


def nvcc() -> str:
    for c in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(os.path.dirname(HERE), "include", "pint.h")]


def _newest_dep() -> float:
    return max(os.path.getmtime(p) for p in _deps())


def _compile(src: str, obj: str, defines: list[str]) -> tuple[str, str]:
    extra = os.environ.get("PINT_NVCC_EXTRA", "").split()      # experiments only (variant builds)
    cmd = [nvcc(), *ARCH, *FLAGS, *extra, *defines, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src} {defines}:\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, jobs: int | None = None, verbose: bool = False,
          defines: list[str] | None = None, lib: str | None = None) -> str:
    """defines/lib: experimental variants (e.g. ["-DPINT_TPASS_MINB=3"], "libpint_minb3.so")."""
    defines = defines or []
    LIB = os.path.join(HERE, lib) if lib else globals()["LIB"]
    # variant objects outside the repo (the repo snapshot shipped to the GPU box stays small)
    build_dir = os.path.join("/tmp", "pint_build_" + os.path.splitext(lib)[0]) if lib else BUILD
    extra = os.environ.get("PINT_NVCC_EXTRA", "").split()
    if extra and not lib:
        raise RuntimeError("PINT_NVCC_EXTRA is for variant builds only: pass lib=<variant name>")
    # the full flag set is stamped next to the library: a change of flags or defines rebuilds it
    stamp = " ".join([nvcc(), *ARCH, *FLAGS, *extra, *defines])
    stamp_path = LIB + ".flags"
    fresh = (os.path.exists(LIB) and os.path.getmtime(LIB) >= _newest_dep() and os.path.exists(stamp_path)
             and open(stamp_path).read() == stamp)
    if not force and fresh:
        return LIB
    os.makedirs(build_dir, exist_ok=True)
    units = [(os.path.join(CSRC, "inst_n.cu"), os.path.join(build_dir, f"inst_{n}.o"), [f"-DPINT_N={n}", *defines])
             for n in NS]
    units += [(os.path.join(CSRC, "dispatch.cu"), os.path.join(build_dir, "dispatch.o"), defines),
              (os.path.join(CSRC, "fused.cu"), os.path.join(build_dir, "fused.o"), defines),
              (os.path.join(CSRC, "newton.cu"), os.path.join(build_dir, "newton.o"), defines),
              (os.path.join(CSRC, "pint.cu"), os.path.join(build_dir, "pint.o"), defines)]
    jobs = jobs or min(len(units), os.cpu_count() or 4)
    logs = []
    with cf.ThreadPoolExecutor(jobs) as ex:
        for obj, log in ex.map(lambda u: _compile(*u), units):
            logs.append((obj, log))
    with open(os.path.join(build_dir, "ptxas.log"), "w") as f:
        for obj, log in logs:
            f.write(f"== {os.path.basename(obj)}\n{log}\n")
    cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", LIB + ".tmp", *[u[1] for u in units]]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(LIB + ".tmp", LIB)
    with open(stamp_path, "w") as f:
        f.write(stamp)
    if verbose:
        print(f"built {LIB}")
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=None)
    ap.add_argument("-D", action="append", default=[], help="extra define (variant builds)")
    ap.add_argument("--lib", default=None, help="variant library file name")
    args = ap.parse_args()
    build(force=args.force, jobs=args.j, verbose=True, defines=[f"-D{d}" for d in args.D], lib=args.lib)
    sys.exit(0)
