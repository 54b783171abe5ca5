"""Build libstencil_b200.so in-tree with nvcc for sm_100a.

Every ``csrc/*.cu`` is compiled separately (in parallel) with
``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo`` and linked into
``paper_2301_11389_b200/libstencil_b200.so``.  ptxas register / spill
reports (``-Xptxas -v``) go to ``build/ptxas_<unit>.log``.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "libstencil_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
              "-Xptxas", "-v", "-I", os.path.join(ROOT, "include")]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _deps_mtime() -> float:
    files = glob.glob(os.path.join(CSRC, "*")) + glob.glob(os.path.join(ROOT, "include", "*.h"))
    return max(os.path.getmtime(f) for f in files)


def _compile(src: str, bdir: str = BUILD, defines: tuple = ()) -> str:
    unit = os.path.splitext(os.path.basename(src))[0]
    obj = os.path.join(bdir, unit + ".o")
    log = os.path.join(bdir, f"ptxas_{unit}.log")
    cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
    p = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + p.stdout + p.stderr)
    if p.returncode:
        sys.stderr.write(p.stderr)
        raise RuntimeError(f"nvcc failed on {unit} (see {log})")
    return obj


def _link(objs, lib: str) -> str:
    tmp = lib + f".tmp{os.getpid()}"
    subprocess.check_call([nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-ldl"])
    os.replace(tmp, lib)
    return lib


def build(force: bool = False, jobs: int | None = None) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _deps_mtime():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    jobs = jobs or min(len(srcs), os.cpu_count() or 4)
    with cf.ThreadPoolExecutor(jobs) as ex:
        objs = list(ex.map(_compile, srcs))
    return _link(objs, LIB)


def build_experiment(name: str, defines: tuple) -> str:
    """A/B builds: the same sources with extra -D flags into
    expbuild/<name>/libstencil_b200.so (git-ignored, travels with gpurun; load
    it with STB200_LIB=<path>)."""
    bdir = os.path.join(ROOT, "expbuild", name)
    os.makedirs(bdir, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(min(len(srcs), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda f: _compile(f, bdir, defines), srcs))
    return _link(objs, os.path.join(bdir, "libstencil_b200.so"))


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--exp":   # --exp NAME DEFINE...
        print(build_experiment(sys.argv[2], tuple(sys.argv[3:])))
    else:
        print(build(force="--force" in sys.argv))
