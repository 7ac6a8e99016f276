"""Build libhp.so (all CUDA kernels + the C ABI) in-tree for sm_100a with nvcc.

SASS only (-gencode arch=compute_100a,code=sm_100a), -lineinfo for ncu source pages,
static cudart (nvcc 12.9 here, torch ships a cu128 runtime), no fast-math.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
SO = os.path.join(HERE, "libhp.so")

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
          "-Xptxas", "-v"] + ARCH
PER_FILE = {"k_feat.cu": ["-fmad=false"], "k_comp.cu": ["-fmad=false"]}


def sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))


def _stale(obj, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, variant: str = "", defines=()) -> str:
    """Build libhp.so; a named variant (extra -D defines, for experiments) builds into
    _build_<variant>/ and libhp_<variant>.so (select it at run time with HP_SO=...)."""
    BUILD = globals()["BUILD"] + (f"_{variant}" if variant else "")
    SO = os.path.join(HERE, f"libhp_{variant}.so") if variant else globals()["SO"]
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(HERE, "..", "include", "hp.h"))
    jobs = []
    for f in sources():
        src = os.path.join(CSRC, f)
        obj = os.path.join(BUILD, f.replace(".cu", ".o"))
        if force or _stale(obj, [src] + headers):
            cmd = [NVCC, "-c", src, "-o", obj] + COMMON + PER_FILE.get(f, []) + list(defines)
            jobs.append((f, cmd))
    logs = {}

    def run(job):
        f, cmd = job
        r = subprocess.run(cmd, capture_output=True, text=True)
        return f, r

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        for f, r in ex.map(run, jobs):
            logs[f] = r.stderr
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {f}")
    objs = [os.path.join(BUILD, f.replace(".cu", ".o")) for f in sources()]
    if force or jobs or not os.path.exists(SO):
        cmd = [NVCC, "-shared", "-o", SO] + objs + ARCH + ["-cudart", "static", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
    if verbose:
        with open(os.path.join(BUILD, "ptxas.log"), "w") as fh:
            for f, log in logs.items():
                fh.write(f"== {f}\n{log}\n")
    return SO


if __name__ == "__main__":
    var = [a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")]
    defs = [a for a in sys.argv if a.startswith("-D")]
    print(build(force="--force" in sys.argv, verbose=True, variant=var[0] if var else "", defines=defs))
