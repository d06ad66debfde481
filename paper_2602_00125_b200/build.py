"""Build libb2.so (sm_100a) in-tree with nvcc.

    python -m paper_2602_00125_b200.build      # or __graft_entry__.build()

Every translation unit is compiled for `-gencode arch=compute_100a,code=sm_100a`
with -lineinfo (ncu source pages). The numerics-critical units (elementwise,
reductions, losses, optimizers) are built with -fmad=false so no FMA
contraction can change a rounding the reference does separately.
"""

from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libb2.so")
BUILD = os.path.join(ROOT, "build", "b2")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NO_FMAD = {"ewise.cu", "reduce.cu", "xent.cu", "optim.cu", "fused_stats.cu"}


def _nvcc():
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found")
    return cand


def _nccl_include():
    import importlib.util

    spec = importlib.util.find_spec("nvidia")
    dirs = []
    if spec and spec.submodule_search_locations:
        for base in spec.submodule_search_locations:
            d = os.path.join(base, "nccl", "include")
            if os.path.exists(os.path.join(d, "nccl.h")):
                dirs.append(d)
    if not dirs:
        raise RuntimeError("nccl.h not found (nvidia/nccl/include)")
    return dirs[0]


def _compile(src, obj, nvcc, incs):
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                    "-Xptxas", "-v" if os.environ.get("B2_PTXAS_V") else "-O3",
                    "--expt-relaxed-constexpr", "-c", src, "-o", obj]
    if os.path.basename(src) in NO_FMAD:
        flags.insert(0, "-fmad=false")
    for i in incs:
        flags += ["-I", i]
    r = subprocess.run([nvcc] + flags, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return r.stderr


def build(verbose=False, force=False):
    nvcc = _nvcc()
    os.makedirs(BUILD, exist_ok=True)
    incs = [os.path.join(ROOT, "include"), CSRC, _nccl_include()]
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    deps = srcs + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "b2.h")]
    newest_dep = max(os.path.getmtime(p) for p in deps)
    if not force and os.path.exists(OUT) and os.path.getmtime(OUT) >= newest_dep:
        return OUT
    objs = []
    jobs = []
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        for s in srcs:
            o = os.path.join(BUILD, os.path.basename(s)[:-3] + ".o")
            objs.append(o)
            jobs.append((s, ex.submit(_compile, s, o, nvcc, incs)))
        for s, j in jobs:
            log = j.result()
            if verbose and log:
                print(f"== {os.path.basename(s)}\n{log}", file=sys.stderr)
    tmp = OUT + ".tmp"
    cmd = [nvcc] + ARCH + ["-shared", "-o", tmp] + objs + ["-ldl", "-lpthread", "-lrt"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
