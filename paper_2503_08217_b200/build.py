"""Build libs3r.so (the CUDA path, sm_100a) in-tree with nvcc.

Flags that are part of the numerical contract (DESIGN.md R-ARITH):
  -fmad=false            no multiply-add contraction; FMAs are explicit
  (no --use_fast_math)   IEEE division and square root (-prec-div/-prec-sqrt)
  -ffp-contract=off      for the host compiler as well

``build_variant(name, defines)`` builds an experimental copy
(``libs3r_<name>.so``, objects under build/<name>/) with extra -D flags; the
binding loads it when the environment variable S3R_LIB points at it.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libs3r.so")
BUILD = os.path.join(HERE, "build")
SOURCES = ["k_filter.cu", "k_project.cu", "k_sort.cu", "k_bin.cu", "k_raster.cu", "k_plan.cu", "k_small.cu",
           "k_backward.cu", "k_neurf.cu", "s3r_api.cu"]
HEADERS = ["s3r_internal.cuh", os.path.join("..", "..", "include", "s3r.h")]
# The backward (config 5) is compared with the oracle at 1e-3, not bit for bit:
# it may contract multiply-adds (its forward recomputation uses explicit
# __fmaf_rn / separate ops where it must match the forward's decisions).
# The NeurF query (bf16 tensor-core contract, R22) likewise.
CONTRACTED = {"k_backward.cu", "k_neurf.cu"}

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-fmad=false", "-prec-div=true", "-prec-sqrt=true",
         "-Xcompiler", "-fPIC,-ffp-contract=off,-O2", "-Xptxas", "-warn-spills"]


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _build(out: str, bdir: str, defines=(), force: bool = False, verbose: bool = False) -> str:
    os.makedirs(bdir, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [__file__]
    dflags = [f"-D{d}" for d in defines]
    objs, jobs = [], []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(bdir, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            flags = list(FLAGS)
            if src in CONTRACTED:      # not part of the bit-exact forward contract
                flags[flags.index("-fmad=false")] = "-fmad=true"
            jobs.append([NVCC, *flags, *dflags, "-c", s, "-o", o])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stdout or r.stderr):
            print(r.stdout + r.stderr, file=sys.stderr)

    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        list(ex.map(run, jobs))
    if force or jobs or _stale(out, objs):
        run([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", out, *objs])
    return out


def build(force: bool = False, verbose: bool = False) -> str:
    return _build(OUT, BUILD, (), force, verbose)


def build_variant(name: str, defines, force: bool = False) -> str:
    return _build(os.path.join(HERE, f"libs3r_{name}.so"), os.path.join(BUILD, name), defines,
                  force)


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
