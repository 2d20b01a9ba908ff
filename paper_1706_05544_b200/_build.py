"""Build libsvmb200.so in-tree with nvcc for sm_100a (no JIT, no torch extension machinery).

The .so lands next to this file so it travels with the repo snapshot to the GPU box.  ptxas
resource usage of every kernel is written to build/ptxas.log.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# SVMB200_BUILD_TAG (diagnostic builds, e.g. the SMO_PROFILE one) puts objects and the library
# under separate names (build_<tag>/, libsvmb200_<tag>.so) next to the product build;
# binding.py loads it only when SVMB200_LIB names it
_TAG = os.environ.get("SVMB200_BUILD_TAG", "")
BUILD = os.path.join(ROOT, "build" + (f"_{_TAG}" if _TAG else ""))
LIB = os.path.join(PKG, "libsvmb200" + (f"_{_TAG}" if _TAG else "") + ".so")
SOURCES = ["smo.cu", "layout.cu", "predict.cu", "capi.cu"]
HEADERS = ["svm_internal.cuh", "layout.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
                "-I" + os.path.join(ROOT, "include"), "-Xptxas", "-v"]
if os.environ.get("SVMB200_PROFILE_BUILD"):  # per-phase clock64 instrumentation of smo.cu
    FLAGS = FLAGS + ["-DSMO_PROFILE"]
if os.environ.get("SVMB200_EXTRA_FLAGS"):  # debugging builds (e.g. -DSMO_POISON=0xffffffffu)
    FLAGS = FLAGS + os.environ["SVMB200_EXTRA_FLAGS"].split()


def _nvcc() -> str:
    for c in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.exists(c) or c == "nvcc":
            return c
    raise RuntimeError("nvcc not found")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "svmb200.h")]
    srcs = [s for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    objs = []
    jobs = []
    for s in srcs:
        src = os.path.join(CSRC, s)
        obj = os.path.join(BUILD, s.replace(".cu", ".o"))
        objs.append(obj)
        if force or _stale(obj, [src] + hdrs):
            jobs.append((src, obj))

    def comp(job):
        src, obj = job
        r = subprocess.run([_nvcc()] + FLAGS + ["-c", src, "-o", obj], capture_output=True,
                           text=True)
        return src, r

    logs = []
    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        for src, r in ex.map(comp, jobs):
            logs.append(f"==== {os.path.basename(src)}\n{r.stderr}")
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {src}")
    if logs:
        with open(os.path.join(BUILD, "ptxas.log"), "w") as f:
            f.write("\n".join(logs))
    if force or jobs or _stale(LIB, objs):
        r = subprocess.run([_nvcc()] + ARCH + ["-shared", "-o", LIB] + objs, capture_output=True,
                           text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link of libsvmb200.so failed")
    if verbose:
        print(LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
