"""Build the sm_100a C-ABI library ``liblnorm.so`` in-tree with nvcc.

``python -m paper_2503_21596_b200.build`` or ``__graft_entry__.build()``.
Each .cu is compiled to an object in parallel (nvcc cross-compiles for
sm_100a without a GPU) and linked with -shared; ``-lineinfo`` keeps the ncu
source page mapped to our code.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
OUT = os.path.join(HERE, "liblnorm.so")
BUILD = os.path.join(HERE, "_build")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-warn-spills",
         "-I" + os.path.join(ROOT, "include")]


def _stale(obj: str, deps) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    sources = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h"))
    jobs = []
    for src in sources:
        obj = os.path.join(BUILD, os.path.basename(src)[:-3] + ".o")
        if force or _stale(obj, [src] + headers):
            jobs.append((src, obj))

    def compile_one(job):
        src, obj = job
        cmd = [NVCC] + ARCH + FLAGS + ["-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        if verbose and r.stderr:
            sys.stderr.write(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
        list(ex.map(compile_one, jobs))
    objs = [os.path.join(BUILD, os.path.basename(s)[:-3] + ".o") for s in sources]
    if force or jobs or not os.path.exists(OUT):
        cmd = [NVCC] + ARCH + ["-shared", "-o", OUT + ".tmp"] + objs + ["-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        os.replace(OUT + ".tmp", OUT)
    return OUT


# Self-check build: the byte binary walk compiled with -G (device debug) and
# LN_SELFCHECK=1 -- every Gray step of unit 0 of every lane is compared with a from-scratch value
# (walk_u8_impl.cuh) -- for the 13-16-column instance only (LN_U8_ONLY_NW=4, seconds to build);
# every other translation unit is the product object.  tests/test_gpu_selfcheck.py loads it.
SELFCHECK_DIR = os.path.join(HERE, "_selfcheck")
SELFCHECK_OUT = os.path.join(SELFCHECK_DIR, "liblnorm_selfcheck.so")
SELFCHECK_TUS = {"abi": ["-O3", "-lineinfo", "-DLN_SELFCHECK=1"],
                 "walk_u8_l1": ["-G", "-DLN_SELFCHECK=1", "-DLN_U8_ONLY_NW=4"],
                 "walk_u8_marg": ["-G", "-DLN_SELFCHECK=1", "-DLN_U8_ONLY_NW=4"],
                 "walk_u8_l2": ["-G", "-DLN_SELFCHECK=1", "-DLN_U8_ONLY_NW=4"]}


def build_selfcheck(force: bool = False) -> str:
    build(force=False)
    os.makedirs(SELFCHECK_DIR, exist_ok=True)
    sources = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h"))
    objs, jobs = [], []
    for src in sources:
        base = os.path.basename(src)[:-3]
        if base in SELFCHECK_TUS:
            obj = os.path.join(SELFCHECK_DIR, base + ".o")
            flags = [f for f in FLAGS if f not in ("-O3", "-lineinfo")] + SELFCHECK_TUS[base]
            if force or _stale(obj, [src] + headers):
                jobs.append([NVCC] + ARCH + flags + ["-c", src, "-o", obj])
            objs.append(obj)
        else:
            objs.append(os.path.join(BUILD, base + ".o"))

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{r.stderr}")

    with cf.ThreadPoolExecutor(max_workers=max(1, len(jobs))) as ex:
        list(ex.map(run, jobs))
    if force or jobs or not os.path.exists(SELFCHECK_OUT) or os.path.getmtime(OUT) > os.path.getmtime(SELFCHECK_OUT):
        r = subprocess.run([NVCC] + ARCH + ["-shared", "-o", SELFCHECK_OUT + ".tmp"] + objs + ["-ldl", "-lpthread"],
                           capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        os.replace(SELFCHECK_OUT + ".tmp", SELFCHECK_OUT)
    return SELFCHECK_OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
    if "--selfcheck" in sys.argv:
        print(build_selfcheck(force="--force" in sys.argv))
