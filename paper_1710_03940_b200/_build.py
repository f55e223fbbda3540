"""Build libdflb200.so in-tree: nvcc for the sm_100a kernels, g++ for the host
setup (no FMA contraction, so the AMG hierarchy matches the reference bit for
bit).  Invoked by ``__graft_entry__.build()`` and ``python -m
paper_1710_03940_b200._build``."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libdflb200.so")
BUILD = os.path.join(REPO, "build", "dflb200")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SOURCES = ["ctx.cu", "ctx_layout.cu", "ctx_comm.cu", "ctx_cycle.cu", "ctx_cg.cu", "ctx_krylov.cu", "ctx_bicg.cu", "ctx_block.cu", "setup_dev.cu", "gen_dev.cu"]
CXX_SOURCES = ["host_setup.cpp", "mmio.cpp"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _cuda_include() -> str:
    return os.path.join(os.path.dirname(os.path.dirname(_nvcc())), "include")  # NVTX 3 headers


def _sources():
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp", ".h"))]
    hdrs.append(os.path.join(REPO, "include", "dflb200.h"))
    return [os.path.join(CSRC, f) for f in CU_SOURCES + CXX_SOURCES] + hdrs


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in _sources())


def build(force: bool = False, verbose: bool = False, out: str | None = None) -> str:
    if out is None and not force and up_to_date():
        return LIB
    bdir = BUILD if out is None else os.path.join(REPO, "build", os.path.basename(out) + ".obj")
    os.makedirs(bdir, exist_ok=True)
    nvcc = _nvcc()
    run = lambda cmd: subprocess.run(cmd, check=True, stdout=None if verbose else subprocess.DEVNULL)
    # only the C ABI of include/dflb200.h (DFL_API) is exported
    jobs = []
    for f in CXX_SOURCES:
        o = os.path.join(bdir, f + ".o")
        jobs.append((o, ["g++", "-O3", "-std=c++17", "-fPIC", "-pthread", "-ffp-contract=off", "-fno-fast-math",
                         "-fvisibility=hidden", "-I", os.path.join(REPO, "include"), "-I", _cuda_include(),
                         "-c", os.path.join(CSRC, f),
                         "-o", o]))
    extra = os.environ.get("DFL_NVCC_FLAGS", "").split()
    for f in CU_SOURCES:
        o = os.path.join(bdir, f + ".o")
        jobs.append((o, [nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", *extra,
                         "-Xcompiler", "-ffp-contract=off", "-Xcompiler", "-fvisibility=hidden",
                         "-I", os.path.join(REPO, "include"), "-c", os.path.join(CSRC, f), "-o", o]))
    with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 1)) as pool:
        list(pool.map(lambda j: run(j[1]), jobs))
    objs = [o for o, _ in jobs]
    target = out or LIB
    tmp = target + ".tmp"
    run([nvcc, *ARCH, "-shared", "-o", tmp, *objs, "-ldl", "-lpthread"])
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    o = None
    if "--out" in sys.argv:
        o = sys.argv[sys.argv.index("--out") + 1]
    print(build(force="--force" in sys.argv, verbose=True, out=o))
