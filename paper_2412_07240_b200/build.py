"""Build libpmf.so (the C-ABI library of include/pmf.h) in-tree for sm_100a.

    python -m paper_2412_07240_b200.build            # incremental
    python -m paper_2412_07240_b200.build --force

nvcc cross-compiles without a GPU. The .so lands next to this file so that it
travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpmf.so")
SOURCES = ["pmf_host.cpp", "pmf_sharded.cpp", "kernels_pencil.cu", "kernels_resident.cu", "kernels_plane.cu", "kernels_fdm.cu",
           "kernels_cluster.cu", "kernels_quad.cu"]
HEADERS = ["plane_common.cuh", "pmf_internal.h", "pmf_ctx_impl.h", "device_common.cuh", "fft_smem.cuh", "fft_reg.cuh", "tma.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills"] + os.environ.get("PMF_NVCC_EXTRA", "").split()


def _stale(obj: str, deps: list[str]) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "pmf.h")]
    objdir = os.path.join(HERE, "build_obj")
    os.makedirs(objdir, exist_ok=True)
    # a change of the compiler flags (e.g. PMF_NVCC_EXTRA) rebuilds everything
    stamp = os.path.join(objdir, "flags.txt")
    flags = " ".join([NVCC, *ARCH, *FLAGS])
    if not os.path.exists(stamp) or open(stamp).read() != flags:
        force = True
        with open(stamp, "w") as fh:
            fh.write(flags)
    objs, cmds = [], []
    for src in SOURCES:
        sp = os.path.join(CSRC, src)
        op = os.path.join(objdir, src + ".o")
        objs.append(op)
        if force or _stale(op, [sp] + hdrs + [__file__]):
            cmd = [NVCC, *ARCH, *FLAGS, "-I", CSRC, "-I", os.path.join(ROOT, "include"), "-c", sp, "-o", op]
            if src.endswith(".cpp"):
                cmd.insert(1, "-x")
                cmd.insert(2, "cu")
            if verbose:
                print(" ".join(cmd))
            cmds.append(cmd)
    # the translation units are independent: compile them in parallel
    with ThreadPoolExecutor(max_workers=max(1, min(len(cmds), os.cpu_count() or 1))) as ex:
        for r in list(ex.map(lambda c: subprocess.run(c), cmds)):
            if r.returncode != 0:
                raise subprocess.CalledProcessError(r.returncode, r.args)
    if force or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-Xcompiler", "-fPIC"]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
