"""Build libztp.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels
with the repo snapshot to the GPU box).  `python -m paper_2401_11469_b200.build`."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libztp.so")
SOURCES = ["ztp_api.cu", "ztp_gemm.cu", "ztp_select.cu", "ztp_misc.cu", "ztp_peer.cu", "ztp_plan.cpp"]
HEADERS = ["ztp_internal.h", "ztp_ptx.cuh"]


def _nccl_dirs():
    import nvidia.nccl  # torch-bundled NCCL 2.28 (the one torch.distributed uses)
    base = nvidia.nccl.__path__[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def nvcc() -> str:
    for c in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.exists(c) or c == "nvcc":
            return c
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "ztp.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = True) -> str:
    if not force and not needs_build():
        return LIB
    inc, libdir = _nccl_dirs()
    objs = []
    bdir = os.path.join(HERE, "build")
    os.makedirs(bdir, exist_ok=True)
    common = ["-std=c++17", "-O3", "-Xcompiler", "-fPIC,-ffp-contract=off", "-I", os.path.join(ROOT, "include"),
              "-I", inc]
    hdr_t = max(os.path.getmtime(d) for d in [os.path.join(CSRC, h) for h in HEADERS] +
                [os.path.join(ROOT, "include", "ztp.h")])
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(bdir, s + ".o")
        objs.append(obj)
        if (not force and os.path.exists(obj) and os.path.getmtime(obj) > max(os.path.getmtime(src), hdr_t)
                and os.environ.get("ZTP_REBUILD_ALL") != "1"):
            continue
        if s.endswith(".cu"):
            cmd = [nvcc(), "-c", src, "-o", obj, "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
                   "--expt-relaxed-constexpr", "-Xptxas", "-v" if os.environ.get("ZTP_PTXAS_V") else "-O3"] + common
        else:
            cmd = [nvcc(), "-c", "-x", "c++", src, "-o", obj] + common
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    link = [nvcc(), "-shared", "-o", LIB] + objs + ["-gencode", "arch=compute_100a,code=sm_100a", "-L", libdir,
                                                    "-l:libnccl.so.2", "-Xlinker", f"-rpath={libdir}",
                                                    "-Xcompiler", "-fPIC"]
    if verbose:
        print(" ".join(link), flush=True)
    subprocess.run(link, check=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
