"""Build libiabn.so in-tree with nvcc for sm_100a (B200).

    python paper_1712_02616_b200/build.py [--force] [--verbose]

The library links the CUDA runtime statically (it coexists with torch's own
cudart) and loads NCCL at run time with dlopen, so it loads on a machine
without a GPU or NCCL (host-side validation still works there).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libiabn.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_include() -> str:
    try:
        import nvidia.nccl  # type: ignore

        for p in nvidia.nccl.__path__:
            inc = os.path.join(p, "include")
            if os.path.exists(os.path.join(inc, "nccl.h")):
                return inc
    except Exception:
        pass
    for inc in ("/usr/include", "/usr/local/include"):
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc
    raise RuntimeError("nccl.h not found (needed for its type definitions only)")


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + [os.path.join(ROOT, "include", "iabn.h")])


def build(force: bool = False, verbose: bool = False, ptxas_v: bool = False) -> str:
    deps = sources()
    if (not force and os.path.exists(LIB)
            and os.path.getmtime(LIB) >= max(os.path.getmtime(d) for d in deps)):
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-O3", "-std=c++17", "-lineinfo", "-shared", "-Xcompiler", "-fPIC",
           "-Xcompiler", "-fvisibility=hidden", "-cudart", "static",
           "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", _nccl_include(),
           "-DIABN_BUILD", "-Xlinker", "--exclude-libs,ALL", "-Xlinker", "-Bsymbolic",
           "-o", tmp, os.path.join(CSRC, "iabn.cu"), "-ldl"]
    if ptxas_v:
        cmd[1:1] = ["-Xptxas", "-v"]
    extra = os.environ.get("IABN_NVCC_EXTRA", "").split()  # experiments (e.g. -DIABN_APPLY_WARPS=4)
    cmd[1:1] = extra
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv,
                ptxas_v="--ptxas-v" in sys.argv))
