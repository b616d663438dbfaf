"""Build the test NCCL (nccl_shim.cu): G ranks as threads of one process on one GPU.

Test infrastructure only.  libiabn.so picks it up through ``IABN_NCCL_LIB`` (read once,
at the library's first NCCL call), so it is used from a subprocess
(``tests/sync_shim_worker.py``) that sets the variable before loading the package.
"""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "nccl_shim.cu")
LIB = os.path.join(HERE, "libnccl_shim.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_include() -> str:
    import nvidia.nccl  # type: ignore

    for p in nvidia.nccl.__path__:
        inc = os.path.join(p, "include")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc
    raise RuntimeError("nccl.h not found")


def build(force: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17",
                    "-shared", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
                    "-cudart", "static", "-I", _nccl_include(), "-o", tmp, SRC], check=True)
    os.replace(tmp, LIB)
    return LIB
