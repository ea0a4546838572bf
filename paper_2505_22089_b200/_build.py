"""In-tree build of libbmg.so for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT = PKG / "libbmg.so"
SOURCES = ["kernels.cu", "vlad.cu", "bmg_api.cpp", "host_random.cpp", "host_synthetic.cpp", "host_io.cpp", "host_sao.cpp"]
HEADERS = ["bmg_internal.h", "../../include/bandmatch_gpu.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++20",
         "-Xcompiler", "-fPIC,-Wall", "-shared", "-cudart", "static"]


def _stale() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + [CSRC / h for h in HEADERS] + [Path(__file__)]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if force or _stale():
        cmd = [NVCC, *FLAGS, "-o", str(OUT), *[str(CSRC / s) for s in SOURCES]]
        if verbose:
            print(" ".join(cmd))
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{r.stdout}\n{r.stderr}")
    return OUT


if __name__ == "__main__":
    print(build(force=True, verbose=True))
