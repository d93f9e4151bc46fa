"""Build the sm_100a C-ABI library ``paper_2411_18889_b200/lib/libsolomon_b200.so``.

Plain ``nvcc -shared`` of ``csrc/*.cu`` -- in-tree, so the built ``.so``
travels with the repo snapshot to the GPU box (it is git-ignored, not
gpurun-ignored). Static cudart keeps the library independent of the CUDA
runtime torch happens to bundle; device pointers and streams are shared
through the driver's primary context.
"""
from __future__ import annotations

import os
import pathlib
import shutil
import subprocess
import sys

PKG = pathlib.Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "lib"
LIB = LIB_DIR / "libsolomon_b200.so"
PROBE = LIB_DIR / "libsolomon_probe.so"
SOURCES = ["nbody.cu", "nbody_small.cu", "diffusion.cu", "diffusion_tb2.cu", "diffusion_resident.cu", "diffusion_halo.cu", "dropin.cu", "ipc.cu", "multicast.cu", "runtime.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and pathlib.Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    if not PROBE.exists():
        return True
    deps = [CSRC / s for s in SOURCES] + [CSRC / "probe.cu"] + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "solomon_b200.h"]
    return any(d.stat().st_mtime > t for d in deps if d.exists())


def build(force: bool = False, verbose: bool = False) -> pathlib.Path:
    if not force and not needs_build():
        return LIB
    LIB_DIR.mkdir(exist_ok=True)
    subprocess.run([nvcc(), *ARCH, "-O3", "-lineinfo", "-shared", "-Xcompiler", "-fPIC",
                    str(CSRC / "probe.cu"), "-o", str(PROBE)], check=True)
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "-Xcompiler", "-fno-fast-math",
           "-DSOLOMON_B200_BUILD", f"-I{ROOT / 'include'}", f"-I{CSRC}",
           *(str(CSRC / s) for s in SOURCES), "-o", str(LIB)]
    extra = os.environ.get("SOLOMON_NVCC_EXTRA")  # A/B builds of compile-time variants (tuning)
    if extra:
        cmd[1:1] = extra.split()
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
