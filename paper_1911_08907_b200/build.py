"""Build libaps.so in-tree with nvcc for sm_100a (no JIT, no torch extension
machinery): the .so travels with the repo to the GPU box.  Each source is
compiled to an object in parallel, then linked."""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = Path(os.environ.get("APS_BUILD_OUT", PKG / "libaps.so"))  # APS_BUILD_OUT / APS_NVCC_EXTRA: A/B variants
SOURCES = [CSRC / "aps_kernels.cu", CSRC / "aps_fused.cu", CSRC / "aps_peer.cu", CSRC / "aps_api.cpp"]
HEADERS = [CSRC / "aps_numerics.cuh", CSRC / "aps_device.cuh", CSRC / "aps_internal.h", CSRC / "aps_peer.h",
           ROOT / "include" / "aps.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs() -> tuple[Path, Path]:
    import nvidia.nccl  # torch's bundled NCCL (one NCCL per process)
    base = Path(list(nvidia.nccl.__path__)[0])
    return base / "include", base / "lib"


def build(force: bool = False, verbose: bool = False) -> Path:
    newest = max(p.stat().st_mtime for p in SOURCES + HEADERS + [Path(__file__)])
    if not force and LIB.exists() and LIB.stat().st_mtime >= newest:
        return LIB
    inc, lib = nccl_dirs()
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    common = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
              "-Xptxas", "-v" if verbose else "-O3", f"-I{ROOT / 'include'}", f"-I{inc}",
              *os.environ.get("APS_NVCC_EXTRA", "").split()]

    def compile_one(src: Path):
        obj = objdir / (src.name + f".{os.getpid()}.{LIB.stem}.o")
        return obj, subprocess.run(common + ["-c", str(src), "-o", str(obj)], capture_output=True, text=True)

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    for (obj, r), src in zip(results, SOURCES):
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src.name}")
        if verbose:
            sys.stderr.write(r.stderr)
    tmp = LIB.with_suffix(f".so.tmp{os.getpid()}")
    cmd = [NVCC, *ARCH, "-shared", *[str(o) for o, _ in results], "-o", str(tmp),
           f"-L{lib}", "-l:libnccl.so.2", "-Xlinker", f"-rpath={lib}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    for o, _ in results:
        o.unlink(missing_ok=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libaps.so")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
