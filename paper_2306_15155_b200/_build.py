"""Build the sm_100a kernel library ``lib/libgnnc.so`` in-tree with nvcc.

Every translation unit is compiled with ``-gencode arch=compute_100a,code=sm_100a``
(plain ``-arch=sm_100`` would drop the ``a`` features and ptxas would reject
``tcgen05.*``) and ``-lineinfo`` so ncu's source page maps to the code.
The objects are linked into one shared library that the Python package binds
through ctypes (see ``_native.py``).  The C ABI is ``include/gnnc.h``.
"""

from __future__ import annotations

import os
import shutil
import subprocess
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "build"
LIB_DIR = PKG / "lib"
LIB = LIB_DIR / "libgnnc.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-O3,-fvisibility=hidden",
    "-I", str(ROOT / "include"),
    "-I", str(CSRC),
]


def nvcc() -> str:
    path = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(path).exists():
        raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libgnnc.so")
    return path


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _stale(lib: Path, deps: list[Path]) -> bool:
    if not lib.exists():
        return True
    t = lib.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, ptxas_verbose: bool = False,
          defines: tuple[str, ...] = (), out: Path | None = None) -> Path:
    """Build ``lib/libgnnc.so`` (or, for A/B experiments, a variant with extra
    ``-D`` ``defines`` written to ``out``; load it with GNNC_LIB_PATH)."""
    deps = sources() + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "gnnc.h", Path(__file__)]
    lib = Path(out) if out is not None else LIB
    if not force and not defines and not _stale(lib, deps):
        return lib
    obj_dir = OBJ if not defines else OBJ / ("v_" + "_".join(d.replace("=", "") for d in defines))
    obj_dir.mkdir(parents=True, exist_ok=True)
    lib.parent.mkdir(parents=True, exist_ok=True)
    cc = nvcc()
    # host compiler: /usr/bin/g++ (the image's CC/CXX point at a gcc without all runtimes)
    host = ["-ccbin", "/usr/bin/g++"] if Path("/usr/bin/g++").exists() else []
    extra = ["-Xptxas", "-v"] if ptxas_verbose else []

    def compile_one(src: Path) -> Path:
        obj = obj_dir / (src.stem + ".o")
        cmd = [cc, *host, *NVCC_FLAGS, *extra, *(f"-D{d}" for d in defines), "-c", str(src),
               "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stdout}\n{r.stderr}")
        if ptxas_verbose and r.stderr:
            print(r.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, sources()))
    tmp = lib.with_suffix(".so.tmp")
    cmd = [cc, *host, *ARCH, "-shared", "-o", str(tmp), *map(str, objs)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    import sys

    print(build(force="--force" in sys.argv, verbose=True, ptxas_verbose="-v" in sys.argv))
