"""In-tree build of the B200 extension (no torch JIT cache: the built .so
files travel to the GPU box with the repo snapshot).

  libtetris_b200.so            CUDA kernels (sm_100a) + C-ABI (include/tetris_b200.h)
                               + the C++ drop-in host API (include/tetris_b200/*.hpp)
  _tetris_b200<ext>.so         pybind11 binding of the C++ API

Usage: python -m paper_2412_13269_b200.build [--force] [-v]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys
import sysconfig
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
BUILD = ROOT / "build" / "tetris_b200"
CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA_HOME / "bin" / "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
LIB = PKG / "libtetris_b200.so"
EXT = sysconfig.get_config_var("EXT_SUFFIX") or ".so"
PYMOD = PKG / f"_tetris_b200{EXT}"

NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", str(INCLUDE),
                     "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]
# tuning experiments only (e.g. TG_NVCC_EXTRA="-DNTT_MIN_BLOCKS=3")
NVCC_FLAGS += os.environ.get("TG_NVCC_EXTRA", "").split()
# Host code is compiled like the reference (g++ -O2, no -march): the
# encoder's FP64 DFT must round exactly as the reference build does.
CXX_FLAGS = ["-O2", "-fPIC", "-std=c++20", "-pthread", "-I", str(INCLUDE), "-I", str(CUDA_HOME / "include")]


def _deps() -> list[Path]:
    return list(INCLUDE.rglob("*.h")) + list(INCLUDE.rglob("*.hpp")) + list(CSRC.rglob("*.cuh")) + \
        list(CSRC.rglob("*.hpp"))


def _stale(target: Path, sources: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(s.stat().st_mtime > t for s in sources)


def _run(cmd: list[str], verbose: bool) -> None:
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd[:3])} ... ({r.returncode})")
    if verbose and (r.stdout or r.stderr):
        sys.stderr.write(r.stdout + r.stderr)


def build(force: bool = False, verbose: bool = False, jobs: int | None = None) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    deps = _deps()
    cu = sorted(CSRC.glob("*.cu"))
    cpp = sorted((CSRC / "host").glob("*.cpp"))
    jobs_list = []
    objs = []
    for src in cu:
        obj = BUILD / (src.stem + ".cu.o")
        objs.append(obj)
        if force or _stale(obj, [src] + deps):
            jobs_list.append([NVCC, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)])
    for src in cpp:
        obj = BUILD / (src.stem + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + deps):
            jobs_list.append(["g++", *CXX_FLAGS, "-c", str(src), "-o", str(obj)])
    with cf.ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 4) as ex:
        list(ex.map(lambda c: _run(c, verbose), jobs_list))
    if force or _stale(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", str(LIB), *map(str, objs), "-lpthread"], verbose)
    pyb = CSRC / "pybind.cpp"
    if force or _stale(PYMOD, [pyb, LIB] + deps):
        import pybind11

        pyinc = sysconfig.get_paths()["include"]
        _run(["g++", *CXX_FLAGS, "-shared", "-I", pybind11.get_include(), "-I", pyinc, str(pyb), "-o", str(PYMOD),
              "-L", str(PKG), "-ltetris_b200", "-Wl,-rpath,$ORIGIN"], verbose)
    return LIB


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    build(force=a.force, verbose=a.verbose)
    print(f"built {LIB.name} and {PYMOD.name}")


if __name__ == "__main__":
    main()
