"""Build libbq.so (sm_100a) in-tree with nvcc.

The product library is compiled straight from ``csrc/*.cu`` into
``paper_2307_02043_b200/lib/libbq.so`` so that it travels with the repo
snapshot to the GPU box (no JIT cache, no site-packages install).

    python -m paper_2307_02043_b200.build          # incremental
    python -m paper_2307_02043_b200.build --force  # rebuild everything
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "lib"
OBJDIR = PKG / "build_obj"
INCLUDE = PKG.parent / "include"
LIB = LIBDIR / "libbq.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-lineinfo",
    "-Xcompiler",
    "-fPIC",
    "-Xcompiler",
    "-fvisibility=hidden",
    "-rdc=false",
]


def _cuda_home() -> Path:
    for cand in (os.environ.get("CUDA_HOME"), "/usr/local/cuda"):
        if cand and Path(cand, "bin", "nvcc").exists():
            return Path(cand)
    nvcc = shutil.which("nvcc")
    if nvcc:
        return Path(nvcc).resolve().parent.parent
    raise RuntimeError("nvcc not found: set CUDA_HOME")


def _headers(src: Path) -> list[Path]:
    return sorted(CSRC.glob("*.cuh")) + [INCLUDE / "bq.h"]


def _needs(obj: Path, deps: list[Path]) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, jobs: int | None = None) -> Path:
    cuda = _cuda_home()
    nvcc = str(cuda / "bin" / "nvcc")
    OBJDIR.mkdir(exist_ok=True)
    LIBDIR.mkdir(exist_ok=True)
    srcs = sorted(CSRC.glob("*.cu"))
    if not srcs:
        raise RuntimeError(f"no CUDA sources under {CSRC}")
    objs = []
    todo = []
    for src in srcs:
        obj = OBJDIR / (src.stem + ".o")
        objs.append(obj)
        if force or _needs(obj, [src] + _headers(src)):
            extra = os.environ.get("BQ_NVCC_EXTRA", "").split()
            cmd = [nvcc, *ARCH, *NVCC_FLAGS, *extra, "-I", str(INCLUDE), "-c", str(src), "-o", str(obj)]
            if verbose:
                cmd += ["-Xptxas", "-v"]
            todo.append((src, cmd))

    def run(item):
        src, cmd = item
        res = subprocess.run(cmd, capture_output=True, text=True)
        return src, cmd, res

    with cf.ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 4) as ex:
        for src, cmd, res in ex.map(run, todo):
            if verbose and res.stderr:
                sys.stderr.write(res.stderr)
            if res.returncode != 0:
                raise RuntimeError(
                    f"nvcc failed on {src.name}:\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}"
                )
    if force or todo or _needs(LIB, objs):
        libdir = cuda / "lib64"
        cmd = [
            nvcc,
            *ARCH,
            "-shared",
            "-o",
            str(LIB),
            *map(str, objs),
            "-L",
            str(libdir),
            "-lcufft",
            "-Xlinker",
            f"-rpath={libdir}",
        ]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    return LIB


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    args = ap.parse_args(argv)
    print(build(force=args.force, verbose=args.verbose))


if __name__ == "__main__":
    main()
