"""Build the in-tree CUDA library libxa_b200.so for sm_100a (no JIT cache).

    python -m paper_2503_03479_b200.build          # or __graft_entry__.build()

nvcc compiles the kernels and the C-ABI engine straight to
paper_2503_03479_b200/libxa_b200.so; the .so is git-ignored but travels to the
GPU box with the repo snapshot. Host code is compiled with -ffp-contract=off
so the view geometry reproduces the reference's double arithmetic exactly.
"""
from __future__ import annotations

import os
import pathlib
import shutil
import subprocess
import sys

PKG = pathlib.Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libxa_b200.so"
SOURCES = ["xa_warp.cu", "xa_orb.cu", "xa_match.cu", "xa_sift.cu", "xa_engine.cu", "xa_multi.cu",
           "xa_image_io.cpp", "xa_homography.cpp"]
# per-file flags: the SIFT replay needs every float op rounded separately
FILE_FLAGS = {"xa_sift.cu": ["--fmad=false"]}
DEPS = SOURCES + ["xa_common.cuh", "xa_kernels.h", "xa_geometry.h", "orb_pattern.inc",
                  "trig_fixups.inc"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and pathlib.Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    hdr = PKG.parent / "include" / "xaffine_b200.h"
    return any((CSRC / f).stat().st_mtime > t for f in DEPS) or hdr.stat().st_mtime > t


def build(force: bool = False, verbose: bool = False, defines=(), out: pathlib.Path = None) -> pathlib.Path:
    """defines/out: A/B variants (tools/build_variant.py) go to build/variants/,
    never to the product library path."""
    lib = pathlib.Path(out) if out else LIB
    if not force and not out and not needs_build():
        return LIB
    objdir = PKG.parent / "build" / ("obj" if not out else "obj_" + lib.stem)
    objdir.mkdir(parents=True, exist_ok=True)
    common = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-ffp-contract=off", "-Xptxas", "-warn-spills",
              *[f"-D{d}" for d in defines]]
    objs = []
    procs = []
    for src in SOURCES:
        obj = objdir / (src + ".o")
        cmd = common + FILE_FLAGS.get(src, []) + ["-c", str(CSRC / src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd))
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                            text=True)))
        objs.append(str(obj))
    failed = []
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            failed.append(f"--- {src}\n{out}")
        elif out.strip() and verbose:
            print(out)
    if failed:
        raise RuntimeError("nvcc failed:\n" + "\n".join(failed))
    lib.parent.mkdir(parents=True, exist_ok=True)
    tmp = lib.with_suffix(".so.tmp")
    link = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *objs, "-ldl", "-lz"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n" + r.stdout + r.stderr)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
