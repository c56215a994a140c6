"""Build libbtp.so in-tree with nvcc for sm_100a (no JIT cache, no torch build system).

The shared library is the product's C-ABI boundary (include/btp.h); it is loaded by
`paper_2512_12131_b200._native` through ctypes. Objects are rebuilt only when a source
or header is newer than the library.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
LIB_DIR = PKG / "_lib"
LIB = LIB_DIR / "libbtp.so"
SOURCES = ("gemm.cu", "gemm_f32.cu", "rowops.cu", "modelops.cu", "peer.cu", "attn.cu", "capi.cu")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h"))
    deps += list(INCLUDE.glob("*.h"))
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    LIB_DIR.mkdir(exist_ok=True)
    nvcc = _nvcc()
    objs = []
    common = ARCH + [
        "-O3",
        "-std=c++17",
        "-lineinfo",
        "-Xcompiler",
        "-fPIC",
        "-I",
        str(INCLUDE),
        "--expt-relaxed-constexpr",
    ]
    if verbose:
        common += ["-Xptxas", "-v"]
    from concurrent.futures import ThreadPoolExecutor

    def compile_one(src):
        obj = LIB_DIR / (Path(src).stem + ".o")
        subprocess.run([nvcc, "-c", str(CSRC / src), "-o", str(obj)] + common, check=True)
        return str(obj)

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as pool:
        objs = list(pool.map(compile_one, SOURCES))
    tmp = LIB.with_suffix(".so.tmp")
    subprocess.run([nvcc, "-shared", "-o", str(tmp)] + objs + ARCH, check=True)
    os.replace(tmp, LIB)
    for o in objs:
        try:
            os.remove(o)
        except OSError:
            pass
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
