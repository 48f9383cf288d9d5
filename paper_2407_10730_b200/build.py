"""Build libconvb200.so in-tree with nvcc for sm_100a (no JIT cache, so it travels).

    python -m paper_2407_10730_b200.build        # or build() from __graft_entry__
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libconvb200.so"
SOURCES = ["capi.cu", "pack_kernels.cu", "conv_tc.cu", "conv_tma.cu", "conv_ts.cu", "conv_gemm_ts.cu", "conv_ffma.cu"]
HEADERS = ["cb_common.cuh", "sm100_ptx.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "convb200.h", Path(__file__)]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile every CUDA source into one shared library next to this file."""
    if not force and not _stale():
        return LIB
    objdir = PKG / "_build"
    objdir.mkdir(exist_ok=True)
    common = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-I", str(ROOT / "include"), "-I", str(CSRC), "--expt-relaxed-constexpr",
              "-Xptxas", "-v" if verbose else "-O3"]
    shared = [CSRC / h for h in HEADERS] + [ROOT / "include" / "convb200.h", Path(__file__)]
    newest_shared = max(p.stat().st_mtime for p in shared)

    def compile_one(src: str) -> str:
        obj = objdir / (Path(src).stem + ".o")
        if (not force and obj.exists() and obj.stat().st_mtime > newest_shared
                and obj.stat().st_mtime > (CSRC / src).stat().st_mtime):
            return str(obj)  # object is newer than its source and every shared header
        cmd = [*common, "-c", str(CSRC / src), "-o", str(obj)]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr, file=sys.stderr)
        return str(obj)

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = LIB.with_suffix(".so.tmp")
    # only the C ABI (cb_*) is exported: the static cudart and the C++ internals stay private
    vscript = objdir / "exports.map"
    vscript.write_text("{ global: cb_*; local: *; };\n")
    cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-Xlinker", "--exclude-libs,ALL",
           "-Xlinker", f"--version-script={vscript}", "-o", str(tmp), *objs, "-lcuda"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    p = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(p)
