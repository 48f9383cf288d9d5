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


def build(force: bool = False, verbose: bool = False, defines: tuple = (), out: Path | None = None) -> Path:
    """Compile every CUDA source into one shared library next to this file.  `defines` /
    `out` build a diagnostics variant elsewhere (e.g. -DCB_MBAR_HINT into _ab/, loaded with
    CB_LIB_PATH for A/B runs)."""
    lib_out = Path(out) if out else LIB
    if not force and not defines and not _stale():
        return LIB
    objdir = PKG / ("_build" if not defines else "_build_" + "_".join(d.strip("-D") for d in defines))
    objdir.mkdir(exist_ok=True)
    common = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-I", str(ROOT / "include"), "-I", str(CSRC), "--expt-relaxed-constexpr",
              "-Xptxas", "-v" if verbose else "-O3", *defines]
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
    lib_out.parent.mkdir(parents=True, exist_ok=True)
    tmp = lib_out.with_suffix(".so.tmp")
    # only the C ABI (cb_*) is exported: the static cudart and the C++ internals stay private
    vscript = objdir / "exports.map"
    vscript.write_text("{ global: cb_*; local: *; };\n")
    cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-Xlinker", "--exclude-libs,ALL",
           "-Xlinker", f"--version-script={vscript}", "-o", str(tmp), *objs, "-lcuda"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, lib_out)
    return lib_out


def trace_lib() -> Path:
    """The diagnostics build with the per-CTA timelines compiled in (-DCB_TRACE), for the
    trace tools (CB_LIB_PATH)."""
    out = ROOT / "_ab" / "libconvb200_trace.so"
    srcs = [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "convb200.h", Path(__file__)]
    if out.exists() and out.stat().st_mtime > max(p.stat().st_mtime for p in srcs):
        return out
    return build(defines=("-DCB_TRACE",), out=out)


if __name__ == "__main__":
    p = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(p)
