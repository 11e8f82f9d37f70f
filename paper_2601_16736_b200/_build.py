"""Build the sm_100a shared library in-tree with nvcc (no JIT cache).

``python -m paper_2601_16736_b200._build`` or ``__graft_entry__.build()``.
The product is ``paper_2601_16736_b200/libadamw_gs_b200.so`` exporting the
C ABI declared in ``include/adamw_gs.h``.
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
LIB = PKG / "libadamw_gs_b200.so"
SOURCES = ("gs_abi.cu", "gs_compact.cu", "gs_step.cu", "gs_step_rows.cu", "gs_step_sh3.cu",
           "gs_step_sh3_m_coupled.cu", "gs_step_sh3_m_sparse.cu", "gs_step_sh3_m_const.cu",
           "gs_step_sh3_m_const_clip.cu", "gs_step_sh3_m_adamw_gs.cu", "gs_state.cu",
           "gs_noise.cu", "gs_rng.cu")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
    "-Xfatbin", "-compress-all",
]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not LIB.exists():
        return True
    mtime = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + [ROOT / "include" / "adamw_gs.h"]
    return any(d.stat().st_mtime > mtime for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    build_dir = PKG / "build"
    build_dir.mkdir(exist_ok=True)
    nvcc = nvcc_path()

    def compile_one(src: str) -> str:
        obj = build_dir / (Path(src).stem + ".o")
        # GS_NVCC_EXTRA: measurement builds only (e.g. -DGS_TRACE=1, -DGS_BUILD_VARIANTS=1)
        extra = os.environ.get("GS_NVCC_EXTRA", "").split()
        cmd = [nvcc, *NVCC_FLAGS, *extra, "-I", str(ROOT / "include"), "-c", str(CSRC / src), "-o",
               str(obj)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}")
        return str(obj)

    # translation units compile in parallel (the SH-3 kernels are split per mode)
    workers = max(1, min(len(SOURCES), os.cpu_count() or 1))
    with ThreadPoolExecutor(max_workers=workers) as pool:
        objs = list(pool.map(compile_one, SOURCES))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(tmp), *objs,
           "-lcudart_static", "-Xcompiler", "-fPIC"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
