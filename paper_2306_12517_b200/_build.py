"""Build libbbx.so in-tree (nvcc for sm_100a + g++ for the host engine).

No JIT cache: the .so lands next to this file so it travels to the GPU box
with the repo snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
LIB = HERE / "libbbx.so"
BUILD = HERE / "_build_obj"

CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = shutil.which("nvcc") or f"{CUDA_HOME}/bin/nvcc"
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]
CXX = os.environ.get("CXX", "g++")

HOST_SOURCES = ["engine.cpp", "format.cpp", "orders.cpp", "jpeg_host.cpp"]
CUDA_SOURCES = ["kernels.cu", "kernels_img_u8.cu", "kernels_img_f32.cu", "kernels_img_f16.cu", "kernels_img_bf16.cu", "jpeg.cu"]
HEADERS = ["bbx_internal.h", "engine.h", "image_kernel.cuh", "jpeg.h"]


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in HOST_SOURCES + CUDA_SOURCES + HEADERS] + [HERE.parent / "include" / "bbx.h",
                                                                       Path(__file__)]
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines: tuple = (), out: Path | None = None) -> Path:
    """Compile libbbx.so.  `defines` / `out`: A/B builds of compile-time constants
    (e.g. ("BBX_CW_STAGES=3",)) into another file, for measurement scripts only."""
    lib = Path(out) if out else LIB
    if not force and not defines and out is None and not _stale():
        return LIB
    build_dir = BUILD if not defines else BUILD.with_name(BUILD.name + "_" + "_".join(d.replace("=", "") for d in defines))
    build_dir.mkdir(exist_ok=True)
    (build_dir / "ptxas.log").write_text("")
    dflags = [f"-D{d}" for d in defines]
    inc = ["-I", str(CSRC), "-I", str(HERE.parent / "include"), "-I", f"{CUDA_HOME}/include"]
    jobs = []
    for src in CUDA_SOURCES:
        obj = build_dir / (src + ".o")
        jobs.append((obj, [NVCC, *GENCODE, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                           *dflags, *inc, "-c", str(CSRC / src), "-o", str(obj)]))
    for src in HOST_SOURCES:
        obj = build_dir / (src + ".o")
        # -ffp-contract=off: the host-side proof of the divide-free normalize
        # (verify_fma_normalize) needs one IEEE subtract + one IEEE divide,
        # never a contracted FMA (pipeline.py:158-160).
        jobs.append((obj, [CXX, "-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-Wall",
                           "-Wno-format-security", *dflags, *inc, "-c", str(CSRC / src), "-o", str(obj)]))
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        list(ex.map(lambda j: _run(j[1], verbose, build_dir), jobs))
    objs = [o for o, _ in jobs]
    tmp = lib.with_suffix(".so.tmp")
    cmd = [NVCC, *GENCODE, "-shared", "-o", str(tmp), *map(str, objs), "-lpthread", "-Xcompiler", "-fPIC"]
    _run(cmd, verbose, build_dir)
    os.replace(tmp, lib)
    return lib


def _run(cmd, verbose, build_dir=BUILD):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or r.returncode:
        print(" ".join(cmd))
        print(r.stdout[-4000:], r.stderr[-8000:])
    if r.returncode:
        raise RuntimeError(f"build step failed: {cmd[0]} {cmd[-3] if len(cmd) > 3 else ''}")
    (build_dir / "ptxas.log").open("a").write(r.stderr)


if __name__ == "__main__":
    import sys
    build(force="--force" in sys.argv, verbose=True)
