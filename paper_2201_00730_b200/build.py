"""Build the sm_100a shared library ``_uot_b200.so`` in-tree with nvcc.

Each ``csrc/*.cu`` is compiled separately (parallel), then linked with NCCL
(the torch-bundled libnccl.so.2; rpath'd so the .so loads anywhere this image
runs).  ``python -m paper_2201_00730_b200.build`` or ``__graft_entry__.build()``.
"""

from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(HERE, "_uot_b200.so")
# Experiment hooks: UOT_NVCC_EXTRA adds nvcc flags (e.g. -DFW_MINB=3) and
# UOT_B200_VARIANT builds _uot_b200_<variant>.so from build_<variant>/ so a
# variant can be loaded side by side (UOT_B200_LIB=... at import time).
VARIANT = os.environ.get("UOT_B200_VARIANT", "")
if VARIANT:
    OUT = os.path.join(HERE, f"_uot_b200_{VARIANT}.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    import importlib.util

    spec = importlib.util.find_spec("nvidia")
    for base in list(spec.submodule_search_locations or []):
        inc = os.path.join(base, "nccl", "include")
        lib = os.path.join(base, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    raise RuntimeError("torch-bundled NCCL headers not found")


def _nvcc():
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def build(verbose=False, force=False):
    srcs = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))
    hdrs = glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + glob.glob(
        os.path.join(ROOT, "include", "*.h"))
    newest = max(os.path.getmtime(p) for p in srcs + hdrs + [__file__])
    if not force and os.path.exists(OUT) and os.path.getmtime(OUT) >= newest:
        return OUT
    inc, lib = _nccl_dirs()
    objdir = os.path.join(HERE, "build" + (f"_{VARIANT}" if VARIANT else ""))
    os.makedirs(objdir, exist_ok=True)
    nvcc = _nvcc()
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-DUOT_WITH_NCCL",
                    "-I" + inc, "--expt-relaxed-constexpr", "-Xptxas", "-v" if verbose else "-O3"]
    flags += os.environ.get("UOT_NVCC_EXTRA", "").split()

    hdr_time = max(os.path.getmtime(p) for p in hdrs + [__file__])

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        if (not force and os.path.exists(obj)
                and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_time)):
            return obj  # up to date (headers are shared, so any header change rebuilds all)
        cmd = [nvcc, "-c", src, "-o", obj] + flags
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
        if verbose and r.stderr:
            sys.stderr.write(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(compile_one, srcs))
    tmp = OUT + ".tmp"
    cmd = [nvcc, "-shared", "-o", tmp] + objs + ARCH + [
        "-L" + lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
