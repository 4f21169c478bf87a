"""Build libfembatch_b200.so in-tree (sm_100a kernels + C ABI + C++ API).

    python -m paper_1103_0066_b200.build [--force] [--verbose]

nvcc cross-compiles for sm_100a without a GPU.  Objects go to build/, the
shared library next to this file so it travels with the repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(ROOT, "build", "fembatch_b200")
LIB = os.path.join(HERE, "libfembatch_b200.so")

CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = shutil.which("nvcc") or os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CU_SOURCES = [
    "fb_kernels_f32_2d.cu",
    "fb_kernels_f32_3d.cu",
    "fb_kernels_f64_2d.cu",
    "fb_kernels_f64_3d.cu",
    "fb_pack.cu",
    "fb_assemble.cu",
    "fb_plan.cu",
    "fb_assemble_g.cu",
]
CPP_SOURCES = ["fb_capi.cpp", "fb_assembly.cpp", "fb_host.cpp", "fembatch_api.cpp", "fembatch_records.cpp"]
CU_HOST_SOURCES = ["fb_tma.cpp"]  # host code that includes the kernel headers (nvcc)
HEADERS = ["fb_internal.h", "fb_kernels.cuh", "fb_launch.cuh", "fb_host.h", "fb_capi_util.h", "fb_asm_store.cuh",
           "fb_devcache.h"]
PUBLIC_HEADERS = [os.path.join(ROOT, "include", "fembatch_b200.h"),
                  os.path.join(ROOT, "include", "fembatch_b200.hpp")]


def _newest(paths):
    return max(os.path.getmtime(p) for p in paths)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build step failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r.stdout + r.stderr


def build(force: bool = False, verbose: bool = False, defines=(), out: str = LIB) -> str:
    """Build the library.  `defines` (e.g. ["FB_PIPE=1"]) and `out` exist for
    same-box A/B experiments (tools/kbench.py with FB_LIB=<path>)."""
    srcs = [os.path.join(CSRC, s) for s in CU_SOURCES + CU_HOST_SOURCES + CPP_SOURCES + HEADERS] + PUBLIC_HEADERS
    if not force and os.path.exists(out) and os.path.getmtime(out) >= _newest(srcs + [__file__]):
        return out
    # A/B builds keep their objects out of the repo snapshot
    build_dir = BUILD if out == LIB else os.path.join("/tmp", "fembatch_build_" + os.path.basename(out).replace(".so", ""))
    os.makedirs(build_dir, exist_ok=True)
    dflags = [f"-D{d}" for d in defines]
    inc = ["-I", CSRC, "-I", os.path.join(ROOT, "include")]
    jobs = []
    for s in CU_SOURCES:
        obj = os.path.join(build_dir, s + ".o")
        jobs.append((obj, [NVCC, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
                           "-Xptxas", "-v", *dflags, *inc, "-c", os.path.join(CSRC, s), "-o", obj]))
    for s in CU_HOST_SOURCES:
        obj = os.path.join(build_dir, s + ".o")
        jobs.append((obj, [NVCC, *ARCH, "-O3", "-std=c++17", "-x", "cu", "-Xcompiler", "-fPIC",
                           *dflags, *inc, "-c", os.path.join(CSRC, s), "-o", obj]))
    for s in CPP_SOURCES:
        obj = os.path.join(build_dir, s + ".o")
        jobs.append((obj, ["g++", "-std=c++20", "-O2", "-fPIC", "-ffp-contract=off", "-pthread",
                           "-I", os.path.join(CUDA_HOME, "include"), *dflags, *inc,
                           "-c", os.path.join(CSRC, s), "-o", obj]))
    logs = []
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        logs.extend(ex.map(lambda j: _run(j[1], verbose), jobs))
    with open(os.path.join(build_dir, "ptxas.log"), "w") as f:
        f.write("\n".join(logs))
    tmp = out + ".tmp"
    _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *[j[0] for j in jobs],
          "-Xlinker", "--no-undefined", "-lpthread", "-ldl", "-lrt"], verbose)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv, defines=defs,
                out=outs[0] if outs else LIB))
