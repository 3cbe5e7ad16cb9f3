"""Builds libfuseplan_b200.so in-tree: C++20 host (planner, executor, C ABI)
plus the sm_100a CUDA kernels, linked against the static CUDA runtime.

    python -m paper_1509_04394_b200.build        # incremental
    python -m paper_1509_04394_b200.build --force

nvcc cross-compiles for sm_100a without a GPU, so this runs in the CPU
container; the built .so travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_build")
# A/B tuning builds: FUSEPLAN_NVCC_EXTRA="-DFP_NF=5 -DFP_NI=6" and
# FUSEPLAN_BUILD_TAG=nf5 build _build_nf5/ + libfuseplan_b200_nf5.so, loaded
# with FUSEPLAN_LIB=<path> (never the shipped library)
_TAG = os.environ.get("FUSEPLAN_BUILD_TAG", "")
if _TAG:
    OBJ = os.path.join(PKG, "_build_" + _TAG)
LIB = os.path.join(PKG, "libfuseplan_b200" + ("_" + _TAG if _TAG else "") + ".so")

CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
CXX = "/usr/bin/g++"
JSON_DIR = os.environ.get(
    "FUSEPLAN_JSON_DIR",
    "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/"
    "thirdparty/nlohmann")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# No fast-math and no implicit contraction: the exact kernels spell out every
# rounding with intrinsics; -fmad=false guards any plain float expression.
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-fmad=false",
                     "-Xcompiler", "-fPIC", "-Xptxas", "-warn-spills"] + \
    os.environ.get("FUSEPLAN_NVCC_EXTRA", "").split()
CXX_FLAGS = ["-std=c++20", "-O2", "-fPIC", "-ffp-contract=off", "-Wall",
             "-Wno-unused-function", f"-I{os.path.join(ROOT, 'include')}", f"-I{JSON_DIR}",
             f"-I{CUDA_HOME}/include"]

HOST_SRCS = ["host/model.cpp", "host/planner.cpp", "host/video.cpp",
             "host/exec.cpp", "host/capi.cpp",
             "host/calibrate.cpp", "host/shard.cpp", "host/simulate.cpp"]
CUDA_SRCS = ["kernels/fc_exact.cu", "kernels/fc_pipe.cu", "kernels/fc_pipe2.cu", "kernels/fc_f12.cu",
             "kernels/fc_track.cu", "kernels/fc_tiled.cu", "kernels/fc_shard.cu",
             "kernels/fc_dispatch.cu"]
HEADERS = ["kernels/fc_pipe.cu", "host/exec.hpp", "host/video.hpp",
           "kernels/fc_kernels.h", "kernels/fc_common.cuh", "kernels/fc_sobel.cuh"]
PUBLIC_HEADERS = ["fuseplan.h", "fuseplan/fuseplan.hpp", "fuseplan/video.hpp",
                  "fuseplan/simulator.hpp"]


def _newest_header() -> float:
    ts = [os.path.getmtime(os.path.join(CSRC, h)) for h in HEADERS
          if os.path.exists(os.path.join(CSRC, h))]
    ts += [os.path.getmtime(os.path.join(ROOT, "include", h)) for h in PUBLIC_HEADERS]
    return max(ts)


def _compile(src: str, force: bool) -> str:
    path = os.path.join(CSRC, src)
    obj = os.path.join(OBJ, src.replace("/", "_") + ".o")
    if (not force and os.path.exists(obj)
            and os.path.getmtime(obj) >= max(os.path.getmtime(path), _newest_header())):
        return obj
    if src.endswith(".cu"):
        cmd = [NVCC] + NVCC_FLAGS + ["-c", path, "-o", obj]
    else:
        cmd = [CXX] + CXX_FLAGS + ["-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if r.stderr.strip():
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = HOST_SRCS + CUDA_SRCS
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), srcs))
    if (force or not os.path.exists(LIB)
            or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs)):
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs + [
            "-Xlinker", "--no-undefined", "-lpthread", "-ldl", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(LIB)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    a = ap.parse_args()
    build(force=a.force, verbose=True)
