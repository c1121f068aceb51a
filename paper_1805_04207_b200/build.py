"""Build the native pieces in-tree (the .so files travel to the GPU box).

    libaiwc_b200.so   CUDA engine + C ABI   (nvcc, sm_100a only)
    _walker*.so       CPython extension: TraceEvent iterable -> columns + stream validation
"""

from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
CU_SOURCES = ["aiwc_ingest.cu", "aiwc_util.cu", "aiwc_memory.cu", "aiwc_dense.cu", "aiwc_branch.cu", "aiwc_capi.cu", "aiwc_synth.cu",
              "aiwc_validate.cu", "aiwc_sim.cu", "aiwc_exchange.cu", "aiwc_bins.cu"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-lnccl"]  # NCCL: the job-mode collectives (aiwc_ctx_set_comm)
LIB = os.path.join(HERE, "libaiwc_b200.so")
WALKER = os.path.join(HERE, "_walker" + (sysconfig.get_config_var("EXT_SUFFIX") or ".so"))


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_engine(force: bool = False) -> str:
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh", ".h"))]
    deps.append(os.path.join(HERE, "..", "include", "aiwc_b200.h"))
    if force or _stale(LIB, deps):
        nvcc = os.environ.get("NVCC", "nvcc")
        cmd = [nvcc, *NVCC_FLAGS, "-o", LIB + ".tmp", *[os.path.join(CSRC, f) for f in CU_SOURCES]]
        subprocess.check_call(cmd)
        os.replace(LIB + ".tmp", LIB)
    return LIB


def build_walker(force: bool = False) -> str:
    src = os.path.join(CSRC, "walker.cpp")
    if force or _stale(WALKER, [src, os.path.join(HERE, "..", "include", "aiwc_b200.h")]):
        inc = sysconfig.get_paths()["include"]
        cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-shared", f"-I{inc}", "-o", WALKER + ".tmp", src]
        subprocess.check_call(cmd)
        os.replace(WALKER + ".tmp", WALKER)
    return WALKER


def build_all(force: bool = False) -> list[str]:
    return [build_engine(force), build_walker(force)]


if __name__ == "__main__":
    print("\n".join(build_all(force="--force" in sys.argv)))
