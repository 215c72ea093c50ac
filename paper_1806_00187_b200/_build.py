"""Build the product library (libsmpu.so) and the GPU input generator for sm_100a, in-tree."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def nccl_paths():
    import nvidia.nccl
    base = list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def _run(cmd):
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=ROOT)


def build_smpu(verbose_ptxas=False):
    inc, lib = nccl_paths()
    cmd = [NVCC, *ARCH, "-O3", "-std=c++17", "-lineinfo", "-shared", "-Xcompiler", "-fPIC,-ffp-contract=off",
           "-I", os.path.join(ROOT, "include"), "-I", inc,
           os.path.join(PKG, "csrc", "smpu.cu"), "-o", os.path.join(PKG, "libsmpu.so"),
           "-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{lib}"]
    if verbose_ptxas:
        cmd += ["-Xptxas", "-v"]
    if os.environ.get("SMPU_L2_HINT"):      # experiment builds only (kernels.cuh)
        cmd += [f"-DSMPU_L2_HINT={int(os.environ['SMPU_L2_HINT'])}"]
    _run(cmd)


def build_synth_gpu():
    _run([NVCC, *ARCH, "-O3", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
          os.path.join(ROOT, "synth", "synth_gpu.cu"), "-o", os.path.join(ROOT, "synth", "libsynth_gpu.so")])


def build_sched():
    _run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-I", os.path.join(ROOT, "include"),
          os.path.join(PKG, "csrc", "sched.cpp"), "-o", os.path.join(PKG, "libsmpu_sched.so")])


def build_all():
    build_smpu()
    build_sched()
    build_synth_gpu()


if __name__ == "__main__":
    build_smpu(verbose_ptxas="-v" in sys.argv)
    build_sched()
    build_synth_gpu()
