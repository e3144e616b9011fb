"""Builds the CUDA library (paper_2406_17248_b200/libsv.so) for sm_100a and the CPU oracle.

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo; the .so is built in-tree so it travels to
the GPU box with the repo snapshot.
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.join(ROOT, "paper_2406_17248_b200")
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsv.so")
SOURCES = ["api.cpp", "gates.cpp", "plan.cpp", "shard.cpp", "kernels.cu", "kernels_reg.cu", "kernels_batch.cu"]
HEADERS = ["sv_internal.h", "sv_handle.h", "cx.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_flags():
    """Link the NCCL that PyTorch loads (the nvidia-nccl wheel, 2.28) rather than the system one
    (2.27): one process can hold only one libnccl.so.2, and torch needs the newer symbols — if this
    library pulled in the system copy first, a later `import torch` would fail."""
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia.nccl")
        for base in (spec.submodule_search_locations or []) if spec else []:
            lib = os.path.join(base, "lib")
            if os.path.exists(os.path.join(lib, "libnccl.so.2")):
                return ["-I", os.path.join(base, "include"), "-L", lib, "-l:libnccl.so.2",
                        "-Xlinker", "-rpath=" + lib]
    except Exception:
        pass
    return ["-lnccl"]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_lib(force=False, verbose=False):
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "sv.h")]
    if not force and not _stale(LIB, deps):
        return LIB
    cmd = [NVCC, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-O2",
           "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-o", LIB, *srcs, *_nccl_flags()]
    cmd[1:1] = os.environ.get("SV_NVCC_DEFS", "").split()  # experiment knobs, e.g. -DSV_DUAL_CTAS=4
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    return LIB


def build_all(force=False):
    build_lib(force=force)
    sys.path.insert(0, ROOT)
    import oracle  # noqa: E402  (test infrastructure; building the checker is not using it)
    oracle.build(force=force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
    print(LIB)
