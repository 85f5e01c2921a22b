"""Build the sm_100a CUDA library (libdeltaserve_b200.so) in-tree with nvcc.

No JIT cache: the .so lives next to this file so it travels with the repo
snapshot to the GPU box (it is git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
# DS_LIB_OUT / DS_NVCC_EXTRA: an instrumented or A/B variant built elsewhere
# (e.g. -DDS_K7_TRACE); the default is the in-tree product library
LIB = os.environ.get("DS_LIB_OUT") or os.path.join(HERE, "libdeltaserve_b200.so")
BUILD = os.path.join(os.path.dirname(LIB), "_build") if os.environ.get("DS_LIB_OUT") else \
    os.path.join(HERE, "_build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include")] + os.environ.get("DS_NVCC_EXTRA", "").split()

SOURCES = ["policy.cu", "kvmeta.cu", "layers.cu", "attn_dispatch.cu", "attn_decode.cu",
           "attn_decode_tc.cu", "attn_prefill_sm100.cu", "gemm_skinny.cu",
           "gemm_stream.cu", "gemm_pair.cu", "tma.cu",
           "runtime.cu"]


def _deps_mtime() -> float:
    paths = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    paths.append(os.path.join(ROOT, "include", "deltaserve_b200.h"))
    return max(os.path.getmtime(p) for p in paths)


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(BUILD, src.replace(".cu", ".o"))
    cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{res.stderr}")
    if verbose and res.stderr:
        sys.stderr.write(res.stderr)
    return obj


HOST_SRC = os.path.join(HERE, "csrc_host", "hostcore.cpp")


def host_lib_path() -> str:
    import sysconfig

    return os.path.join(HERE, "_hostcore" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_host(force: bool = False) -> str:
    """The native host core (radix trie + cell allocator, pybind11) - g++,
    in-tree next to the CUDA library."""
    import sysconfig

    import pybind11

    out = host_lib_path()
    if not force and os.path.exists(out) and os.path.getmtime(out) >= os.path.getmtime(HOST_SRC):
        return out
    tmp = out + ".tmp"
    cmd = ["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-fvisibility=hidden",
           "-I" + pybind11.get_include(), "-I" + sysconfig.get_paths()["include"], HOST_SRC,
           "-o", tmp]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"g++ failed for hostcore.cpp:\n{res.stderr}")
    os.replace(tmp, out)
    return out


def build(force: bool = False, verbose: bool = False) -> str:
    if not os.environ.get("DS_LIB_OUT"):  # variant builds: the CUDA library only
        build_host(force)
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _deps_mtime():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), SOURCES))
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-L/usr/local/cuda/lib64", "-lcublas", "-lcublasLt", "-lcudart",
           "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
