"""Build libbitdelta_b200.so in-tree for sm_100a (nvcc; no torch JIT cache).

    python -m paper_2402_10193_b200.build [--force]

Objects go to paper_2402_10193_b200/_build/, the shared library next to this
file (both git-ignored; the .so travels to the GPU box with the snapshot).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libbitdelta_b200.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dir() -> str:
    """NCCL 2.28 shipped with torch (nvidia-nccl wheel): headers + libnccl.so.2."""
    import importlib.util

    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        d = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("NCCL headers not found (expected site-packages/nvidia/nccl)")


NCCL = _nccl_dir()
FLAGS = ["-O3", "-std=c++20", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", f"-I{INCLUDE}", f"-I{CSRC}", f"-I{NCCL}/include"]
LDFLAGS = [f"-L{NCCL}/lib", "-l:libnccl.so.2", f"-Xlinker=-rpath={NCCL}/lib"]


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    hs += [os.path.join(INCLUDE, "bitdelta", f) for f in os.listdir(os.path.join(INCLUDE, "bitdelta"))]
    return hs


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    if _stale(obj, [src] + _headers()):
        cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
        if src.endswith(".cpp"):
            cmd = [NVCC, *ARCH, *FLAGS, "-x", "cu", "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        log = os.path.join(OBJ, os.path.basename(src) + ".ptxas.txt")
        with open(log, "w") as f:
            f.write(r.stderr)
        if verbose:
            print(f"[build] {os.path.basename(src)}", file=sys.stderr)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = _sources()
    if force:
        for f in os.listdir(OBJ):
            os.remove(os.path.join(OBJ, f))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if force or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, *LDFLAGS]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    _build_cpp_test(force)
    return LIB


def _build_cpp_test(force: bool) -> None:
    """tests/cpp/test_deltakit_gpu: the deltakit_gpu C++ mirror's parity program."""
    root = os.path.dirname(HERE)
    src = os.path.join(root, "tests", "cpp", "test_deltakit_gpu.cpp")
    out = os.path.join(root, "tests", "cpp", "test_deltakit_gpu")
    if not os.path.exists(src):
        return
    hdr = os.path.join(INCLUDE, "deltakit_gpu", "deltakit_gpu.hpp")
    if not force and not _stale(out, [src, hdr, LIB]):
        return
    cmd = ["g++", "-std=c++20", "-O2", f"-I{INCLUDE}", "-I/usr/local/cuda/include", src, f"-L{HERE}",
           "-lbitdelta_b200", "-Wl,-rpath,$ORIGIN/../../paper_2402_10193_b200", "-L/usr/local/cuda/lib64",
           "-lcudart", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"C++ shim test build failed:\n{r.stderr}")


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
