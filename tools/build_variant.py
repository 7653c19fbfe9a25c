"""Build an A/B variant of libbitdelta_b200.so with extra nvcc defines (experiments only).

    python tools/build_variant.py NAME -DBD_LUT_PF=2 -DBD_LUT_REGS=112

Objects go to _ab/NAME/, the library to _ab/libbitdelta_NAME.so (git-ignored as *.so, travels
to the GPU box with the snapshot). Select it at run time with BD_LIB=_ab/libbitdelta_NAME.so.
"""
import concurrent.futures as cf
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2402_10193_b200 import build as B  # noqa: E402


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    obj_dir = os.path.join(ROOT, "_ab", name)
    os.makedirs(obj_dir, exist_ok=True)
    lib = os.path.join(ROOT, "_ab", f"libbitdelta_{name}.so")

    def comp(src):
        obj = os.path.join(obj_dir, os.path.basename(src) + ".o")
        cmd = [B.NVCC, *B.ARCH, *B.FLAGS, *defs]
        if src.endswith(".cpp"):
            cmd += ["-x", "cu"]
        r = subprocess.run(cmd + ["-c", src, "-o", obj], capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(r.stderr)
        open(obj + ".ptxas.txt", "w").write(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(8) as ex:
        objs = list(ex.map(comp, B._sources()))
    r = subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", lib, *objs, *B.LDFLAGS], capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(r.stderr)
    print(lib)


if __name__ == "__main__":
    main()
