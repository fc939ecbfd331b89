"""Build the sm_100a shared library in-tree: paper_1511_08463_b200/libphasefrac_b200.so.

Each translation unit compiles to its own object (in parallel, rebuilt only when its source or a
shared header changed), then nvcc links the shared library."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = ["pf_core.cu", "pf_ops2d.cu", "pf_strip2.cu", "pf_ops3d.cu", "pf_gmg.cu", "pf_gmg3.cu", "pf_newton.cu",
       "pf_umesh.cu"]
HDR = ["pf_internal.cuh", "pf_elem.cuh", "pf_strip2d.cuh"]
LIB = os.path.join(HERE, "libphasefrac_b200.so")
OBJ = os.path.join(HERE, "_obj")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
                "-Xptxas", "-v"]


def _nvcc():
    return os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def build(verbose=False, force=False):
    srcs = [os.path.join(HERE, "csrc", s) for s in SRC]
    hdrs = [os.path.join(HERE, "csrc", h) for h in HDR] + [
        os.path.join(os.path.dirname(HERE), "include", "phasefrac_b200.h")]
    hdr_t = max(os.path.getmtime(h) for h in hdrs)
    os.makedirs(OBJ, exist_ok=True)
    objs = [os.path.join(OBJ, os.path.splitext(s)[0] + ".o") for s in SRC]
    todo = [(s, o) for s, o in zip(srcs, objs)
            if force or not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(s), hdr_t)]
    if not todo and os.path.exists(LIB) and os.path.getmtime(LIB) >= max(os.path.getmtime(o) for o in objs):
        return LIB

    def compile_one(so):
        s, o = so
        r = subprocess.run([_nvcc()] + FLAGS + ["-c", s, "-o", o + ".tmp"], capture_output=True, text=True)
        if r.returncode == 0:
            os.replace(o + ".tmp", o)
        return s, r

    with ThreadPoolExecutor(max_workers=len(SRC)) as ex:
        results = list(ex.map(compile_one, todo))
    failed = False
    for s, r in results:
        if verbose or r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
        failed |= r.returncode != 0
    if failed:
        raise RuntimeError("nvcc failed building libphasefrac_b200.so")
    r = subprocess.run([_nvcc()] + ARCH + ["-shared", "-Xcompiler", "-fPIC"] + objs + ["-o", LIB + ".tmp"],
                       capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed linking libphasefrac_b200.so")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print(LIB)
