"""Build the in-tree C-ABI library ``libppf.so`` for sm_100a with nvcc.

    python -m paper_2401_06684_b200.build        (or __graft_entry__.build())

Every CUDA translation unit is compiled with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3``; the host C++ files
go through nvcc's host compiler.  NCCL is the torch-bundled one (same
libnccl.so.2 that torch.distributed loads), linked with an rpath.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "libppf.so")
BUILD = os.path.join(PKG, "_build")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    import nvidia.nccl
    base = list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    return "nvcc"


def build(verbose: bool = False, force: bool = False) -> str:
    inc, lib = _nccl_dirs()
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    hdrs = glob.glob(os.path.join(CSRC, "*.h")) + [os.path.join(ROOT, "include", "ppf.h")]
    newest = max(os.path.getmtime(p) for p in srcs + hdrs + [__file__])
    if not force and os.path.exists(OUT) and os.path.getmtime(OUT) >= newest:
        return OUT
    os.makedirs(BUILD, exist_ok=True)
    nvcc = _nvcc()
    common = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"),
              "-I", inc]
    objs = []
    cmds = []
    for s in srcs:
        o = os.path.join(BUILD, os.path.basename(s) + ".o")
        objs.append(o)
        cmd = [nvcc, *ARCH, "-lineinfo", *common, "-c", s, "-o", o]
        if s.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        else:
            # host C++: complex multiply/divide inline (no __muldc3 inf/nan
            # recovery calls) -- the host dense kernels (dense.cpp) are built
            # on std::complex and are 5-10x slower otherwise
            cmd += ["-Xcompiler", "-fcx-fortran-rules"]
        cmds.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        if verbose and (r.stdout or r.stderr):
            sys.stderr.write(r.stdout + r.stderr)

    with ThreadPoolExecutor(len(cmds)) as ex:
        list(ex.map(run, cmds))
    link = [nvcc, *ARCH, "-shared", "-o", OUT + ".tmp", *objs, "-L", lib, "-l:libnccl.so.2",
            "-Xlinker", f"-rpath,{lib}", "-lcudart"]
    run(link)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
