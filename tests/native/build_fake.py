"""TEST INFRASTRUCTURE: link ``tests/native/libppf_fakenccl.so`` -- the product's
own object files (paper_2401_06684_b200/_build/*.o, built by build.py) with
tests/native/fake_nccl.cpp in place of libnccl.so.2, so that several processes
can drive the library's NCCL code path on one GPU (tests/test_gpu_multirank.py).
The product libppf.so is never touched."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "libppf_fakenccl.so")


def build() -> str:
    from paper_2401_06684_b200 import build as pb
    pb.build()
    objs = sorted(o for o in glob.glob(os.path.join(pb.BUILD, "*.o")) if ".test." not in o)
    if not objs:                      # libppf.so present but its objects are not
        pb.build(force=True)
        objs = sorted(o for o in glob.glob(os.path.join(pb.BUILD, "*.o")) if ".test." not in o)
    src = os.path.join(HERE, "fake_nccl.cpp")
    newest = max(os.path.getmtime(p) for p in objs + [src, pb.OUT])
    if os.path.exists(OUT) and os.path.getmtime(OUT) >= newest:
        return OUT
    inc, _ = pb._nccl_dirs()
    nvcc = pb._nvcc()
    fobj = os.path.join(pb.BUILD, "fake_nccl.test.o")
    for cmd in ([nvcc, "-O2", "-std=c++17", "-Xcompiler", "-fPIC", "-I", inc, "-c", src, "-o", fobj],
                [nvcc, *pb.ARCH, "-shared", "-o", OUT + ".tmp", *objs, fobj, "-lcudart",
                 # bind the library's nccl* calls to the fake even if torch has
                 # already loaded the real libnccl.so.2 into the process
                 "-Xlinker", "-Bsymbolic"]):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("fake NCCL build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build())
