#!/usr/bin/env python
"""Write tests/golden/fullsize/<key>.npz: the ORACLE's results on the full
BASELINE.json workloads (tests/fullsize_oracle.py; calls only oracle/ and the
seeded generators in inputs/, never the CUDA path).

    python tools/make_fullsize_goldens.py [KEY ...]     # default: all keys
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from tests import fullsize_oracle as fo  # noqa: E402


def main():
    keys = sys.argv[1:] or list(fo.KEYS)
    for key in keys:
        t0 = time.perf_counter()
        d = fo.compute(key, log=lambda s: print(s, flush=True))
        p = fo.save(d)
        print(f"{key}: wrote {os.path.relpath(p, ROOT)} ({os.path.getsize(p) / 1e6:.2f} MB, "
              f"{time.perf_counter() - t0:.0f} s, {d['threads']} threads)", flush=True)


if __name__ == "__main__":
    main()
