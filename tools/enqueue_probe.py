#!/usr/bin/env python
"""Host enqueue cost of one sharded SpMV (ppf_spmv on a row slab: halo push
on the communication stream, diagonal block, stream wait on the peers'
arrival counters, halo block) -- the work ppf_run repeats 2 deg + 1 times per
step.  R ranks are emulated as R contexts of this process on one GPU (as in
tests/test_gpu_peer.py), one host thread each; every thread times K calls
that only enqueue (no synchronisation inside the loop), minus the cost of a
bare ctypes call.  The device time per call of the same slab alone (one rank,
the diagonal block's size) is printed next to it.

    python tools/enqueue_probe.py C4 8
"""
import os
import sys
import threading
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2401_06684_b200 as pp  # noqa: E402
from paper_2401_06684_b200 import _lib  # noqa: E402
from inputs import configs  # noqa: E402
from tests.test_gpu_peer import _make_ranks  # noqa: E402


def main(name, world, K=32, reps=5):
    cfg = configs.CONFIGS[name]
    A, b, _ = configs.build(name)
    bounds, ranks = _make_ranks(A, b, cfg, world)
    for R in ranks:
        R["y"] = torch.empty_like(R["bd"])
    torch.cuda.synchronize()
    lib = _lib.load()
    t0 = time.perf_counter()
    for _ in range(10000):
        lib.ppf_abi_version()
    t_ct = (time.perf_counter() - t0) / 10000
    per = [[] for _ in ranks]
    barrier = threading.Barrier(world)

    def body(r):
        R = ranks[r]
        for rep in range(reps):
            barrier.wait()
            t = time.perf_counter()
            for k in range(K):
                if k % 2 == 0:
                    R["M"].spmv(R["bd"], R["y"])
                else:
                    R["M"].spmv(R["y"], R["bd"])
            per[r].append((time.perf_counter() - t) / K)
            R["st"].synchronize()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(300)
    host_us = 1e6 * (np.median([min(p) for p in per]) - t_ct)
    # device time of one rank's SpMV when it has the GPU alone: the slab as an
    # unsharded matrix of the same rows (diagonal + halo columns as local)
    lo, hi = bounds[0], bounds[1]
    sl = slice(int(A.row_ptr[lo]), int(A.row_ptr[hi]))
    rp = A.row_ptr[lo:hi + 1] - A.row_ptr[lo]
    cols = A.col[sl] - lo
    keep = (cols >= 0) & (cols < hi - lo)
    # (drop the halo columns: the diagonal block, what overlaps the exchange)
    nn = hi - lo
    rows = np.repeat(np.arange(nn), np.diff(rp))
    import scipy.sparse as sp
    S = sp.csr_matrix((A.val[sl][keep], (rows[keep], cols[keep])), shape=(nn, nn))
    ctx = pp.Context(0)
    fmt = "sell"
    M = pp.Matrix(ctx, pp.Plan(S.indptr.astype(np.int64), S.indices.astype(np.int64), S.data,
                               n_global=nn, fmt=fmt, C_=64 if not np.iscomplexobj(S.data) else 32))
    x = ranks[0]["bd"].clone()
    y = torch.empty_like(x)
    for _ in range(5):
        M.spmv(x, y)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        for _ in range(K):
            M.spmv(x, y)
        ts.append((time.perf_counter() - t) / K)
        torch.cuda.synchronize()
    host1_us = 1e6 * (min(ts) - t_ct)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(ctx.stream)
    for _ in range(50):
        M.spmv(x, y)
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    dev_us = 1e3 * e0.elapsed_time(e1) / 50
    print(f"{name} R={world}: host enqueue per sharded SpMV {host_us:.1f} us (ctypes call "
          f"{1e6 * t_ct:.2f} us subtracted); device time of one rank's diagonal block alone "
          f"{dev_us:.1f} us ({nn} rows); host enqueue of that unsharded SpMV {host1_us:.1f} us")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
