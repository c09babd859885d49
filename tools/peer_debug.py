"""Diagnose the peer-memory exchange (csrc/peer.cu) with R emulated ranks in one
process: enqueue sharded SpMVs of all ranks from ONE host thread (the waits are
device-side, so no host thread ever blocks), poll the streams with a deadline
and dump every window's counters if they stall.  Exits the process on a stall
so the context is torn down."""
import ctypes as C
import os
import struct
import sys
import time

# every emulated rank's streams on their own hardware queue: a stream blocked
# in a wait must not hold up the stream whose push would release it
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_06684_b200 as pp  # noqa: E402
from inputs import configs  # noqa: E402
from tests.test_gpu_multirank import _slab_bounds  # noqa: E402

cudart = C.CDLL("libcudart.so.12")


_side = C.c_void_p()
_pin = C.c_void_p()


def counters(desc):
    """The window's counters, read on a private non-blocking stream (a legacy
    stream copy would wait behind a stalled blocking stream)."""
    if not _side.value:
        cudart.cudaStreamCreateWithFlags(C.byref(_side), 1)
        cudart.cudaMallocHost(C.byref(_pin), C.c_size_t(1024))   # pageable copies sync
    win = struct.unpack_from("<Q", desc, 32)[0]
    buf = C.cast(_pin, C.POINTER(C.c_uint32))
    rc = cudart.cudaMemcpyAsync(_pin, C.c_void_p(win), C.c_size_t(1024), 2, _side)
    t0 = time.time()
    while cudart.cudaStreamQuery(_side) != 0:
        if time.time() - t0 > 5:
            return "read stalled"
        time.sleep(0.01)
    return rc, [buf[i] for i in range(4)] + [buf[64 + i] for i in range(4)] + [buf[128]]


def main(name="C3s", world=2, steps=5, threads=False):
    import faulthandler
    faulthandler.dump_traceback_later(40, exit=True)
    A, b, _ = configs.build(name)
    cfg = configs.CONFIGS[name]
    bounds = _slab_bounds(cfg, A.n, world)
    plans = []
    for r in range(world):
        lo, hi = bounds[r], bounds[r + 1]
        rp = A.row_ptr[lo:hi + 1] - A.row_ptr[lo]
        sl = slice(int(A.row_ptr[lo]), int(A.row_ptr[hi]))
        plans.append(pp.Plan(rp, A.col[sl], A.val[sl], row_bounds=bounds, rank=r))
    needs = [{p: plans[r].halo_recv(p) for p in range(world)} for r in range(world)]
    for r in range(world):
        for p in range(world):
            plans[r].set_halo_send(p, needs[p][r] - bounds[r])
    ranks = []
    for r in range(world):
        h = C.c_void_p()
        assert cudart.cudaStreamCreateWithFlags(C.byref(h), 1) == 0
        st = torch.cuda.ExternalStream(h.value)
        ctx = pp.Context(0, rank=r, nranks=world, stream=st)
        ranks.append(dict(ctx=ctx, M=pp.Matrix(ctx, plans[r]), st=st))
    descs = [R["M"].peer_window() for R in ranks]
    for R in ranks:
        R["M"].peer_connect(descs)
    print("connected", [counters(d) for d in descs], flush=True)
    yd = torch.from_numpy(b).cuda()
    for r, R in enumerate(ranks):
        R["x"] = yd[bounds[r]:bounds[r + 1]].clone()
        R["y"] = torch.empty_like(R["x"])
    torch.cuda.synchronize()
    for k in range(steps):
        for r, R in enumerate(ranks):
            print("enqueue rank", r, flush=True)
            R["M"].spmv(R["x"], R["y"])
            print("  enqueued; stream idle:", R["st"].query(), counters(descs[r]), flush=True)
        t0 = time.time()
        while not all(R["st"].query() for R in ranks) or not all(
                R["ctx"].comm_query() if hasattr(R["ctx"], "comm_query") else True for R in ranks):
            if time.time() - t0 > 10:
                print("STALL at step", k, [counters(d) for d in descs], flush=True)
                os._exit(3)
            time.sleep(0.01)
        print("step", k, "ok", [counters(d)[1] for d in descs], flush=True)
        xs = np.concatenate([R["x"].cpu().numpy() for R in ranks])
        ys = np.concatenate([R["y"].cpu().numpy() for R in ranks])
        ref = A.to_scipy() @ xs
        bad = np.nonzero(np.abs(ys - ref) > 1e-9 * np.abs(ref).max())[0]
        print("  wrong rows:", len(bad), bad[:8], bad[-8:] if len(bad) else "",
              "slab bounds", bounds, flush=True)
        for R in ranks:
            R["x"], R["y"] = R["y"], R["x"]
    print("done", flush=True)


if __name__ == "__main__":
    main(*(a if i == 0 else int(a) for i, a in enumerate(sys.argv[1:])))
