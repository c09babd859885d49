"""Host logic of the sharded (N > 1) path on the CPU with world size 2 over gloo:
row-slab plans, exchange of halo index lists through
torch.distributed, and a host emulation of one halo exchange + slab SpMV that
must equal the unsharded product."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytest.importorskip("paper_2401_06684_b200")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, family, q):
    try:
        import sys
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        import torch.distributed as dist
        from inputs import operators as ops
        from paper_2401_06684_b200.api import Plan

        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        if family == "conv":
            N = 8
            A = ops.convdiff(N, 3, (10.0, 10.0, 10.0))
            planes = N * N
            bounds = [0, 5 * planes, N**3]            # uneven z-slabs
        else:
            L = 3
            A = ops.wilson_dirac(L, -1.0, seed=3)       # periodic in t: both neighbours
            per_t = 12 * L**3
            bounds = [0, 2 * per_t, 3 * per_t]
        lo, hi = bounds[rank], bounds[rank + 1]
        rp = A.row_ptr[lo:hi + 1] - A.row_ptr[lo]
        sl = slice(A.row_ptr[lo], A.row_ptr[hi])
        plan = Plan(rp, A.col[sl], A.val[sl], row_bounds=bounds, rank=rank)
        need = {p: plan.halo_recv(p) for p in range(world)}
        allneed = [None] * world
        dist.all_gather_object(allneed, need)
        # what peer p needs from me -> my local send rows
        sends = {}
        for p in range(world):
            g = allneed[p][rank]
            assert np.all((g >= lo) & (g < hi))
            sends[p] = g - lo
            plan.set_halo_send(p, sends[p])
        # host emulation of one exchange + SpMV on the slab
        rng = np.random.default_rng(0)
        x = rng.standard_normal(A.n) + (1j * rng.standard_normal(A.n) if np.iscomplexobj(A.val) else 0)
        x_local = x[lo:hi]
        payload = {p: x_local[sends[p]] for p in range(world)}
        recv = [None] * world
        dist.all_gather_object(recv, payload)
        x_full_view = np.zeros_like(x)
        x_full_view[lo:hi] = x_local
        for p in range(world):
            if p == rank:
                continue
            x_full_view[need[p]] = recv[p][rank]
        S = A.to_scipy()[lo:hi]
        y_slab = S @ x_full_view
        y_ref = A.to_scipy() @ x
        ok = np.allclose(y_slab, y_ref[lo:hi], rtol=0, atol=1e-12 * np.abs(y_ref).max())
        info = plan.info()
        dist.destroy_process_group()
        q.put((rank, ok, info["halo_total"], {p: len(v) for p, v in need.items()}))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e), None, None))


@pytest.mark.parametrize("family", ["conv", "wilson"])
def test_two_rank_halo_plan_gloo(family):
    mp = torch.multiprocessing.get_context("spawn")
    q = mp.Queue()
    port = _free_port()
    procs = [mp.Process(target=_worker, args=(r, 2, port, family, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    res.sort()
    for rank, ok, halo_total, counts in res:
        assert ok is True, (rank, ok)
        if family == "conv":
            assert halo_total == 64                   # one neighbouring z-plane of 8x8
        else:
            # periodic t, L = 3: rank 0 owns t = 0, 1 and needs only t = 2 (as t+1 of
            # t = 1 and t-1 of t = 0); rank 1 owns t = 2 and needs t = 1 and t = 0
            assert halo_total == (12 * 27 if rank == 0 else 2 * 12 * 27)
