"""Sharded (row-slab) SpMV on the GPU, all ranks in one process on one device
(SURVEY §8(e)): each rank's plan/matrix/context (nranks > 1, no NCCL
communicator), halo index lists exchanged on the host, boundary entries packed
by the library's kernel, moved by the test, then the diagonal-block SpMV + halo
block.  The concatenated slabs must equal the unsharded product."""
import numpy as np
import pytest

from inputs import operators as ops

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2401_06684_b200 as pp  # noqa: E402
from paper_2401_06684_b200 import api  # noqa: E402


def _shard(A, bounds, fmt):
    R = len(bounds) - 1
    plans = []
    for r in range(R):
        lo, hi = bounds[r], bounds[r + 1]
        rp = A.row_ptr[lo:hi + 1] - A.row_ptr[lo]
        sl = slice(A.row_ptr[lo], A.row_ptr[hi])
        plans.append(pp.Plan(rp, A.col[sl], A.val[sl], row_bounds=bounds, rank=r, fmt=fmt[0],
                             C_=fmt[1]))
    recv = [[plans[r].halo_recv(p) for p in range(R)] for r in range(R)]
    for r in range(R):
        for p in range(R):
            plans[r].set_halo_send(p, recv[p][r] - bounds[r])
    return plans, recv


@pytest.mark.parametrize("fmt", [("sell", 64), ("sell", 32), ("csr", 32)])
@pytest.mark.parametrize("case", ["conv3d_2", "conv3d_3", "wilson_2", "lap3d_4"])
def test_sharded_spmv(fmt, case):
    if case.startswith("conv3d"):
        N = 24
        A = ops.convdiff(N, 3, (10.0, 10.0, 10.0))
        R = int(case[-1])
        cuts = np.linspace(0, N, R + 1).astype(int)
        bounds = [int(c) * N * N for c in cuts]
    elif case == "lap3d_4":
        N = 20
        A = ops.laplacian(N, 3)
        bounds = [0, 3 * N * N, 9 * N * N, 15 * N * N, N**3]
    else:
        L = 4
        A = ops.wilson_dirac(L, -1.0, seed=21)
        bounds = [0, 12 * L**3, 12 * L**4]
    if np.iscomplexobj(A.val) and fmt == ("sell", 64):
        pytest.skip("C = 64 is the fp64 layout")
    R = len(bounds) - 1
    plans, recv = _shard(A, bounds, fmt)
    ctxs = [pp.Context(0, rank=r, nranks=R) for r in range(R)]
    mats = [pp.Matrix(ctxs[r], plans[r]) for r in range(R)]
    rng = np.random.default_rng(5)
    x = rng.standard_normal(A.n)
    if np.iscomplexobj(A.val):
        x = x + 1j * rng.standard_normal(A.n)
    xs = [torch.from_numpy(x[bounds[r]:bounds[r + 1]].copy()).cuda() for r in range(R)]
    send_tot = [sum(len(recv[p][r]) for p in range(R)) for r in range(R)]
    recv_tot = [sum(len(recv[r][p]) for p in range(R)) for r in range(R)]
    bufs = [api.halo_buffers(mats[r], send_tot[r], recv_tot[r]) for r in range(R)]
    for r in range(R):
        api.halo_pack(ctxs[r], mats[r], xs[r])
    torch.cuda.synchronize()
    # move segments: rank r's send segment for peer p -> rank p's recv segment for r
    for r in range(R):
        soff = 0
        for p in range(R):
            cnt = len(recv[p][r])
            if cnt:
                roff = sum(len(recv[p][q]) for q in range(r))
                bufs[p][1][roff:roff + cnt].copy_(bufs[r][0][soff:soff + cnt])
            soff += cnt
    torch.cuda.synchronize()
    ys = []
    for r in range(R):
        y = torch.full_like(xs[r], float("nan"))
        api.spmv_local(ctxs[r], mats[r], xs[r], y)
        ys.append(y)
    torch.cuda.synchronize()
    got = np.concatenate([y.cpu().numpy() for y in ys])
    ref = A.to_scipy() @ x
    absA = abs(A.to_scipy()) @ np.abs(x)
    assert np.all(np.abs(got - ref) <= 1e-14 * absA)
