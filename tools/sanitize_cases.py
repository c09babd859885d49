#!/usr/bin/env python
"""Small runs of the hot path for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck), each checked against the oracle so a run that
"passes" the sanitizer also computed the right thing:

  c1          C1 (2D Laplacian 32^2, Chebyshev deg 4, Lanczos, SELL-32)
  c2_tiled    C2 deg 5 (65,536 rows), CGS2 through the TMA/mbarrier-ring tiled
              sweeps (PPF_CGS_FLAT=0), 30 steps = two column tiles, SELL-32
  c2_flat     the same through the flat sweeps (PPF_CGS_FLAT=1)
  c4s_sell64  C4s (32^3 conv-diff, sqrt) in SELL-64 with the sell2 prefetch/PDL
  c5s         C5s (complex Wilson 4^4, Ritz-Newton setup on the device, CGS2)
  peer3       C4s on 3 emulated ranks of one process (peer-memory windows,
              push kernels, stream waits on the counters, rank-order sums)

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py c2_tiled
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2401_06684_b200 as pp  # noqa: E402
from inputs import configs  # noqa: E402
from oracle import chebyshev, krylov, newton  # noqa: E402
from oracle.spmv import Operator  # noqa: E402


def check(x, ref, what):
    e = np.linalg.norm(x - ref) / np.linalg.norm(ref)
    print(f"{what}: rel err vs oracle {e:.2e}")
    assert e <= 1e-10, e


def cheb_case(name, deg, m, C_=32, flat=None):
    if flat is not None:
        os.environ["PPF_CGS_FLAT"] = "1" if flat else "0"
    cfg = configs.CONFIGS[name]
    A, b, iv = configs.build(name)
    ctx = pp.Context(0)
    M = pp.Matrix(ctx, pp.Plan.from_csr(A, fmt="sell", C_=C_))
    x, rep = pp.run(ctx, M, pp.Poly.chebyshev(*iv, deg), torch.from_numpy(b).cuda(),
                    func=cfg.func, krylov=cfg.krylov, m_max=m, stop="fixed")
    torch.cuda.synchronize()
    r = krylov.run(Operator(A.to_scipy()), b, chebyshev.coefficients(*iv, deg), func=cfg.func,
                   krylov=cfg.krylov, m_max=m)
    check(x.cpu().numpy(), r.x, f"{name} deg {deg} m {m}")


def c5s():
    A, b, _ = configs.build("C5s")
    ctx = pp.Context(0)
    M = pp.Matrix(ctx, pp.Plan.from_csr(A))
    bd = torch.from_numpy(b).cuda()
    q = pp.Poly.ritz_newton(ctx, M, bd, 16)
    x, rep = pp.run(ctx, M, q, bd, func="invsqrt", krylov="cgs2", m_max=4, stop="fixed")
    torch.cuda.synchronize()
    op = Operator(A.to_scipy())
    qo, _, _ = newton.ritz_newton(op, b, 16)
    r = krylov.run(op, b, qo, func="invsqrt", krylov="cgs2", m_max=4)
    check(x.cpu().numpy(), r.x, "C5s Ritz-Newton m 4")


def peer3():
    os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
    from tests.test_gpu_multirank import CASES, oracle_case
    from tests.test_gpu_peer import child_run
    import tempfile
    d = tempfile.mkdtemp()
    case = "c4s_cgs2_sqrt" if "c4s_cgs2_sqrt" in CASES else sorted(CASES)[0]
    q_path = os.path.join(d, "q.npy")
    out = os.path.join(d, "out.npz")
    child_run(case, q_path, out, world=3)
    print(f"peer3: {case} on 3 emulated ranks finished")


if __name__ == "__main__":
    c = sys.argv[1]
    if c == "c1":
        cheb_case("C1", 4, 20)
    elif c == "c2_tiled":
        cheb_case("C2", 5, 30, flat=False)
    elif c == "c2_flat":
        cheb_case("C2", 5, 30, flat=True)
    elif c == "c4s_sell64":
        cheb_case("C4s", 20, 12, C_=64)
    elif c == "c5s":
        c5s()
    elif c == "peer3":
        peer3()
    else:
        sys.exit(f"unknown case {c}")
