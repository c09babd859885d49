#!/usr/bin/env python
"""Micro-benchmark of the fused SpMV chain (ppf_poly_apply) on a BASELINE
config's operator: per-launch device time from the library's CUDA events and
the algorithmic bytes -> GB/s.  Profiling aid, not the bench.

    python tools/spmv_micro.py [--config C4] [--deg 20] [--reps 5] [--split 0]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from inputs import configs  # noqa: E402
import paper_2401_06684_b200 as pp  # noqa: E402
from paper_2401_06684_b200 import api  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--deg", type=int, default=20)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--split", type=int, default=0)
    ap.add_argument("--fmt", default="sell64")
    ap.add_argument("--sigma", type=int, default=1, help="SELL sorting window (0: all rows)")
    ap.add_argument("--eval", default=None, choices=["horner", "basis", "pairs"])
    a = ap.parse_args()
    cfg = configs.CONFIGS[a.config]
    A, iv = configs.operator(cfg)
    fmt = {"sell32": ("sell", 32), "sell64": ("sell", 64), "csr": ("csr", 32)}[a.fmt]
    if cfg.complex_ and fmt[1] == 64:
        fmt = ("sell", 32)
    ctx = pp.Context(0)
    sigma = a.sigma if a.sigma > 0 else 32 * ((A.n + 31) // 32)
    M = pp.Matrix(ctx, pp.Plan.from_csr(A, fmt=fmt[0], C_=fmt[1], sigma=sigma))
    M.set_split(a.split)
    dt = torch.complex128 if cfg.complex_ else torch.float64
    x = torch.randn(A.n, dtype=dt, device="cuda")
    if cfg.poly == "ritz":
        q = pp.Poly.ritz_newton(ctx, M, x, a.deg)
        if a.eval:
            q.set_newton_eval(a.eval)
    else:
        q = pp.Poly.chebyshev(*iv, a.deg)
    y = torch.empty_like(x)
    for _ in range(2):
        q.apply(ctx, M, x, y)
    torch.cuda.synchronize()
    api.profile_enable(ctx, True)
    for _ in range(a.reps):
        q.apply(ctx, M, x, y)
    torch.cuda.synchronize()
    p = api.profile_read(ctx)["spmv"]
    api.profile_enable(ctx, False)
    print(f"{a.config} deg {a.deg} fmt {a.fmt}: {p['launches']} launches, "
          f"{p['ms'] / p['launches'] * 1e3:.1f} us/launch, {p['bytes'] / (p['ms'] * 1e-3) / 1e9:.0f} GB/s")


if __name__ == "__main__":
    main()
