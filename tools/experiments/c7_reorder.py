#!/usr/bin/env python
"""Timing experiment: does a symmetric renumbering of the graph's vertices
(P L P^T, the caller's choice before ppf_plan_create; the library takes any CSR) speed up the
gather-bound C7 SpMV chain?  Orders: the generator's, reverse Cuthill-McKee on L + L^T, and hub
sorting (vertices by how often their x entry is gathered, i.e. by column count, descending).

    python tools/experiments/c7_reorder.py [--reps 5]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from inputs import configs  # noqa: E402
from inputs.operators import CSR  # noqa: E402
import paper_2401_06684_b200 as pp  # noqa: E402
from paper_2401_06684_b200 import api  # noqa: E402


def permuted(A: CSR, perm: np.ndarray) -> CSR:
    S = A.to_scipy()[perm][:, perm].tocsr()
    S.sort_indices()
    return CSR(A.n, S.indptr.astype(np.int64), S.indices.astype(np.int64), S.data.copy())


def chain_us(ctx, A: CSR, deg: int, reps: int) -> float:
    sigma = 32 * ((A.n + 31) // 32)
    M = pp.Matrix(ctx, pp.Plan.from_csr(A, fmt="sell", C_=32, sigma=sigma))
    x = torch.randn(A.n, dtype=torch.float64, device="cuda")
    q = pp.Poly.ritz_newton(ctx, M, x, deg)
    y = torch.empty_like(x)
    for _ in range(2):
        q.apply(ctx, M, x, y)
    torch.cuda.synchronize()
    api.profile_enable(ctx, True)
    for _ in range(reps):
        q.apply(ctx, M, x, y)
    torch.cuda.synchronize()
    p = api.profile_read(ctx)["spmv"]
    api.profile_enable(ctx, False)
    return p["ms"] / p["launches"] * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    cfg = configs.CONFIGS["C7"]
    A, _ = configs.operator(cfg)
    ctx = pp.Context(0)
    from scipy.sparse.csgraph import reverse_cuthill_mckee
    S = A.to_scipy()
    orders = {
        "generator": np.arange(A.n),
        "rcm": np.asarray(reverse_cuthill_mckee((S + S.T).tocsr(), symmetric_mode=True)),
        "hub": np.argsort(-np.bincount(A.col, minlength=A.n), kind="stable"),
        "random": np.random.default_rng(1).permutation(A.n),
    }
    for name, perm in orders.items():
        B = A if name == "generator" else permuted(A, perm)
        print(f"C7 deg 15, order {name}: {chain_us(ctx, B, 15, a.reps):.1f} us per SpMV", flush=True)


if __name__ == "__main__":
    main()
