"""The five BASELINE.json workloads and scaled-down
variants of the same operator families used for element-wise parity tests.

``build(name)`` returns ``(A: CSR, b: ndarray, interval: (a, b) or None)``.
The interval is the operator's closed-form spectral interval (problem data; the
3D Laplacian formula is PAPER.md:419), passed to the Chebyshev construction.
"""
from __future__ import annotations

from dataclasses import dataclass, field

from . import operators as ops
from .vectors import gaussian_vector


@dataclass(frozen=True)
class Config:
    name: str
    family: str                  # "laplacian" | "convdiff" | "wilson" | "overlap" | "graph"
    params: dict = field(default_factory=dict)
    func: str = "invsqrt"        # "invsqrt" | "sqrt" (= A^{-1/2}(Ab)) | "sign"
                                 # (= Q (Q^2)^{-1/2} b)
    degs: tuple = (4,)           # degree of q (deg = d-1 in the paper's notation, reading Q1)
    krylov: str = "lanczos"      # "lanczos" | "cgs2"
    poly: str = "chebyshev"      # "chebyshev" | "ritz"
    tol: float = 1e-8
    m_max: int = 60
    b_seed: int = 0

    @property
    def complex_(self) -> bool:
        return self.family in ("wilson", "overlap")


CONFIGS = {
    # BASELINE.json configs[0..4]
    "C1": Config("C1", "laplacian", dict(N=32, dim=2), "invsqrt", (4,), "lanczos", "chebyshev", 1e-10, 60, 101),
    "C2": Config("C2", "convdiff", dict(N=256, dim=2, beta=(20.0, 20.0)), "sqrt", (5, 10, 20), "cgs2",
                 "chebyshev", 1e-8, 120, 102),
    "C3": Config("C3", "laplacian", dict(N=200, dim=3), "invsqrt", (10, 20, 40), "lanczos", "chebyshev",
                 1e-8, 80, 103),
    "C4": Config("C4", "convdiff", dict(N=256, dim=3, beta=(10.0, 10.0, 10.0)), "sqrt", (20,), "cgs2",
                 "chebyshev", 1e-8, 60, 104),
    "C5": Config("C5", "wilson", dict(L=16, m0=-1.0, link_seed=205), "invsqrt", (16,), "cgs2", "ritz",
                 1e-8, 30, 105),
    # the paper's headline application (§6.2): sign(Q)b for the
    # overlap kernel Q = Γ5 D_w(m_w = -1.4, mu = 0.3) (P:473 values) on a 16^4 Haar
    # lattice (the SFB-TRR55 ensemble is not available), Ritz-Newton q of Q^2
    # (P:475), d = 16 (Table 2 row), Arnoldi CGS2 (context workload, not a BASELINE config)
    "C6": Config("C6", "overlap", dict(L=16, m_w=-1.4, mu=0.3, link_seed=206), "sign", (15,),
                 "cgs2", "ritz", 1e-8, 60, 106),
    # Ex. 6.3's setting: L^{1/2} b for the in-degree Laplacian of a
    # directed graph, a seeded synthetic web-like graph standing in for Kamvar/Stanford
    # (n = 281,903, ~2.59M nnz; the dataset is not available), Ritz-Newton q from
    # L b (implicit desingularisation, Thm 4.1), Arnoldi with reorthogonalisation,
    # tol 1e-7, k = 32/d (context workload, not a BASELINE config)
    "C7": Config("C7", "graph", dict(n=281903, avg_deg=8.97, graph_seed=207, ritz_start="Ab"),
                 "sqrt", (15, 7), "cgs2", "ritz", 1e-7, 200, 107),
    # PAPER.md Table 1's own workload (§6.1): 3D Laplacian 100^3, tol 1e-12,
    # right preconditioning, d = deg+1 in {1..64}, k = 64/d (context workload)
    "T1": Config("T1", "laplacian", dict(N=100, dim=3), "invsqrt", (7,), "lanczos", "chebyshev",
                 1e-12, 600, 100),
    # scaled-down members of the same families (oracle finishes in seconds)
    "C3s": Config("C3s", "laplacian", dict(N=30, dim=3), "invsqrt", (10, 20), "lanczos", "chebyshev",
                  1e-8, 80, 203),
    # L2-resident member of the C4 family (micro-benchmarks of the SpMV chain)
    "C4m": Config("C4m", "convdiff", dict(N=80, dim=3, beta=(10.0, 10.0, 10.0)), "sqrt", (20,), "cgs2",
                  "chebyshev", 1e-8, 60, 404),
    "C4s": Config("C4s", "convdiff", dict(N=32, dim=3, beta=(10.0, 10.0, 10.0)), "sqrt", (20, 5), "cgs2",
                  "chebyshev", 1e-8, 60, 204),
    "C6s": Config("C6s", "overlap", dict(L=4, m_w=-1.4, mu=0.3, link_seed=306), "sign", (15, 7),
                  "cgs2", "ritz", 1e-8, 60, 206),
    "C7s": Config("C7s", "graph", dict(n=2000, avg_deg=8.97, graph_seed=307, ritz_start="Ab"),
                  "sqrt", (7, 3), "cgs2", "ritz", 1e-7, 200, 207),
    # convection-dominated 2D convection-diffusion (cell Peclet 3 > 1): a real
    # operator with complex eigenvalues and complex-pair Ritz values, for the
    # real conjugate-pair Newton form
    "C8s": Config("C8s", "convdiff", dict(N=32, dim=2, beta=(200.0, 200.0)), "sqrt", (9,), "cgs2",
                  "ritz", 1e-8, 120, 208),
    "C5s": Config("C5s", "wilson", dict(L=4, m0=-1.0, link_seed=305), "invsqrt", (16, 4), "cgs2", "ritz",
                  1e-8, 30, 205),
}


def operator(cfg: Config):
    p = cfg.params
    if cfg.family == "laplacian":
        return ops.laplacian(p["N"], p["dim"]), ops.laplacian_interval(p["N"], p["dim"])
    if cfg.family == "convdiff":
        A = ops.convdiff(p["N"], p["dim"], p["beta"])
        # a real spectral interval exists only for cell Peclet numbers < 1
        if max(abs(b) for b in p["beta"]) / (2.0 * (p["N"] + 1)) >= 1.0:
            return A, None
        return A, ops.convdiff_interval(p["N"], p["dim"], p["beta"])
    if cfg.family == "wilson":
        return ops.wilson_dirac(p["L"], p["m0"], seed=p["link_seed"]), None
    if cfg.family == "graph":
        return ops.directed_graph_laplacian(p["n"], p["avg_deg"], p["graph_seed"]), None
    if cfg.family == "overlap":
        return ops.overlap_kernel(p["L"], p["m_w"], p["mu"], seed=p["link_seed"]), None
    raise ValueError(cfg.family)


def build(name_or_cfg):
    cfg = CONFIGS[name_or_cfg] if isinstance(name_or_cfg, str) else name_or_cfg
    A, interval = operator(cfg)
    b = gaussian_vector(A.n, cfg.b_seed, cfg.complex_)
    return A, b, interval
