"""Sparse test operators of the paper's workloads, as plain CSR arrays.

Every operator is returned as a ``CSR`` (0-based ``row_ptr`` int64, ``col``
int64 sorted within each row, ``val`` float64 or complex128).  Grid index is
``i = ix + N*iy (+ N^2*iz)`` (x fastest), lattice site ``x + L*y + L^2*z + L^3*t``.

Operators (BASELINE.json configs):
  * ``laplacian(N, dim)``   -- unscaled Dirichlet 5/7-point Laplacian; the
    operator of the paper's §3.2 example and Example 6.1
    (PAPER.md:419).  Diagonal 2*dim, off-diagonal -1 (reading Q14).
  * ``convdiff(N, dim, beta, h)`` -- centred  -Δu + β·∇u  scaled by 1/h^2
    (BASELINE.json configs 2 and 4; reading Q15).
  * ``wilson_dirac(L, m0, seed)`` -- D = (4+m0)I - 1/2 Σ_μ[(1-γ_μ)U_μ(x)δ_{x+μ,y}
    + (1+γ_μ)U_μ(x-μ)^† δ_{x-μ,y}] on a periodic L^4 lattice, chiral γ basis,
    Haar SU(3) links (BASELINE.json config 5; reading Q16).  Stand-in for the
    paper's Example 6.2 Wilson-Dirac operator, whose gauge
    ensemble is not available.

The spectral intervals are closed forms of the operator (problem data, the 3D
formula is printed at PAPER.md:419), not part of the method.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class CSR:
    n: int
    row_ptr: np.ndarray  # int64 [n+1]
    col: np.ndarray      # int64 [nnz], sorted within rows
    val: np.ndarray      # float64 or complex128 [nnz]

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    @property
    def dtype(self):
        return self.val.dtype

    def to_scipy(self):
        import scipy.sparse as sp
        idx = np.int32 if self.n < 2**31 - 1 and self.nnz < 2**31 - 1 else np.int64
        m = sp.csr_matrix((self.val, self.col.astype(idx), self.row_ptr.astype(idx)),
                          shape=(self.n, self.n))
        m.has_sorted_indices = True
        return m


def _stencil(N: int, dim: int, diag: float, lower, upper) -> CSR:
    """Nearest-neighbour stencil on an N^dim Dirichlet grid.

    ``lower[d]`` is the coefficient of u at coordinate-1 along axis d,
    ``upper[d]`` the coefficient at coordinate+1.  Columns come out sorted
    because the offsets are visited in increasing order.
    """
    n = N ** dim
    idx = np.arange(n, dtype=np.int64)
    coords = []
    rem = idx
    for _ in range(dim):
        coords.append(rem % N)
        rem = rem // N
    # offsets in increasing column order: -N^{dim-1} ... -1, 0, +1 ... +N^{dim-1}
    entries = []
    for d in reversed(range(dim)):
        entries.append((-(N ** d), coords[d] > 0, lower[d]))
    entries.append((0, None, diag))
    for d in range(dim):
        entries.append((N ** d, coords[d] < N - 1, upper[d]))
    counts = np.zeros(n, dtype=np.int64)
    for off, mask, _ in entries:
        counts += 1 if mask is None else mask
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    nnz = int(row_ptr[-1])
    col = np.empty(nnz, dtype=np.int64)
    val = np.empty(nnz, dtype=np.float64)
    pos = row_ptr[:-1].copy()
    for off, mask, v in entries:
        if mask is None:
            rows = idx
        else:
            rows = idx[mask]
        p = pos[rows]
        col[p] = rows + off
        val[p] = v
        pos[rows] += 1
    return CSR(n, row_ptr, col, val)


def laplacian(N: int, dim: int) -> CSR:
    """Unscaled Dirichlet Laplacian: diagonal 2*dim, neighbours -1 (Q14)."""
    return _stencil(N, dim, 2.0 * dim, [-1.0] * dim, [-1.0] * dim)


def convdiff(N: int, dim: int, beta, h: float | None = None) -> CSR:
    """Centred -Δu + β·∇u on the unit square/cube, Dirichlet, h = 1/(N+1) (Q15).

    Row i: diagonal 2*dim/h^2; neighbour -x: -1/h^2 - β_x/(2h);
    neighbour +x: -1/h^2 + β_x/(2h) (likewise y, z).
    """
    if h is None:
        h = 1.0 / (N + 1)
    beta = list(beta)
    assert len(beta) == dim
    ih2 = 1.0 / (h * h)
    lower = [-ih2 - b / (2.0 * h) for b in beta]
    upper = [-ih2 + b / (2.0 * h) for b in beta]
    return _stencil(N, dim, 2.0 * dim * ih2, lower, upper)


def laplacian_interval(N: int, dim: int):
    """Exact spectral interval [λ_min, λ_max] of ``laplacian(N, dim)``.

    dim=3 is PAPER.md:419: [6(1-cos(π/(N+1))), 12 - 6(1-cos(π/(N+1)))].
    """
    c = np.cos(np.pi / (N + 1))
    return dim * (2.0 - 2.0 * c), dim * (2.0 + 2.0 * c)


def convdiff_interval(N: int, dim: int, beta, h: float | None = None):
    """Exact real spectral interval of ``convdiff`` with equal β per axis.

    The 1D factor h^-2 tridiag(-(1+P), 2, -(1-P)), P = β h/2 < 1, is similar to a
    symmetric tridiagonal matrix with off-diagonal -sqrt(1-P^2), so
    σ_k = (2 - 2 sqrt(1-P^2) cos(kπ/(N+1)))/h^2 and the dim-D spectrum is the
    sum over axes.
    """
    if h is None:
        h = 1.0 / (N + 1)
    c = np.cos(np.pi / (N + 1))
    lo = hi = 0.0
    for b in beta:
        P = b * h / 2.0
        assert abs(P) < 1.0
        s = np.sqrt(1.0 - P * P)
        lo += (2.0 - 2.0 * s * c) / (h * h)
        hi += (2.0 + 2.0 * s * c) / (h * h)
    return lo, hi


# ----------------------------------------------------------------------------
# Wilson-Dirac operator (reading Q16)
# ----------------------------------------------------------------------------

def _gammas():
    """Chiral-basis Euclidean gamma matrices γ_1..γ_4 (Hermitian, anticommuting)."""
    s1 = np.array([[0, 1], [1, 0]], dtype=np.complex128)
    s2 = np.array([[0, -1j], [1j, 0]], dtype=np.complex128)
    s3 = np.array([[1, 0], [0, -1]], dtype=np.complex128)
    Z = np.zeros((2, 2), dtype=np.complex128)
    I2 = np.eye(2, dtype=np.complex128)
    g = []
    for s in (s1, s2, s3):
        g.append(np.block([[Z, -1j * s], [1j * s, Z]]))
    g.append(np.block([[Z, I2], [I2, Z]]))
    return g


def gamma5():
    g = _gammas()
    return g[0] @ g[1] @ g[2] @ g[3]


def haar_su3(rng: np.random.Generator, count: int) -> np.ndarray:
    """``count`` Haar-distributed SU(3) matrices: QR of a complex Ginibre matrix,
    phases fixed by diag(R)/|diag(R)|, divided by det^{1/3} (Q16)."""
    z = rng.standard_normal((count, 3, 3, 2))
    Z = (z[..., 0] + 1j * z[..., 1]) / np.sqrt(2.0)
    Q, R = np.linalg.qr(Z)
    d = np.diagonal(R, axis1=1, axis2=2)
    ph = d / np.abs(d)
    Q = Q * ph[:, None, :]
    det = np.linalg.det(Q)
    Q = Q / np.power(det, 1.0 / 3.0)[:, None, None]
    return Q


def wilson_dirac(L: int, m0: float, seed: int | None = None, links: np.ndarray | None = None,
                 mu: float = 0.0) -> CSR:
    """Wilson-Dirac matrix on a periodic L^4 lattice (12 dof/site, 49 nnz/row).

    ``links`` has shape (4, L^4, 3, 3); if None, Haar SU(3) links are drawn from
    ``seed`` in (μ, site) order.  ``links = identity`` gives the free operator.
    ``mu`` is a chemical potential: the forward time hop
    (direction 4) carries e^{mu}, the backward one e^{-mu}, which makes
    Γ5 D non-Hermitian.  Requires L >= 3 so that the +μ and -μ neighbours are
    distinct sites.
    """
    assert L >= 3
    V = L ** 4
    if links is None:
        rng = np.random.default_rng(seed)
        links = haar_su3(rng, 4 * V).reshape(4, V, 3, 3)
    return _wilson_assemble(L, m0, links, mu)


def overlap_kernel(L: int, m_w: float, mu: float = 0.0, seed: int | None = None,
                   links: np.ndarray | None = None) -> CSR:
    """Q = Γ5 D_w(m_w, mu), the argument of the sign function in the overlap
    operator D_ov = I + ρ Γ5 sign(Q).  Γ5 = γ1γ2γ3γ4 =
    diag(1, 1, -1, -1) on the spins in this chiral basis (the identity on spins
    1, 2 and minus the identity on spins 3, 4): rows of spin 3, 4
    of D_w are negated.  Hermitian for mu = 0."""
    D = wilson_dirac(L, m_w, seed=seed, links=links, mu=mu)
    rows = np.repeat(np.arange(D.n), np.diff(D.row_ptr))
    sign = np.where(((rows % 12) // 3) >= 2, -1.0, 1.0)
    return CSR(D.n, D.row_ptr.copy(), D.col.copy(), D.val * sign)


def _wilson_assemble(L: int, m0: float, links: np.ndarray, mu_c: float = 0.0) -> CSR:
    V = L ** 4
    site = np.arange(V, dtype=np.int64)
    coord = [(site // L ** k) % L for k in range(4)]

    def shift(mu, step):
        c = coord[mu]
        return site + (((c + step) % L) - c) * L ** mu

    g = _gammas()
    I4 = np.eye(4, dtype=np.complex128)
    K = 49
    cols = np.empty((V, 4, 3, K), dtype=np.int64)
    vals = np.empty((V, 4, 3, K), dtype=np.complex128)
    spin = np.arange(4)
    colour = np.arange(3)
    cols[..., 0] = 12 * site[:, None, None] + 3 * spin[None, :, None] + colour[None, None, :]
    vals[..., 0] = 4.0 + m0
    for s in range(4):
        e = 1
        for mu in range(4):
            fwd = shift(mu, +1)
            bwd = shift(mu, -1)
            ef, eb = (np.exp(mu_c), np.exp(-mu_c)) if mu == 3 else (1.0, 1.0)
            for nb, P, Cm, ex in ((fwd, I4 - g[mu], links[mu], ef),
                                  (bwd, I4 + g[mu], np.conj(np.swapaxes(links[mu][bwd], 1, 2)), eb)):
                for sp in np.nonzero(P[s])[0]:
                    coef = -0.5 * P[s, sp] * ex
                    for b in range(3):
                        cols[:, s, :, e] = (12 * nb + 3 * sp + b)[:, None]
                        vals[:, s, :, e] = coef * Cm[:, :, b]
                        e += 1
        assert e == K
    n = 12 * V
    cols = cols.reshape(n, K)
    vals = vals.reshape(n, K)
    order = np.argsort(cols, axis=1, kind="stable")
    cols = np.take_along_axis(cols, order, axis=1)
    vals = np.take_along_axis(vals, order, axis=1)
    assert np.all(np.diff(cols, axis=1) > 0), "duplicate columns (L too small?)"
    row_ptr = np.arange(0, n * K + 1, K, dtype=np.int64)
    return CSR(n, row_ptr, cols.reshape(-1), vals.reshape(-1))


# ----------------------------------------------------------------------------
# In-degree graph Laplacian of a directed graph (Ex. 6.3)
# ----------------------------------------------------------------------------
def directed_graph_laplacian(n: int, avg_deg: float, seed: int, alpha: float = 2.1,
                             max_out: int = 255) -> CSR:
    """L = D_in - A for a seeded synthetic directed graph (it
    stands in for SuiteSparse Kamvar/Stanford, which is not available and is
    not reproduced).  A_ij = 1 for an edge i -> j; D_in = diag(column sums of
    A), so every column of L sums to zero and L is singular.

    Web-crawl-like degree structure: out-degrees (the row lengths of L) follow
    a power law truncated at ``max_out`` (crawlers cap the links followed per
    page), in-degrees are heavy-tailed (targets drawn with weights
    w_k ∝ k^{-1/(alpha-1)}); self loops dropped, duplicates merged; plus the
    cycle i -> i+1 (mod n), so the graph is strongly connected and the
    eigenvalue 0 of L is simple (hence semi-simple, the hypothesis of
    Theorem 4.1)."""
    rng = np.random.default_rng(seed)
    # out-degrees: P(d) ∝ d^{-2.2} on 1..max_out, rescaled to the mean avg_deg - 1
    d = np.arange(1, max_out + 1, dtype=np.float64)
    pd = d ** -2.2
    pd /= pd.sum()
    outdeg = rng.choice(np.arange(1, max_out + 1), size=n, p=pd).astype(np.float64)
    outdeg = np.clip(np.round(outdeg * (avg_deg - 1.0) / outdeg.mean()), 0, max_out).astype(np.int64)
    k = np.arange(1, n + 1, dtype=np.float64)
    win = k ** (-1.0 / (alpha - 1.0))
    rng.shuffle(win)
    src = np.repeat(np.arange(n, dtype=np.int64), outdeg)
    dst = rng.choice(n, size=len(src), p=win / win.sum())
    keep = src != dst
    src = np.concatenate([src[keep], np.arange(n)])
    dst = np.concatenate([dst[keep], (np.arange(n) + 1) % n])
    key = np.unique(src * n + dst)
    src, dst = key // n, key % n
    din = np.bincount(dst, minlength=n).astype(np.float64)
    # rows of L: diagonal din[i] and -1 at (i, j) for every edge i -> j
    rows = np.concatenate([np.arange(n), src])
    cols = np.concatenate([np.arange(n), dst])
    vals = np.concatenate([din, -np.ones(len(src))])
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=row_ptr[1:])
    return CSR(n, row_ptr, cols.astype(np.int64), vals)
