"""The stored full-size oracle results (tests/golden/fullsize/*.npz, written by
tools/make_fullsize_goldens.py from oracle/ only) are self-consistent and
match what the oracle's definitions fix, without a GPU:
  * the sampled rows are inputs.vectors.sample_indices(n, 65536, seed) and the
    q coefficients are the oracle's Chebyshev construction for the config;
  * m* is the FIRST m with true error <= tol (error history above tol before it),
    the estimate-stop m the first checkpoint with estimate <= tol;
  * H_m has the Arnoldi/Lanczos shape and a positive subdiagonal; the two runs
    of one config agree on their common leading block (same process, same
    rounding up to the stop);
  * the iteration counts of the headline configs (C4: 23 / 23)."""
import numpy as np
import pytest

from inputs import configs
from inputs.vectors import sample_indices
from oracle import chebyshev

from . import fullsize_oracle as fo


@pytest.mark.parametrize("key", list(fo.KEYS))
def test_golden_consistency(key):
    g = fo.load(key)
    name, deg, k, _, _ = fo.KEYS[key]
    cfg = configs.CONFIGS[name]
    assert g["config"] == name and g["deg"] == deg and g["check_every"] == k
    assert np.array_equal(g["idx"], sample_indices(int(g["n"]), fo.SAMPLE_K, fo.SAMPLE_SEED))
    if cfg.poly == "chebyshev":
        _, _, iv = (None, None, configs.operator(cfg)[1])
        q = chebyshev.coefficients(*iv, deg)
        assert np.array_equal(q.c, g["q_c"])
    tol = float(g["tol"])
    modes = [m for m in ("true", "est") if f"{m}_m" in g]
    for mode in modes:
        m = int(g[f"{mode}_m"])
        H = g[f"{mode}_H"]
        assert H.shape == (m + 1, m)
        sub = np.abs(np.diag(H, -1))
        assert np.all(sub > 0)
        assert np.allclose(np.tril(H, -2), 0)                  # upper Hessenberg
        hm, he, hr = g[f"{mode}_hist_m"], g[f"{mode}_hist_est"], g[f"{mode}_hist_err"]
        assert hm[-1] == m and np.all(np.diff(hm) == k)
        if mode == "true":
            assert hr[-1] <= tol and np.all(hr[:-1] > tol)     # the FIRST m below tol
        else:
            ok = ~np.isnan(he)
            assert he[ok][-1] <= tol and np.all(he[ok][:-1] > tol)
        assert g[f"{mode}_mvms"] > m
    if len(modes) == 2:
        mm = min(int(g["true_m"]), int(g["est_m"]))
        Ht, He = g["true_H"], g["est_H"]
        assert np.array_equal(Ht[: mm + 1, :mm], He[: mm + 1, :mm])
        assert g["true_beta0"] == g["est_beta0"]


def test_headline_iteration_counts():
    """BASELINE configs[3] (C4, seed 104): m* = 23 by the true error and 23 by
    the paper's estimate -- the m bench.py's C4 line reports; C3 deg 10/20/40
    (seed 103): m* 51 / 27 / 14; C5: 3 (estimate 4)."""
    g = fo.load("C4_deg20")
    assert g["true_m"] == 23 and g["est_m"] == 23 and g["est_mvms"] == 964
    assert [fo.load(f"C3_deg{d}")["true_m"] for d in (10, 20, 40)] == [51, 27, 14]
    g5 = fo.load("C5_deg16")
    assert g5["true_m"] == 3 and g5["est_m"] == 4
