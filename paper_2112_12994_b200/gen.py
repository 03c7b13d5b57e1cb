"""Synthetic series for the BASELINE.json configs (input plumbing, host side).

BASELINE's generator is root-based, which the reference does not have (its
own generator is partials -> Levinson, series.cpp:58-87).  Roots r_k with
|r_k| ~ U[lo, hi] and a fair sign define Phi(z) = prod_k (1 - z / r_k); the
series is simulated in cascade form (one first-order section per root,
x_t = x_{t-1} / r_k + in_t) because the direct form is numerically unsafe
when |phi| reaches ~1e8 (SURVEY.md §7 hard part 1).  Innovations are N(0,1)
(or Student-t(3)/sqrt(3) for C3), burn-in 1000 samples.  Seeds are derived
with the reference's derive_seed so every stream is reproducible.
"""
from __future__ import annotations

import numpy as np
from scipy.signal import lfilter



def _derive_py(seed: int, tag: int) -> int:
    """Pure-Python derive_seed (rng.hpp:82-84) so generation works without the GPU library."""
    M = (1 << 64) - 1

    def mix(z):
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)

    child = mix(seed ^ mix((tag + 0x632BE59BD9B4E019) & M))
    return mix((child + 0x9E3779B97F4A7C15) & M)


def ar_roots(q: int, lo: float, hi: float, seed: int) -> np.ndarray:
    g = np.random.default_rng(_derive_py(seed, 0x7007))
    mag = g.uniform(lo, hi, size=q)
    sign = np.where(g.random(q) < 0.5, -1.0, 1.0)
    return mag * sign


def ar_coefficients(roots) -> np.ndarray:
    """phi with y_t = sum_j phi_j y_{t-j} + e_t, from Phi(z) = prod(1 - z / r)."""
    poly = np.array([1.0])
    for r in roots:
        poly = np.convolve(poly, np.array([1.0, -1.0 / r]))
    return -poly[1:]


def simulate_roots(roots, n: int, seed: int, innovations: str = "normal", burn_in: int = 1000,
                   outlier_frac: float = 0.0) -> np.ndarray:
    g = np.random.default_rng(_derive_py(seed, 0xDA7A))
    total = n + burn_in
    if innovations == "normal":
        e = g.standard_normal(total)
    elif innovations == "t3":
        e = g.standard_t(3, size=total) / np.sqrt(3.0)
    else:
        raise ValueError(innovations)
    x = e
    for r in roots:  # cascade of first-order sections
        x = lfilter([1.0], [1.0, -1.0 / r], x)
    y = np.ascontiguousarray(x[burn_in:])
    if outlier_frac > 0.0:
        go = np.random.default_rng(_derive_py(seed, 0x0071))
        k = int(round(outlier_frac * n))
        pos = go.choice(n, size=k, replace=False)
        sigma = float(np.std(y))  # sigma of the clean series (recorded choice)
        y[pos] += 10.0 * sigma * np.where(go.random(k) < 0.5, -1.0, 1.0)
    return y


CONFIGS = {
    # name: (q, lo, hi, n, p_bar, c_list, innovations, outliers)
    "C1": (20, 1.2, 3.0, 1_000_000, 100, [20_000], "normal", 0.0),
    "C2": (50, 1.2, 3.0, 10_000_000, 200, [10_000, 100_000], "normal", 0.0),
    "C3": (50, 1.2, 3.0, 100_000_000, 200, [100_000], "t3", 0.01),
    "C4": (100, 1.05, 2.0, 1_000_000_000, 500, [200_000], "normal", 0.0),
}


def make_config_series(name: str, seed: int = 2112_12994, n: int | None = None):
    q, lo, hi, n0, p_bar, cs, inn, out = CONFIGS[name]
    roots = ar_roots(q, lo, hi, seed)
    y = simulate_roots(roots, n or n0, seed, inn, outlier_frac=out)
    return y, ar_coefficients(roots), p_bar, cs
