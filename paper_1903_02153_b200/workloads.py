"""Seeded synthetic inputs for the BASELINE.json configurations.

BASELINE.json names no public dataset (the paper also uses uniform random
clouds), so every config is a seeded NumPy recipe; the
recipes follow SURVEY.md §8(d) draw for draw.  C1 fixes seed 0 in
BASELINE.json; seed 0 for C2..C5 is the survey's choice.

``scale=k`` gives the density-preserving reduced variant used for parity
runs (N / 8**k points, k fewer tree levels, same order / kernel / columns),
SURVEY.md §8(c)(7).  Check targets are always
``default_rng(1).choice(N, 1000, replace=False)``.
"""

from __future__ import annotations

import numpy as np

#: name -> (N, levels, order, scheme, eps, kernel key, ncols)
CONFIGS = {
    "C1": (20_000, 3, 4, "chebyshev", 1e-5, "laplacian", 1),
    "C2": (1_000_000, 5, 5, "chebyshev", 1e-7, "gauss02", 1),
    "C3": (4_000_000, 6, 6, "uniform", 1e-5, "exp03", 16),
    "C4": (8_000_000, 7, 6, "chebyshev", 1e-5, "laplacianforce", 1),
    "C5": (64_000_000, 8, 5, "chebyshev", 1e-5, "laplacian", 1),
}

DESCRIPTION = {
    "C1": "Laplace 1/r, N=20k uniform [-1,1]^3, L=3, Chebyshev p=4, eps 1e-5",
    "C2": "Gaussian exp(-(r/0.2)^2), N=1M uniform [-1,1]^3, L=5, Chebyshev p=5, eps 1e-7",
    "C3": "exp(-r/0.3), N=4M uniform [0,1]^3, L=6, uniform p=6 FFT M2L, 16 RHS",
    "C4": "1/r^4, N=8M sphere + 32 clusters, L=7, Chebyshev p=6",
    "C5": "Laplace 1/r, N=64M uniform [-1,1]^3, L=8, Chebyshev p=5",
}


def domain_from_points(X):
    """Smallest common-center cube around the points (oct:53-65)."""
    lo = X.min(axis=0)
    hi = X.max(axis=0)
    length = float(np.max(hi - lo))
    if length == 0.0:
        length = 1.0
    return tuple(float(c) for c in 0.5 * (lo + hi)), length


def make(name: str, scale: int = 0, n_override: int | None = None):
    """Return a dict with points, weights, plan parameters and check indices."""
    N, L, p, scheme, eps, kern, m = CONFIGS[name]
    N = N // (8 ** scale)
    L = L - scale
    if n_override is not None:
        N = int(n_override)
    g = np.random.default_rng(0)
    if name == "C1":
        X = g.uniform(-1, 1, (N, 3))
        w = g.uniform(-1, 1, N)
        center, length = (0.0, 0.0, 0.0), 2.0
    elif name == "C2":
        X = g.uniform(-1, 1, (N, 3))
        w = g.standard_normal(N)
        center, length = (0.0, 0.0, 0.0), 2.0
    elif name == "C3":
        X = g.uniform(0, 1, (N, 3))
        w = g.standard_normal((N, m))
        center, length = (0.5, 0.5, 0.5), 1.0
    elif name == "C4":
        half = N // 2
        v = g.standard_normal((half, 3))
        S = v / np.linalg.norm(v, axis=1, keepdims=True)
        C = g.uniform(-1, 1, (32, 3))
        per = half // 32
        X2 = C[np.repeat(np.arange(32), per)] + 0.02 * g.standard_normal((per * 32, 3))
        X = np.vstack([S, X2])
        N = X.shape[0]
        w = g.uniform(-1, 1, N)
        center, length = domain_from_points(X)
    elif name == "C5":
        X = g.uniform(-1, 1, (N, 3))
        w = g.uniform(-1, 1, N)
        center, length = (0.0, 0.0, 0.0), 2.0
    else:  # pragma: no cover
        raise KeyError(name)
    idx = np.random.default_rng(1).choice(N, min(1000, N), replace=False)
    return {
        "name": name, "scale": scale, "points": X, "weights": w,
        "levels": L, "order": p, "scheme": scheme, "eps": eps,
        "kernel": kern, "ncols": m, "center": center, "length": length,
        "check_idx": idx,
    }
