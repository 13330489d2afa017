"""Host-side interpolation setup (reference interpolation.py:47-155).

Only small p x p / p^3 x p^3 factors are built here; the per-point weights
are evaluated on the device (csrc/interp.cu) from the coefficients this
module uploads.
"""

from __future__ import annotations

import numpy as np

from .errors import ConfigurationError, DomainError
from .plan import SchemeKind

_EDGE_TOL = 1e-12


def nodes_1d(p: int, scheme: SchemeKind) -> np.ndarray:
    """Ascending Chebyshev roots cos(pi (2k-1) / 2p), or p equispaced
    points on [-1, 1] (interpolation.py:47-56)."""
    if p < 1:
        raise ConfigurationError(f"interpolation order must be >= 1, got {p}")
    if p == 1:
        return np.zeros(1)
    if scheme is SchemeKind.CHEBYSHEV:
        return np.cos(np.pi * (2 * np.arange(p, 0, -1) - 1) / (2 * p))
    return np.linspace(-1.0, 1.0, p)


def chebyshev_coefficients(p: int) -> np.ndarray:
    """S[n, j] = c_n T_n(x_j), c_0 = 1/p, c_n = 2/p, so that the weight of
    node j at x is sum_n T_n(x) S[n, j] (interpolation.py:59-66, 80-83)."""
    nd = nodes_1d(p, SchemeKind.CHEBYSHEV)
    tn = np.cos(np.outer(np.arange(p), np.arccos(np.clip(nd, -1.0, 1.0))))
    c = np.full(p, 2.0 / p)
    c[0] = 1.0 / p
    return c[:, None] * tn


def interp_matrix_1d(x, p: int, scheme: SchemeKind) -> np.ndarray:
    """W[i, j]: weight of node j at x[i] (interpolation.py:66-90)."""
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    if x.size and np.max(np.abs(x)) > 1.0 + _EDGE_TOL:
        raise DomainError(f"interpolation point {x[np.argmax(np.abs(x))]} outside [-1, 1]")
    nd = nodes_1d(p, scheme)
    if scheme is SchemeKind.CHEBYSHEV:
        tx = np.cos(np.outer(np.arange(p), np.arccos(np.clip(x, -1.0, 1.0))))
        return tx.T @ chebyshev_coefficients(p)
    w = np.ones((x.size, p))
    for j in range(p):
        for k in range(p):
            if k != j:
                w[:, j] *= (x - nd[k]) / (nd[j] - nd[k])
    return w


def interp_matrix_3d(points, p: int, scheme: SchemeKind) -> np.ndarray:
    """Row a = (i*p + j)*p + k: weight of node (x_i, y_j, z_k)."""
    pts = np.atleast_2d(np.asarray(points, dtype=np.float64))
    w = [interp_matrix_1d(pts[:, a], p, scheme) for a in range(3)]
    return (w[0][:, :, None, None] * w[1][:, None, :, None]
            * w[2][:, None, None, :]).reshape(pts.shape[0], p ** 3)


def nodes_3d(p: int, scheme: SchemeKind, half_width: float = 1.0) -> np.ndarray:
    nd = nodes_1d(p, scheme)
    g = np.meshgrid(nd, nd, nd, indexing="ij")
    return half_width * np.stack([a.ravel() for a in g], axis=1)


def half_interval_matrices(p: int, scheme: SchemeKind) -> np.ndarray:
    """H[s][a, b]: weight of parent node a at the child node b of the lower
    (s = 0) or upper (s = 1) half; T[o] = kron(H[ox], H[oy], H[oz])
    (interpolation.py:136-155)."""
    nd = nodes_1d(p, scheme)
    return np.stack([interp_matrix_1d(0.5 * sign + 0.5 * nd, p, scheme).T
                     for sign in (-1.0, 1.0)])


def child_transfer_matrices(p: int, scheme: SchemeKind) -> np.ndarray:
    """Dense (8, p^3, p^3) transfers, for tests and diagnostics only; the
    device applies the Kronecker factors."""
    H = half_interval_matrices(p, scheme)
    out = np.empty((8, p ** 3, p ** 3))
    for o in range(8):
        out[o] = np.kron(H[(o >> 2) & 1], np.kron(H[(o >> 1) & 1], H[o & 1]))
    return out


def device_interp_blob(p: int, scheme: SchemeKind) -> np.ndarray:
    """The host array bfmm_p2m / bfmm_l2p take: p nodes then p*p S."""
    S = chebyshev_coefficients(p) if scheme is SchemeKind.CHEBYSHEV else np.zeros((p, p))
    return np.ascontiguousarray(np.concatenate([nodes_1d(p, scheme), S.ravel()]))
