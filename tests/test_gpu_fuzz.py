"""Seeded randomized parity sweep: the CUDA path against the CPU oracle.

Each case draws a configuration (tree depth, order, scheme, kernel, weight
columns, shared or distinct targets, uniform or clustered cloud, domain
offset and size) from a fixed seed and compares phi at rel-L2 1e-10, the
bar of SURVEY §8(c)(5).  Sizes stay small so the NumPy oracle finishes in
seconds; the oracle itself is pinned to the reference in
tests/test_oracle_golden.py.
"""

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1903_02153_b200 as bf  # noqa: E402
from oracle import fmm_oracle as O  # noqa: E402

KERNELS = ["laplacian", "laplacianforce", "gaussian", "exponential", "logarithm"]


def _case(seed):
    g = np.random.default_rng(1000 + seed)
    levels = int(g.integers(2, 5))
    order = int(g.integers(2, 7))
    scheme = "uniform" if g.random() < 0.35 else "chebyshev"
    kernel = bf.kernel_by_name(KERNELS[int(g.integers(0, len(KERNELS)))])
    m = int(g.choice([1, 1, 2, 3]))
    n = int(g.integers(200, 2500))
    center = g.uniform(-2, 2, 3)
    length = float(g.uniform(0.5, 4.0))
    lo = center - length / 2
    if g.random() < 0.4:  # clustered: a few tight blobs plus background
        k = int(g.integers(2, 5))
        cents = lo + length * g.uniform(0.15, 0.85, (k, 3))
        pts = cents[g.integers(0, k, n)] + 0.03 * length * g.standard_normal((n, 3))
        pts = np.clip(pts, lo, lo + length)
    else:
        pts = lo + length * g.random((n, 3))
    w = g.standard_normal((n, m))
    tgt = None
    if g.random() < 0.3:
        tgt = lo + length * g.random((int(g.integers(50, 800)), 3))
    eps = float(g.choice([1e-5, 1e-7, 1e-9]))
    return dict(levels=levels, order=order, scheme=scheme, kernel=kernel, pts=pts, w=w,
                tgt=tgt, center=tuple(center), length=length, eps=eps)


@pytest.mark.parametrize("seed", range(48))
def test_random_config_matches_oracle(seed, cache_dir):
    c = _case(seed)
    plan = bf.FmmPlan(levels=c["levels"], order=c["order"], scheme=c["scheme"], eps=c["eps"],
                      domain_center=c["center"], domain_length=c["length"])
    ev = bf.FmmEvaluator(c["kernel"], plan, cache_dir=cache_dir)
    got = ev.evaluate(c["pts"], targets=c["tgt"], weights=c["w"])
    orc = O.OracleFMM(c["kernel"], c["levels"], c["order"], c["scheme"], c["eps"], c["center"],
                      c["length"])
    ref = orc.matvec(c["pts"], targets=c["tgt"], weights=c["w"])
    assert got.shape == ref.shape
    assert rel_l2(got, ref) < 1e-10, {k: v for k, v in c.items() if k not in ("pts", "w", "tgt")}
