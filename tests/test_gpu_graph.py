"""CUDA-graph replay of the device step (FmmEvaluator.use_graph): the same
kernels on the same buffers, so phi is bitwise equal to the eager path, for
host, pinned and device inputs, and across replays with new data."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1903_02153_b200 as bf  # noqa: E402
from paper_1903_02153_b200 import workloads  # noqa: E402
from paper_1903_02153_b200.kernel import workload_kernel  # noqa: E402


def _ev(name, scale, cache_dir):
    wl = workloads.make(name, scale)
    plan = bf.FmmPlan(levels=wl["levels"], order=wl["order"], scheme=wl["scheme"], eps=wl["eps"],
                      domain_center=wl["center"], domain_length=wl["length"], n_cols=wl["ncols"])
    return wl, bf.FmmEvaluator(workload_kernel(wl["kernel"]), plan, cache_dir=cache_dir)


@pytest.mark.parametrize("name,scale", [("C1", 0), ("C2", 1)])
def test_graph_replay_bitwise_equals_eager(name, scale, cache_dir):
    wl, ev = _ev(name, scale, cache_dir)
    X, w = wl["points"], np.ascontiguousarray(wl["weights"])
    eager = ev.evaluate(X, weights=w)
    ev.use_graph = True
    for _ in range(2):  # capture, then replay
        got = ev.evaluate(X, weights=w)
        assert np.array_equal(got, eager)
    assert ev.timings["near_pairs"] > 0
    # stage timings come from event nodes inside the graph (eng:505-533 keys)
    for k in ("distribute", "upward", "far_field", "downward"):
        assert ev.timings[k] > 0.0, k
    assert ev.timings["total"] > 0.0
    # device tensors in, device tensor out
    dX, dw = torch.from_numpy(X).cuda(), torch.from_numpy(w).cuda()
    got = ev.evaluate(dX, weights=dw)
    assert got.is_cuda and np.array_equal(got.cpu().numpy(), eager)
    # pinned host tensors
    hX, hw = torch.from_numpy(X).pin_memory(), torch.from_numpy(w).pin_memory()
    got = ev.evaluate(hX, weights=hw)
    assert got.device.type == "cpu" and np.array_equal(got.numpy(), eager)
    # new data through the same graph
    g = np.random.default_rng(5)
    w2 = g.standard_normal(w.shape)
    X2 = np.clip(X + 1e-3 * g.standard_normal(X.shape), -0.999, 0.999) if name != "C3" else X
    ev.use_graph = False
    eager2 = ev.evaluate(X2, weights=w2)
    ev.use_graph = True
    assert np.array_equal(ev.evaluate(X2, weights=w2), eager2)


def test_graph_multi_column_and_fallbacks(cache_dir):
    wl, ev = _ev("C1", 0, cache_dir)
    X = wl["points"]
    w = np.random.default_rng(2).standard_normal((X.shape[0], 3))
    eager = ev.evaluate(X, weights=w)
    ev.use_graph = True
    assert np.array_equal(ev.evaluate(X, weights=w), eager)
    # distinct targets are not captured: the eager path runs
    t = X[:500] * 0.5
    ev.use_graph = False
    ref = ev.evaluate(X, targets=t, weights=w)
    ev.use_graph = True
    assert np.array_equal(ev.evaluate(X, targets=t, weights=w), ref)
    # errors still surface (a point outside the box)
    bad = X.copy()
    bad[7] = 5.0
    with pytest.raises(ValueError):
        ev.evaluate(bad, weights=w)


def test_graph_recaptures_when_a_knob_changes(cache_dir):
    """The graph key holds every knob that changes the captured kernels: a
    change after a capture re-captures instead of replaying stale kernels."""
    wl, ev = _ev("C2", 1, cache_dir)
    X, w = wl["points"], np.ascontiguousarray(wl["weights"])
    ev.m2l_mode = "dmma"
    dmma = ev.evaluate(X, weights=w)
    ev.m2l_mode = "i8"
    i8 = ev.evaluate(X, weights=w)
    assert not np.array_equal(dmma, i8)  # the engines differ in the last bits
    ev.use_graph = True
    assert np.array_equal(ev.evaluate(X, weights=w), i8)
    ev.m2l_mode = "dmma"
    assert np.array_equal(ev.evaluate(X, weights=w), dmma)
    assert len(ev._graphs) == 2
