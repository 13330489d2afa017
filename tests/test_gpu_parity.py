"""GPU parity: the CUDA path (through libbfmm.so) against the golden
fixtures of the real reference and against the CPU oracle.

Bars (BASELINE.json north_star): tree and lists bit-exact; phi within
relative L2 1e-10 in FP64 of the reference's own output.
"""

import hashlib

import numpy as np
import pytest

from conftest import golden, rel_l2, small_plan, unit_cloud

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1903_02153_b200 as bf  # noqa: E402
from paper_1903_02153_b200 import workloads  # noqa: E402
from paper_1903_02153_b200.kernel import workload_kernel  # noqa: E402
from oracle import fmm_oracle as O  # noqa: E402

PHI_TOL = 1e-10


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def plan_of(wl):
    return bf.FmmPlan(levels=wl["levels"], order=wl["order"], scheme=wl["scheme"],
                      eps=wl["eps"], domain_center=wl["center"], domain_length=wl["length"],
                      n_cols=wl["ncols"])


@pytest.fixture(scope="module")
def c1_eval(tmp_path_factory):
    wl = workloads.make("C1")
    ev = bf.FmmEvaluator(workload_kernel(wl["kernel"]), plan_of(wl),
                         cache_dir=str(tmp_path_factory.mktemp("c")))
    return wl, ev


# ---------------------------------------------------------------------------
# tree + lists: bit-exact

@pytest.mark.parametrize("tag,name,scale", [("c1", "C1", 0), ("c4s2", "C4", 2), ("c2s1", "C2", 1)])
def test_partition_bit_exact(tag, name, scale, cache_dir):
    g = golden("tree")
    wl = workloads.make(name, scale)
    ev = bf.FmmEvaluator(workload_kernel(wl["kernel"]), plan_of(wl), cache_dir=cache_dir)
    part = ev.partition(wl["points"])
    assert sha(part["perm"].astype(np.int64)) == str(g[f"{tag}_perm_sha"])
    assert np.array_equal(part["leaves"], g[f"{tag}_leaves"])
    assert np.array_equal(part["starts"], g[f"{tag}_starts"])
    assert np.array_equal(part["counts"], g[f"{tag}_counts"])
    if tag == "c1":
        assert np.array_equal(part["perm"], g["c1_perm"].astype(np.int64))


def test_partition_face_conventions(cache_dir):
    g = golden("tree")
    plan = bf.FmmPlan(levels=2, order=2, domain_center=(0.5, 0.5, 0.5), domain_length=1.0)
    ev = bf.FmmEvaluator(bf.LAPLACIAN, plan, cache_dir=cache_dir)
    part = ev.partition(g["faces_pts"])
    ids = np.empty(len(g["faces_pts"]), np.int64)
    for leaf, s, c in zip(part["leaves"], part["starts"], part["counts"]):
        ids[part["perm"][s:s + c]] = leaf
    assert np.array_equal(ids, g["faces_ids"])
    with pytest.raises(bf.DomainError):
        ev.partition(np.array([[1.1, 0.5, 0.5]]))


@pytest.mark.parametrize("lev", [2, 3, 4, 5])
def test_far_lists_bit_exact(lev, c1_eval):
    g = golden("lists")
    _, ev = c1_eval
    tgs, srs = [], []
    for j in range(316):
        tg, sr = ev.far_pairs(lev, j)
        tgs.append(tg)
        srs.append(sr)
    assert np.array_equal([len(a) for a in tgs], g[f"l{lev}_counts"])
    assert sha(np.concatenate(tgs)) == str(g[f"l{lev}_tg_sha"])
    assert sha(np.concatenate(srs)) == str(g[f"l{lev}_sr_sha"])
    if lev <= 3:
        assert np.array_equal(np.concatenate(tgs), g[f"l{lev}_tg"].astype(np.int64))


def test_near_lists_bit_exact(c1_eval):
    g = golden("lists")
    wl, ev = c1_eval
    ts, ss = [], []
    for t in range(27):
        a, b = ev.near_segments(wl["points"], t)
        ts.append(a)
        ss.append(b)
    assert np.array_equal([len(a) for a in ts], g["c1_near_counts"])
    assert np.array_equal(np.concatenate(ts), g["c1_near_tseg"].astype(np.int64))
    assert np.array_equal(np.concatenate(ss), g["c1_near_sseg"].astype(np.int64))


# ---------------------------------------------------------------------------
# phi parity against the reference's own outputs

def test_c1_phi_matches_reference(c1_eval):
    g = golden("c1_s0")
    wl, ev = c1_eval
    phi = ev.evaluate(wl["points"], weights=wl["weights"])
    assert rel_l2(phi, g["phi"]) < PHI_TOL
    acc = rel_l2(phi[wl["check_idx"]], g["direct_idx"])
    assert acc <= float(g["rel_l2_vs_direct"]) * 1.01 + 1e-15
    assert ev.timings["near_pairs"] == int(g["timings"][5])


@pytest.mark.parametrize("name", ["laplacian", "laplacianforce", "gaussian", "exponential",
                                  "logarithm"])
def test_builtin_kernels_match_reference_chebyshev(name, cache_dir):
    g = golden("engine")
    ev = bf.FmmEvaluator(bf.kernel_by_name(name), small_plan(), cache_dir=cache_dir)
    phi = ev.evaluate(g["cloud1500_pts"], weights=g["cloud1500_w"])
    assert rel_l2(phi, g[f"phi_{name}_chebyshev"]) < PHI_TOL
    assert rel_l2(phi, g[f"direct_{name}"]) < 1e-3


@pytest.mark.parametrize("name", ["laplacian", "laplacianforce", "gaussian", "exponential",
                                  "logarithm"])
def test_builtin_kernels_match_reference_uniform(name, cache_dir):
    g = golden("engine")
    ev = bf.FmmEvaluator(bf.kernel_by_name(name), small_plan(scheme="uniform"), cache_dir=cache_dir)
    phi = ev.evaluate(g["cloud1500_pts"], weights=g["cloud1500_w"])
    assert rel_l2(phi, g[f"phi_{name}_uniform"]) < PHI_TOL
    assert rel_l2(phi, g[f"direct_{name}"]) < 1e-3


def test_uniform_level4_multicolumn_matches_reference(cache_dir):
    g = golden("engine")
    plan = bf.FmmPlan(levels=4, order=5, scheme="uniform", eps=1e-6,
                      domain_center=(0.5, 0.5, 0.5), domain_length=1.0)
    ev = bf.FmmEvaluator(bf.EXPONENTIAL, plan, cache_dir=cache_dir)
    got = ev.evaluate(g["u4_pts"], weights=g["u4_w"])
    assert got.shape == (4000, 3)
    assert rel_l2(got, g["u4_phi"]) < PHI_TOL


def test_distinct_targets_match_reference(cache_dir):
    g = golden("engine")
    ev = bf.FmmEvaluator(bf.LAPLACIAN, small_plan(), cache_dir=cache_dir)
    got = ev.evaluate(g["tgt_src"], targets=g["tgt_t"], weights=g["tgt_w"])
    assert got.shape == (300,)
    assert rel_l2(got, g["tgt_phi"]) < PHI_TOL


@pytest.mark.parametrize("nc", [4, 20])
def test_multi_column_matches_reference(nc, cache_dir):
    g = golden("engine")
    ev = bf.FmmEvaluator(bf.LAPLACIAN, small_plan(), cache_dir=cache_dir)
    got = ev.evaluate(g["mc_pts"], weights=g[f"mc{nc}_w"])
    assert got.shape == (800, nc)
    assert rel_l2(got, g[f"mc{nc}_phi"]) < PHI_TOL
    for c in (0, nc - 1):
        single = ev.evaluate(g["mc_pts"], weights=g[f"mc{nc}_w"][:, c])
        assert np.max(np.abs(got[:, c] - single)) <= 1e-13 * np.max(np.abs(single))


def test_nonsymmetric_kernel_matches_reference(cache_dir):
    g = golden("engine")
    ks = bf.KernelSpec(name="skew", diff_func=lambda dx, dy, dz: np.exp(-(dx + 2 * dy) ** 2 - dz * dz),
                       symmetry=0, cuda_expr="exp(-(dx + 2.0 * dy) * (dx + 2.0 * dy) - dz * dz)",
                       cuda_arg="diff")
    plan = bf.FmmPlan(levels=3, order=4, scheme="chebyshev", eps=1e-7,
                      domain_center=(0.5, 0.5, 0.5), domain_length=1.0)
    ev = bf.FmmEvaluator(ks, plan, cache_dir=cache_dir)
    assert rel_l2(ev.evaluate(g["skew_pts"], weights=g["skew_w"]), g["skew_phi"]) < PHI_TOL


def test_order_sweep_matches_reference(cache_dir):
    g = golden("engine")
    for p in (2, 4, 6):
        plan = bf.FmmPlan(levels=3, order=p, scheme="chebyshev", eps=1e-10,
                          domain_center=(0.5, 0.5, 0.5), domain_length=1.0)
        got = bf.FmmEvaluator(bf.LAPLACIAN, plan, cache_dir=cache_dir).evaluate(
            g["ord_pts"], weights=g["ord_w"])
        assert rel_l2(got, g[f"ord{p}_phi"]) < PHI_TOL, p


@pytest.mark.parametrize("name,scale", [("C2", 1), ("C5", 3), ("C4", 2), ("C3", 2), ("C3", 1),
                                        ("C5", 2), ("C4", 1), ("C5", 1)])
def test_scaled_configs_match_reference(name, scale, cache_dir):
    g = golden(f"{name.lower()}_s{scale}")
    wl = workloads.make(name, scale)
    ev = bf.FmmEvaluator(workload_kernel(wl["kernel"]), plan_of(wl), cache_dir=cache_dir)
    phi = ev.evaluate(wl["points"], weights=wl["weights"])
    idx = wl["check_idx"]
    assert rel_l2(phi[idx], g["phi_idx"]) < PHI_TOL
    assert abs(np.linalg.norm(phi) - float(g["phi_norm"])) <= PHI_TOL * float(g["phi_norm"])
    acc = rel_l2(phi[idx], g["direct_idx"])
    assert acc <= float(g["rel_l2_vs_direct"]) * 1.01 + 1e-15
    assert ev.timings["near_pairs"] == int(g["timings"][5])


def test_c2_full_matches_reference(cache_dir):
    g = golden("c2_s0")
    wl = workloads.make("C2")
    ev = bf.FmmEvaluator(workload_kernel(wl["kernel"]), plan_of(wl), cache_dir=cache_dir)
    phi = ev.evaluate(wl["points"], weights=wl["weights"])
    idx = wl["check_idx"]
    assert rel_l2(phi[idx], g["phi_idx"]) < PHI_TOL
    assert rel_l2(phi[idx], g["direct_idx"]) <= float(g["rel_l2_vs_direct"]) * 1.01


# ---------------------------------------------------------------------------
# stage parity against the oracle (moments / locals per level)

def test_stage_moments_and_locals_match_oracle(cache_dir):
    wl = workloads.make("C2", 2)
    k = workload_kernel(wl["kernel"])
    plan = plan_of(wl)
    ev = bf.FmmEvaluator(k, plan, cache_dir=cache_dir)
    ev.keep_stages = True
    phi = ev.evaluate(wl["points"], weights=wl["weights"])
    orc = O.OracleFMM(k, wl["levels"], wl["order"], wl["scheme"], wl["eps"], wl["center"],
                      wl["length"], threads=4)
    ref = orc.matvec(wl["points"], weights=wl["weights"])
    assert rel_l2(phi, ref) < PHI_TOL
    p3 = wl["order"] ** 3
    for lev, mom in orc.stage["M"].items():
        got = ev.stages["moments"][lev].view(-1, 1, p3).cpu().numpy().transpose(0, 2, 1)
        assert rel_l2(got, mom) < 1e-12, lev
    # per-level locals after M2L + L2L, every level 2..L
    assert sorted(orc.stage["locals"]) == list(range(2, wl["levels"] + 1))
    for lev, loc in orc.stage["locals"].items():
        got = ev.stages["locals"][lev].view(-1, 1, p3).cpu().numpy().transpose(0, 2, 1)
        assert rel_l2(got, loc) < 1e-12, lev


# ---------------------------------------------------------------------------
# behaviour restated from the reference's engine tests (T/test_engine.py)

def test_single_point_self_interaction_is_zero(cache_dir):
    ev = bf.FmmEvaluator(bf.LAPLACIAN, small_plan(levels=2), cache_dir=cache_dir)
    out = ev.evaluate(np.array([[0.5, 0.5, 0.5]]), weights=np.array([3.0]))
    assert out.shape == (1,) and out[0] == 0.0


def test_constant_kernel_sums_weights(cache_dir):
    k = bf.KernelSpec(name="flatone", profile=lambda r: np.ones_like(r), symmetry=1,
                      cuda_expr="1.0", cuda_arg="r2")
    pts, w = unit_cloud(2000, seed=3)
    out = bf.FmmEvaluator(k, small_plan(), cache_dir=cache_dir).evaluate(pts, weights=w)
    assert np.allclose(out, w.sum(), rtol=0, atol=1e-10 * abs(w.sum()))


def test_repeat_runs_are_bitwise_identical(cache_dir):
    pts, w = unit_cloud(1000, seed=5)
    ev = bf.FmmEvaluator(bf.LAPLACIAN, small_plan(), cache_dir=cache_dir)
    assert np.array_equal(ev.evaluate(pts, weights=w), ev.evaluate(pts, weights=w))


def test_linearity_in_weights(cache_dir):
    pts, _ = unit_cloud(900, seed=12)
    gen = np.random.default_rng(13)
    u, v = gen.standard_normal(900), gen.standard_normal(900)
    ev = bf.FmmEvaluator(bf.EXPONENTIAL, small_plan(), cache_dir=cache_dir)
    lhs = ev.evaluate(pts, weights=2.5 * u - 0.75 * v)
    rhs = 2.5 * ev.evaluate(pts, weights=u) - 0.75 * ev.evaluate(pts, weights=v)
    # the int8 M2L cuts z under one power-of-two scale per column, so the
    # three evaluations truncate at different absolute levels (six 8-bit
    # digits: ~2^-40 of the scale); 1e-11 still sits 10x inside the 1e-10
    # parity bar
    assert np.max(np.abs(lhs - rhs)) / np.max(np.abs(rhs)) < 1e-11


def test_far_field_actually_contributes(cache_dir):
    pts, w = unit_cloud(1500, seed=14)
    ev = bf.FmmEvaluator(bf.LAPLACIAN, small_plan(), cache_dir=cache_dir)
    full = ev.evaluate(pts, weights=w)
    ev._disable_far_field = True
    near_only = ev.evaluate(pts, weights=w)
    ev._disable_far_field = False
    assert np.max(np.abs(full - near_only)) > 1e-3 * np.max(np.abs(full))
    orc = O.OracleFMM(bf.LAPLACIAN, 3, 4, "chebyshev", 1e-6, (0.5, 0.5, 0.5), 1.0)
    orc.disable_far = True
    assert rel_l2(near_only, orc.matvec(pts, weights=w)) < 1e-13


def test_nonfinite_kernel_value_reports_indices(cache_dir):
    k = bf.KernelSpec(name="rawinv", profile=lambda r: 1.0 / r, homogen=-1.0, symmetry=1,
                      cuda_expr="1.0 / r", cuda_arg="r")
    pts, w = unit_cloud(100, seed=16)
    ev = bf.FmmEvaluator(k, small_plan(levels=2, order=2), cache_dir=cache_dir)
    with pytest.raises(bf.KernelEvaluationError) as err:
        ev.evaluate(pts, targets=pts[37:38].copy(), weights=w)
    assert "target 0" in str(err.value) and "source 37" in str(err.value)
    assert err.value.indices == (0, 37)


@pytest.mark.parametrize("expr,edge", [("exp(-(r2 * 4.0e4))", "underflow"),
                                       ("exp(1.0 / r2)", "inf")])
def test_exp_out_of_range_arguments(expr, edge, cache_dir):
    """exp() arguments beyond the fast path (|x| >= 708, inf, NaN) take the
    exact path for their tile: tiny terms flush to 0 like NumPy's exp; an
    infinite exponent still reports the offending pair."""
    import numpy as _np
    if edge == "underflow":
        k = bf.KernelSpec(name="sharp", profile=lambda r: _np.exp(-(r * r) * 4.0e4),
                          homogen=0.0, symmetry=1, cuda_expr=expr, cuda_arg="r2")
        pts, w = unit_cloud(6000, seed=23)
        w = w[:, 0]
        plan = small_plan(levels=3, order=4)
        ev = bf.FmmEvaluator(k, plan, cache_dir=cache_dir)
        ev._disable_far_field = True
        got = ev.evaluate(pts, weights=w)
        # brute-force near field: sources in the 27 neighbour leaves (L = 3)
        cell = _np.clip(_np.floor(pts * 8.0).astype(_np.int64), 0, 7)
        ref = _np.zeros(len(pts))
        for i0 in range(0, len(pts), 500):
            d2 = ((pts[i0:i0 + 500, None, :] - pts[None, :, :]) ** 2).sum(-1)
            near = (_np.abs(cell[i0:i0 + 500, None, :] - cell[None, :, :]) <= 1).all(-1)
            ref[i0:i0 + 500] = (_np.where(near, _np.exp(-d2 * 4.0e4), 0.0) * w[None, :]).sum(1)
        assert rel_l2(got, ref) < 1e-12
    else:
        # finite on the far-field node grids, +inf at the self pairs (r = 0)
        k = bf.KernelSpec(name="blowup", profile=lambda r: _np.exp(1.0 / (r * r)),
                          homogen=0.0, symmetry=1, cuda_expr=expr, cuda_arg="r2")
        pts, w = unit_cloud(200, seed=24)
        ev = bf.FmmEvaluator(k, small_plan(levels=2, order=2), cache_dir=cache_dir)
        with pytest.raises(bf.KernelEvaluationError):
            ev.evaluate(pts, weights=w)


def _near_brute(pts, tgt, w, levels, fn):
    """Brute-force near field on the unit cube: sources in the 27 neighbour
    leaves of each target, K(0) = 0 (kernel.py:149-180)."""
    n = 1 << levels
    cs = np.clip(np.floor(pts * n).astype(np.int64), 0, n - 1)
    ct = np.clip(np.floor(tgt * n).astype(np.int64), 0, n - 1)
    out = np.zeros(len(tgt))
    for i0 in range(0, len(tgt), 400):
        d2 = ((tgt[i0:i0 + 400, None, :] - pts[None, :, :]) ** 2).sum(-1)
        near = (np.abs(ct[i0:i0 + 400, None, :] - cs[None, :, :]) <= 1).all(-1)
        with np.errstate(divide="ignore", invalid="ignore"):
            kv = np.where(d2 == 0.0, 0.0, fn(d2))
        out[i0:i0 + 400] = (np.where(near, kv, 0.0) * w[None, :]).sum(1)
    return out


@pytest.mark.parametrize("kname,distinct", [("laplacian", False), ("laplacianforce", False),
                                            ("laplacian", True), ("laplacianforce", True)])
def test_singular_kernels_crowded_leaves_and_coincident_points(kname, distinct, cache_dir):
    """The flag-free 1/r and 1/r^4 bodies (csrc/p2p.cuh, accum_fast): leaves
    of hundreds of points (64-target wide units plus 32-target remainders),
    exact duplicates inside a leaf (r = 0 contributes 0, kernel.py:149-180)
    and -- with distinct targets -- targets that coincide with sources."""
    gen = np.random.default_rng(77)
    crowd = np.clip(0.55 + 0.02 * gen.standard_normal((2500, 3)), 0.0, 1.0 - 1e-12)
    pts = np.vstack([crowd, gen.random((3000, 3)), crowd[:40], crowd[100:103]])
    w = gen.standard_normal(len(pts))
    fn = (lambda d2: 1.0 / np.sqrt(d2)) if kname == "laplacian" else (lambda d2: 1.0 / (d2 * d2))
    kern = bf.LAPLACIAN if kname == "laplacian" else workload_kernel("laplacianforce")
    ev = bf.FmmEvaluator(kern, small_plan(levels=3, order=3), cache_dir=cache_dir)
    ev._disable_far_field = True
    if distinct:
        tgt = np.vstack([pts[5:900:3], gen.random((700, 3)), crowd[2000:2200]])
        got = ev.evaluate(pts, targets=tgt, weights=w)
    else:
        tgt = pts
        got = ev.evaluate(pts, weights=w)
    ref = _near_brute(pts, tgt, w, 3, fn)
    assert np.all(np.isfinite(got))
    assert rel_l2(got, ref) < 1e-12


def test_laplace_subnormal_distances_take_exact_path(cache_dir):
    """Pairs whose r^2 is subnormal (points ~1e-160 apart next to the origin)
    break the hardware rsqrt seed (flush-to-zero): the sum turns non-finite,
    which is the flag that sends the tile through the exact body."""
    gen = np.random.default_rng(78)
    pts = gen.random((2000, 3))
    # on one axis, so r^2 = dx * dx is a single rounding on both sides
    tiny = np.array([[0.0, 0.0, 0.0], [1e-160, 0.0, 0.0], [3e-160, 0.0, 0.0],
                     [7e-160, 0.0, 0.0]])
    pts = np.vstack([pts, tiny])
    w = gen.standard_normal(len(pts))
    ev = bf.FmmEvaluator(bf.LAPLACIAN, small_plan(levels=3, order=3), cache_dir=cache_dir)
    ev._disable_far_field = True
    got = ev.evaluate(pts, weights=w)
    ref = _near_brute(pts, pts, w, 3, lambda d2: 1.0 / np.sqrt(d2))
    assert np.all(np.isfinite(got))
    # elementwise: the four tiny targets sum three ~1e160 terms of mixed sign
    assert np.max(np.abs(got - ref) / np.abs(ref)) < 1e-10
    assert np.max(np.abs(got[-4:])) > 1e150


def test_nvtx_ranges_do_not_change_results(cache_dir):
    """ev.nvtx (or BFMM_NVTX=1) wraps the stages and far-field levels in NVTX
    ranges for Nsight timelines; the matvec itself is untouched."""
    pts, w = unit_cloud(5000, seed=33)
    ev = bf.FmmEvaluator(bf.LAPLACIAN, small_plan(levels=3, order=4), cache_dir=cache_dir)
    a = ev.evaluate(pts, weights=w)
    ev.nvtx = True
    b = ev.evaluate(pts, weights=w)
    assert np.array_equal(a, b)
    assert set(ev.timings) >= {"distribute", "upward", "far_field", "downward", "near_field"}


def test_rejects_bad_inputs(cache_dir):
    pts, w = unit_cloud(100, seed=0)
    ev = bf.FmmEvaluator(bf.LAPLACIAN, small_plan(), cache_dir=cache_dir)
    with pytest.raises(bf.ConfigurationError):
        ev.evaluate(pts)
    with pytest.raises(bf.ConfigurationError):
        ev.evaluate(pts, weights=w[:50])
    bad = w.copy()
    bad[3] = np.nan
    with pytest.raises(bf.ConfigurationError):
        ev.evaluate(pts, weights=bad)
    out = pts.copy()
    out[0] = (2.5, 0.5, 0.5)
    with pytest.raises(bf.DomainError):
        ev.evaluate(out, weights=w)
    with pytest.raises(bf.ConfigurationError):
        ev.evaluate(pts[:, :2], weights=w)


def test_device_tensors_round_trip(cache_dir):
    pts, w = unit_cloud(3000, seed=31)
    ev = bf.FmmEvaluator(bf.LAPLACIAN, small_plan(), cache_dir=cache_dir)
    host = ev.evaluate(pts, weights=w[:, 0])
    dev = ev.evaluate(torch.from_numpy(pts).cuda(), weights=torch.from_numpy(w[:, 0]).cuda())
    assert dev.is_cuda and np.array_equal(dev.cpu().numpy(), host)


def _dipole():
    def dipole(dx, dy, dz):
        r2 = dx * dx + dy * dy + dz * dz
        with np.errstate(divide="ignore", invalid="ignore"):
            v = dx / (r2 * np.sqrt(r2))
        return np.where(r2 == 0, 0.0, v)
    return bf.KernelSpec(name="xdipole", diff_func=dipole, symmetry=-1, homogen=-2.0,
                         cuda_expr="(dx * dx + dy * dy + dz * dz) == 0.0 ? 0.0 : dx / "
                                   "((dx * dx + dy * dy + dz * dz) * sqrt(dx * dx + dy * dy + dz * dz))",
                         cuda_arg="diff")


@pytest.mark.parametrize("kname", ["gauss02", "laplacian", "dipole"])
def test_symmetric_near_field_matches_full(kname, cache_dir):
    """Transpose replay (reference engine.py:361-364) vs all 27 offsets, like
    T/test_engine.py::test_near_field_transpose_reuse_is_faithful."""
    kernel = _dipole() if kname == "dipole" else workload_kernel(kname)
    pts, w = unit_cloud(40000, seed=61)
    plan = bf.FmmPlan(levels=3, order=4, eps=1e-6, domain_center=(0.5, 0.5, 0.5),
                      domain_length=1.0)
    ev = bf.FmmEvaluator(kernel, plan, cache_dir=cache_dir)
    ev._disable_far_field = True
    ev.near_mode = "symmetric"
    a = ev.evaluate(pts, weights=w[:, 0])
    ev.near_mode = "full"
    b = ev.evaluate(pts, weights=w[:, 0])
    assert np.max(np.abs(a - b)) <= 1e-13 * np.max(np.abs(b))


def test_symmetric_near_field_falls_back_on_crowded_leaves(cache_dir):
    gen = np.random.default_rng(71)
    pts = np.clip(0.3 + 0.002 * gen.standard_normal((500, 3)), 0, 1)  # one crowded leaf
    pts = np.vstack([pts, gen.random((4000, 3))])
    w = gen.standard_normal(len(pts))
    plan = bf.FmmPlan(levels=3, order=3, eps=1e-6, domain_center=(0.5, 0.5, 0.5),
                      domain_length=1.0)
    ev = bf.FmmEvaluator(bf.LAPLACIAN, plan, cache_dir=cache_dir)
    ev.near_mode = "symmetric"
    a = ev.evaluate(pts, weights=w)
    ev.near_mode = "full"
    b = ev.evaluate(pts, weights=w)
    # device-side fallback: the plain P2P over all leaves (its chunk kernel
    # for every leaf, where "full" sends leaves of <= 8 points to the
    # thread-per-target kernel: same pairs, different summation order)
    assert rel_l2(a, b) < 1e-14


def test_empty_leaves_and_clusters(cache_dir):
    """Ragged occupancy: most leaves empty, a few crowded (C4-like)."""
    gen = np.random.default_rng(41)
    pts = np.clip(0.5 + 0.01 * gen.standard_normal((3000, 3)), 0, 1)
    pts = np.vstack([pts, gen.random((50, 3))])
    w = gen.standard_normal(len(pts))
    plan = bf.FmmPlan(levels=5, order=3, eps=1e-6, domain_center=(0.5, 0.5, 0.5),
                      domain_length=1.0)
    got = bf.FmmEvaluator(bf.LAPLACIAN, plan, cache_dir=cache_dir).evaluate(pts, weights=w)
    ref = O.OracleFMM(bf.LAPLACIAN, 5, 3, "chebyshev", 1e-6, (0.5, 0.5, 0.5), 1.0).matvec(
        pts, weights=w)
    assert rel_l2(got, ref) < PHI_TOL


@pytest.mark.parametrize("ncols,distinct", [(1, False), (3, False), (1, True)])
def test_active_far_field_matches_dense(ncols, distinct, cache_dir):
    """M2L over the ancestors of occupied target leaves only (far_mode
    "active") gives the dense result: empty cells' locals never reach a
    target (engine.py:206-226)."""
    gen = np.random.default_rng(83)
    pts = np.vstack([np.clip(c + 0.02 * gen.standard_normal((4000, 3)), 0, 1)
                     for c in (0.2, 0.55, 0.8)])
    w = gen.standard_normal((len(pts), ncols))
    tg = np.clip(0.6 + 0.05 * gen.standard_normal((3000, 3)), 0, 1) if distinct else None
    plan = bf.FmmPlan(levels=5, order=4, eps=1e-7, domain_center=(0.5, 0.5, 0.5),
                      domain_length=1.0)
    ev = bf.FmmEvaluator(bf.EXPONENTIAL, plan, cache_dir=cache_dir)
    res = {}
    for mode in ("dense", "active", "auto"):
        ev.far_mode = mode
        res[mode] = ev.evaluate(pts, targets=tg, weights=w)
    assert rel_l2(res["active"], res["dense"]) < 1e-14
    assert rel_l2(res["auto"], res["dense"]) < 1e-14
    if not distinct:
        ref = O.OracleFMM(bf.EXPONENTIAL, 5, 4, "chebyshev", 1e-7, (0.5, 0.5, 0.5), 1.0).matvec(
            pts, weights=w)
        assert rel_l2(res["active"], ref.reshape(res["active"].shape)) < PHI_TOL


@pytest.mark.parametrize("scheme", ["chebyshev", "uniform"])
def test_l2p_point_and_warp_kernels_agree_bitwise(scheme, cache_dir):
    """The thread-per-point and leaf-cell-chunk L2P (sparse clouds) and the
    warp-per-leaf one do the same arithmetic: identical phi, including 3
    columns and crowded leaves (> 32 points)."""
    gen = np.random.default_rng(97)
    pts = np.vstack([gen.random((3000, 3)),
                     np.clip(0.4 + 0.01 * gen.standard_normal((400, 3)), 0, 1)])
    w = gen.standard_normal((len(pts), 3))
    plan = bf.FmmPlan(levels=4, order=4, scheme=scheme, eps=1e-6,
                      domain_center=(0.5, 0.5, 0.5), domain_length=1.0)
    ev = bf.FmmEvaluator(bf.EXPONENTIAL, plan, cache_dir=cache_dir)
    ev.l2p_mode = "warp"
    a = ev.evaluate(pts, weights=w)
    ev.l2p_mode = "point"
    b = ev.evaluate(pts, weights=w)
    assert np.array_equal(a, b)
    ev.l2p_mode = "cells"  # leaf-cell chunks, locals staged in shared memory
    c = ev.evaluate(pts, weights=w)
    assert np.array_equal(a, c)


@pytest.mark.parametrize("name,scale", [("C5", 2), ("C4", 2)])
def test_p2m_cell_chunks_equal_warp_per_leaf(name, scale, cache_dir):
    """The sparse-cloud P2M over leaf-cell chunks (bfmm_p2m_cells, zeros for
    empty cells, no memset) gives the warp-per-leaf kernel's moments: the
    same products in the same order (bitwise where a chunk's points fit one
    batch, C5; crowded C4 chunks split the sums)."""
    wl = workloads.make(name, scale)
    ev = bf.FmmEvaluator(workload_kernel(wl["kernel"]), plan_of(wl), cache_dir=cache_dir)
    ev.keep_stages = True
    out = {}
    for mode in ("leaf", "cells"):
        ev.p2m_mode = mode
        phi = ev.evaluate(wl["points"], weights=wl["weights"])
        out[mode] = (phi, ev.stages["moments"][wl["levels"]].cpu().numpy())
    if name == "C5":
        assert np.array_equal(out["leaf"][1], out["cells"][1])
    else:
        assert rel_l2(out["cells"][1], out["leaf"][1]) < 1e-14
    assert rel_l2(out["cells"][0], out["leaf"][0]) < 1e-13


@pytest.mark.parametrize("name,scale", [("C5", 2), ("C4", 2)])
def test_grouped_near_field_matches(name, scale, cache_dir):
    """The one-thread-per-target near field (p2p_group_kernel, which
    bfmm_p2p runs for leaves of <= 8 points) against the 32-target-chunk
    kernel for every leaf and against the reference fixture."""
    g = golden(f"{name.lower()}_s{scale}")
    wl = workloads.make(name, scale)
    ev = bf.FmmEvaluator(workload_kernel(wl["kernel"]), plan_of(wl), cache_dir=cache_dir)
    ev.keep_stages = True
    out = {}
    for mode in ("auto", "grouped"):
        ev.near_mode = mode
        phi = ev.evaluate(wl["points"], weights=wl["weights"])
        out[mode] = (phi, ev.stages["near"].cpu().numpy())
        assert rel_l2(phi[wl["check_idx"]], g["phi_idx"]) < PHI_TOL
    assert rel_l2(out["grouped"][1], out["auto"][1]) < 1e-14


@pytest.mark.parametrize("name,scale", [("C5", 2), ("C4", 2), ("C4", 3)])
def test_tiled_near_field_bitwise_equals_untiled(name, scale, cache_dir, monkeypatch):
    """p2p_tile_kernel (sources of a 4 x 4 x 4 block's halo staged in shared
    memory; clustered blocks over kTileCap points stream from global memory):
    its thread-per-target mode sums the same pairs in the same order as
    p2p_group_kernel (bitwise equal near fields, uniform C5 and clustered C4,
    both paths); the default warp-per-cell mode (lane partial sums, fixed
    butterfly) agrees to rounding."""
    wl = workloads.make(name, scale)
    ev = bf.FmmEvaluator(workload_kernel(wl["kernel"]), plan_of(wl), cache_dir=cache_dir)
    ev.keep_stages = True
    near = {}
    for mode in ("auto", "untiled", "auto0"):
        if mode == "auto0":
            monkeypatch.setenv("BFMM_TILE_MODE", "0")
        ev.near_mode = mode[:4] if mode == "auto0" else mode
        ev.evaluate(wl["points"], weights=wl["weights"])
        near[mode] = ev.stages["near"].cpu().numpy()
    assert np.array_equal(near["auto0"], near["untiled"])
    assert rel_l2(near["auto"], near["untiled"]) < 1e-14


@pytest.mark.parametrize("name,scale", [("C5", 2), ("C4", 2), ("uniform", 0)])
def test_leaf_pair_matches_separate_passes(name, scale, cache_dir):
    """Leaf-pair P2M / L2P (parent moments straight from the points, the
    parent's locals evaluated through its own basis -- no L -> L-1 M2M and
    no L-1 -> L L2L) against the separate passes, and against the reference
    fixture where one exists (engine.py:176-204, 296-327)."""
    if name == "uniform":
        pts, w = unit_cloud(20000, seed=77)
        w = w[:, 0]
        plan = bf.FmmPlan(levels=5, order=4, scheme="uniform", eps=1e-6,
                          domain_center=(0.5, 0.5, 0.5), domain_length=1.0)
        kern, g = bf.EXPONENTIAL, None
    else:
        wl = workloads.make(name, scale)
        pts, w, plan = wl["points"], wl["weights"], plan_of(wl)
        kern, g = workload_kernel(wl["kernel"]), golden(f"{name.lower()}_s{scale}")
    ev = bf.FmmEvaluator(kern, plan, cache_dir=cache_dir)
    out = {}
    for mode in ("pair", "plain"):
        ev.leaf_mode = mode
        out[mode] = ev.evaluate(pts, weights=w)
    assert rel_l2(out["pair"], out["plain"]) < 1e-13
    if g is not None:
        assert rel_l2(out["pair"][wl["check_idx"]], g["phi_idx"]) < PHI_TOL


def test_stencil_variants_bitwise(cache_dir, monkeypatch):
    """The three FFT-M2L stencil kernels -- stencil_kernel (4 same-parity z
    targets per thread), stencil2_kernel (two x targets per thread) and the
    default stencil3_kernel (a whole z column per thread) -- apply the same
    taps in the same order per target, so phi is bitwise equal (uniform
    scheme, engine.py:258-292).  Level 5 has interior and boundary tiles;
    level 2 (n = 4) is smaller than a tile."""
    pts, w = unit_cloud(30000, seed=91, ncols=3)
    plan = bf.FmmPlan(levels=5, order=4, scheme="uniform", eps=1e-6,
                      domain_center=(0.5, 0.5, 0.5), domain_length=1.0)
    ev = bf.FmmEvaluator(bf.EXPONENTIAL, plan, cache_dir=cache_dir)
    out = {}
    for mode in ("3", "1", "2"):
        monkeypatch.setenv("BFMM_STENCIL", mode)
        out[mode] = ev.evaluate(pts, weights=w)
    assert np.array_equal(out["3"], out["1"])
    assert np.array_equal(out["2"], out["1"])
