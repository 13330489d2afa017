"""The int8 tensor-core M2L (csrc/m2l_i8.cuh, m2l_mode "i8") against the
FP64 tensor-core M2L (m2l_mode "dmma") and the reference fixtures.

The i8 path is exact integer arithmetic on digit planes, so its error
against FP64 is the digit truncation: about 2^(-7S) of the operand scales
(S digits of 7 bits) or 2^(-8S+1) (six 8-bit digits, BFMM_I8_BASE256), and
it is bitwise repeatable.
"""

import numpy as np
import pytest

from conftest import golden, rel_l2

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1903_02153_b200 as bf  # noqa: E402
from paper_1903_02153_b200 import _native, workloads  # noqa: E402
from paper_1903_02153_b200.engine import _i8_core_slices  # noqa: E402
from paper_1903_02153_b200.kernel import workload_kernel  # noqa: E402

PHI_TOL = 1e-10


def _run_both(level, rp, m, S, ns, seed=0, gather=False, bits=7):
    lib = _native.load()
    st = _native.C.c_void_p(torch.cuda.current_stream().cuda_stream)
    g = np.random.default_rng(seed)
    ncell = 8 ** level
    # rows of very different magnitude (as z of empty vs crowded cells)
    z = g.standard_normal((ncell * m, rp)) * np.exp(g.uniform(-4, 0, (ncell * m, 1)))
    cores = g.standard_normal((316, rp, rp)) * np.logspace(0, -7, rp)[None, :, None]
    dz, dc = torch.from_numpy(z).cuda(), torch.from_numpy(cores).cuda()
    nq = ncell // 8
    ref = torch.zeros(ncell * m * rp, dtype=torch.float64, device="cuda")
    _native.check(lib.bfmm_m2l_cheb(dz.data_ptr(), ref.data_ptr(), level, m, rp, 1, 0, nq,
                                    dc.data_ptr(), st), "cheb")
    cs, cpow = _i8_core_slices(cores, S, bits)
    Sarg = S | (_native.I8_BASE256 if bits == 8 else 0)
    dcs, dcp = torch.from_numpy(cs.reshape(-1)).cuda(), torch.from_numpy(cpow).cuda()
    rows = ncell * m
    zs = torch.empty(int(lib.bfmm_m2l_i8_zs_bytes(rows, rp, Sarg)), dtype=torch.int8, device="cuda")
    zmax = torch.empty(m, dtype=torch.int64, device="cuda")
    _native.check(lib.bfmm_m2l_i8_slice_z(dz.data_ptr(), rows, m, rp, Sarg, zs.data_ptr(),
                                          zmax.data_ptr(), st), "slice")
    outs = []
    if gather:  # diagnostic switch: force the gather kernel on a dense level
        import os
        os.environ["BFMM_I8_GATHER"] = "1"
    for _ in range(2):
        lt = torch.full((rows * ns * rp,), float("nan"), dtype=torch.float64, device="cuda")
        _native.check(lib.bfmm_m2l_i8(zs.data_ptr(), zmax.data_ptr(), dcs.data_ptr(),
                                      dcp.data_ptr(), lt.data_ptr(), level, m, rp, Sarg, ns, 0, nq,
                                      st), "i8")
        outs.append(lt)
    torch.cuda.synchronize()
    if gather:
        del os.environ["BFMM_I8_GATHER"]
    assert torch.equal(outs[0], outs[1]), "i8 M2L not bitwise repeatable"
    got = outs[0].view(rows, ns, rp).sum(1).cpu().numpy()
    return got, ref.view(rows, rp).cpu().numpy(), outs[0]


@pytest.mark.parametrize("ncell,nact,p3,rp,m,bits", [(4096, 300, 216, 168, 1, 7), (512, 40, 125, 61, 3, 8),
                                                      (4096, 1, 64, 37, 1, 8)])
def test_listed_cell_projection_and_slicing_equal_dense(ncell, nact, p3, rp, m, bits):
    """Sparse clouds (C ABI): bfmm_rows_gemm_cells and
    bfmm_m2l_i8_slice_z_cells over the listed (occupied) cells against the
    dense bfmm_rows_gemm / bfmm_m2l_i8_slice_z over every cell, the other
    cells' moments being zero: z rows, digit scale and digit planes bitwise
    equal (engine.py:233; the evaluator's active far field on a shared tree)."""
    lib = _native.load()
    st = _native.C.c_void_p(torch.cuda.current_stream().cuda_stream)
    g = np.random.default_rng(ncell + nact)
    cells = np.sort(g.choice(ncell, nact, replace=False)).astype(np.int64)
    mom = np.zeros((ncell * m, p3))
    for c in cells:
        mom[c * m:(c + 1) * m] = g.standard_normal((m, p3)) * np.exp(g.uniform(-6, 2))
    V = g.standard_normal((p3, rp))
    dm, dV, dc = torch.from_numpy(mom).cuda(), torch.from_numpy(V).cuda(), torch.from_numpy(cells).cuda()
    z_dense = torch.full((ncell * m, rp), float("nan"), dtype=torch.float64, device="cuda")
    _native.check(lib.bfmm_rows_gemm(dm.data_ptr(), ncell * m, p3, dV.data_ptr(), rp,
                                     z_dense.data_ptr(), 1.0, 0.0, 1, st), "rows_gemm")
    z_list = torch.zeros((ncell * m, rp), dtype=torch.float64, device="cuda")
    _native.check(lib.bfmm_rows_gemm_cells(dm.data_ptr(), nact * m, p3, dV.data_ptr(), rp,
                                           z_list.data_ptr(), 1.0, dc.data_ptr(), m, st),
                  "rows_gemm_cells")
    torch.cuda.synchronize()
    assert torch.equal(z_dense, z_list)
    S = 6 if bits == 8 else 7
    Sarg = S | (_native.I8_BASE256 if bits == 8 else 0)
    nbytes = int(lib.bfmm_m2l_i8_zs_bytes(ncell * m, rp, Sarg))
    zs_d = torch.full((nbytes,), 55, dtype=torch.int8, device="cuda")
    zs_l = torch.zeros(nbytes, dtype=torch.int8, device="cuda")
    zm_d = torch.empty(m, dtype=torch.int64, device="cuda")
    zm_l = torch.empty(m, dtype=torch.int64, device="cuda")
    _native.check(lib.bfmm_m2l_i8_slice_z(z_dense.data_ptr(), ncell * m, m, rp, Sarg,
                                          zs_d.data_ptr(), zm_d.data_ptr(), st), "slice")
    _native.check(lib.bfmm_m2l_i8_slice_z_cells(z_list.data_ptr(), nact * m, m, rp, Sarg,
                                                zs_l.data_ptr(), zm_l.data_ptr(), dc.data_ptr(),
                                                st), "slice_cells")
    torch.cuda.synchronize()
    assert torch.equal(zm_d, zm_l)
    assert torch.equal(zs_d, zs_l)


@pytest.mark.parametrize("level,rp,m,S,ns", [(3, 56, 1, 7, 1), (3, 104, 1, 7, 3),
                                             (3, 64, 3, 6, 2), (2, 168, 1, 8, 1),
                                             (4, 56, 1, 5, 4), (2, 8, 2, 7, 189),
                                             (5, 56, 1, 7, 1), (5, 104, 2, 7, 3),
                                             (4, 104, 1, 7, 1), (4, 48, 3, 6, 2),
                                             (5, 64, 1, 8, 2), (6, 24, 1, 6, 1)])
def test_i8_translation_matches_dmma(level, rp, m, S, ns):
    got, ref, _ = _run_both(level, rp, m, S, ns)
    assert np.all(np.isfinite(got))
    # per weight column (each has its own digit scale)
    for c in range(m):
        err = rel_l2(got[c::m], ref[c::m])
        print(f"S={S} column {c}: rel-L2 {err:.3e}")
        # digit truncation (one scale for rows spanning e^-4 costs ~7 bits)
        # or the FP64 floor
        assert err < max(2.0 ** (8 - 7 * S), 1e-14), (c, err)


@pytest.mark.parametrize("level,rp,m,ns", [(3, 56, 1, 1), (3, 64, 2, 2), (5, 64, 1, 1),
                                          (4, 48, 3, 2), (6, 24, 1, 1), (5, 96, 1, 3)])
def test_i8_base256_digits_match_dmma(level, rp, m, ns):
    """Six signed 8-bit digits (21 digit products; csrc/m2l_i8.cuh
    z_slice_kernel<6, 8>, engine._i8_core_slices(bits=8)) where the int32
    accumulation bound allows it."""
    got, ref, _ = _run_both(level, rp, m, 6, ns, bits=8)
    assert np.all(np.isfinite(got))
    for c in range(m):
        err = rel_l2(got[c::m], ref[c::m])
        assert err < max(2.0 ** (10 - 8 * 6), 1e-14), (c, err)
    if level >= 4:  # plane kernel == gather kernel, bitwise
        _, _, a = _run_both(level, rp, m, 6, 1, bits=8)
        _, _, b = _run_both(level, rp, m, 6, 1, gather=True, bits=8)
        assert torch.equal(a, b)


def test_i8_base256_rejects_plans_past_the_int32_bound():
    lib = _native.load()
    st = _native.C.c_void_p(torch.cuda.current_stream().cuda_stream)
    rc = lib.bfmm_m2l_i8(None, None, None, None, None, 4, 1, 128, 6 | _native.I8_BASE256, 1, 0,
                         8 ** 3, st)
    assert rc == 2 and b"8-bit digits" in lib.bfmm_last_error()


def test_i8_split_blocks_past_the_last_offset_are_zero():
    # 189 offsets over 100 splits of 2: splits 95..99 have no offsets
    got, ref, _ = _run_both(2, 56, 1, 7, 100)
    assert np.abs(got - ref).max() < 1e-12 * np.abs(ref).max()
    # the plane kernel's splits run over 56 (chunk, plane) units
    got, ref, _ = _run_both(5, 56, 1, 7, 16)
    assert np.abs(got - ref).max() < 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("level,rp,m,S", [(5, 56, 1, 7), (5, 40, 2, 6), (4, 104, 1, 7),
                                          (4, 64, 2, 8)])
def test_i8_plane_and_gather_kernels_agree_bitwise(level, rp, m, S):
    """Dense levels >= 4 use the plane-buffered kernel (1 x 16 x 8 tiles, or
    2 x 8 x 8 at level 4); its int32 sums are the gather kernel's integers,
    so the lt blocks are bitwise equal."""
    _, _, a = _run_both(level, rp, m, S, 1)
    _, _, b = _run_both(level, rp, m, S, 1, gather=True)
    assert torch.equal(a, b)


@pytest.mark.parametrize("level,rp,m", [(5, 64, 1), (5, 96, 2), (6, 64, 1)])
def test_i8_cta_pair_variants_agree_bitwise(level, rp, m, monkeypatch):
    """Six 8-bit digits at dense levels >= 5 run the CTA-pair kernel
    (m2l_i8p2_kernel).  Its default form issues the three a + 2k = 5 digit
    pairs as N = 64 MMAs (exactly the 21 products); the unsplit form
    (BFMM_I8P2_N128) runs 24 and drops 3 in an unread accumulator; the
    single-CTA plane kernel (BFMM_I8_1CTA) runs the 21 one CTA at a time.
    Same integer sums in accumulators 0..5, so all three are bitwise equal."""
    outs = []
    for env in ({}, {"BFMM_I8P2_N128": "1"}, {"BFMM_I8_1CTA": "1"}):
        for k in ("BFMM_I8P2_N128", "BFMM_I8_1CTA"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        got, ref, lt = _run_both(level, rp, m, 6, 1, bits=8)
        for c in range(m):
            assert rel_l2(got[c::m], ref[c::m]) < 2.0 ** (10 - 8 * 6)
        outs.append(lt)
    assert torch.equal(outs[0], outs[1])
    assert torch.equal(outs[0], outs[2])


@pytest.mark.parametrize("name,scale", [("C2", 1), ("C5", 3), ("C4", 2)])
@pytest.mark.parametrize("mode,S", [("dmma", 7), ("i8", 6), ("i8", 7), ("i8", 8)])
def test_m2l_engines_match_reference(name, scale, mode, S, cache_dir):
    """Both M2L engines (and other digit counts than the default) meet the
    phi bar against the reference fixtures."""
    g = golden(f"{name.lower()}_s{scale}")
    wl = workloads.make(name, scale)
    plan = bf.FmmPlan(levels=wl["levels"], order=wl["order"], scheme=wl["scheme"], eps=wl["eps"],
                      domain_center=wl["center"], domain_length=wl["length"], n_cols=wl["ncols"])
    ev = bf.FmmEvaluator(workload_kernel(wl["kernel"]), plan, cache_dir=cache_dir)
    ev.m2l_mode, ev.i8_slices = mode, S
    if S == 7:
        ev.i8_digits = "base128"  # the 7-bit split itself (auto would use 8-bit digits)
    phi = ev.evaluate(wl["points"], weights=wl["weights"])
    idx = wl["check_idx"]
    assert rel_l2(phi[idx], g["phi_idx"]) < PHI_TOL


def test_i8_and_dmma_agree_on_c2_scaled(cache_dir):
    wl = workloads.make("C2", 1)
    plan = bf.FmmPlan(levels=wl["levels"], order=wl["order"], eps=wl["eps"],
                      domain_center=wl["center"], domain_length=wl["length"])
    ev = bf.FmmEvaluator(workload_kernel(wl["kernel"]), plan, cache_dir=cache_dir)
    res = {}
    for mode in ("dmma", "i8"):
        ev.m2l_mode = mode
        res[mode] = ev.evaluate(wl["points"], weights=wl["weights"])
    assert rel_l2(res["i8"], res["dmma"]) < 1e-12


@pytest.mark.parametrize("rows,K,N", [(1000, 125, 64), (777, 64, 125), (300, 8, 8),
                                      (129, 100, 104), (5000, 27, 16)])
def test_int8_projection_matches_fp64(rows, K, N):
    """bfmm_rows_gemm_i8 (per-row digit scales, six 8-bit digits, csrc/
    proj_i8.cuh) against the FP64 product: rows of very different magnitude
    (empty vs crowded cells), a zero row and a non-finite row; the zmax
    epilogue equals max |C|."""
    lib = _native.load()
    st = _native.C.c_void_p(torch.cuda.current_stream().cuda_stream)
    g = np.random.default_rng(rows + K)
    A = g.standard_normal((rows, K)) * np.exp(g.uniform(-30, 5, (rows, 1)))
    A[3] = 0.0
    B = g.standard_normal((K, N)) * np.logspace(0, -6, N)[None, :]
    d, pw = _i8_core_slices(np.ascontiguousarray(B.T)[None], 6, 8)
    dA = torch.from_numpy(A).cuda()
    dd, dp = torch.from_numpy(d.reshape(-1)).cuda(), torch.from_numpy(pw).cuda()
    C = torch.full((rows, N), float("nan"), dtype=torch.float64, device="cuda")
    zmax = torch.zeros(1, dtype=torch.int64, device="cuda")
    _native.check(lib.bfmm_rows_gemm_i8(dA.data_ptr(), rows, K, dd.data_ptr(), dp.data_ptr(), N,
                                        C.data_ptr(), 0.5, zmax.data_ptr(), st), "gemm_i8")
    got = C.cpu().numpy()
    want = 0.5 * (A @ B)
    # per row, relative to the row's scale (|A_r| |B|): the digit truncation
    scale = np.abs(A).max(axis=1, keepdims=True) * np.abs(B).max() * K
    assert np.all(np.abs(got - want) <= 1e-12 * scale + 1e-300)
    assert np.all(got[3] == 0.0)
    zm = zmax.cpu().numpy().view(np.float64)[0]
    assert zm == np.abs(got).max()
    # a non-finite row propagates (NaN), the others are untouched
    A[7, 2] = np.inf
    dA = torch.from_numpy(A).cuda()
    _native.check(lib.bfmm_rows_gemm_i8(dA.data_ptr(), rows, K, dd.data_ptr(), dp.data_ptr(), N,
                                        C.data_ptr(), 0.5, None, st), "gemm_i8")
    got2 = C.cpu().numpy()
    assert np.isnan(got2[7]).all()
    assert np.array_equal(np.delete(got2, 7, axis=0), np.delete(got, 7, axis=0))


@pytest.mark.parametrize("name,scale", [("C2", 1), ("C5", 2), ("C4", 2)])
def test_int8_projections_match_fp64_projections(name, scale, cache_dir):
    """proj_mode "i8" (z = M V and locals = s lt U^T on the int8 tensor
    cores) against the FP64 DMMA projections, and against the reference."""
    wl = workloads.make(name, scale)
    plan = bf.FmmPlan(levels=wl["levels"], order=wl["order"], scheme=wl["scheme"], eps=wl["eps"],
                      domain_center=wl["center"], domain_length=wl["length"], n_cols=wl["ncols"])
    ev = bf.FmmEvaluator(workload_kernel(wl["kernel"]), plan, cache_dir=cache_dir)
    out = {}
    for mode in ("i8", "fp64"):
        ev.proj_mode = mode
        out[mode] = ev.evaluate(wl["points"], weights=wl["weights"])
    assert rel_l2(out["i8"], out["fp64"]) < 1e-12
    g = golden(f"{name.lower()}_s{scale}")
    assert rel_l2(out["i8"][wl["check_idx"]], g["phi_idx"]) < PHI_TOL
