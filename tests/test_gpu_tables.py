"""M2L tables built on the GPU (reference operators.py:244-341):
the dense family and the difference grids evaluated by the device functor,
the stacked QR on the device, SVD + rank cut on the host.  Same ranks and
the same operators (dense blocks U C_t V^T) as the reference's own tables
(tests/golden/tables.npz), for symmetric, antisymmetric and non-symmetric
kernels, Chebyshev and uniform."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1903_02153_b200 as bf  # noqa: E402
from paper_1903_02153_b200 import _native, workloads  # noqa: E402
from paper_1903_02153_b200.kernel import workload_kernel  # noqa: E402
from paper_1903_02153_b200.tables import DeviceTableBuilder, precompute_m2l  # noqa: E402


def _builder(kernel):
    ev_like = bf.FmmEvaluator.__new__(bf.FmmEvaluator)
    ev_like.kernel, ev_like.lib = kernel, _native.load()
    handle = ev_like._kernel_handle()
    return DeviceTableBuilder(kernel, handle, ev_like.lib, torch.device("cuda"),
                              bf.FmmEvaluator._stream)


@pytest.mark.parametrize("tag,name", [("c1", "C1"), ("c2", "C2"), ("c5", "C5"), ("c3", "C3"),
                                      ("c4", "C4")])
def test_device_tables_match_reference_golden(tag, name):
    g = golden("tables")
    probe = [tuple(t) for t in g["probe_offsets"]]
    wl = workloads.make(name, n_override=8)
    if name == "C4":
        wl["center"], wl["length"] = (0.04243, 0.00945, -0.01194), 2.14973
    plan = bf.FmmPlan(levels=wl["levels"], order=wl["order"], scheme=wl["scheme"],
                      eps=wl["eps"], domain_center=wl["center"], domain_length=wl["length"])
    k = workload_kernel(wl["kernel"])
    b = _builder(k)
    t = precompute_m2l(k, plan, use_cache=False, builder=b)
    assert b.fallbacks == 0
    assert t.single_level == bool(g[f"{tag}_single"])
    assert t.nbytes() == int(g[f"{tag}_nbytes"])
    for lev in g[f"{tag}_levels"]:
        if f"{tag}_rank_{lev}" in g:
            assert t.blocks[int(lev)].rank == int(g[f"{tag}_rank_{lev}"])
    for lev in (2, 3, 4):
        key = f"{tag}_dense_{lev}"
        if key not in g:
            continue
        for j, off in enumerate(probe[:g[key].shape[0]]):
            d = t.dense(off, lev)
            ref = g[key][j]
            assert np.max(np.abs(d - ref)) <= 1e-11 * np.max(np.abs(ref)), (tag, lev, off)


def test_device_tables_nonsymmetric_and_antisymmetric():
    g = golden("tables")
    probe = [tuple(t) for t in g["probe_offsets"]]
    dip = bf.KernelSpec(
        name="xdipole", symmetry=-1, homogen=-2.0,
        diff_func=lambda dx, dy, dz: np.where(dx * dx + dy * dy + dz * dz == 0, 0.0,
                                              dx / ((dx * dx + dy * dy + dz * dz) ** 1.5)),
        cuda_expr="(dx * dx + dy * dy + dz * dz) == 0.0 ? 0.0 : dx / ((dx * dx + dy * dy + "
                  "dz * dz) * sqrt(dx * dx + dy * dy + dz * dz))", cuda_arg="diff")
    skew = bf.KernelSpec(name="skew", symmetry=0,
                         diff_func=lambda dx, dy, dz: np.exp(-(dx + 2 * dy) ** 2 - dz * dz),
                         cuda_expr="exp(-(dx + 2.0 * dy) * (dx + 2.0 * dy) - dz * dz)",
                         cuda_arg="diff")
    for kern, tag, lev in ((dip, "dipole", 2), (skew, "skew", 2)):
        plan = bf.FmmPlan(levels=2, order=3, scheme="chebyshev", eps=1e-7)
        b = _builder(kern)
        t = precompute_m2l(kern, plan, use_cache=False, builder=b)
        blk = t.blocks[min(t.blocks)]
        assert blk.rank == int(g[f"{tag}_rank"])
        for j, off in enumerate(probe):
            ref = g[f"{tag}_dense"][j]
            assert np.max(np.abs(t.dense(off, lev) - ref)) <= 1e-11 * np.max(np.abs(ref))


def test_device_build_is_the_default_and_matches_host_build(cache_dir):
    plan = bf.FmmPlan(levels=3, order=8, eps=1e-10, domain_center=(0.5, 0.5, 0.5),
                      domain_length=1.0)
    ev = bf.FmmEvaluator(bf.LAPLACIAN, plan, use_cache=False)
    assert ev.table_builder is not None and ev.table_builder.fallbacks == 0
    host = precompute_m2l(bf.LAPLACIAN, plan, use_cache=False)
    assert ev.table.blocks[0].rank == host.blocks[0].rank == 288
    for off in [(2, 0, 0), (3, -1, 2), (-3, -3, -3)]:
        a, r = ev.table.dense(off, 3), host.dense(off, 3)
        assert np.max(np.abs(a - r)) <= 1e-12 * np.max(np.abs(r))
