"""Pin the CPU oracle (oracle/fmm_oracle.py) to the REAL reference.

The fixtures were produced by importing the reference (boxfmm) in the
builder container (tests/golden/make_golden.py).  CPU only.
"""

import hashlib

import numpy as np
import pytest

from conftest import golden, rel_l2
from oracle import fmm_oracle as O
from paper_1903_02153_b200 import workloads
from paper_1903_02153_b200.kernel import kernel_by_name, workload_kernel


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("tag,name,scale", [("c1", "C1", 0), ("c4s2", "C4", 2), ("c2s1", "C2", 1)])
def test_oracle_partition_bit_exact(tag, name, scale):
    g = golden("tree")
    wl = workloads.make(name, scale)
    assert np.array_equal(g[f"{tag}_center"], np.array(wl["center"]))
    b = O.Binned(wl["points"], wl["center"], wl["length"], wl["levels"])
    assert sha(b.perm.astype(np.int64)) == str(g[f"{tag}_perm_sha"])
    assert np.array_equal(b.leaves, g[f"{tag}_leaves"])
    assert np.array_equal(b.starts, g[f"{tag}_starts"])
    assert np.array_equal(b.counts, g[f"{tag}_counts"])


def test_oracle_face_conventions():
    g = golden("tree")
    ids = O.leaf_of(g["faces_pts"], (0.5, 0.5, 0.5), 1.0, 2)
    assert np.array_equal(ids, g["faces_ids"])


@pytest.mark.parametrize("lev", [2, 3, 4, 5])
def test_oracle_far_lists_bit_exact(lev):
    g = golden("lists")
    assert np.array_equal(O.FAR, g["offsets"])
    tg = [O.offset_pairs(lev, t)[0] for t in O.FAR]
    sr = [O.offset_pairs(lev, t)[1] for t in O.FAR]
    assert np.array_equal([len(a) for a in tg], g[f"l{lev}_counts"])
    assert sha(np.concatenate(tg)) == str(g[f"l{lev}_tg_sha"])
    assert sha(np.concatenate(sr)) == str(g[f"l{lev}_sr_sha"])


def test_oracle_tables_match_reference():
    g = golden("tables")
    probe = [tuple(t) for t in g["probe_offsets"]]
    for tag, name in (("c1", "C1"), ("c2", "C2"), ("c5", "C5")):
        wl = workloads.make(name, n_override=8)
        k = workload_kernel(wl["kernel"])
        blocks, single = O.build_tables(k, wl["levels"], wl["order"], wl["scheme"], wl["eps"],
                                        wl["length"])
        assert bool(single) == bool(g[f"{tag}_single"])
        for lev in g[f"{tag}_levels"]:
            assert blocks[int(lev)]["u"].shape[1] == int(g[f"{tag}_rank_{lev}"])
        for lev in (2, 3, 4):
            key = f"{tag}_dense_{lev}"
            if key not in g:
                continue
            blk = blocks[0] if single else blocks[lev]
            s = O.level_scale(k, single, wl["length"], lev)
            for j, t in enumerate(probe[:g[key].shape[0]]):
                jj = [tuple(x) for x in O.FAR].index(t)
                d = s * blk["u"] @ blk["cores"][jj] @ blk["v"].T
                ref = g[key][j]
                assert np.max(np.abs(d - ref)) <= 1e-12 * np.max(np.abs(ref))


def _oracle_for(wl, threads=1):
    k = workload_kernel(wl["kernel"])
    return O.OracleFMM(k, wl["levels"], wl["order"], wl["scheme"], wl["eps"],
                       wl["center"], wl["length"], threads=threads)


def test_oracle_c1_matches_reference():
    g = golden("c1_s0")
    wl = workloads.make("C1")
    phi = _oracle_for(wl).matvec(wl["points"], weights=wl["weights"])
    assert rel_l2(phi, g["phi"]) < 1e-12
    d = O.direct_sum(kernel_by_name("laplacian"), wl["points"],
                     targets=wl["points"][wl["check_idx"]], weights=wl["weights"])
    assert rel_l2(d, g["direct_idx"]) < 1e-14


@pytest.mark.parametrize("name,scale", [("C2", 1), ("C5", 3)])
def test_oracle_scaled_configs_match_reference(name, scale):
    g = golden(f"{name.lower()}_s{scale}")
    wl = workloads.make(name, scale)
    phi = _oracle_for(wl, threads=O.default_threads()).matvec(wl["points"], weights=wl["weights"])
    assert rel_l2(phi[wl["check_idx"]], g["phi_idx"]) < 1e-12


def test_oracle_engine_cases_match_reference():
    g = golden("engine")
    pts, w = g["cloud1500_pts"], g["cloud1500_w"]
    for name in ("laplacian", "gaussian", "logarithm"):
        k = kernel_by_name(name)
        for scheme in ("chebyshev", "uniform"):
            fmm = O.OracleFMM(k, 3, 4, scheme, 1e-6, (0.5, 0.5, 0.5), 1.0)
            phi = fmm.matvec(pts, weights=w)
            assert rel_l2(phi, g[f"phi_{name}_{scheme}"]) < 1e-12, (name, scheme)
    # non-symmetric kernel (distinct U / V)
    from paper_1903_02153_b200 import KernelSpec
    ks = KernelSpec(name="skew", diff_func=lambda dx, dy, dz: np.exp(-(dx + 2 * dy) ** 2 - dz * dz),
                    symmetry=0)
    fmm = O.OracleFMM(ks, 3, 4, "chebyshev", 1e-7, (0.5, 0.5, 0.5), 1.0)
    assert rel_l2(fmm.matvec(g["skew_pts"], weights=g["skew_w"]), g["skew_phi"]) < 1e-12
    # distinct targets
    fmm = O.OracleFMM(kernel_by_name("laplacian"), 3, 4, "chebyshev", 1e-6, (0.5, 0.5, 0.5), 1.0)
    got = fmm.matvec(g["tgt_src"], targets=g["tgt_t"], weights=g["tgt_w"])
    assert rel_l2(got, g["tgt_phi"]) < 1e-12
    # multi-column (m = 20)
    got = fmm.matvec(g["mc_pts"], weights=g["mc20_w"])
    assert rel_l2(got, g["mc20_phi"]) < 1e-12
