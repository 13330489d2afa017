"""Kernel-level check: bfmm_m2l_i8 vs bfmm_m2l_cheb (DMMA) on random z and
cores (development helper; run on the GPU box)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1903_02153_b200 import _native  # noqa: E402
from paper_1903_02153_b200.engine import _i8_core_slices  # noqa: E402

lib = _native.load()
st = _native.C.c_void_p(0)
g = np.random.default_rng(0)
import os
for level, rp, m, S in [(4, 104, 1, 7), (4, 56, 2, 7), (5, 56, 1, 7), (4, 128, 1, 8), (3, 56, 1, 7)]:
    ncell = 8 ** level
    z = g.standard_normal((ncell * m, rp)) * np.exp(g.uniform(-3, 0, (ncell * m, 1)))
    cores = g.standard_normal((316, rp, rp)) * np.logspace(0, -6, rp)[None, :, None]
    dz = torch.from_numpy(z).cuda()
    dc = torch.from_numpy(cores).cuda()
    nq = ncell // 8
    lt_ref = torch.zeros(ncell * m * rp, dtype=torch.float64, device="cuda")
    _native.check(lib.bfmm_m2l_cheb(dz.data_ptr(), lt_ref.data_ptr(), level, m, rp, 1, 0, nq,
                                    dc.data_ptr(), st), "cheb")
    cs, cpow = _i8_core_slices(cores, S)
    dcs = torch.from_numpy(cs.reshape(-1)).cuda()
    dcp = torch.from_numpy(cpow).cuda()
    rows = ncell * m
    zs = torch.empty(int(lib.bfmm_m2l_i8_zs_bytes(rows, rp, S)), dtype=torch.int8, device="cuda")
    zmax = torch.empty(m, dtype=torch.int64, device="cuda")
    _native.check(lib.bfmm_m2l_i8_slice_z(dz.data_ptr(), rows, m, rp, S, zs.data_ptr(),
                                          zmax.data_ptr(), st), "slice")
    for ns in (1, 3):
        lt = torch.full((ncell * m * ns * rp,), float("nan"), dtype=torch.float64, device="cuda")
        _native.check(lib.bfmm_m2l_i8(zs.data_ptr(), zmax.data_ptr(), dcs.data_ptr(),
                                      dcp.data_ptr(), lt.data_ptr(), level, m, rp, S, ns, 0, nq,
                                      st), "i8")
        torch.cuda.synchronize()
        for rep in range(5):  # bitwise repeatable (exact int32 accumulation)
            lt2 = torch.full_like(lt, float("nan"))
            _native.check(lib.bfmm_m2l_i8(zs.data_ptr(), zmax.data_ptr(), dcs.data_ptr(),
                                          dcp.data_ptr(), lt2.data_ptr(), level, m, rp, S, ns, 0,
                                          nq, st), "i8")
            assert torch.equal(lt, lt2), "not repeatable"
        os.environ["BFMM_I8_GATHER"] = "1"
        ltg = torch.full_like(lt, float("nan"))
        _native.check(lib.bfmm_m2l_i8(zs.data_ptr(), zmax.data_ptr(), dcs.data_ptr(),
                                      dcp.data_ptr(), ltg.data_ptr(), level, m, rp, S, ns, 0,
                                      nq, st), "i8 gather")
        del os.environ["BFMM_I8_GATHER"]
        torch.cuda.synchronize()
        if ns == 1:
            print("  plane == gather bitwise:", torch.equal(lt, ltg))
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e2 = torch.cuda.Event(enable_timing=True)
        e0.record()
        _native.check(lib.bfmm_m2l_i8(zs.data_ptr(), zmax.data_ptr(), dcs.data_ptr(),
                                      dcp.data_ptr(), lt.data_ptr(), level, m, rp, S, ns, 0,
                                      nq, st), "i8")
        e1.record()
        os.environ["BFMM_I8_GATHER"] = "1"
        _native.check(lib.bfmm_m2l_i8(zs.data_ptr(), zmax.data_ptr(), dcs.data_ptr(),
                                      dcp.data_ptr(), ltg.data_ptr(), level, m, rp, S, ns, 0,
                                      nq, st), "i8 gather")
        del os.environ["BFMM_I8_GATHER"]
        e2.record(); torch.cuda.synchronize()
        print(f"  ms: default {e0.elapsed_time(e1):.3f}  gather {e1.elapsed_time(e2):.3f}")
        a = lt.view(ncell * m, ns, rp).sum(1).cpu().numpy()
        b = lt_ref.view(ncell * m, rp).cpu().numpy()
        err = np.abs(a - b).max() / np.abs(b).max()
        bad = np.argwhere(np.abs(a - b) > 1e-6 * np.abs(b).max())
        print(f"level {level} rp {rp} m {m} S {S} ns {ns}: max rel err {err:.3e}; "
              f"bad entries {len(bad)} first {bad[:4].tolist()}", flush=True)
