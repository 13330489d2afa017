"""Stage timeline of one m2l_i8 CTA (level-5 sized problem), from a
-DBFMM_I8_TRACE build (development helper)."""
import ctypes as C
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1903_02153_b200 import _native
from paper_1903_02153_b200.engine import _i8_core_slices
lib = _native.load(_native.LIB_PATH.replace("libbfmm.so", "libbfmm_trace.so"))
lib.bfmm_i8_trace_read.argtypes = [C.c_void_p]
st = C.c_void_p(0)
g = np.random.default_rng(0)
level, rp, m, S = 5, 56, 1, 7
ncell = 8 ** level
z = torch.from_numpy(g.standard_normal((ncell, rp))).cuda()
cores = g.standard_normal((316, rp, rp))
cs, cpow = _i8_core_slices(cores, S)
dcs = torch.from_numpy(cs.reshape(-1)).cuda(); dcp = torch.from_numpy(cpow).cuda()
zs = torch.empty(int(lib.bfmm_m2l_i8_zs_bytes(ncell, rp, S)), dtype=torch.int8, device="cuda")
zmax = torch.empty(m, dtype=torch.int64, device="cuda")
_native.check(lib.bfmm_m2l_i8_slice_z(z.data_ptr(), ncell, m, rp, S, zs.data_ptr(), zmax.data_ptr(), st), "slice")
ns = int(sys.argv[1]) if len(sys.argv) > 1 else 4
lt = torch.empty(ncell * ns * rp, dtype=torch.float64, device="cuda")
for it in range(3):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    _native.check(lib.bfmm_m2l_i8(zs.data_ptr(), zmax.data_ptr(), dcs.data_ptr(), dcp.data_ptr(),
                                  lt.data_ptr(), level, m, rp, S, ns, 0, ncell // 8, st), "i8")
    e1.record(); torch.cuda.synchronize()
    print("kernel ms", e0.elapsed_time(e1))
tr = np.zeros(8192, dtype=np.int64)
lib.bfmm_i8_trace_read(tr.ctypes.data)
nst = (189 + ns - 1) // ns * 2
mma = tr[:nst]; t0 = mma[0]
prod = [tr[1024 * (1 + w):1024 * (1 + w) + nst] for w in range(4)]
print("steps", nst, "MMA full-wait-done deltas (clk):", np.diff(mma)[:40].tolist())
print("median MMA stage period", np.median(np.diff(mma)))
for w in range(4):
    print(f"warp {w} issue - t0:", (prod[w][:24] - t0).tolist())
print("issue->full lag (steps 5..):", (mma[5:40] - prod[0][5:40]).tolist())
print("total clk", mma[-1] - prod[0][0])
