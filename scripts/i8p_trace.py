"""Wait-time trace of one m2l_i8p CTA's MMA warp (plane-buffer and core-block
waits, clock64) from a -DBFMM_I8_TRACE build -- development helper."""
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
cs, cpow = _i8_core_slices(g.standard_normal((316, rp, rp)), S)
dcs = torch.from_numpy(cs.reshape(-1)).cuda(); dcp = torch.from_numpy(cpow).cuda()
zs = torch.empty(int(lib.bfmm_m2l_i8_zs_bytes(ncell, rp, S)), dtype=torch.int8, device="cuda")
zmax = torch.empty(1, dtype=torch.int64, device="cuda")
_native.check(lib.bfmm_m2l_i8_slice_z(z.data_ptr(), ncell, 1, rp, S, zs.data_ptr(), zmax.data_ptr(), st), "s")
ns = int(sys.argv[1]) if len(sys.argv) > 1 else 1
lt = torch.empty(ncell * ns * rp, dtype=torch.float64, device="cuda")
for it in range(2):
    _native.check(lib.bfmm_m2l_i8(zs.data_ptr(), zmax.data_ptr(), dcs.data_ptr(), dcp.data_ptr(),
                                  lt.data_ptr(), level, m, rp, S, ns, 0, ncell // 8, st), "i8")
torch.cuda.synchronize()
tr = np.zeros(8192, dtype=np.int64)
lib.bfmm_i8_trace_read(tr.ctypes.data)
ev = tr[:8000].reshape(-1, 2)
ev = ev[ev[:, 0] != 0]
plane = ev[:, 1] < 0
t0, t1 = ev[:, 0], np.abs(ev[:, 1])
wait = t1 - t0
print("events", len(ev), "plane waits", plane.sum(), "core waits", (~plane).sum())
span = t1.max() - t0.min()
print("CTA span (clk)", span, "plane wait total", wait[plane].sum(), "core wait total", wait[~plane].sum())
bw = t1[~plane]
print("core-stage period (median clk)", np.median(np.diff(bw)))
print("first 40 waits:", [(('P' if p else 'B'), int(w)) for p, w in zip(plane[:40], wait[:40])])
