"""tcgen05 int8 self-test against an exact CPU product (diagnostic)."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1903_02153_b200 import _native  # noqa: E402

lib = _native.load()
g = np.random.default_rng(0)
for K in (32, 64, 256, 12096):
    A = g.integers(-64, 65, (128, K), dtype=np.int8)
    B = g.integers(-64, 65, (64, K), dtype=np.int8)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    D = torch.zeros((128, 64), dtype=torch.int32, device="cuda")
    rc = lib.bfmm_tc_i8_selftest(dA.data_ptr(), dB.data_ptr(), K, D.data_ptr(),
                                 C.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    ref = A.astype(np.int64) @ B.astype(np.int64).T
    got = D.cpu().numpy()
    print(K, rc, "exact" if np.array_equal(got, ref) else
          f"MISMATCH max|d|={np.abs(got - ref).max()} got[0,:4]={got[0,:4]} ref[0,:4]={ref[0,:4]}",
          flush=True)
