"""Measured tcgen05 kind::i8 peak (bfmm_device_i8_probe) -- diagnostic."""
import ctypes as C
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
from paper_1903_02153_b200 import _native  # noqa: E402
lib = _native.load()
v = C.c_double(0)
for _ in range(3):
    rc = lib.bfmm_device_i8_probe(C.byref(v), C.c_void_p(torch.cuda.current_stream().cuda_stream))
    print("rc", rc, "int8 TOPS", round(v.value, 1), flush=True)
for N in (64, 128, 192, 256):
    rc = lib.bfmm_device_i8_probe_n(N, C.byref(v), C.c_void_p(torch.cuda.current_stream().cuda_stream))
    print("N", N, "rc", rc, "int8 TOPS", round(v.value, 1), flush=True)
