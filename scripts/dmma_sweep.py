import sys, ctypes as C
sys.path.insert(0, ".")
import torch
from paper_1903_02153_b200 import _native
lib = _native.load()
f = lib.bfmm_device_dmma_sweep
f.restype = C.c_int; f.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_double), C.c_void_p]
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for w in (4, 8, 16, 32):
    row = []
    for ch in (1, 2, 4, 8, 16):
        g = C.c_double(0); f(w, ch, C.byref(g), s); row.append(f"{g.value/1e3:6.1f}")
    print(f"warps/SM {w:2d}: chains 1,2,4,8,16 ->", " ".join(row), "TF")
