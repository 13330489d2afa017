import sys, ctypes as C
sys.path.insert(0, ".")
import torch
from paper_1903_02153_b200 import _native
lib = _native.load()
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for name in ("bfmm_device_fp64_probe", "bfmm_device_dmma_probe"):
    g = C.c_double(0)
    _native.check(getattr(lib, name)(C.byref(g), s), name)
    print(name, f"{g.value/1e3:.2f} TFLOP/s")
