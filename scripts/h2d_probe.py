import time, numpy as np, torch, sys
sys.path.insert(0, ".")
x = torch.empty(32 * 1024 * 1024 // 8, dtype=torch.float64).pin_memory()
d = torch.empty_like(x, device="cuda")
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(x, non_blocking=True); torch.cuda.synchronize()
    print("H2D 32MB %.3f ms -> %.1f GB/s" % ((time.perf_counter()-t0)*1e3, 32*1.048576e6/((time.perf_counter()-t0)*1e9)))
import subprocess
print(subprocess.run(["nvidia-smi", "--query-gpu=pci.link.gen.current,pci.link.width.current", "--format=csv"], capture_output=True, text=True).stdout)
