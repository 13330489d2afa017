"""Build libbfmm.so (the C-ABI of include/bfmm.h) in-tree for sm_100a.

    python -m paper_1903_02153_b200.build [--force]

nvcc cross-compiles without a GPU; the resulting .so lives next to the
package (paper_1903_02153_b200/_lib/libbfmm.so) so it travels to the GPU
box with the repository snapshot.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(OUT_DIR, "libbfmm.so")
OBJ_DIR = os.path.join(ROOT, "build", "obj")

SOURCES = ["tree.cu", "interp.cu", "m2l_cheb.cu", "m2l_fft.cu", "p2p.cu", "misc.cu"]
HEADERS = ["common.cuh", "p2p.cuh", "m2l_ws.cuh", "m2l_i8.cuh", "proj_i8.cuh", "tcgen05.cuh",
           "leaf_kernels.cuh", "transfer_kernels.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def _embed_p2p_source():
    src = open(os.path.join(CSRC, "p2p.cuh")).read()
    inc = os.path.join(CSRC, "p2p_src.inc")
    text = 'R"BFMMSRC(' + src + ')BFMMSRC"\n'
    if not os.path.exists(inc) or open(inc).read() != text:
        with open(inc, "w") as f:
            f.write(text)


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OUT_DIR, exist_ok=True)
    os.makedirs(OBJ_DIR, exist_ok=True)
    _embed_p2p_source()
    # every header under csrc/ (a new .cuh is tracked without listing it)
    hdrs = sorted({os.path.join(CSRC, h) for h in HEADERS} |
                  {os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")}) + [
        os.path.join(ROOT, "include", "bfmm.h"), os.path.join(CSRC, "p2p_src.inc")]
    objs, jobs = [], []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(OBJ_DIR, s.replace(".cu", ".o"))
        objs.append(obj)
        if force or _stale(obj, [src] + hdrs):
            jobs.append([nvcc(), *ARCH, *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"),
                         "-c", src, "-o", obj])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        return r.stderr

    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        logs = list(ex.map(run, jobs))
    if verbose:
        for log in logs:
            sys.stderr.write(log)
    if force or jobs or _stale(LIB, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", LIB, *objs, "-lnvrtc", "-ldl",
               "-Xlinker", "-rpath=/usr/local/cuda/lib64"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
