#!/bin/bash
# Build variant libraries of the leaf-pair kernels (P2M / L2P) -- batch size
# and occupancy floor -- into paper_1903_02153_b200/_lib/var/ (run here, the
# .so files travel to the GPU box), then time each on C5 with
#   BFMM_LIB=... BFMM_PROFILE=1 python scripts/one_config.py C5
set -e
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
cd "$ROOT"
python -m paper_1903_02153_b200.build > /dev/null
mkdir -p build/var paper_1903_02153_b200/_lib/var
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I include"
for v in "64 4" "48 4" "32 4" "32 6" "32 8" "48 6"; do
  set -- $v
  tag=b$1_m$2
  nvcc $FLAGS -DBFMM_PAIR_BATCH=$1 -DBFMM_PAIR_MINB=$2 -Xptxas -v -c paper_1903_02153_b200/csrc/interp.cu -o build/var/interp_$tag.o 2> build/var/interp_$tag.log &
done
wait
for v in "64 4" "48 4" "32 4" "32 6" "32 8" "48 6"; do
  set -- $v
  tag=b$1_m$2
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_1903_02153_b200/_lib/var/libbfmm_$tag.so \
    build/var/interp_$tag.o build/obj/tree.o build/obj/m2l_cheb.o build/obj/m2l_fft.o build/obj/p2p.o build/obj/misc.o \
    -lnvrtc -ldl -Xlinker -rpath=/usr/local/cuda/lib64
  echo "$tag: $(grep -A1 'pair_kernelILi5' build/var/interp_$tag.log | grep -o 'Used [0-9]* registers\|[0-9]* bytes stack' | tr '\n' ' ')"
done
