#!/bin/bash
# Focused ncu of the leaf-pair and tiled near-field kernels on C5/64.
O=gpurun_out/r2f
mkdir -p $O
python scripts/one_config.py C5 2 > $O/plain.log 2>&1
for k in p2m_pair_kernel l2p_pair_kernel p2p_tile_kernel; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o $O/$k python scripts/one_config.py C5 2 > $O/ncu_$k.log 2>&1
done
BFMM_TILE_MODE=0 timeout 300 ncu --set full --clock-control none --import-source on -k regex:p2p_tile -s 1 -c 1 \
      -o $O/p2p_tile_mode0 python scripts/one_config.py C5 2 > $O/ncu_tile0.log 2>&1
for f in $O/*.ncu-rep; do python scripts/ncu_summary.py $f > ${f%.ncu-rep}_summary.txt 2>&1; done
echo done
