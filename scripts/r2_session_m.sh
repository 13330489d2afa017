#!/bin/bash
# Round-2 session M: full-size C5 ncu captures of the non-M2L kernels
# (leaf-pair P2M / L2P, tiled P2P, near-pair count).
O=gpurun_out/r2m
mkdir -p $O
for k in p2m_pair l2p_pair p2p_tile near_count gather_weights; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o $O/$k python scripts/one_config.py C5 > $O/ncu_$k.log 2>&1
done
for f in $O/*.ncu-rep; do python scripts/ncu_summary.py $f > ${f%.ncu-rep}_summary.txt 2>&1; done
echo done
