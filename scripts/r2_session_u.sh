#!/bin/bash
# Round-2 session U: ncu --set full of the dominant kernels with the current code (DRAM traffic for bench.py's roofline objects).
O=gpurun_out/r2u
mkdir -p $O
# C5: level-8 CTA-pair M2L = 4th m2l_i8p2 launch of an evaluate (levels 5..8); second evaluate -> skip 7
timeout 900 ncu --set full --clock-control none --import-source on -k regex:m2l_i8p2_kernel -s 7 -c 1 \
      -o $O/c5_m2l_l8 python scripts/one_config.py C5 > $O/ncu_c5_m2l.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:p2p_tile_kernel -s 1 -c 1 \
      -o $O/c5_p2p_tile python scripts/one_config.py C5 > $O/ncu_c5_tile.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_kernel -s 1 -c 1 \
      -o $O/c4_p2p python scripts/one_config.py C4 > $O/ncu_c4_p2p.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:p2p_kernel -s 1 -c 1 \
      -o $O/c2_p2p python scripts/one_config.py C2 > $O/ncu_c2_p2p.log 2>&1
for f in $O/*.ncu-rep; do python scripts/ncu_summary.py $f > ${f%.ncu-rep}_summary.txt 2>&1; done
echo done
