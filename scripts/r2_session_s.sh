#!/bin/bash
# Round-2 session S: ncu --set full of the level-6 stencil launch of full C3, stencil3 vs stencil.
O=gpurun_out/r2s
mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil3_kernel -s 4 -c 1 \
      -o $O/stencil3 python scripts/one_config.py C3 > $O/ncu3.log 2>&1
BFMM_STENCIL=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil_kernel -s 4 -c 1 \
      -o $O/stencil1 python scripts/one_config.py C3 > $O/ncu1.log 2>&1
for f in $O/*.ncu-rep; do python scripts/ncu_summary.py $f > ${f%.ncu-rep}_summary.txt 2>&1; done
echo done
