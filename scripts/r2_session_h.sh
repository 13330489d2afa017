#!/bin/bash
O=gpurun_out/r2h
mkdir -p $O
BFMM_PROFILE=1 timeout 300 python scripts/one_config.py C5 > $O/c5.log 2>&1
BFMM_PROFILE=1 BFMM_TILE_MODE=0 timeout 300 python scripts/one_config.py C5 > $O/c5_tile0.log 2>&1
BFMM_PROFILE=1 timeout 300 python scripts/one_config.py C4 > $O/c4.log 2>&1
BFMM_PROFILE=1 timeout 300 python scripts/one_config.py C2 > $O/c2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:p2p_tile -s 1 -c 1 \
      -o $O/p2p_tile python scripts/one_config.py C5 2 > $O/ncu_tile.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:proj_i8 -s 4 -c 2 \
      -o $O/proj_i8 python scripts/one_config.py C5 2 > $O/ncu_proj.log 2>&1
for f in $O/*.ncu-rep; do python scripts/ncu_summary.py $f > ${f%.ncu-rep}_summary.txt 2>&1; done
timeout 1500 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider --timeout 600 -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
echo done
