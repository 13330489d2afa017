#!/bin/bash
# Round-2 session R: stencil3 (both z parities per thread, skewed halo) -- bitwise test, uniform-scheme tests, C3 kernel times, ncu.
O=gpurun_out/r2r
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -rfE -p no:cacheprovider -x --timeout 600 -k "stencil or uniform or C3 or scaled" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for sv in 3 1; do
  BFMM_STENCIL=$sv BFMM_PROFILE=1 timeout 600 python scripts/one_config.py C3 > $O/C3_stencil$sv.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stencil3_kernel -s 4 -c 1 \
      -o $O/stencil3b python scripts/one_config.py C3 > $O/ncu3.log 2>&1
for f in $O/*.ncu-rep; do python scripts/ncu_summary.py $f > ${f%.ncu-rep}_summary.txt 2>&1; done
echo done
