#!/bin/bash
# Quick loop: targeted tests, per-kernel times of full C5 / C3, ncu of the
# rewritten leaf-pair / tile kernels on C5/64.
O=gpurun_out/r2g
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider --timeout 600 \
  -k "pair or tile or stencil or grouped or full_configs or sharded or symmetric" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
BFMM_PROFILE=1 timeout 300 python scripts/one_config.py C5 > $O/c5.log 2>&1
BFMM_PROFILE=1 timeout 300 python scripts/one_config.py C3 > $O/c3.log 2>&1
BFMM_PROFILE=1 BFMM_STENCIL=2 timeout 300 python scripts/one_config.py C3 > $O/c3_s2.log 2>&1
for k in p2m_pair_kernel l2p_pair_kernel p2p_tile_kernel; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o $O/$k python scripts/one_config.py C5 2 > $O/ncu_$k.log 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:stencil -s 2 -c 1 \
      -o $O/stencil python scripts/one_config.py C3 1 > $O/ncu_stencil.log 2>&1
for f in $O/*.ncu-rep; do python scripts/ncu_summary.py $f > ${f%.ncu-rep}_summary.txt 2>&1; done
echo done
