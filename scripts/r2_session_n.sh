#!/bin/bash
# Round-2 session N: split CTA-pair M2L (N = 64 for the a + 2k = 5 pairs) --
# correctness (i8 tests) and C5 per-kernel times against the unsplit variant.
O=gpurun_out/r2n
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_m2l_i8.py -q -rfE -p no:cacheprovider -x > $O/pytest_i8.log 2>&1; echo "rc=$?" >> $O/pytest_i8.log
BFMM_PROFILE=1 timeout 300 python scripts/one_config.py C5 > $O/c5_split.log 2>&1
BFMM_PROFILE=1 BFMM_I8P2_N128=1 timeout 300 python scripts/one_config.py C5 > $O/c5_n128.log 2>&1
BFMM_PROFILE=1 timeout 300 python scripts/one_config.py C5 > $O/c5_split2.log 2>&1
echo done
