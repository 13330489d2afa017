#!/bin/bash
# Round-2 session X2: branch-free sqrt in the hot loop -- parity tests, C3 kernel times.
O=gpurun_out/r2x2
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_consumers.py -q -rfE -p no:cacheprovider -x --timeout 600 > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
BFMM_PROFILE=1 timeout 600 python scripts/one_config.py C3 > $O/C3.log 2>&1
BFMM_PROFILE=1 timeout 600 python scripts/one_config.py C2 > $O/C2.log 2>&1
echo done
