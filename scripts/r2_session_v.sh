#!/bin/bash
# Round-2 session V: FFT transforms with per-P thread counts: uniform-scheme tests, C3 kernel times + launch list.
O=gpurun_out/r2v
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -rfE -p no:cacheprovider -x --timeout 600 -k "stencil or uniform or C3 or scaled or fuzz" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
BFMM_PROFILE=1 timeout 600 python scripts/one_config.py C3 > $O/C3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/c3_launches.csv python scripts/one_config.py C3 > $O/c3_ncu.log 2>&1
echo done
