#!/bin/bash
O=gpurun_out/r2i
mkdir -p $O
BFMM_PROFILE=1 timeout 300 python scripts/one_config.py C5 > $O/c5.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 1800 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider --timeout 900 > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
echo done
