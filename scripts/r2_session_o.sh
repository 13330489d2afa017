#!/bin/bash
# Round-2 session O: HEAD (split CTA-pair M2L) on the B200: bench C5, gpu suite, launch list.
O=gpurun_out/r2o
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $O/smi.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 1800 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider --timeout 900 > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
BFMM_PROFILE=1 timeout 300 python scripts/one_config.py C5 > $O/c5_kernels.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --secondary none --no-cpu-baseline > $O/ncu_bench.log 2>&1
echo done
