#!/bin/bash
O=gpurun_out/r2k
mkdir -p $O
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 1800 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider --timeout 900 > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:m2l_i8p2 -s 3 -c 1 \
    -o $O/m2l_l8 python scripts/one_config.py C5 > $O/ncu_m2l.log 2>&1
python scripts/ncu_summary.py $O/m2l_l8.ncu-rep > $O/m2l_l8_summary.txt 2>&1
echo done
