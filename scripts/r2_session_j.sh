#!/bin/bash
# Bench lines of the secondary configs with the current kernels + the C5
# launch list (serialised, cold) for the kernel shares.
O=gpurun_out/r2j
mkdir -p $O
for c in C4 C3 C2 C1; do
  timeout 900 python bench.py --config $c --secondary none --no-cpu-baseline --steps 5 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C5.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --secondary none > $O/ncu_C5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:m2l_i8p -s 7 -c 1 \
    -o $O/m2l_l8 python scripts/one_config.py C5 > $O/ncu_m2l.log 2>&1
python scripts/ncu_summary.py $O/m2l_l8.ncu-rep > $O/m2l_l8_summary.txt 2>&1
echo done
