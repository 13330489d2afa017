#!/bin/bash
# Round-2 GPU session B: tests, bench lines (C5 headline with the reference
# CPU baseline, C3, C4), ncu launch lists of one C5 and one C3 matvec.
O=gpurun_out/r2b
mkdir -p $O
python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
python bench.py --steps 10 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err
python bench.py --config C3 --secondary none --no-cpu-baseline --no-e2e --steps 3 --warmup 2 > $O/bench_c3.json 2> $O/bench_c3.err
python bench.py --config C4 --secondary none --no-cpu-baseline --no-e2e --steps 5 --warmup 2 > $O/bench_c4.json 2> $O/bench_c4.err
for c in C5 C3; do
  python scripts/one_config.py $c > $O/one_$c.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$c.csv \
      python scripts/one_config.py $c > $O/ncu_$c.log 2>&1
done
echo done
