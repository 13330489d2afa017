#!/bin/bash
# Round-2 GPU session B: C3 reference fixture (CPU, background, 12 threads);
# tests; bench lines C5 / C3 / C4 with the new kernels; digit-mode A/B on C5;
# ncu launch lists of one C5 and one C3 matvec.
O=gpurun_out/r2b
mkdir -p $O
(BOXFMM_THREADS=12 nice -n 5 bash scripts/gen_full_fixtures.sh c3full > $O/c3full.log 2>&1) &
FIX=$!
( while kill -0 $FIX 2>/dev/null; do free -g | awk 'NR==2{print $3}' >> $O/mem_trace.txt; sleep 30; done ) &
python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
python bench.py --no-cpu-baseline --steps 10 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err
python bench.py --config C3 --secondary none --no-cpu-baseline --no-e2e --steps 3 --warmup 2 > $O/bench_c3.json 2> $O/bench_c3.err
python bench.py --config C4 --secondary none --no-cpu-baseline --no-e2e --steps 5 --warmup 2 > $O/bench_c4.json 2> $O/bench_c4.err
BFMM_PROFILE=1 BFMM_I8_DIGITS=base128 python scripts/one_config.py C5 > $O/c5_base128.log 2>&1
BFMM_PROFILE=1 python scripts/one_config.py C5 > $O/c5_auto.log 2>&1
for c in C5 C3; do
  python scripts/one_config.py $c > $O/one_$c.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$c.csv \
      python scripts/one_config.py $c > $O/ncu_$c.log 2>&1
done
wait $FIX
cp tests/golden/c3_full.npz $O/ 2>/dev/null
echo done
