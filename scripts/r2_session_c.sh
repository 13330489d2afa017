#!/bin/bash
# Round-2 GPU session C: the full-size C5 reference fixture (CPU, background,
# unmodified reference from baseline/_ref) while the GPU runs the tests, the
# bench lines of every config and the C5 ncu launch list.
O=gpurun_out/r2c
mkdir -p $O
{ nproc; free -g; lscpu | grep -i "model name\|socket\|core\|numa"; nvidia-smi; } > $O/host.txt 2>&1
AVAIL=$(free -g | awk 'NR==2{print $7}')
T=2; [ "$AVAIL" -gt 120 ] && T=4; [ "$AVAIL" -gt 160 ] && T=6
echo "fixture threads $T (avail $AVAIL GB)" >> $O/host.txt
(BOXFMM_THREADS=$T timeout ${FIX_LIMIT:-5400} nice -n 5 bash scripts/gen_full_fixtures.sh c5full > $O/c5full.log 2>&1; echo "rc=$?" >> $O/c5full.log) &
FIX=$!
( while kill -0 $FIX 2>/dev/null; do free -g | awk 'NR==2{print $3}' >> $O/mem_trace.txt; sleep 30; done ) &
timeout 2400 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider --timeout 900 > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err
for c in C2 C3 C4 C1; do
  timeout 900 python bench.py --config $c --secondary none --no-cpu-baseline --steps 5 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C5.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --secondary none > $O/ncu_C5.log 2>&1
wait $FIX
echo done
