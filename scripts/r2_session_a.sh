#!/bin/bash
# Round-2 GPU session A: C5 reference fixture (CPU, background) + GPU tests,
# bench lines of C5 (headline), C3, C4, C1, P2P flop counts.
O=gpurun_out/r2a
mkdir -p $O
free -g > $O/free.txt
(BOXFMM_THREADS=2 nice -n 5 bash scripts/gen_full_fixtures.sh c5full > $O/c5full.log 2>&1; free -g >> $O/free.txt) &
FIX=$!
( while kill -0 $FIX 2>/dev/null; do free -g | awk 'NR==2{print $3}' >> $O/mem_trace.txt; sleep 20; done ) &
python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
python bench.py --no-cpu-baseline --steps 10 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err
python bench.py --config C3 --secondary none --no-cpu-baseline --no-e2e --steps 3 --warmup 2 > $O/bench_c3.json 2> $O/bench_c3.err
python bench.py --config C4 --secondary none --no-cpu-baseline --no-e2e --steps 5 --warmup 2 > $O/bench_c4.json 2> $O/bench_c4.err
python bench.py --config C1 --secondary none --no-cpu-baseline --steps 20 --warmup 5 > $O/bench_c1.json 2> $O/bench_c1.err
bash scripts/p2p_flops.sh $O/p2pflops
wait $FIX
echo done
