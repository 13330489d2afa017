#!/bin/bash
# Round-2 session W (final evidence run; last output directory r2w6): evidence of the current tree -- bench C5 (headline, with C2 secondary and the
# reference cpu_baseline), bench C1..C4, the reference arm, the gpu suite, the C5 launch list.
O=gpurun_out/r2w6
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $O/smi.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err
for c in C4 C3 C2 C1; do
  timeout 900 python bench.py --config $c --secondary none --no-cpu-baseline --steps 5 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 1800 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider --timeout 900 > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
BFMM_PROFILE=1 timeout 300 python scripts/one_config.py C5 > $O/c5_kernels.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --secondary none --no-cpu-baseline > $O/ncu_bench.log 2>&1
echo done
