#!/bin/bash
# Round-2 session W3: exp range flag on kd -- gpu suite, bench C5 (+C2 secondary), C2, C3.
O=gpurun_out/r2w3
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider --timeout 900 > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err
for c in C3 C2; do
  timeout 900 python bench.py --config $c --secondary none --no-cpu-baseline --steps 5 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
done
echo done
