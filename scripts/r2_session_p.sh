#!/bin/bash
# Round-2 session P: flag-free singular P2P bodies + 64-target wide units:
# near-field tests, then C4 / C1 / C5 / C2 kernel times.
O=gpurun_out/r2p
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -rfE -p no:cacheprovider -x --timeout 600 > $O/pytest_parity.log 2>&1; echo "rc=$?" >> $O/pytest_parity.log
for c in C4 C1 C5 C2; do
  BFMM_PROFILE=1 timeout 600 python scripts/one_config.py $c > $O/${c}_kernels.log 2>&1
done
timeout 900 python bench.py --config C4 --secondary none --no-cpu-baseline --steps 5 --warmup 3 > $O/bench_C4.json 2> $O/bench_C4.err
echo done
