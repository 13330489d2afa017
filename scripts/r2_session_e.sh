#!/bin/bash
# Round-2 GPU session E: tests (tile / pair / stencil2 / full C3), bench lines
# C5 (headline, + C2 secondary), C3, C4; launch lists; targeted ncu captures.
O=gpurun_out/r2e
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider --timeout 900 > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 python bench.py --config C3 --secondary none --no-cpu-baseline --steps 3 --warmup 3 > $O/bench_C3.json 2> $O/bench_C3.err
timeout 900 python bench.py --config C4 --secondary none --no-cpu-baseline --steps 5 --warmup 3 > $O/bench_C4.json 2> $O/bench_C4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C5.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --secondary none > $O/ncu_C5.log 2>&1
for k in m2l_i8p_kernel p2p_tile_kernel p2m_pair_kernel l2p_pair_kernel proj_gemm_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
      -o $O/c5_$k python scripts/one_config.py C5 > $O/ncu_c5_$k.log 2>&1
done
for k in stencil2_kernel fft_fwd_kernel fft_inv_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o $O/c3_$k python scripts/one_config.py C3 1 > $O/ncu_c3_$k.log 2>&1
done
for f in $O/*.ncu-rep; do python scripts/ncu_summary.py $f > ${f%.ncu-rep}_summary.txt 2>&1; done
echo done
