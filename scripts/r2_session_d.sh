#!/bin/bash
# Round-2 GPU session D: tests, the C5 bench line, then (CPU, background) the
# full-size C3 reference fixture while the GPU runs the P2P flop counts, the
# C5 launch list, ncu --set full of the top C5 kernels and compute-sanitizer.
O=gpurun_out/r2d
mkdir -p $O
{ nproc; free -g; } > $O/host.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rfE -p no:cacheprovider --timeout 900 > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err
(BOXFMM_THREADS=${FIX_T:-14} timeout ${FIX_LIMIT:-2900} nice -n 5 bash scripts/gen_full_fixtures.sh c3full > $O/c3full.log 2>&1; echo "rc=$?" >> $O/c3full.log) &
FIX=$!
( while kill -0 $FIX 2>/dev/null; do free -g | awk 'NR==2{print $3}' >> $O/mem_trace.txt; sleep 30; done ) &
timeout 600 bash scripts/p2p_flops.sh $O/p2pflops
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C5.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --secondary none > $O/ncu_C5.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:"m2l_i8p_kernel|p2p_tile_kernel|p2m_cells_kernel|proj_gemm_kernel|l2p_cells_kernel|l2l_warp_kernel|z_slice" \
    -s 10 -c 9 -o $O/c5_top python scripts/one_config.py C5 > $O/ncu_full_c5.log 2>&1
python scripts/ncu_summary.py $O/c5_top.ncu-rep > $O/c5_top_summary.txt 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_case.py \
      > $O/sanitizer_$tool.txt 2>&1
  echo "rc=$?" >> $O/sanitizer_$tool.txt
done
wait $FIX
echo done
