#!/bin/bash
# FP64 thread instructions of the P2P kernel per pair, one config per kernel
# functor (freezes bench.py P2P_FLOPS_PER_PAIR; profiles/r02_p2p_flops.txt).
# Usage (GPU box): bash scripts/p2p_flops.sh OUTDIR
set -u
OUT=${1:-gpurun_out/p2pflops}
mkdir -p "$OUT"
M=smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum
for cs in "C5 2" "C4 2" "C3 2" "C2 1"; do
  set -- $cs
  tag="$1s$2"
  python scripts/one_config.py $1 $2 > "$OUT/$tag.plain.log" 2>&1 &&
  ncu --metrics $M --clock-control none -k regex:p2p_kernel -s 1 -c 1 --csv \
      --log-file "$OUT/$tag.csv" python scripts/one_config.py $1 $2 > "$OUT/$tag.ncu.log" 2>&1
done
