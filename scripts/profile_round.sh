#!/bin/bash
# Round profile capture (run under gpurun): plain bench, launch list of the
# bench command, and one ncu --set full capture of the top kernels.
# Usage: bash scripts/profile_round.sh r01
set -u
R=${1:-r01}
OUT=gpurun_out/$R
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt
python bench.py > $OUT/bench.json 2> $OUT/bench.err
echo "bench rc=$?"
# launch list of a short run of the same command (cold-cache, serialised)
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
    > $OUT/ncu_launches.log 2>&1
echo "launches rc=$?"
python scripts/launches.py $OUT/launches.csv > $OUT/launch_shares.txt
# one full capture of the dominant kernels of a steady-state C2 step
python scripts/quick_c2.py C2 > $OUT/plain_quick.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"p2p_kernel|m2l_i8p_kernel|m2l_i8_kernel|l2p_warp|p2m_leaf" -s 14 -c 7 \
    -o $OUT/top python scripts/quick_c2.py C2 > $OUT/ncu_full.log 2>&1
echo "ncu full rc=$?"
python scripts/ncu_summary.py $OUT/top.ncu-rep > $OUT/top_summary.txt 2>&1
