#!/bin/bash
# Round profile capture (run under gpurun): plain bench, launch list of the
# bench command, and one ncu --set full capture of the two top kernels.
# Usage: bash scripts/profile_round.sh r01
set -u
R=${1:-r01}
OUT=gpurun_out/$R
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu.txt
python bench.py --steps 5 --warmup 3 > $OUT/bench.json 2> $OUT/bench.err
echo "bench rc=$?"
# launch list of a short run of the same command (cold-cache, serialised)
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $OUT/plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
    > $OUT/ncu_launches.log 2>&1
echo "launches rc=$?"
python scripts/quick_c2.py C2 > $OUT/plain_quick.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"p2p_kernel|m2l_ws" -s 6 -c 5 \
    -o $OUT/top python scripts/quick_c2.py C2 > $OUT/ncu_full.log 2>&1
echo "ncu full rc=$?"
