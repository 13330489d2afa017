python scripts/h2d_probe.py
for i in 1 2 3; do python bench.py --no-cpu-baseline --steps 5 > gpurun_out/b$i.log 2>&1; tail -1 gpurun_out/b$i.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['ms_per_step'])"; done
