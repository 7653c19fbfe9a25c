# glue latency-chain changes: parity, step time, attribution
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for sk in 0 0 24 1 2 4; do
BD_SKIP=$sk timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/v.json 2>gpurun_out/v.err
python -c "
import json;d=json.load(open('gpurun_out/v.json'));print('skip=$sk', d['value'], d['ms_per_step'])" 2>/dev/null || tail -2 gpurun_out/v.err
done
