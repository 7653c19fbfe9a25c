set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
for rep in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/v.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/v.json'));p=d.get('profile_ms_per_step',{});print(d['value'],d['ms_per_step'],' '.join(f'{k}={v}' for k,v in p.items() if v))"
done
