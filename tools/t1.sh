python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for rep in 1 2; do
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/v.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/v.json'));p=d['profile_ms_per_step'];print(d['value'],d['ms_per_step'],' '.join(f'{k}={v}' for k,v in p.items() if v))"
done
