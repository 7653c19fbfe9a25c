for c in 0 1 2 3; do for rep in 1 2; do
BD_CARVEOUT=$c python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/v.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/v.json'));p=d['profile_ms_per_step'];print('carve=$c', d['value'],d['ms_per_step'],' '.join(f'{k}={v}' for k,v in p.items() if v))"
done; done
