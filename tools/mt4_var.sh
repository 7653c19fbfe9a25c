for dbg in 0 1 2 3 4 8 15; do
BD_DELTA=mt4 BD_MT4_DEBUG=$dbg timeout 120 python bench.py --workload l7_layer --tenants 16 --batch 16 --ctx 8 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/v.json 2>gpurun_out/v.err
python -c "
import json;d=json.load(open('gpurun_out/v.json'));p=d['profile_ms_per_step'];print('dbg=$dbg', ' '.join(f'{k}={v}' for k,v in p.items() if v))" 2>/dev/null || tail -2 gpurun_out/v.err
done
