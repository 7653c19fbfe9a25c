for sk in 29 31 27 30; do
BD_SKIP=$sk python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/v.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/v.json'));print('skip=$sk', d['value'],d['ms_per_step'])"
done
