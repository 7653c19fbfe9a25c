# timing attribution: BD_SKIP drops launches (results wrong) - 1 norm, 2 attn, 4 silu, 8 K3, 16 K2
for sk in 0 1 2 4 7 8 16 24 31; do
BD_SKIP=$sk timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/v.json 2>gpurun_out/v.err
python -c "
import json;d=json.load(open('gpurun_out/v.json'));print('skip=$sk', d['value'], d['ms_per_step'])" 2>/dev/null || tail -2 gpurun_out/v.err
done
