# other BASELINE configs (the bench line is configs[2]); one JSON line each
timeout 300 python bench.py --workload l7_layer --steps 50 --warmup 5 > gpurun_out/cfg_l7_layer.json 2>gpurun_out/cfg_l7_layer.err
for T in 1 4 16 64; do
timeout 900 python bench.py --workload m7_stack --tenants $T --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_m7_T$T.json 2>gpurun_out/cfg_m7_T$T.err
done
for f in gpurun_out/cfg_*.json; do python -c "
import json,sys;d=json.load(open('$f'));print('$f', d['value'], d['ms_per_step'], d['config'].get('tenants'), d['roofline']['kernel'], d['roofline']['frac'], d['step_roofline']['frac_of_measured_hbm'])" 2>/dev/null || (echo "$f failed"; tail -2 ${f%.json}.err); done
