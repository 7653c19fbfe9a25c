for rep in 1 2 3 4; do
python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/v.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/v.json'));print(d['value'],d['ms_per_step'],d['clocks'])"
done
ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:lut_kernel|base_gemm|attn_kernel|norm_kernel|resid_kernel|silu|embed_kernel|logits_kernel|combine" -c 600 --csv --log-file gpurun_out/launches2.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
