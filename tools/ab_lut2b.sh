# LUT alone (BD_SKIP=16 drops K2; results wrong) and together, v1 vs v2; ncu of lut2 on one layer
for sk in 0 16; do for v in 1 0; do
  BD_SKIP=$sk BD_LUT_V1=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['profile_ms_per_step']; print('skip=$sk v1=$v', d['value'], d['ms_per_step'], {k:v for k,v in p.items() if v})"
done; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"lut2_kernel" -s 8 -c 4 \
    -o gpurun_out/r02_lut2 python bench.py --workload l7_layer --tenants 16 --batch 16 --ctx 8 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_lut2.log 2>&1
BD_SKIP=16 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"lut2_kernel" -s 8 -c 4 \
    -o gpurun_out/r02_lut2_alone python bench.py --workload l7_layer --tenants 16 --batch 16 --ctx 8 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_lut2b.log 2>&1
ls gpurun_out
