# A/B of the byte-LUT v1 vs v2 on the default workload + LUT parity tests
set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "multitenant" > gpurun_out/lut2_tests.log 2>&1; tail -3 gpurun_out/lut2_tests.log
timeout 600 python -m pytest tests/test_gpu_pool.py -q -x > gpurun_out/lut2_pool.log 2>&1; tail -3 gpurun_out/lut2_pool.log
for i in 1 2; do
  BD_LUT_V1=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('v1', d['value'], d['ms_per_step'], d['profile_ms_per_step'], d['clocks']['sm_mhz'])"
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('v2', d['value'], d['ms_per_step'], d['profile_ms_per_step'], d['clocks']['sm_mhz'])"
done
