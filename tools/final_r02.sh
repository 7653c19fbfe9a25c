timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/gputest_r02c.log
python bench.py > gpurun_out/bench_r02c.json 2> gpurun_out/bench_r02c.err
for T in 1 2 4 8 16 32 64; do timeout 600 python bench.py --workload m7_stack --tenants $T --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/m7_sweep_r02c.jsonl; done
