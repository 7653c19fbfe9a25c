#!/bin/bash
# Other BASELINE configs on one B200 (profiles/r02_bench_other_configs.jsonl)
out=gpurun_out/r02_configs.jsonl; : > $out
run() { timeout 900 python bench.py "$@" --no-cpu-baseline 2>>gpurun_out/configs_err.log | tail -1 >> $out; }
run --workload l7_layer --steps 50 --warmup 5
run --workload l7_stack --steps 20 --warmup 5 --backbone int8
for T in 1 4 16 64; do run --workload m7_stack --tenants $T --steps 10 --warmup 3; done
run --workload l70_stack --layers 8 --steps 10 --warmup 3
run --workload compress_f32 --steps 20 --warmup 3
run --workload compress_l70 --layers 2 --steps 5 --warmup 3
