#!/bin/bash
# Round-2 closing evidence on one box: GPU suite, smoke, default bench (with the CPU baseline),
# launch list of one decode step, M7 sweep.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02g_gputest.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02g_smoke.log 2>&1
python bench.py > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err
for T in 1 2 4 8 16 32 64; do
  timeout 600 python bench.py --workload m7_stack --tenants $T --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/r02g_m7_sweep.jsonl
done
timeout 900 python bench.py --workload l70_stack --layers 8 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/r02g_other.jsonl
timeout 900 python bench.py --workload l7_layer --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/r02g_other.jsonl
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"lut2|base_gemm|resid_norm|attn128|silu|quant_pieces|mt4_kernel" -s 3200 -c 400 --csv \
    --log-file gpurun_out/r02g_launches_l7stack.csv python bench.py --ctx 8 --steps 2 --warmup 1 --no-cpu-baseline \
    > gpurun_out/r02g_ncu_launch.log 2>&1
python tools/launch_summary.py gpurun_out/r02g_launches_l7stack.csv > gpurun_out/r02g_launches_summary.txt 2>&1
