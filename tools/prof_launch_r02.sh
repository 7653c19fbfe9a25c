#!/bin/bash
# launch list (serialised, cold) of the decode kernels over ~one step of the default stack workload
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"lut2|base_gemm|resid_norm|attn128|silu|quant_pieces|mt4_kernel" -s 3200 -c 400 --csv \
    --log-file gpurun_out/r02_launches_l7stack.csv python bench.py --ctx 8 --steps 2 --warmup 1 --no-cpu-baseline \
    > gpurun_out/ncu_launch.log 2>&1
python tools/launch_summary.py gpurun_out/r02_launches_l7stack.csv > gpurun_out/r02_launches_summary.txt 2>&1
cat gpurun_out/r02_launches_summary.txt
