# launch list (serialised, cold) of our kernels over ~one decode step of the default stack workload
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"lut_kernel|base_gemm|resid_norm|attn128|silu4|mt4_kernel|xp_prep|embed|logits|combine" \
    -s 2700 -c 400 --csv --log-file gpurun_out/r01_launches_l7stack.csv \
    python bench.py --ctx 8 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_c.log 2>&1
tail -2 gpurun_out/ncu_c.log
