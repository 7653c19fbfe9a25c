# ncu evidence for round 1 (one GPU; never multi-rank)
set -x
W="--workload l7_layer --tenants 16 --batch 16 --ctx 8 --steps 2 --warmup 1 --no-cpu-baseline"
# full sections for the LUT (K3) and the base GEMM (K2) of the gate/up group, and K23 (FP4 tensor-core) forced
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"lut_kernel|base_gemm_kernel" -s 10 -c 8 \
    -o gpurun_out/r01_lut_k2 python bench.py $W > gpurun_out/ncu_a.log 2>&1
BD_DELTA=mt4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:mt4_kernel -s 4 -c 4 \
    -o gpurun_out/r01_mt4 python bench.py $W > gpurun_out/ncu_b.log 2>&1
# launch list of the default workload (serialised, cold): per-kernel device time
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -s 3000 -c 600 --csv --log-file gpurun_out/r01_launches_l7stack.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_c.log 2>&1
ls -la gpurun_out/
