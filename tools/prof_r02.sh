#!/bin/bash
# ncu evidence for round 2 (one GPU; never multi-rank). Reports -> gpurun_out/, summaries -> profiles/
W="--workload l7_layer --tenants 16 --batch 16 --ctx 8 --steps 2 --warmup 1 --no-cpu-baseline"
# full sections: K3 LUT + K2 of every projection group (bf16), and K2 int8 beside the LUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lut2_kernel|base_gemm_kernel" -s 16 -c 8 \
    -o gpurun_out/r02_lut_k2 python bench.py $W > gpurun_out/ncu_a.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"base_gemm_kernel|quant_pieces" -s 16 -c 8 \
    -o gpurun_out/r02_k2_int8 python bench.py $W --backbone int8 > gpurun_out/ncu_b.log 2>&1
# K1 compressor (configs[0] f32 4096^2 and the L70 matrix set) and K6 backward
timeout 600 ncu --set full --clock-control none -k regex:"compress_kernel" -s 3 -c 2 \
    -o gpurun_out/r02_k1 python bench.py --workload compress_f32 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_c.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"compress_kernel" -s 3 -c 1 \
    -o gpurun_out/r02_k1_l70 python bench.py --workload compress_l70 --layers 1 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_d.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"transpose_acc|dot_f64" -c 4 \
    -o gpurun_out/r02_k6 python -m pytest tests/test_gpu_backward.py -q -k "large and 11008" > gpurun_out/ncu_e.log 2>&1
# launch list of the default workload (serialised, cold): per-kernel device time and DRAM bytes
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -s 3000 -c 600 --csv --log-file gpurun_out/r02_launches_l7stack.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_f.log 2>&1
for r in r02_lut_k2 r02_k2_int8 r02_k1 r02_k1_l70 r02_k6; do
  [ -f gpurun_out/$r.ncu-rep ] && python tools/ncu_summary.py gpurun_out/$r.ncu-rep --stalls > gpurun_out/${r}_summary.txt 2>&1
done
python tools/launch_summary.py gpurun_out/r02_launches_l7stack.csv > gpurun_out/r02_launches_summary.txt 2>&1
ls -la gpurun_out/*.ncu-rep
