# TP loopback test, compressor bench lines + ncu of the compressor, default bench
timeout 900 python -m pytest tests/test_gpu_tp.py -q -x > gpurun_out/r02_tp.log 2>&1; tail -5 gpurun_out/r02_tp.log
timeout 300 python bench.py --workload compress_f32 --steps 20 --warmup 3 > gpurun_out/r02_compress_f32.json 2> gpurun_out/r02_compress_f32.err; tail -1 gpurun_out/r02_compress_f32.json; tail -3 gpurun_out/r02_compress_f32.err
timeout 300 python bench.py --workload compress_l70 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_compress_l70.json 2> gpurun_out/r02_compress_l70.err; tail -1 gpurun_out/r02_compress_l70.json; tail -3 gpurun_out/r02_compress_l70.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:compress_kernel -s 3 -c 2 -o gpurun_out/r02_compress_l70 python bench.py --workload compress_l70 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_compress.log 2>&1; tail -2 gpurun_out/ncu_compress.log
timeout 300 python bench.py --impl reference --workload compress_f32 --steps 1 --warmup 0 | tail -1
