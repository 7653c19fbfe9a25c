# K2 variants: tests, per-kernel durations (ncu, serialised), step A/B (experiments only)
timeout 900 python -m pytest tests -m gpu -x -q -k "gemm or int8 or config or pool" 2>&1 | tail -3
for lib in prev base; do
  if [ $lib = base ]; then unset BD_LIB; else export BD_LIB=_ab/libbitdelta_$lib.so; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"base_gemm" --csv --log-file gpurun_out/k2_ncu_${lib}_m7.csv \
    python bench.py --workload m7_stack --tenants 1 --layers 1 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
unset BD_LIB
tools/ab.sh k2_ab_l7.txt 2 "--steps 20 --warmup 5" prev base
for T in 1 4 16; do tools/ab.sh k2_ab_m7_T$T.txt 1 "--workload m7_stack --tenants $T --steps 10 --warmup 3" prev base; done
