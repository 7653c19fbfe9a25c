# K3d variants: per-kernel durations (ncu, serialised), step A/B (experiments only)
for T in 1 4; do
for lib in base ww; do
  if [ $lib = base ]; then unset BD_LIB; else export BD_LIB=_ab/libbitdelta_$lib.so; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"mtd_kernel" --csv --log-file gpurun_out/k3d_ncu6_${lib}_T$T.csv \
    python bench.py --workload m7_stack --tenants $T --layers 1 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
done
unset BD_LIB
for T in 1 4; do tools/ab.sh k3d_ab6_T$T.txt 1 "--workload m7_stack --tenants $T --steps 10 --warmup 3" base ww; done
tools/ab.sh k3d_ab6_T8.txt 1 "--workload m7_stack --tenants 8 --steps 10 --warmup 3" base
BD_DELTA=mtd tools/ab.sh k3d_ab6_T8mtd.txt 1 "--workload m7_stack --tenants 8 --steps 10 --warmup 3" base ww
