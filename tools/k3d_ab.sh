# K3d A/B against the HEAD build (experiments only)
timeout 600 python -m pytest tests -m gpu -x -q -k "k3d or config3 or mtd" 2>&1 | tail -3
for T in 1 4 16; do tools/ab.sh k3d_ab3_T$T.txt 2 "--workload m7_stack --tenants $T --steps 10 --warmup 3" head base; done
