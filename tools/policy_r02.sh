for T in 8 16; do
  tools/ab.sh pol_T$T.txt 2 "--workload m7_stack --tenants $T --steps 10 --warmup 3" base
  BD_DELTA=mtd tools/ab.sh pol_T${T}_mtd.txt 2 "--workload m7_stack --tenants $T --steps 10 --warmup 3" base
done
