bash tools/k1var/build_variants.sh > /tmp/k1var_build.log 2>&1 || tail -5 /tmp/k1var_build.log
for rep in 1 2 3; do for v in c4_2 c8_4 c16_8 c32_16; do
  echo "== $v rep $rep"; timeout 300 python tools/k1_probe.py /tmp/k1var/$v/libbitdelta_b200.so 2>&1 | grep -v "^$" | sed -n '1p;3p;$p'
done; done
