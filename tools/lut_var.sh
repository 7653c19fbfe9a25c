# LUT occupancy variants: rebuild lut.cu with -D overrides, relink, bench
cd $GRAFT_REPO_ROOT
for cfg in "512 96" "640 88" "768 72"; do
  set -- $cfg
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -Xptxas -v -DBD_LUT_THREADS=$1 -DBD_LUT_REGS=$2 -Iinclude -Ipaper_2402_10193_b200/csrc -c paper_2402_10193_b200/csrc/lut.cu -o paper_2402_10193_b200/_build/lut.cu.o 2>&1 | grep -i "error\|spill" | sort | uniq -c | head -3
  touch paper_2402_10193_b200/_build/lut.cu.o
  python -c "from paper_2402_10193_b200 import build as b; b.build()" > /dev/null 2>&1
  timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/v.json 2>gpurun_out/v.err
  python -c "
import json;d=json.load(open('gpurun_out/v.json'));print('lut $1 $2', d['value'], d['ms_per_step'])" 2>/dev/null || tail -2 gpurun_out/v.err
done
