# K3b binary tensor-core delta: parity, then occupancy variants vs the byte LUT in the full step
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for v in "lut" "b1"; do
  if [ $v = lut ]; then export BD_LUT_B1=0; else export BD_LUT_B1=1; fi
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/v.json 2>gpurun_out/v.err
  python -c "
import json;d=json.load(open('gpurun_out/v.json'));p=d.get('profile_ms_per_step',{});print('$v',d['value'],d['ms_per_step'],' '.join(f'{k}={v}' for k,v in p.items() if v))" 2>/dev/null || tail -3 gpurun_out/v.err
done
export BD_LUT_B1=1
for cfg in "512 112" "128 255"; do
  set -- $cfg
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -Xptxas -v -DBD_B1_THREADS=$1 -DBD_B1_REGS=$2 -Iinclude -Ipaper_2402_10193_b200/csrc -c paper_2402_10193_b200/csrc/bmma.cu -o paper_2402_10193_b200/_build/bmma.cu.o 2>&1 | grep -i "error\|spill" | sort | uniq -c | head -3
  touch paper_2402_10193_b200/_build/bmma.cu.o
  python -c "from paper_2402_10193_b200 import build as b; b.build()" > /dev/null 2>&1
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/v.json 2>gpurun_out/v.err
  python -c "
import json;d=json.load(open('gpurun_out/v.json'));p=d.get('profile_ms_per_step',{});print('b1 $1 $2',d['value'],d['ms_per_step'],' '.join(f'{k}={v}' for k,v in p.items() if v))" 2>/dev/null || tail -3 gpurun_out/v.err
done
