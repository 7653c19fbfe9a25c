# LUT: alpha-late vs per-word alpha; down-projection row alignment (11008 = 1376-B rows vs 11264 = 1408-B rows)
cd $GRAFT_REPO_ROOT
run() {
  timeout 300 env "$@" python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/v.json 2>gpurun_out/v.err
  python -c "
import json;d=json.load(open('gpurun_out/v.json'));p=d.get('profile_ms_per_step',{});print('$*',d['value'],d['ms_per_step'],' '.join(f'{k}={v}' for k,v in p.items() if v))" 2>/dev/null || tail -3 gpurun_out/v.err
}
run ALPHA=late
run BD_BENCH_INTER=11264
run BD_BENCH_INTER=10240
run BD_BENCH_INTER=11008 BD_SERIAL=1
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -DBD_LUT_ALPHA_LATE=0 -Iinclude -Ipaper_2402_10193_b200/csrc -c paper_2402_10193_b200/csrc/lut.cu -o paper_2402_10193_b200/_build/lut.cu.o
touch paper_2402_10193_b200/_build/lut.cu.o
python -c "from paper_2402_10193_b200 import build as b; b.build()" > /dev/null 2>&1
run ALPHA=early
