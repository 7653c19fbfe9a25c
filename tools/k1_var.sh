# K1 variants: 16-byte loads per tensor per thread per block, rebuilt on the box
cd $GRAFT_REPO_ROOT
for v in "8 4" "16 8" "8 8" "4 4"; do
  set -- $v
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -DBD_K1_VPT_BF16=$1 -DBD_K1_VPT_F32=$2 -Iinclude -Ipaper_2402_10193_b200/csrc -c paper_2402_10193_b200/csrc/compress.cu -o paper_2402_10193_b200/_build/compress.cu.o
  touch paper_2402_10193_b200/_build/compress.cu.o
  python -c "from paper_2402_10193_b200 import build as b; b.build()" > /dev/null 2>&1
  for rep in 1 2; do for w in compress_l70 compress_f32; do
    timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('vpt=$1/$2', '$w', d['value'], d['ms_per_step'], d['parity_first_matrix_bits_exact'])"
  done; done
done
