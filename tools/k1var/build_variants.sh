# Build full libbitdelta_b200.so variants that differ only in the K1 compressor source / flags
# into /tmp/k1var/<name>/ (probe: tools/k1_probe.py <lib>...)
cd $GRAFT_REPO_ROOT
B=paper_2402_10193_b200/_build
NCCL=$(python -c "import paper_2402_10193_b200.build as b; print(b.NCCL)")
objs=$(ls $B/*.o | grep -v compress.cu.o)
mk() {  # name src flags
  mkdir -p /tmp/k1var/$1
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr $3 -Iinclude -Ipaper_2402_10193_b200/csrc -I$NCCL/include -c $2 -o /tmp/k1var/$1/compress.o
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /tmp/k1var/$1/libbitdelta_b200.so $objs /tmp/k1var/$1/compress.o -L$NCCL/lib -l:libnccl.so.2 -Xlinker=-rpath=$NCCL/lib
}
mk c8_4 paper_2402_10193_b200/csrc/compress.cu "-DBD_K1_VPT_BF16=8 -DBD_K1_VPT_F32=4"
mk c16_8 paper_2402_10193_b200/csrc/compress.cu "-DBD_K1_VPT_BF16=16 -DBD_K1_VPT_F32=8"
mk c4_2 paper_2402_10193_b200/csrc/compress.cu "-DBD_K1_VPT_BF16=4 -DBD_K1_VPT_F32=2"
mk c32_16 paper_2402_10193_b200/csrc/compress.cu "-DBD_K1_VPT_BF16=32 -DBD_K1_VPT_F32=16"
