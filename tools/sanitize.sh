#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over a small cross-section of the GPU
# tests: K1 compress, K3 LUT + K2 linear, K6 backward, K2 int8, the device pool (toy
# reference tenants, CUDA graph + PDL; raw and >4-plane projections), K3d (L7 shapes, 2 layers; its inputs
# written by the glue kernels), grouped-query attention (4 query heads per KV head, two K/V chunks). Logs -> gpurun_out/sanitize_<tool>.log
mkdir -p gpurun_out
SEL="tests/test_gpu_kernels.py::test_compress_golden_f32 tests/test_gpu_kernels.py::test_multitenant_linear_each_delta_path tests/test_gpu_backward.py::test_transpose_accumulate_golden tests/test_gpu_backward.py::test_delta_linear_backward_vs_reference tests/test_gpu_int8.py::test_int8_matmul_nt_vs_reference tests/test_gpu_pool.py::test_shared_matches_reference_logits tests/test_gpu_pool.py::test_int8_backbone_toy_matches_port tests/test_gpu_pool.py::test_raw_projection_deltas_match_port tests/test_gpu_pool.py::test_more_than_four_planes_match_port tests/test_gpu_configs.py::test_k3d_many_requests_per_tenant[arch2-2-3-40] tests/test_gpu_pool.py::test_head_dim_128_long_context_matches_port[512-4-256]"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
      python -m pytest $SEL -q -x -p no:cacheprovider > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/sanitize_$tool.log | tail -4 >> gpurun_out/sanitize_summary.txt
done
