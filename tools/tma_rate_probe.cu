// Microbenchmark: HBM streaming rate of a persistent TMA ring (no compute), per box shape,
// ring depth and CTAs per SM.  Box = [rows x 128 B] SW128 of a [R_total x 8192 B] u8 matrix.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include "../paper_2402_10193_b200/csrc/common.cuh"
using namespace bd;
namespace bd { void set_error(const std::string&) {} }

__global__ void stream(const __grid_constant__ CUtensorMap map, int box_rows, int stages, long long n_boxes_total,
                       int row_boxes, int col_boxes, int warp_issue, int n_prod) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + 4 * stages * box_rows * 128);
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { for (int s = 0; s < stages * n_prod; ++s) mbar_init(&full[s], 1); fence_mbar_init(); }
  __syncthreads();
  const int unit = blockIdx.x * n_prod + warp;
  const int n_units = gridDim.x * n_prod;
  long long b0 = n_boxes_total * unit / n_units, b1 = n_boxes_total * (unit + 1) / n_units;
  if (warp < n_prod) { full += warp * stages; smem += size_t(warp) * stages * box_rows * 128; }
  const uint32_t bytes = box_rows * 128;
  if (warp < n_prod) {
    long long i = 0;
    // prologue
    for (long long b = b0; b < b1 && i < stages; ++b, ++i) {
      int s = int(i);
      int r = int(b / col_boxes) % row_boxes, c = int(b % col_boxes);
      if (warp_issue) { mbar_arrive_expect_tx_w(&full[s], bytes); tma_load_2d_w(smem + s * bytes, &map, &full[s], c * 128, r * box_rows, policy_evict_first()); }
      else if (lane == 0) { mbar_arrive_expect_tx(&full[s], bytes); tma_load_2d_hint(smem + s * bytes, &map, &full[s], c * 128, r * box_rows, policy_evict_first()); }
      __syncwarp();
    }
    for (long long b = b0 + stages, j = 0; b < b1 + stages; ++b, ++j) {
      int s = int(j % stages); uint32_t ph = uint32_t((j / stages) & 1);
      mbar_wait(&full[s], ph);
      if (b < b1) {
        int r = int(b / col_boxes) % row_boxes, c = int(b % col_boxes);
        if (warp_issue) { mbar_arrive_expect_tx_w(&full[s], bytes); tma_load_2d_w(smem + s * bytes, &map, &full[s], c * 128, r * box_rows, policy_evict_first()); }
        else if (lane == 0) { mbar_arrive_expect_tx(&full[s], bytes); tma_load_2d_hint(smem + s * bytes, &map, &full[s], c * 128, r * box_rows, policy_evict_first()); }
        __syncwarp();
      }
    }
  }
}

int main() {
  const size_t cols = 8192, rows = 262144;  // 2 GiB
  uint8_t* buf; cudaMalloc(&buf, cols * rows); cudaMemset(buf, 1, cols * rows);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  PFN_cuTensorMapEncodeTiled_v12000 enc; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  for (int box_rows : {32, 64, 128}) for (int stages : {2, 4}) for (int n_prod : {1, 2, 4}) {
    int per_sm = 1, wi = 1;
    size_t smem = size_t(4 * stages) * box_rows * 128 + 1024 + 512;
    if (smem > 227 * 1024) continue;
    CUtensorMap m;
    cuuint64_t dims[2] = {cols, rows}, strides[1] = {cols};
    cuuint32_t box[2] = {128, cuuint32_t(box_rows)}, es[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    long long nb = (long long)(cols / 128) * (rows / box_rows);
    int grid = 148 * per_sm;
    stream<<<grid, 32 * n_prod, smem>>>(m, box_rows, stages, nb, int(rows / box_rows), int(cols / 128), wi, n_prod);
    cudaEventRecord(e0);
    stream<<<grid, 32 * n_prod, smem>>>(m, box_rows, stages, nb, int(rows / box_rows), int(cols / 128), wi, n_prod);
    cudaEventRecord(e1);
    cudaError_t e = cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("box %3d x 128B stages %2d producers %d: %7.1f GB/s  %s\n", box_rows, stages, n_prod,
           cols * rows / ms / 1e6, e ? cudaGetErrorString(e) : "");
  }
  return 0;
}
