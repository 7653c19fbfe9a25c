// Probe: where tcgen05.mma kind::mxf4.block32 reads B's ue8m0 scale factors in TMEM.
// A = +1 everywhere (scales 1.0); B row n = +1 only in K-block kb; B-scale region
// (4 columns x 128 lanes x 4 bytes) filled with 127 + code(lane, col, byte).
// D[m][n] = 32 * 2^code  ->  code of the byte used for (n, kb).
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2402_10193_b200/csrc/common.cuh"
using namespace bd;
namespace bd { void set_error(const std::string&) {} }

__device__ __forceinline__ void mma_mxf4_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc,
                                            uint32_t sfa, uint32_t sfb, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %6, 0;\n"
    "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%4], [%5], p;\n}\n"
    :: "r"(d), "r"(a), "l"(bdesc), "r"(idesc), "r"(sfa), "r"(sfb), "r"(acc) : "memory");
}

__global__ void probe(int N, int kb, int mode, int sfid, float* D) {
  __shared__ __align__(1024) uint8_t bs[128 * 128];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  int t = threadIdx.x, w = t >> 5, l = t & 31;
  for (int i = t; i < 128 * 128; i += 128) bs[i] = 0;
  __syncthreads();
  for (int i = t; i < N * 32; i += 128) {
    int r = i / 32, byte = i % 32, chunk = byte / 16;
    int phys = ((chunk ^ (r & 7)) * 16) + byte % 16;
    bs[r * 128 + phys] = (byte / 16 == kb) ? 0x22 : 0x00;  // block kb = bytes [16kb, 16kb+16)
  }
  if (w == 0) tmem_alloc<256>(&slot);
  if (t == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  uint32_t tb = slot, lane_base = (w * 32) << 16;
  uint32_t a[8], s[8], z[8];
  for (int j = 0; j < 8; ++j) { a[j] = 0x22222222u; s[j] = 0x7F7F7F7Fu; z[j] = 0; }
  tmem_st8(tb + lane_base + 0, a);
  tmem_st8(tb + lane_base + 64, s);   // A scales: cols 64..71 all 1.0
  uint32_t b[8];
  for (int c = 0; c < 8; ++c) {
    uint32_t v = 0;
    for (int by = 0; by < 4; ++by) {
      int code = mode == 0 ? (l) : (c * 4 + by);
      v |= uint32_t(127 - 40 + code) << (8 * by);
    }
    b[c] = v;
  }
  tmem_st8(tb + lane_base + 72, b);   // B scales: cols 72..79
  for (int c0 = 0; c0 < 128; c0 += 8) tmem_st8(tb + lane_base + 128 + c0, z);
  tmem_st_wait();
  fence_proxy_async();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (t == 0) {
    uint32_t idesc = (uint32_t(sfid) << 4) | (1u << 7) | (1u << 10) | ((uint32_t(N) >> 3) << 17) | (1u << 23) |
                     ((128u >> 4) << 24);
    mma_mxf4_ts(tb + 128, tb + 0, sdesc_k128(bs), idesc, tb + 64, tb + 72, 0);
    tc_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t v[16];
    tmem_ld16(tb + lane_base + 128 + c0, v);
    tmem_ld_wait();
    for (int n = 0; n < 16 && c0 + n < N; ++n) D[t * N + c0 + n] = __uint_as_float(v[n]);
  }
  tc_fence_before(); __syncthreads();
  if (w == 0) tmem_dealloc<256>(tb);
}

int main() {
  float* dD; cudaMalloc(&dD, 128 * 128 * 4);
  std::vector<float> D(128 * 128);
  for (int sfid : {0})
  for (int N : {64, 128}) for (int kb : {0}) {
    int codes[2][128];
    for (int mode : {0, 1}) {
      probe<<<1, 128>>>(N, kb, mode, sfid, dD);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("sfid=%d N=%d err %s\n", sfid, N, cudaGetErrorString(e)); return 1; }
      cudaMemcpy(D.data(), dD, 128 * N * 4, cudaMemcpyDeviceToHost);
      for (int n = 0; n < N; ++n) {
        double v = D[0 * N + n] / 32.0;
        codes[mode][n] = v > 0 ? int(std::lround(std::log2(v))) + 40 : -999;
        // consistency across rows m
        for (int m = 1; m < 128; ++m) if (D[m * N + n] != D[n]) { codes[mode][n] = -777; break; }
      }
    }
    printf("sfid=%d N=%2d kb=%d: ", sfid, N, kb);
    for (int n = 0; n < N; ++n) {
      int c1 = codes[1][n];
      if (n % 8 == 0 || n == 31 || n == 32 || n == 33) printf("n%d[l%d c%d b%d] ", n, codes[0][n], c1 / 4, c1 % 4);
    }
    printf("\n");
  }
  return 0;
}
