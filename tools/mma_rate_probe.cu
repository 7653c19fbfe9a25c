// Microbenchmark: issue rate and completion time of back-to-back tcgen05.mma from one thread.
#include <cstdio>
#include <cstdint>
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
__device__ __forceinline__ void mma_bf16_ss_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                            uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_mxf4_ts_elect(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc,
                                            uint32_t sfa, uint32_t sfb, uint32_t acc) {
  asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %6, 0;\n"
    "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%4], [%5], p;\n}\n"
    :: "r"(d), "r"(a), "l"(bdesc), "r"(idesc), "r"(sfa), "r"(sfb), "r"(acc) : "memory");
}
__device__ __forceinline__ long long clk() { long long t; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)); return t; }

// mode 0: bf16 SS N=n same D; 1: bf16 SS, 4 different D; 2: mxf4 TS N=8 same D
__global__ void k(int mode, int n_mma, int N, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar, bar2[8], bar3;
  __shared__ uint32_t slot;
  int t = threadIdx.x, w = t >> 5;
  for (int i = t; i < 64 * 1024; i += blockDim.x) sm[i] = 0;
  if (w == 0) tmem_alloc<512>(&slot);
  if (t == 0) { mbar_init(&bar, 1); for (int i = 0; i < 8; ++i) mbar_init(&bar2[i], 1 << 20); mbar_init(&bar3, 1); mbar_arrive(&bar3); fence_mbar_init(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  uint32_t tb = slot;
  if (w == 0 && mode >= 3) {
    const uint32_t idb = idesc_bf16_f32(128, N);
    const uint32_t idm = (1u << 7) | (1u << 10) | ((8u >> 3) << 17) | (1u << 23) | ((128u >> 4) << 24);
    uint8_t* a = sm; uint8_t* b = sm + 32768;
    const uint64_t da0 = sdesc_k128(a), db0 = sdesc_k128(b);
    __syncwarp();
    long long t0 = clk();
    if (mode == 7) {            // commit alone
      for (int i = 0; i < n_mma; ++i) tc_commit_w(&bar2[i & 7]);
    } else if (mode == 8) {     // try_wait (vote) on a completed barrier
      for (int i = 0; i < n_mma; ++i) mbar_wait_w(&bar3, 0);
    } else if (mode == 9) {     // 16 mxf4 MMAs + 1 commit per iteration
      for (int i = 0; i < n_mma; i += 16) {
#pragma unroll
        for (int j = 0; j < 16; ++j)
          mma_mxf4_ts_elect(tb, tb + 256 + 8 * j, db0 + 2 * (j & 3), idm | ((2u * (j & 1)) << 4), tb + 240, tb + 242 + 2 * (j >> 1), (i + j) > 0);
        tc_commit_w(&bar2[(i >> 4) & 7]);
      }
    } else if (mode == 11) {    // per-thread try_wait loop on a completed barrier
      for (int i = 0; i < n_mma; ++i) mbar_wait(&bar3, 0);
    } else if (mode == 12) {    // test_wait (non-blocking) per thread
      for (int i = 0; i < n_mma; ++i) {
        uint32_t ok;
        asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}" : "=r"(ok) : "r"(smem_u32(&bar3)), "r"(0) : "memory");
        if (!ok) break;
      }
    } else if (mode == 13) {    // 4 independent try_waits then use
      for (int i = 0; i < n_mma; i += 4) {
        bool a0 = mbar_try(&bar3, 0), a1 = mbar_try(&bar3, 0), a2 = mbar_try(&bar3, 0), a3 = mbar_try(&bar3, 0);
        if (!(a0 && a1 && a2 && a3)) break;
      }
    } else if (mode == 10) {    // fence::after_thread_sync alone
      for (int i = 0; i < n_mma; ++i) tc_fence_after();
    } else if (mode == 5) {
      for (int i = 0; i < n_mma; i += 16) {
#pragma unroll
        for (int j = 0; j < 16; ++j)
          mma_bf16_ss_elect(tb, da0 + 256 * (j & 7) + 2 * (j & 3), db0 + 2 * (j & 3), idb, (i + j) > 0);
      }
    } else if (mode == 6) {
      for (int i = 0; i < n_mma; i += 16) {
#pragma unroll
        for (int j = 0; j < 16; ++j)
          mma_mxf4_ts_elect(tb, tb + 256 + 8 * j, db0 + 2 * (j & 3), idm | ((2u * (j & 1)) << 4), tb + 240, tb + 242 + 2 * (j >> 1), (i + j) > 0);
      }
    } else if (mode == 3) {
      for (int i = 0; i < n_mma; ++i)
        mma_bf16_ss_elect(tb, da0 + 256 * (i & 7) + 2 * (i & 3), db0 + 2 * (i & 3), idb, i > 0);
    } else {
      for (int i = 0; i < n_mma; ++i)
        mma_mxf4_ts_elect(tb, tb + 256 + 8 * (i & 15), db0 + 2 * (i & 3), idm, tb + 240, tb + 242, i > 0);
    }
    __syncwarp();
    long long t1 = clk();
    if (t == 0) { tc_commit(&bar); }
    mbar_wait(&bar, 0);
    long long t2 = clk();
    if (t == 0) { out[blockIdx.x * 2] = t1 - t0; out[blockIdx.x * 2 + 1] = t2 - t0; }
  }
  if (t == 0 && mode < 3) {
    const uint32_t idb = idesc_bf16_f32(128, N);
    const uint32_t idm = (1u << 7) | (1u << 10) | ((8u >> 3) << 17) | (1u << 23) | ((128u >> 4) << 24);
    uint8_t* a = sm; uint8_t* b = sm + 32768;
    long long t0 = clk();
    for (int i = 0; i < n_mma; ++i) {
      if (mode == 0) mma_bf16_ss(tb, sdesc_k128(a + (i & 7) * 4096) + 2 * (i & 3), sdesc_k128(b) + 2 * (i & 3), idb, i > 0);
      else if (mode == 1) mma_bf16_ss(tb + 64 * (i & 3), sdesc_k128(a + (i & 7) * 4096) + 2 * (i & 3), sdesc_k128(b) + 2 * (i & 3), idb, i > 3);
      else mma_mxf4_ts(tb, tb + 256 + 8 * (i & 15), sdesc_k128(b) + 2 * (i & 3), idm, tb + 240, tb + 242, i > 0);
    }
    long long t1 = clk();
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clk();
    out[blockIdx.x * 2] = t1 - t0; out[blockIdx.x * 2 + 1] = t2 - t0;
  }
  tc_fence_before(); __syncthreads();
  if (w == 0) tmem_dealloc<512>(tb);
}

int main() {
  long long* d; cudaMalloc(&d, 148 * 16);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  long long h[2];
  for (int mode : {8, 11, 12, 13}) for (int N : {16}) for (int n : {16, 256}) {
    k<<<1, 128, 70000>>>(mode, n, N, d); // warm
    k<<<1, 128, 70000>>>(mode, n, N, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("mode %d N %3d n_mma %3d: issue %6lld cyc (%.1f/mma)  complete %6lld cyc (%.1f/mma)\n", mode, N, n, h[0], double(h[0]) / n, h[1], double(h[1]) / n);
  }
  return 0;
}
