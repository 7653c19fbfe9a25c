// The INT8 RTN backbone (P:src/int8.cpp, P:src/serve.cpp:99-108,120-125):
//
//  * rtn_quantize_kernel — rtn_quantize (int8.cpp:15-42), bit-exact: per row
//    s = amax / 127 (f32), q = clamp(nearbyint(double(w) / double(s)), -127, 127), a zero
//    row gets s = 0 and q = 0; non-finite entries are reported (errc::non_finite).
//  * quant_pieces_kernel — the activations for the kind::i8 base GEMM (gemm.cu, K2 with
//    kI8): per request row, x = sum_p 2^-(S + 7p) q_p with S chosen so max|x| * 2^S lies in
//    [32, 64): q_0 = rint(x 2^S), then each residual (|r| <= 1/2) times 2^7 is rounded to the
//    next piece, so |q_p| <= 64 and 4 pieces carry x to 2^-27 of the row maximum (exact for
//    the row's largest elements; f32 has 24 bits). The tensor cores accumulate
//    W_q . q_p exactly in s32 and the GEMM epilogue recombines in fp64, so the product
//    matches int8_matmul_nt's f32 sum (int8.cpp:67-81) to its own rounding level.
#include <cmath>

#include "common.cuh"
#include "kernels.h"

namespace bd {

void note_launch();

namespace {

constexpr int kQThreads = 256;

__device__ __forceinline__ float block_max(float v, float* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        float w = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) w = fmaxf(w, __shfl_xor_sync(0xffffffffu, w, o));
        if (threadIdx.x == 0) red[32] = w;
    }
    __syncthreads();
    return red[32];
}

__global__ void __launch_bounds__(kQThreads)
    rtn_quantize_kernel(const float* __restrict__ W, uint64_t cols, int8_t* __restrict__ q, uint64_t ldq,
                        float* __restrict__ scales, int* __restrict__ bad) {
    __shared__ float red[33];
    const float* row = W + blockIdx.x * cols;
    float amax = 0.0f;
    bool finite = true;
    for (uint64_t c = threadIdx.x; c < cols; c += kQThreads) {
        const float w = row[c];
        finite &= isfinite(w);
        amax = fmaxf(amax, fabsf(w));
    }
    if (!finite) atomicExch(bad, 1);
    amax = block_max(amax, red);
    const float s = amax / 127.0f;
    if (threadIdx.x == 0) scales[blockIdx.x] = s;
    int8_t* out = q + blockIdx.x * ldq;
    const double sd = static_cast<double>(s);
    for (uint64_t c = threadIdx.x; c < cols; c += kQThreads) {
        int8_t v = 0;
        if (s != 0.0f) {
            // double quotient + ties-to-even, like the reference
            const double r = fmin(fmax(nearbyint(static_cast<double>(row[c]) / sd), -127.0), 127.0);
            v = static_cast<int8_t>(r);
        }
        out[c] = v;
    }
}

// grid (batch, column chunks of 1024): every CTA takes the row maximum over the whole row
// (16-byte loads, served from L2 after the first CTA) and writes its chunk's pieces
constexpr int kQChunk = 1024;
__global__ void __launch_bounds__(kQThreads)
    quant_pieces_kernel(const void* __restrict__ X, int x_f32, int ldx, int K, int8_t* __restrict__ Xq, int ldq,
                        float* __restrict__ piece_scale) {
    __shared__ float red[33];
    const int b = blockIdx.x;
    auto load = [&](int k) -> float {
        if (k >= K) return 0.0f;
        return x_f32 ? static_cast<const float*>(X)[size_t(b) * ldx + k]
                     : bf16_to_f32(static_cast<const uint16_t*>(X)[size_t(b) * ldx + k]);
    };
    griddep_wait();  // PDL: X comes from the previous kernel
    float m = 0.0f;
    if (!x_f32 && ldx % 8 == 0) {
        const uint4* row = reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(X) + size_t(b) * ldx);
        for (int k8 = threadIdx.x; k8 * 8 < K; k8 += kQThreads) {
            const uint4 u = row[k8];
            const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int h = 0; h < 8; ++h) {
                const float v = __uint_as_float((h & 1 ? w[h >> 1] & 0xFFFF0000u : w[h >> 1] << 16));
                if (k8 * 8 + h < K) m = fmaxf(m, fabsf(v));
            }
        }
    } else {
        for (int k = threadIdx.x; k < K; k += kQThreads) m = fmaxf(m, fabsf(load(k)));
    }
    m = block_max(m, red);
    int S = 0;
    if (m > 0.0f) {
        int e;
        frexpf(m, &e);  // m = f 2^e, f in [0.5, 1)
        S = 6 - e;      // m 2^S in [32, 64)
    }
    if (blockIdx.y == 0 && threadIdx.x < kPieces)
        piece_scale[b * kPieces + threadIdx.x] = m > 0.0f ? ldexpf(1.0f, -(S + 7 * int(threadIdx.x))) : 0.0f;
    int8_t* q0 = Xq + size_t(b) * kPieces * ldq;
    const int k_end = min(ldq, int(blockIdx.y + 1) * kQChunk);
    for (int k = blockIdx.y * kQChunk + threadIdx.x; k < k_end; k += kQThreads) {
        float v = m > 0.0f ? ldexpf(load(k), S) : 0.0f;
#pragma unroll
        for (int p = 0; p < kPieces; ++p) {
            const float qp = rintf(v);
            q0[size_t(p) * ldq + k] = static_cast<int8_t>(qp);
            v = (v - qp) * 128.0f;  // exact: |v - qp| <= 1/2
        }
    }
}

}  // namespace

void rtn_quantize_launch(const float* W, uint64_t rows, uint64_t cols, int8_t* q, uint64_t ldq,
                         float* row_scales, cudaStream_t stream) {
    require(W && q && row_scales, BD_ERR_BAD_ARGUMENT, "rtn_quantize: null pointer");
    require(ldq >= cols, BD_ERR_BAD_ARGUMENT, "rtn_quantize: row stride < cols");
    if (rows == 0) return;
    require(rows <= 0x7fffffffull, BD_ERR_BAD_ARGUMENT, "rtn_quantize: too many rows");
    int* bad = nullptr;
    BD_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&bad), sizeof(int), stream));
    BD_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), stream));
    rtn_quantize_kernel<<<unsigned(rows), kQThreads, 0, stream>>>(W, cols, q, ldq, row_scales, bad);
    note_launch();
    BD_CUDA(cudaGetLastError());
    int h = 0;
    BD_CUDA(cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, stream));
    BD_CUDA(cudaFreeAsync(bad, stream));
    BD_CUDA(cudaStreamSynchronize(stream));
    require(h == 0, BD_ERR_NON_FINITE, "rtn_quantize: non-finite entries");
}

void quant_pieces_launch(const void* X, bool x_f32, int ldx, int K, int batch, int8_t* Xq, int ldq,
                         float* piece_scale, cudaStream_t stream) {
    require(ldq >= K && ldq % 16 == 0, BD_ERR_BAD_ARGUMENT, "int8 pieces: bad row stride");
    if (batch <= 0) return;
    BD_CUDA(launch_pdl(quant_pieces_kernel, dim3(batch, (ldq + kQChunk - 1) / kQChunk), dim3(kQThreads), 0, stream,
                       X, x_f32 ? 1 : 0, ldx, K, Xq, ldq, piece_scale));
    note_launch();
    BD_CUDA(cudaGetLastError());
}

}  // namespace bd
