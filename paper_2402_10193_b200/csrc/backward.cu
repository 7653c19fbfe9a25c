// K6 — the BitDelta distillation backward on the GPU, the two
// packed-plane pieces of linear_backward's PackedDelta branch (P:src/model.cpp:87-107):
//
//  (1) packed_signed_accumulate_t (P:src/delta.cpp:105-131), the transpose product
//        out[v][j] (+)= scale * float( sum_i s_ij y_v[i] ),  s = +1 for bit 1, -1 for bit 0,
//      which linear_backward uses as dx[t] += alpha_pl * S_pl^T dy[t];
//  (2) the scale (alpha) gradient g_pl += sum_i double(dy_i) * u_pl_i (model.cpp:92-95),
//      u_pl = the forward's S_pl x (LinearTape::plane_u).
//
// (1) Each thread owns 32 consecutive columns (one 32-bit window of a row's bits, any
//     bit offset: rows need not start on a byte) and walks a chunk of rows (8 row words in
//     flight), adding +-y_i into 32 fp64 accumulators (the reference keeps its column sums
//     in double too); chunks are sized so the grid is ~4 CTAs per SM;
//     chunk partials [chunk][vec][col] are summed in chunk order by a second kernel and
//     rounded to f32 once (deterministic, no atomics). HBM: the plane is read once per
//     vector, rows * cols / 8 bytes.
// (2) fp64 products of f32 pairs are exact; per-block tree sums, then the block partials
//     in index order (deterministic).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace bd {

void note_launch();

namespace {

constexpr int kTtThreads = 128;     // 128 x 32 = 4096 columns per block
constexpr int kTtBlocks = 4 * kNumSMs;  // target grid: row chunks sized so the grid fills the GPU

__device__ __forceinline__ uint32_t window32(const uint8_t* __restrict__ bits, uint64_t nbytes,
                                             uint64_t pos, bool aligned) {
    if (aligned) return __ldg(reinterpret_cast<const uint32_t*>(bits) + (pos >> 5));
    const uint64_t b = pos >> 3;
    uint64_t v = 0;
#pragma unroll
    for (int i = 0; i < 5; ++i)
        if (b + i < nbytes) v |= static_cast<uint64_t>(__ldg(bits + b + i)) << (8 * i);
    return static_cast<uint32_t>(v >> (pos & 7));
}

// grid (column blocks, row chunks of chunk_rows, vectors); part[(chunk * n_vec + v) * cols + j]
__global__ void __launch_bounds__(kTtThreads)
    transpose_acc_kernel(const uint8_t* __restrict__ bits, uint64_t rows, uint64_t cols,
                         const float* __restrict__ y, uint64_t n_vec, uint64_t chunk_rows,
                         double* __restrict__ part) {
    const uint64_t v = blockIdx.z, chunk = blockIdx.y;
    const uint64_t r0 = chunk * chunk_rows, r1 = min(rows, r0 + chunk_rows);
    const float* yv = y + v * rows;
    const uint64_t c0 = (uint64_t(blockIdx.x) * kTtThreads + threadIdx.x) * 32;
    if (c0 >= cols) return;
    const int take = cols - c0 < 32 ? int(cols - c0) : 32;
    const uint64_t nbytes = (rows * cols + 7) / 8;
    const bool aligned = (cols % 32) == 0 && (reinterpret_cast<uintptr_t>(bits) & 3) == 0;
    double acc[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) acc[k] = 0.0;
    // 8 row words in flight per batch (the row loop is otherwise one dependent load per row)
    for (uint64_t rb = r0; rb < r1; rb += 8) {
        uint32_t w[8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
            w[i] = rb + i < r1 ? window32(bits, nbytes, (rb + i) * cols + c0, aligned) : 0u;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (rb + i >= r1) break;
            const double yr = __ldg(yv + rb + i);  // one address per warp: broadcast
#pragma unroll
            for (int k = 0; k < 32; ++k) acc[k] += ((w[i] >> k) & 1u) ? yr : -yr;
        }
    }
    double* out = part + (chunk * n_vec + v) * cols + c0;
#pragma unroll
    for (int k = 0; k < 32; ++k)
        if (k < take) out[k] = acc[k];
}

// out[v][j] = (overwrite ? 0 : out[v][j]) + scale * float(sum over chunks, in order)
__global__ void transpose_reduce_kernel(const double* __restrict__ part, uint64_t n_chunks,
                                        uint64_t n_vec, uint64_t cols, float* __restrict__ out,
                                        float scale, int overwrite) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n_vec * cols) return;
    double s = 0.0;
    const uint64_t stride = n_vec * cols;
    uint64_t c = 0;
    for (; c + 8 <= n_chunks; c += 8) {  // 8 loads in flight, added in chunk order
        double t[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) t[k] = part[(c + k) * stride + i];
#pragma unroll
        for (int k = 0; k < 8; ++k) s += t[k];
    }
    for (; c < n_chunks; ++c) s += part[c * stride + i];
    const float col = static_cast<float>(s);
    out[i] = overwrite ? scale * col : out[i] + scale * col;
}

constexpr int kDotThreads = 256;
constexpr int kDotBlocks = 296;  // 2 per SM

__global__ void __launch_bounds__(kDotThreads)
    dot_f64_kernel(const float* __restrict__ a, const float* __restrict__ b, uint64_t n,
                   double* __restrict__ part) {
    __shared__ double red[kDotThreads];
    double s = 0.0;
    for (uint64_t i = uint64_t(blockIdx.x) * kDotThreads + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * kDotThreads)
        s += static_cast<double>(a[i]) * static_cast<double>(b[i]);
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = kDotThreads / 2; o > 0; o >>= 1) {
        if (int(threadIdx.x) < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

// acc[0] += sum of the block partials in index order (one thread: 296 additions)
__global__ void dot_final_kernel(const double* __restrict__ part, int n, double* __restrict__ acc) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += part[i];
    acc[0] += s;
}

}  // namespace

void packed_transpose_launch(const uint8_t* bits, uint64_t rows, uint64_t cols, const float* y,
                             uint64_t n_vec, float* out, float scale, bool overwrite, cudaStream_t s) {
    require(bits && y && out, BD_ERR_BAD_ARGUMENT, "packed_signed_accumulate_t: null pointer");
    if (n_vec == 0 || cols == 0) return;
    if (rows == 0) {
        if (overwrite) BD_CUDA(cudaMemsetAsync(out, 0, n_vec * cols * sizeof(float), s));
        return;
    }
    require(n_vec <= 65535, BD_ERR_BAD_ARGUMENT, "packed_signed_accumulate_t: too many vectors");
    const uint64_t col_blocks = (cols + 32ull * kTtThreads - 1) / (32ull * kTtThreads);
    // enough row chunks to fill the GPU, and no more: the fp64 partials are chunks x vectors x cols
    const uint64_t want = std::max<uint64_t>(1, kTtBlocks / (col_blocks * n_vec));
    uint64_t chunk_rows = (rows + want - 1) / want;
    chunk_rows = std::max<uint64_t>(64, (chunk_rows + 7) / 8 * 8);  // >= 64: bounded partial sums
    const uint64_t n_chunks = (rows + chunk_rows - 1) / chunk_rows;
    require(n_chunks <= 65535 && col_blocks <= 0x7fffffffull, BD_ERR_BAD_ARGUMENT,
            "packed_signed_accumulate_t: shape too large");
    double* part = nullptr;
    BD_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&part), n_chunks * n_vec * cols * sizeof(double), s));
    const dim3 grid{unsigned(col_blocks), unsigned(n_chunks), unsigned(n_vec)};
    transpose_acc_kernel<<<grid, kTtThreads, 0, s>>>(bits, rows, cols, y, n_vec, chunk_rows, part);
    note_launch();
    BD_CUDA(cudaGetLastError());
    const uint64_t n = n_vec * cols;
    transpose_reduce_kernel<<<unsigned((n + 255) / 256), 256, 0, s>>>(part, n_chunks, n_vec, cols, out, scale,
                                                                       overwrite ? 1 : 0);
    note_launch();
    BD_CUDA(cudaGetLastError());
    BD_CUDA(cudaFreeAsync(part, s));
}

void dot_f64_launch(const float* a, const float* b, uint64_t n, double* acc, cudaStream_t s) {
    require(a && b && acc, BD_ERR_BAD_ARGUMENT, "scale gradient: null pointer");
    if (n == 0) return;
    const int blocks = int(std::min<uint64_t>(kDotBlocks, (n + kDotThreads - 1) / kDotThreads));
    double* part = nullptr;
    BD_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&part), blocks * sizeof(double), s));
    dot_f64_kernel<<<blocks, kDotThreads, 0, s>>>(a, b, n, part);
    note_launch();
    BD_CUDA(cudaGetLastError());
    dot_final_kernel<<<1, 1, 0, s>>>(part, blocks, acc);
    note_launch();
    BD_CUDA(cudaGetLastError());
    BD_CUDA(cudaFreeAsync(part, s));
}

}  // namespace bd
