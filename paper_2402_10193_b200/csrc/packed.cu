// K3 — packed sign-plane application.
//
// (1) packed_accumulate_kernel: the drop-in for deltakit::packed_signed_accumulate
//     (P:src/delta.cpp:80-103) and packed_matvec (delta.cpp:72-78). Any shape:
//     rows need not start on a byte (the layout is a flat bit stream), so bits
//     are read through a 32-bit window at an arbitrary bit offset. Signed sums
//     are accumulated in fp64 like the reference (which keeps 2*sum_set - total
//     in double) and rounded to f32 once per row.
// (2) delta_units_kernel: the per-projection multi-tenant delta of
//     ServingPool::decode_shared (apply_delta_correction, P:src/serve.cpp:19-36,
//     called per request at serve.cpp:250-254), segmented by tenant: a unit is
//     (tenant planes, output-row range, the tenant's requests), so one tenant's
//     bits are streamed once for all of its requests in the batch.
// (3) combine_kernel: Y = sum of split-K base partials + delta.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace bd {

void note_launch();

namespace {

// bits [pos, pos+32) of a flat LSB-first stream of nbytes bytes (zero past end)
__device__ __forceinline__ uint32_t bit_window(const uint8_t* __restrict__ bits, uint64_t nbytes,
                                               uint64_t pos) {
    const uint64_t b = pos >> 3;
    uint64_t v = 0;
#pragma unroll
    for (int i = 0; i < 5; ++i)
        if (b + i < nbytes) v |= static_cast<uint64_t>(__ldg(bits + b + i)) << (8 * i);
    return static_cast<uint32_t>(v >> (pos & 7));
}

constexpr int kPaThreads = 256;

template <bool kSmemX>
__global__ void __launch_bounds__(kPaThreads)
    packed_accumulate_kernel(const uint8_t* __restrict__ bits, uint64_t rows, uint64_t cols,
                             const float* __restrict__ x, float* __restrict__ out, float scale,
                             int overwrite, int aligned) {
    extern __shared__ float xs[];  // transposed: xs[k * nchunk + chunk] = x[32*chunk + k]
    const uint64_t v = blockIdx.y;
    const float* xv = x + v * cols;
    const uint64_t nchunk = (cols + 31) / 32;
    if (kSmemX) {
        for (uint64_t c = threadIdx.x; c < cols; c += blockDim.x)
            xs[(c & 31) * nchunk + (c >> 5)] = xv[c];
        for (uint64_t c = cols + threadIdx.x; c < nchunk * 32; c += blockDim.x)
            xs[(c & 31) * nchunk + (c >> 5)] = 0.0f;
        __syncthreads();
    }
    const uint64_t nbytes = (rows * cols + 7) / 8;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warps = uint64_t(gridDim.x) * (kPaThreads / 32);
    for (uint64_t r = uint64_t(blockIdx.x) * (kPaThreads / 32) + (threadIdx.x >> 5); r < rows;
         r += warps) {
        double acc = 0.0;
        for (uint64_t ch = lane; ch < nchunk; ch += 32) {
            const uint64_t c0 = ch * 32;
            const uint32_t w = aligned ? __ldg(reinterpret_cast<const uint32_t*>(bits) +
                                               ((r * cols + c0) >> 5))
                                       : bit_window(bits, nbytes, r * cols + c0);
            const int take = cols - c0 < 32 ? static_cast<int>(cols - c0) : 32;
#pragma unroll 8
            for (int k = 0; k < take; ++k) {
                const float xk = kSmemX ? xs[k * nchunk + ch] : __ldg(xv + c0 + k);
                acc += ((w >> k) & 1u) ? static_cast<double>(xk) : -static_cast<double>(xk);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) {
            float* o = out + v * rows + r;
            if (overwrite)
                *o = scale * static_cast<float>(acc);
            else
                *o = *o + scale * static_cast<float>(acc);  // scale == 1 for a7
        }
    }
}

// ---------------------------------------------------------------- units --
constexpr int kMaxUnitsPerLaunch = 160;
struct UnitTable {
    int n_units;
    int cols, ldx, batch, out_rows;
    int rows_per_block;
    int accumulate;                      // D += (units of a projection's planes 5, 6, ...)
    int block0[kMaxUnitsPerLaunch + 1];  // prefix of row-blocks per unit
    DeltaUnit u[kMaxUnitsPerLaunch];
};

constexpr int kDuThreads = 256;

__global__ void __launch_bounds__(kDuThreads)
    delta_units_kernel(const __grid_constant__ UnitTable tab, const uint16_t* __restrict__ X,
                       float* __restrict__ D) {
    extern __shared__ float xs[];  // [q][k][chunk]
    int ui = 0;
    while (ui + 1 < tab.n_units && int(blockIdx.x) >= tab.block0[ui + 1]) ++ui;
    const DeltaUnit& u = tab.u[ui];
    const int rb = blockIdx.x - tab.block0[ui];
    const int cols = tab.cols;
    const int nchunk = (cols + 31) / 32;
    const int nq = u.n_req;
    for (int q = 0; q < nq; ++q) {
        const uint16_t* xr = X + static_cast<size_t>(u.req[q]) * tab.ldx;
        for (int c = threadIdx.x; c < nchunk * 32; c += kDuThreads)
            xs[(q * 32 + (c & 31)) * nchunk + (c >> 5)] = c < cols ? bf16_to_f32(xr[c]) : 0.0f;
    }
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool aligned = (cols % 32) == 0;
    const uint64_t nbytes = (static_cast<uint64_t>(u.rows) * cols + 7) / 8;
    const int r_begin = rb * tab.rows_per_block;
    const int r_end = min(u.rows, r_begin + tab.rows_per_block);
    for (int r = r_begin + warp; r < r_end; r += kDuThreads / 32) {
        float tot[kMaxReqPerUnit];
#pragma unroll
        for (int q = 0; q < kMaxReqPerUnit; ++q) tot[q] = 0.0f;
        for (int p = 0; p < u.n_planes; ++p) {
            const uint8_t* bits = u.bits[p];
            const bool al = aligned && ((reinterpret_cast<uintptr_t>(bits) & 3) == 0);
            float acc[kMaxReqPerUnit];
#pragma unroll
            for (int q = 0; q < kMaxReqPerUnit; ++q) acc[q] = 0.0f;
            for (int ch = lane; ch < nchunk; ch += 32) {
                const uint64_t pos = static_cast<uint64_t>(r) * cols + ch * 32;
                const uint32_t w = al ? __ldg(reinterpret_cast<const uint32_t*>(bits) + (pos >> 5))
                                      : bit_window(bits, nbytes, pos);
                const int take = min(32, cols - ch * 32);
#pragma unroll
                for (int q = 0; q < kMaxReqPerUnit; ++q) {
                    if (q >= nq) break;
                    const float* xq = xs + q * 32 * nchunk + ch;
                    float a = 0.0f;
#pragma unroll 8
                    for (int k = 0; k < take; ++k) {
                        const float xk = xq[k * nchunk];
                        a += ((w >> k) & 1u) ? xk : -xk;
                    }
                    acc[q] += a;
                }
            }
#pragma unroll
            for (int q = 0; q < kMaxReqPerUnit; ++q) {
                float a = acc[q];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
                tot[q] += u.alpha[p] * a;
            }
        }
        if (lane == 0)
            for (int q = 0; q < nq; ++q)
                D[static_cast<size_t>(u.req[q]) * tab.out_rows + u.row0 + r] =
                    tab.accumulate ? D[static_cast<size_t>(u.req[q]) * tab.out_rows + u.row0 + r] + tot[q] : tot[q];
    }
}

__global__ void combine_kernel(const float* __restrict__ P, int splits, const float* __restrict__ D,
                               int dsplits, int batch, int M, float* __restrict__ Y) {
    const size_t n = static_cast<size_t>(batch) * M;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x) {
        float s = 0.0f;
        for (int k = 0; k < splits; ++k) s += P[k * n + i];
        if (D)
            for (int k = 0; k < dsplits; ++k) s += D[k * n + i];
        Y[i] = s;
    }
}

// ------------------------------------------------------------------ K5 --
// fp32 multi-tenant linear (BASELINE configs[0]: the reference's f32 path at 1e-5):
//   Y[b][r] = float(sum_j W[r][j] x_b[j]) + alpha_t(b) * float(sum_j s_t(b)[r][j] x_b[j])
// mirroring matmul_nt (P:src/matrix.cpp:26-41) then apply_delta_correction's
// y += alpha * packed_signed_accumulate (P:src/serve.cpp:19-36, delta.cpp:80-103), with
// fp64 accumulation of both sums (the reference rounds a sequential f32 / f64 sum).
// tcgen05 has no f32 kind, so this is a SIMT kernel; it is HBM-bound on W (4 B/weight,
// read once for up to kF32Req requests) plus each request's tenant plane.
// Warp per row, lane l covers columns [c0 + 4l, c0 + 4l + 4) of every 128-column step.
constexpr int kF32Threads = 256;
constexpr int kF32Req = 8;  // requests per pass over W
struct F32Linear {
    const float* W;
    const float* X;  // [batch][cols]
    float* Y;        // [batch][rows]
    uint64_t rows, cols;
    int batch;
    int n_req;  // requests in this pass
    int req[kF32Req];
    const uint8_t* bits[kF32Req];  // tenant plane of each request (null = base only)
    float alpha[kF32Req];
};

__global__ void __launch_bounds__(kF32Threads) f32_linear_kernel(const __grid_constant__ F32Linear a) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warps = uint64_t(gridDim.x) * (kF32Threads / 32);
    const bool vec = (a.cols % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.W) | reinterpret_cast<uintptr_t>(a.X)) % 16 == 0);
    for (uint64_t r = uint64_t(blockIdx.x) * (kF32Threads / 32) + (threadIdx.x >> 5); r < a.rows; r += warps) {
        double base[kF32Req], del[kF32Req];
#pragma unroll
        for (int q = 0; q < kF32Req; ++q) base[q] = del[q] = 0.0;
        const float* wr = a.W + r * a.cols;
        const uint64_t nbytes = (a.rows * a.cols + 7) / 8;
        for (uint64_t c = 4 * lane; c < a.cols; c += 128) {
            float w[4];
            const int take = a.cols - c < 4 ? int(a.cols - c) : 4;
            if (vec) {
                const float4 v = __ldcs(reinterpret_cast<const float4*>(wr + c));
                w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) w[k] = k < take ? wr[c + k] : 0.0f;
            }
#pragma unroll
            for (int q = 0; q < kF32Req; ++q) {
                if (q >= a.n_req) break;
                const float* xr = a.X + size_t(a.req[q]) * a.cols + c;
                float x[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) x[k] = k < take ? __ldg(xr + k) : 0.0f;
                uint32_t sb = 0;
                if (a.bits[q]) sb = bit_window(a.bits[q], nbytes, r * a.cols + c);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    base[q] = fma(double(w[k]), double(x[k]), base[q]);
                    if (k < take) del[q] += ((sb >> k) & 1u) ? double(x[k]) : -double(x[k]);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < kF32Req; ++q) {
            if (q >= a.n_req) break;
            double b = base[q], d = del[q];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                b += __shfl_xor_sync(0xffffffffu, b, o);
                d += __shfl_xor_sync(0xffffffffu, d, o);
            }
            if (lane == 0) {
                float y = float(b);
                if (a.bits[q]) y = y + a.alpha[q] * float(d);
                a.Y[size_t(a.req[q]) * a.rows + r] = y;
            }
        }
    }
}

}  // namespace

void f32_linear_launch(const float* W, uint64_t rows, uint64_t cols, const uint8_t* const* req_bits,
                       const float* req_alpha, int batch, const float* X, float* Y, cudaStream_t stream) {
    if (rows == 0 || batch == 0) return;
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((rows + 7) / 8, kNumSMs * 8));
    for (int first = 0; first < batch; first += kF32Req) {
        F32Linear a{};
        a.W = W;
        a.X = X;
        a.Y = Y;
        a.rows = rows;
        a.cols = cols;
        a.batch = batch;
        a.n_req = std::min(kF32Req, batch - first);
        for (int q = 0; q < a.n_req; ++q) {
            a.req[q] = first + q;
            a.bits[q] = req_bits[first + q];
            a.alpha[q] = req_alpha[first + q];
        }
        f32_linear_kernel<<<grid, kF32Threads, 0, stream>>>(a);
        note_launch();
        BD_CUDA(cudaGetLastError());
    }
}

void packed_accumulate_launch(const uint8_t* bits, uint64_t rows, uint64_t cols, const float* x,
                              uint64_t n_vec, float* out, float scale, bool overwrite,
                              cudaStream_t stream) {
    if (rows == 0 || n_vec == 0) return;
    require(cols == 0 || (bits && x && out), BD_ERR_BAD_ARGUMENT, "packed: null pointer");
    if (cols == 0) {  // empty rows: sum is 0
        if (overwrite) BD_CUDA(cudaMemsetAsync(out, 0, rows * n_vec * sizeof(float), stream));
        return;
    }
    require(n_vec <= 65535, BD_ERR_BAD_ARGUMENT, "packed: n_vec must be <= 65535");
    const uint64_t nchunk = (cols + 31) / 32;
    const size_t smem = nchunk * 32 * sizeof(float);
    const bool use_smem = smem <= 96 * 1024;
    const int aligned = ((cols % 32) == 0 && (reinterpret_cast<uintptr_t>(bits) & 3) == 0) ? 1 : 0;
    const uint64_t blocks_needed = (rows + (kPaThreads / 32) - 1) / (kPaThreads / 32);
    dim3 grid(static_cast<unsigned>(std::min<uint64_t>(blocks_needed, kNumSMs * 8)),
              static_cast<unsigned>(n_vec));
    if (use_smem) {
        static bool attr = false;
        if (!attr) {
            BD_CUDA(cudaFuncSetAttribute(packed_accumulate_kernel<true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
            attr = true;
        }
        packed_accumulate_kernel<true><<<grid, kPaThreads, smem, stream>>>(
            bits, rows, cols, x, out, scale, overwrite ? 1 : 0, aligned);
    } else {
        packed_accumulate_kernel<false><<<grid, kPaThreads, 0, stream>>>(
            bits, rows, cols, x, out, scale, overwrite ? 1 : 0, aligned);
    }
    note_launch();
    BD_CUDA(cudaGetLastError());
}

namespace {

// raw projection deltas: block = 8 rows of one job (warp = row), f32 weights, bf16
// activations, f32 sums (the reference sums in f32 too, serve.cpp:30-33), added to D
constexpr int kRawJobsPerLaunch = 32;
constexpr int kRawRowsPerBlock = 8;
struct RawTable {
    int n_jobs, cols, ldx, out_rows;
    int block0[kRawJobsPerLaunch + 1];
    RawJob j[kRawJobsPerLaunch];
};

__global__ void __launch_bounds__(32 * kRawRowsPerBlock)
    raw_delta_kernel(const __grid_constant__ RawTable t, const uint16_t* __restrict__ X, float* __restrict__ D) {
    int ji = 0;
    while (ji + 1 < t.n_jobs && int(blockIdx.x) >= t.block0[ji + 1]) ++ji;
    const RawJob& J = t.j[ji];
    const int r = (int(blockIdx.x) - t.block0[ji]) * kRawRowsPerBlock + int(threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (r >= J.rows) return;
    const float* w = J.W + static_cast<size_t>(r) * t.cols;
    for (int q0 = 0; q0 < J.n_req; q0 += 4) {
        float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        for (int c = lane; c < t.cols; c += 32) {
            const float wv = __ldg(w + c);
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (q0 + i < J.n_req) acc[i] += wv * bf16_to_f32(X[static_cast<size_t>(J.req[q0 + i]) * t.ldx + c]);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            float v = acc[i];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0 && q0 + i < J.n_req) D[static_cast<size_t>(J.req[q0 + i]) * t.out_rows + J.row0 + r] += v;
        }
    }
}

}  // namespace

void raw_delta_launch(const RawJob* jobs, int n_jobs, const void* X, int ldx, int cols, float* D, int out_rows,
                      cudaStream_t stream) {
    for (int first = 0; first < n_jobs; first += kRawJobsPerLaunch) {
        RawTable tab{};
        tab.n_jobs = std::min(kRawJobsPerLaunch, n_jobs - first);
        tab.cols = cols;
        tab.ldx = ldx;
        tab.out_rows = out_rows;
        int blocks = 0;
        for (int i = 0; i < tab.n_jobs; ++i) {
            tab.j[i] = jobs[first + i];
            require(tab.j[i].W && tab.j[i].n_req >= 1 && tab.j[i].n_req <= kRawMaxReq, BD_ERR_BAD_ARGUMENT,
                    "raw delta: bad job");
            tab.block0[i] = blocks;
            blocks += (tab.j[i].rows + kRawRowsPerBlock - 1) / kRawRowsPerBlock;
        }
        tab.block0[tab.n_jobs] = blocks;
        if (blocks == 0) continue;
        raw_delta_kernel<<<blocks, 32 * kRawRowsPerBlock, 0, stream>>>(tab, static_cast<const uint16_t*>(X), D);
        note_launch();
        BD_CUDA(cudaGetLastError());
    }
}

void delta_units_launch(const DeltaUnit* units, int n_units, const void* X, int ldx, int cols,
                        int batch, float* D, int out_rows, cudaStream_t stream, bool accumulate) {
    if (!accumulate) BD_CUDA(cudaMemsetAsync(D, 0, static_cast<size_t>(batch) * out_rows * sizeof(float), stream));
    if (n_units == 0) return;
    const int nchunk = (cols + 31) / 32;
    static bool attr = false;
    if (!attr) {
        BD_CUDA(cudaFuncSetAttribute(delta_units_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     200 * 1024));
        attr = true;
    }
    for (int first = 0; first < n_units; first += kMaxUnitsPerLaunch) {
        const int cnt = std::min(kMaxUnitsPerLaunch, n_units - first);
        UnitTable tab{};
        tab.n_units = cnt;
        tab.cols = cols;
        tab.ldx = ldx;
        tab.batch = batch;
        tab.out_rows = out_rows;
        tab.rows_per_block = 64;
        tab.accumulate = accumulate ? 1 : 0;
        int blocks = 0, max_q = 1;
        for (int i = 0; i < cnt; ++i) {
            tab.u[i] = units[first + i];
            require(tab.u[i].n_req >= 1 && tab.u[i].n_req <= kMaxReqPerUnit, BD_ERR_BAD_ARGUMENT,
                    "delta unit: bad request count");
            require(tab.u[i].n_planes >= 1 && tab.u[i].n_planes <= kMaxPlanesPerUnit,
                    BD_ERR_BAD_ARGUMENT, "delta unit: bad plane count");
            tab.block0[i] = blocks;
            blocks += (tab.u[i].rows + tab.rows_per_block - 1) / tab.rows_per_block;
            max_q = std::max(max_q, tab.u[i].n_req);
        }
        tab.block0[cnt] = blocks;
        const size_t smem = static_cast<size_t>(max_q) * 32 * nchunk * sizeof(float);
        require(smem <= 200 * 1024, BD_ERR_BAD_ARGUMENT, "delta unit: activations exceed smem");
        delta_units_kernel<<<blocks, kDuThreads, smem, stream>>>(
            tab, static_cast<const uint16_t*>(X), D);
        note_launch();
        BD_CUDA(cudaGetLastError());
    }
}

void combine_launch(const float* P, int splits, const float* D, int batch, int M, float* Y,
                    cudaStream_t stream, int dsplits) {
    const size_t n = static_cast<size_t>(batch) * M;
    const unsigned grid = static_cast<unsigned>(std::min<size_t>((n + 255) / 256, kNumSMs * 8));
    combine_kernel<<<grid, 256, 0, stream>>>(P, splits, D, dsplits, batch, M, Y);
    note_launch();
    BD_CUDA(cudaGetLastError());
}

}  // namespace bd
