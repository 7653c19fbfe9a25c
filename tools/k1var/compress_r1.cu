// K1 — delta compressor (replaces deltakit::compress_delta / compress_tensor,
// P:src/delta.cpp:16-34, and compress_stack, delta.cpp:57-70).
//
// The packed layout is a flat bit stream over the row-major elements, so the
// kernel is a pure streaming pass over n = rows*cols elements: 16-byte
// vectorised loads of base/fine, delta in f32 (exactly like sub(),
// P:src/matrix.cpp:72-77), sign bit = delta > 0 (NaN/0/-0 -> 0, no FTZ), bits
// assembled into little-endian 32-bit words with warp shuffles, and
// alpha = float(sum |double(delta)| / n). The alpha sum is a deterministic
// two-level fp64 reduction: fixed per-thread order, fixed block tree, and the
// last block of each job sums the block partials in index order.
//
// Algorithmic bytes per element: 2*s_in read + 1/8 written.
#include <cuda_bf16.h>

#include <algorithm>
#include <vector>

#include "common.cuh"

namespace bd {

namespace {

constexpr int kThreads = 256;
#ifndef BD_K1_VPT
#define BD_K1_VPT 4
#endif
constexpr int kVecPerThread = BD_K1_VPT;  // 16-byte loads per tensor per thread per chunk
constexpr int kMaxJobsPerLaunch = 192;

struct Job {
    const void* base;
    const void* fine;
    uint64_t n;          // elements
    uint8_t* bits;       // ceil(n/8) bytes
    float* alpha;
    uint64_t block0;     // first global block of this job
    uint64_t nblocks;
    double* partial;     // nblocks doubles
    unsigned int* counter;
};

struct JobTable {
    int n_jobs;
    Job jobs[kMaxJobsPerLaunch];
};

template <bool kBf16>
struct Elt;
template <>
struct Elt<false> {
    static constexpr int kPerVec = 4;
    __device__ static float load(const void* p, uint64_t i) {
        return static_cast<const float*>(p)[i];
    }
    __device__ static void load_vec(const void* p, uint64_t i, float (&v)[4]) {
        const float4 q = __ldcs(reinterpret_cast<const float4*>(static_cast<const float*>(p) + i));
        v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    }
};
template <>
struct Elt<true> {
    static constexpr int kPerVec = 8;
    __device__ static float load(const void* p, uint64_t i) {
        return bf16_to_f32(static_cast<const uint16_t*>(p)[i]);
    }
    __device__ static void load_vec(const void* p, uint64_t i, float (&v)[8]) {
        const uint4 q = __ldcs(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(p) + i));
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            v[2 * k] = __uint_as_float(w[k] << 16);
            v[2 * k + 1] = __uint_as_float(w[k] & 0xFFFF0000u);
        }
    }
};

// Writes byte-granular tail of a word (when the word straddles ceil(n/8)).
__device__ __forceinline__ void store_word(uint8_t* bits, uint64_t word_idx, uint32_t w,
                                           uint64_t nbytes, bool aligned) {
    const uint64_t b0 = word_idx * 4;
    if (aligned && b0 + 4 <= nbytes) {
        reinterpret_cast<uint32_t*>(bits)[word_idx] = w;
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (b0 + k < nbytes) bits[b0 + k] = static_cast<uint8_t>(w >> (8 * k));
    }
}

template <bool kBf16>
__global__ void __launch_bounds__(kThreads) compress_kernel(const __grid_constant__ JobTable tab) {
    using E = Elt<kBf16>;
    constexpr int P = E::kPerVec;              // elements per 16-byte vector
    constexpr int kChunk = kThreads * kVecPerThread * P;  // elements per block
    __shared__ double s_red[kThreads / 32];
    __shared__ bool s_last;

    // locate job (tables are small; linear scan is uniform across the block)
    int j = 0;
    while (j + 1 < tab.n_jobs && blockIdx.x >= tab.jobs[j + 1].block0) ++j;
    const Job& job = tab.jobs[j];
    const uint64_t blk = blockIdx.x - job.block0;
    const uint64_t n = job.n;
    const uint64_t nbytes = (n + 7) / 8;
    const bool bits_aligned = (reinterpret_cast<uintptr_t>(job.bits) & 3) == 0;
    const bool vec_ok = ((reinterpret_cast<uintptr_t>(job.fine) |
                          reinterpret_cast<uintptr_t>(job.base)) & 15) == 0;

    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double abs_sum = 0.0;

    // warp-span layout: each iteration a warp covers 32*P consecutive elements
    // (lane l holds elements l*P .. l*P+P-1 of the span).
#pragma unroll
    for (int it = 0; it < kVecPerThread; ++it) {
        const uint64_t span0 = blk * kChunk + (uint64_t(it) * (kThreads / 32) + warp) * 32 * P;
        const uint64_t e0 = span0 + lane * P;
        float f[P], b[P];
        if (vec_ok && e0 + P <= n) {
            E::load_vec(job.fine, e0, f);
            if (job.base) E::load_vec(job.base, e0, b);
        } else {
#pragma unroll
            for (int k = 0; k < P; ++k) {
                const bool in = e0 + k < n;
                f[k] = in ? E::load(job.fine, e0 + k) : 0.0f;
                b[k] = (in && job.base) ? E::load(job.base, e0 + k) : 0.0f;
            }
        }
        uint32_t mybits = 0;
#pragma unroll
        for (int k = 0; k < P; ++k) {
            const float d = job.base ? __fsub_rn(f[k], b[k]) : f[k];  // sub(), matrix.cpp:72-77
            mybits |= (d > 0.0f ? 1u : 0u) << k;                        // sign_of, delta.hpp:18
            abs_sum += fabs(static_cast<double>(d));
        }
        // assemble 32-element words: word w of the span = lanes w*(32/P) ...
        constexpr int kLanesPerWord = 32 / P;  // 8 (f32) or 4 (bf16)
        uint32_t w = mybits << (P * (lane % kLanesPerWord));
#pragma unroll
        for (int o = 1; o < kLanesPerWord; o <<= 1) w |= __shfl_xor_sync(0xffffffffu, w, o);
        if (lane % kLanesPerWord == 0) {
            const uint64_t word_idx = span0 / 32 + lane / kLanesPerWord;
            if (word_idx * 32 < n) store_word(job.bits, word_idx, w, nbytes, bits_aligned);
        }
    }

    // block reduction (fixed tree) -> partial[blk]
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) abs_sum += __shfl_xor_sync(0xffffffffu, abs_sum, o);
    if (lane == 0) s_red[warp] = abs_sum;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < kThreads / 32; ++i) s += s_red[i];
        job.partial[blk] = s;
        __threadfence();
        const unsigned int done = atomicAdd(job.counter, 1u);
        s_last = (done == job.nblocks - 1);
    }
    __syncthreads();
    if (!s_last) return;

    // last block: sum partials in index order (deterministic), write alpha
    __threadfence();
    double s = 0.0;
    const volatile double* part = job.partial;
    for (uint64_t i = threadIdx.x; i < job.nblocks; i += kThreads) s += part[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) s_red[warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double tot = 0.0;
        for (int i = 0; i < kThreads / 32; ++i) tot += s_red[i];
        *job.alpha = n == 0 ? 0.0f : static_cast<float>(tot / static_cast<double>(n));
        *job.counter = 0;  // re-arm
    }
}

// residual -= decompress(plane) (compress_stack, delta.cpp:63-66)
__global__ void residual_update_kernel(float* res, const uint8_t* bits, const float* alpha,
                                       uint64_t n) {
    const float a = *alpha;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const bool pos = (bits[i >> 3] >> (i & 7)) & 1u;
        res[i] = __fsub_rn(res[i], pos ? a : -a);
    }
}

__global__ void diff_kernel(float* res, const void* base, const void* fine, bool bf16,
                            uint64_t n) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const float f = bf16 ? Elt<true>::load(fine, i) : Elt<false>::load(fine, i);
        const float b = base ? (bf16 ? Elt<true>::load(base, i) : Elt<false>::load(base, i)) : 0.0f;
        res[i] = base ? __fsub_rn(f, b) : f;
    }
}

}  // namespace

void note_launch();

void compress_launch(const bd_compress_job* jobs, int n_jobs, bd_dtype dtype,
                     cudaStream_t stream) {
    require(dtype == BD_F32 || dtype == BD_BF16, BD_ERR_UNSUPPORTED_DTYPE,
            "compress: dtype must be BD_F32 or BD_BF16");
    const bool bf16 = dtype == BD_BF16;
    const uint64_t chunk = uint64_t(kThreads) * kVecPerThread * (bf16 ? 8 : 4);
    for (int first = 0; first < n_jobs; first += kMaxJobsPerLaunch) {
        const int cnt = std::min(kMaxJobsPerLaunch, n_jobs - first);
        JobTable tab{};
        tab.n_jobs = 0;
        uint64_t total_blocks = 0, total_partials = 0;
        for (int i = 0; i < cnt; ++i) {
            const bd_compress_job& in = jobs[first + i];
            require(in.fine != nullptr && in.bits != nullptr && in.alpha != nullptr,
                    BD_ERR_BAD_ARGUMENT, "compress: null fine/bits/alpha pointer");
            const uint64_t n = in.rows * in.cols;
            Job& j = tab.jobs[tab.n_jobs++];
            j.base = in.base;
            j.fine = in.fine;
            j.n = n;
            j.bits = in.bits;
            j.alpha = in.alpha;
            j.block0 = total_blocks;
            j.nblocks = std::max<uint64_t>(1, (n + chunk - 1) / chunk);
            total_blocks += j.nblocks;
            total_partials += j.nblocks;
        }
        // workspace: partial sums + one counter per job (stream-ordered)
        const size_t ws_bytes = total_partials * sizeof(double) + cnt * sizeof(unsigned int) + 16;
        char* ws = nullptr;
        BD_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ws), ws_bytes, stream));
        BD_CUDA(cudaMemsetAsync(ws + total_partials * sizeof(double), 0,
                                cnt * sizeof(unsigned int), stream));
        uint64_t off = 0;
        for (int i = 0; i < tab.n_jobs; ++i) {
            tab.jobs[i].partial = reinterpret_cast<double*>(ws) + off;
            off += tab.jobs[i].nblocks;
            tab.jobs[i].counter =
                reinterpret_cast<unsigned int*>(ws + total_partials * sizeof(double)) + i;
        }
        if (bf16)
            compress_kernel<true><<<static_cast<unsigned>(total_blocks), kThreads, 0, stream>>>(tab);
        else
            compress_kernel<false><<<static_cast<unsigned>(total_blocks), kThreads, 0, stream>>>(tab);
        note_launch();
        BD_CUDA(cudaGetLastError());
        BD_CUDA(cudaFreeAsync(ws, stream));
    }
}

void compress_stack_launch(const void* base, const void* fine, bd_dtype dtype, uint64_t rows,
                           uint64_t cols, uint64_t planes, uint8_t* bits, float* alphas,
                           cudaStream_t stream) {
    require(planes >= 1, BD_ERR_BAD_ARGUMENT, "compress_stack: plane count must be >= 1");
    const uint64_t n = rows * cols, nb = (n + 7) / 8;
    float* res = nullptr;
    BD_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&res), std::max<uint64_t>(n, 1) * 4, stream));
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256 + 1, 148 * 16));
    diff_kernel<<<grid, 256, 0, stream>>>(res, base, fine, dtype == BD_BF16, n);
    note_launch();
    for (uint64_t k = 0; k < planes; ++k) {
        bd_compress_job j{nullptr, res, rows, cols, bits + k * nb, alphas + k};
        compress_launch(&j, 1, BD_F32, stream);
        if (k + 1 < planes) {
            residual_update_kernel<<<grid, 256, 0, stream>>>(res, bits + k * nb, alphas + k, n);
            note_launch();
        }
    }
    BD_CUDA(cudaGetLastError());
    BD_CUDA(cudaFreeAsync(res, stream));
}

}  // namespace bd
