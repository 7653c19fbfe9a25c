// K3 (few requests per tenant) — byte-LUT signed accumulation on the CUDA cores.
//
// Replaces per request r of tenant t (P:src/serve.cpp:250-254):
//   apply_delta_correction -> packed_signed_accumulate (P:src/delta.cpp:80-103)
//   y_r[m] += alpha_t * sum_j s_t[m][j] x_r[j]
// reading every plane row with fully coalesced 128-byte warp loads straight from
// the reference layout (flat row-major bits, LSB first), no re-tiling.
//
// A CTA owns (job = one request and its tenant's planes, 1024-column slice,
// chunk of rows). It first builds, for the slice's x values, 128 byte-tables
// T[k][e][l] = sum_{i<8} (bit_i(e) ? +x : -x)[32 l + 8 k + i]   (128 KB smem)
// laid out so that lane l always reads bank l (conflict-free), then for every
// row each lane loads its 32-bit word of the row slice and adds 4 table
// entries. 32 rows are accumulated per warp and reduced with a transposing
// butterfly (31 shuffles per 32 rows). Cost per 8 bits: 2 ALU + 1 LDS + 1 FADD.
// Output: one f32 partial per (slice, request, row), already scaled by alpha;
// the consumer kernel sums slices in a fixed order (deterministic).
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace bd {

void note_launch();

namespace {

constexpr int kLutThreads = 512;
constexpr int kSliceCols = 1024;
constexpr size_t kTableBytes = 4 * 256 * 32 * sizeof(float);  // 128 KB

__global__ void __launch_bounds__(kLutThreads, 1)
    lut_kernel(const __grid_constant__ LutParams p, const uint16_t* __restrict__ X,
               float* __restrict__ out) {
    extern __shared__ float T[];  // [4][256][32]
    __shared__ float xs[kSliceCols];
    // locate (job, slice, chunk)
    const int per_job = p.slices * p.n_chunks;
    const int job_i = blockIdx.x / per_job;
    const int rem = blockIdx.x % per_job;
    const int slice = rem / p.n_chunks;
    const int chunk = rem % p.n_chunks;
    const LutJob& job = p.jobs[job_i];
    const int c0 = slice * kSliceCols;
    // x of this slice (bf16 -> f32), zero past cols
    const uint16_t* xr = X + static_cast<size_t>(job.req) * p.ldx;
    for (int i = threadIdx.x; i < kSliceCols; i += kLutThreads)
        xs[i] = (c0 + i < p.cols) ? bf16_to_f32(xr[c0 + i]) : 0.0f;
    __syncthreads();
    // build the 128 tables: thread t -> table (k, l) = t/4, quarter t%4 of its 256 entries
    {
        const int tb = threadIdx.x >> 2, quarter = threadIdx.x & 3;
        const int k = tb >> 5, l = tb & 31;
        const float* xv = xs + 32 * l + 8 * k;
        float lo[16], hi[4];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            float s = 0.0f;
#pragma unroll
            for (int i = 0; i < 4; ++i) s += (e >> i & 1) ? xv[i] : -xv[i];
            lo[e] = s;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int eh = quarter * 4 + e;
            float s = 0.0f;
#pragma unroll
            for (int i = 0; i < 4; ++i) s += (eh >> i & 1) ? xv[4 + i] : -xv[4 + i];
            hi[e] = s;
        }
        float* Tk = T + (k * 256) * 32 + l;
#pragma unroll
        for (int eh = 0; eh < 4; ++eh)
#pragma unroll
            for (int el = 0; el < 16; ++el) Tk[((quarter * 4 + eh) * 16 + el) * 32] = hi[eh] + lo[el];
    }
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int seg = p.chunk_seg[chunk];
    const int r_begin = p.chunk_begin[chunk], r_end = p.chunk_end[chunk];  // rows within seg
    const int n_planes = job.n_planes[seg];
    const bool lane_on = c0 + 32 * lane < p.cols;
    const size_t words_per_row = p.cols / 32;
    const float* T0 = T + lane;
    constexpr int R = 16;                       // rows per warp batch
    constexpr int kWarps = kLutThreads / 32;
    float* outp = out + (static_cast<size_t>(slice) * p.batch + job.req) * p.M + p.seg_row0[seg];
    for (int pl = 0; pl < n_planes; ++pl) {
        const uint32_t* bits = reinterpret_cast<const uint32_t*>(job.bits[seg][pl]) + slice * 32 + lane;
        const float a = job.alpha[seg][pl];
        auto load = [&](int rb, uint32_t (&w)[R]) {
#pragma unroll
            for (int j = 0; j < R; ++j) {
                const int r = rb + j;
                w[j] = (lane_on && r < r_end) ? __ldcs(bits + static_cast<size_t>(r) * words_per_row) : 0u;
            }
        };
        uint32_t wn[R];
        int rb = r_begin + warp * R;
        if (rb < r_end) load(rb, wn);
        for (; rb < r_end; rb += kWarps * R) {
            uint32_t w[R];
#pragma unroll
            for (int j = 0; j < R; ++j) w[j] = wn[j];
            if (rb + kWarps * R < r_end) load(rb + kWarps * R, wn);  // prefetch next batch
            float acc[R];
#pragma unroll
            for (int j = 0; j < R; ++j) {
                const uint32_t v = w[j];
                acc[j] = a * (T0[(v & 0xFF) * 32] + T0[(256 + ((v >> 8) & 0xFF)) * 32] +
                              T0[(512 + ((v >> 16) & 0xFF)) * 32] + T0[(768 + (v >> 24)) * 32]);
            }
            // transposing butterfly over lane bits 4..1, then pair-sum: lanes 2i, 2i+1 hold row i
#pragma unroll
            for (int o = 16, n = R / 2; o >= 2; o >>= 1, n >>= 1) {
                const bool upper = (lane & o) != 0;
#pragma unroll
                for (int j = 0; j < n; ++j) {
                    const float send = upper ? acc[j] : acc[j + n];
                    const float keep = upper ? acc[j + n] : acc[j];
                    acc[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                }
            }
            const float tot = acc[0] + __shfl_xor_sync(0xffffffffu, acc[0], 1);
            // row held by lane: bits 4..1 of the lane select 8,4,2,1
            const int row = rb + ((lane >> 1) & 15);
            if ((lane & 1) == 0 && row < r_end) {
                if (pl == 0) outp[row] = tot;
                else outp[row] += tot;
            }
        }
    }
}
}  // namespace

size_t lut_smem_bytes() { return kTableBytes; }

bool plan_lut(LutParams& p, const int* seg_rows, int n_segs, int cols, int ldx, int batch) {
    if (cols % 32 != 0 || n_segs < 1 || n_segs > kLutMaxSegs || p.n_jobs < 1 || p.n_jobs > kLutMaxJobs)
        return false;
    for (int j = 0; j < p.n_jobs; ++j)
        for (int s = 0; s < n_segs; ++s)
            for (int k = 0; k < p.jobs[j].n_planes[s]; ++k)
                if (reinterpret_cast<uintptr_t>(p.jobs[j].bits[s][k]) % 4) return false;
    p.cols = cols;
    p.ldx = ldx;
    p.batch = batch;
    p.slices = (cols + kSliceCols - 1) / kSliceCols;
    int total = 0;
    for (int s = 0; s < n_segs; ++s) {
        p.seg_row0[s] = total;
        total += seg_rows[s];
    }
    p.M = total;
    // enough CTAs for ~2 waves at 1 CTA/SM, chunks of >= 512 rows (table build amortised)
    const int units = p.n_jobs * p.slices;
    const int want = std::max(1, (2 * kNumSMs + units - 1) / units);
    int chunk = std::max(512, ((total + want - 1) / want + 31) / 32 * 32);
    for (;;) {
        int n = 0;
        for (int s = 0; s < n_segs; ++s) n += (seg_rows[s] + chunk - 1) / chunk;
        if (n <= kLutMaxChunks) break;
        chunk *= 2;
    }
    p.n_chunks = 0;
    for (int s = 0; s < n_segs; ++s)
        for (int r = 0; r < seg_rows[s]; r += chunk) {
            p.chunk_seg[p.n_chunks] = s;
            p.chunk_begin[p.n_chunks] = r;
            p.chunk_end[p.n_chunks] = std::min(seg_rows[s], r + chunk);
            ++p.n_chunks;
        }
    return true;
}

void lut_launch(const LutParams& p, const void* X, float* out, cudaStream_t stream) {
    static bool attr = false;
    if (!attr) {
        BD_CUDA(cudaFuncSetAttribute(lut_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(kTableBytes)));
        attr = true;
    }
    const int grid = p.n_jobs * p.slices * p.n_chunks;
    if (grid == 0) return;
    lut_kernel<<<grid, kLutThreads, kTableBytes, stream>>>(p, static_cast<const uint16_t*>(X), out);
    note_launch();
    BD_CUDA(cudaGetLastError());
}

}  // namespace bd
