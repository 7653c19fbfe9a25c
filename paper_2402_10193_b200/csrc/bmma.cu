// K3b — tenant deltas on the binary tensor-core path (mma.sync m16n8k256 .b1, AND + POPC).
//
// Replaces, per request r of tenant t (P:src/serve.cpp:250-254):
//   apply_delta_correction -> packed_signed_accumulate (P:src/delta.cpp:80-103)
//   y_r[m] += alpha_t * sum_j s_t[m][j] x_r[j],   s = 2 bit - 1
// with the same work decomposition and output as the byte-LUT (lut.cu): a
// persistent grid over the flattened (request x 1024-column slice, stacked row)
// space, one f32 partial per (slice, request, row) with alpha applied.
//
// The sign plane is the A operand AS STORED: the words of the reference layout
// (flat row-major, LSB first) are loaded with coalesced 16-byte loads straight
// into the A fragment registers — no expansion at all. The activations of a
// (request, slice) become 24 bit planes of a two's-complement fixed-point copy
//   q_j = round(x_j * 2^e),  |q_j| < 2^23,  e = 23 - ceil-exponent(max_j |x_j|)
// (exact for every bf16 x_j within 2^-16 of the slice max, else rounded at
// 2^-24 of the max), which form the B operand: MMA column n of plane group g is
// bit plane 8g + n. One MMA per (16 rows, 256 columns, 8 planes):
//   C[row][n] += popc(bits_row & plane_{8g+n})  (s32)
// and the row's signed sum is rebuilt exactly in integers:
//   sum_j bit_j q_j = sum_p w_p C_p   (w_p = 2^p, w_23 = -2^23)
//   sum_j s_j q_j   = 2 sum_j bit_j q_j - sum_j q_j
//   y = alpha * 2^-e * that                      (one rounding, in double)
// Per 16 rows x 1024 bits a warp issues 4 LDG.128 + 12 MMA + ~40 integer ops
// (the LUT: 64 LDS + 16 SHFL + ~200 ALU).
//
// MEASURED on B200 (tools/b1_var.sh, L7 stack T=16 B=16): correct (all delta-only
// parity cases <= 1e-5, exact integer reconstruction), but the legacy .b1 mma.sync
// runs at ~75 SM cycles per m16n8k256 (not at tensor-core rate on sm_100a):
// 22.7 ms/step vs 6.39 with the byte LUT (512x112 and 128x255 occupancy variants
// no better). Kept opt-in (BD_LUT_B1=1) as the record of that measurement.
// The K order inside an MMA is free (A and B are permuted alike): thread
// (gid, tig) feeds row gid words [4 tig, +4) and [16 + 4 tig, +4) of the slice,
// and the B fragments are built with the same permutation.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace bd {

void note_launch();

namespace {

#ifndef BD_B1_THREADS
#define BD_B1_THREADS 256
#endif
#ifndef BD_B1_REGS
#define BD_B1_REGS 168  // 256 x 168 + the K2 CTA beside it (128 threads x 32) fit the 64K register file
#endif
constexpr int kB1Threads = BD_B1_THREADS;
constexpr int kB1Warps = kB1Threads / 32;
constexpr int kSlice = 1024;   // columns per unit (= 32 words of a plane row)
constexpr int kQBits = 24;     // fixed-point bits of the activations (3 MMA column groups of 8)

__device__ __forceinline__ void mma_b1(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                       uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc "
        "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint4 ld_stream4(const uint32_t* p) {
    uint4 v;
    asm volatile("ld.global.cs.v4.u32 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ uint32_t u4(const uint4& v, int j) {
    return j == 0 ? v.x : (j == 1 ? v.y : (j == 2 ? v.z : v.w));
}

template <int kWPR>  // words per plane row (cols / 32); 0 = runtime value
__global__ void __maxnreg__(BD_B1_REGS)
    b1_kernel(const __grid_constant__ LutParams p, const uint16_t* __restrict__ X, float* __restrict__ out) {
    __shared__ uint2 frag[3][4][32];  // B fragments [group][k-block j][lane]
    __shared__ float cw_max[32];      // per column-word max |x|
    __shared__ int cw_sum[32];        // per column-word sum of q
    griddep_wait();                   // PDL: X comes from the previous kernel; D is still read by it
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gid = lane >> 2, tig = lane & 3;
    const int wpr = kWPR ? kWPR : p.cols / 32;
    // integer column weights of this thread's two MMA columns (2 tig, 2 tig + 1) per group;
    // plane 23 (group 2, column 7) is the two's-complement sign plane
    const int w_lo = 1 << (2 * tig), w_hi_std = 1 << (2 * tig + 1);
    const int w_hi_top = tig == 3 ? -(1 << 7) : w_hi_std;
    const long long total = static_cast<long long>(p.n_jobs) * p.slices * p.M;
    const long long g0 = total * blockIdx.x / gridDim.x;
    const long long g1 = total * (blockIdx.x + 1) / gridDim.x;
    int cur = -1;
    uint2 bf[3][4];
    long long qsum = 0;
    int e = 0;
    for (long long g = g0; g < g1;) {
        const int u = static_cast<int>(g / p.M);
        const int ra = static_cast<int>(g % p.M);
        const int rb = static_cast<int>(std::min<long long>(p.M, ra + (g1 - g)));
        const int job_i = u / p.slices, slice = u % p.slices;
        const LutJob& job = p.jobs[job_i];
        const int c0 = slice * kSlice;
        const int nw = min(32, wpr - slice * 32);  // words of this slice (multiple of 4)
        if (u != cur) {
            // ---- activations of (request, slice) -> 24 bit-plane B fragments ----
            __syncthreads();  // every warp holds its copy of the previous fragments
            const uint16_t* xr = X + static_cast<size_t>(job.req) * p.ldx + c0;
            // warp w owns column-words w and w + 16 (lane = column inside the word)
            float xv[32 / kB1Warps];
#pragma unroll
            for (int k = 0; k < 32 / kB1Warps; ++k) {
                const int cw = warp + k * kB1Warps;
                xv[k] = cw < nw ? bf16_to_f32(xr[32 * cw + lane]) : 0.0f;
                float m = fabsf(xv[k]);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
                if (lane == 0) cw_max[cw] = m;
            }
            __syncthreads();
            float m = cw_max[lane];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            int ex = 0;
            if (m > 0.0f) frexpf(m, &ex);  // m < 2^ex
            e = m > 0.0f ? (kQBits - 1) - ex : 0;
#pragma unroll
            for (int k = 0; k < 32 / kB1Warps; ++k) {
                const int cw = warp + k * kB1Warps;
                const int q = __float2int_rn(ldexpf(xv[k], e));
                int s = q;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                if (lane == 0) cw_sum[cw] = s;
                // column-word cw feeds k-block j = cw & 3 of thread tig = (cw & 15) >> 2, half cw >> 4
                const int j = cw & 3, ftig = (cw & 15) >> 2, half = cw >> 4;
                uint32_t mine = 0;
#pragma unroll
                for (int pl = 0; pl < kQBits; ++pl) {
                    const uint32_t b = __ballot_sync(0xffffffffu, (q >> pl) & 1);
                    mine = lane == pl ? b : mine;
                }
                if (lane < kQBits) {
                    const int fg = lane >> 3, fgid = lane & 7;
                    reinterpret_cast<uint32_t*>(&frag[fg][j][fgid * 4 + ftig])[half] = mine;
                }
            }
            __syncthreads();
#pragma unroll
            for (int fg = 0; fg < 3; ++fg)
#pragma unroll
                for (int j = 0; j < 4; ++j) bf[fg][j] = frag[fg][j][lane];
            long long s = cw_sum[lane];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            qsum = s;
            cur = u;
        }
        float* out_u = out + (static_cast<size_t>(slice) * p.batch + job.req) * p.M;
        const bool lo_on = 4 * tig < nw, hi_on = 16 + 4 * tig < nw;
        for (int sg = 0; sg < p.n_segs; ++sg) {
            const int s0 = p.seg_row0[sg], s1 = p.seg_row0[sg + 1];
            const int la = std::max(ra, s0) - s0, lb = std::min(rb, s1) - s0;
            if (la >= lb) continue;
            const int n_planes = job.n_planes[sg];
            for (int pl = 0; pl < n_planes; ++pl) {
                const uint32_t* plane = reinterpret_cast<const uint32_t*>(job.bits[sg][pl]) + slice * 32 + 4 * tig;
                const double scale = ldexp(static_cast<double>(job.alpha[sg][pl]), -e);
                auto load = [&](int r0, uint4 (&w)[4]) {
                    const int rA = r0 + gid, rB = r0 + gid + 8;
                    const uint4 z = make_uint4(0u, 0u, 0u, 0u);
                    w[0] = (lo_on && rA < lb) ? ld_stream4(plane + static_cast<size_t>(rA) * wpr) : z;
                    w[1] = (hi_on && rA < lb) ? ld_stream4(plane + static_cast<size_t>(rA) * wpr + 16) : z;
                    w[2] = (lo_on && rB < lb) ? ld_stream4(plane + static_cast<size_t>(rB) * wpr) : z;
                    w[3] = (hi_on && rB < lb) ? ld_stream4(plane + static_cast<size_t>(rB) * wpr + 16) : z;
                };
                uint4 wn[4];
                int r0 = la + warp * 16;
                if (r0 < lb) load(r0, wn);
                for (; r0 < lb; r0 += kB1Warps * 16) {
                    uint4 w[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) w[k] = wn[k];
                    if (r0 + kB1Warps * 16 < lb) load(r0 + kB1Warps * 16, wn);
                    int acc[3][4];
#pragma unroll
                    for (int fg = 0; fg < 3; ++fg)
#pragma unroll
                        for (int k = 0; k < 4; ++k) acc[fg][k] = 0;
#pragma unroll
                    for (int j = 0; j < 4; ++j)
#pragma unroll
                        for (int fg = 0; fg < 3; ++fg)
                            mma_b1(acc[fg], u4(w[0], j), u4(w[2], j), u4(w[1], j), u4(w[3], j), bf[fg][j].x,
                                   bf[fg][j].y);
                    // C layout: c0,c1 = (row gid, cols 2tig, 2tig+1); c2,c3 = (row gid+8, same cols)
                    int G[3][2];
#pragma unroll
                    for (int fg = 0; fg < 3; ++fg) {
                        const int wh = fg == 2 ? w_hi_top : w_hi_std;
                        G[fg][0] = acc[fg][0] * w_lo + acc[fg][1] * wh;
                        G[fg][1] = acc[fg][2] * w_lo + acc[fg][3] * wh;
#pragma unroll
                        for (int o = 1; o <= 2; o <<= 1) {
                            G[fg][0] += __shfl_xor_sync(0xffffffffu, G[fg][0], o);
                            G[fg][1] += __shfl_xor_sync(0xffffffffu, G[fg][1], o);
                        }
                    }
                    // lane tig 0 stores row gid, lane tig 1 row gid + 8
                    const int h = tig & 1;
                    const long long S = (static_cast<long long>(G[2][h]) << 16) +
                                        (static_cast<long long>(G[1][h]) << 8) + G[0][h];
                    const float y = static_cast<float>(static_cast<double>(2 * S - qsum) * scale);
                    const int r = r0 + gid + 8 * h;
                    if (tig < 2 && r < lb) {
                        if (pl == 0) out_u[s0 + r] = y;
                        else out_u[s0 + r] += y;  // same thread wrote it for plane 0
                    }
                }
            }
        }
        g += rb - ra;
    }
}

}  // namespace

bool b1_supported(const LutParams& p) {
    // opt-in (BD_LUT_B1=1): measured 3.6x slower than the byte LUT on B200 (see header)
    static const bool on = std::getenv("BD_LUT_B1") && std::getenv("BD_LUT_B1")[0] == '1';
    if (!on || p.cols % 128 != 0) return false;
    for (int j = 0; j < p.n_jobs; ++j)
        for (int s = 0; s < p.n_segs; ++s)
            for (int k = 0; k < p.jobs[j].n_planes[s]; ++k)
                if (reinterpret_cast<uintptr_t>(p.jobs[j].bits[s][k]) % 16) return false;
    return true;
}

template <int kWPR>
static void b1_launch_t(const LutParams& p, const void* X, float* out, cudaStream_t stream) {
    static bool attr = false;
    if (!attr) {
        // the K2 GEMM CTA beside it on every SM takes the shared memory
        BD_CUDA(cudaFuncSetAttribute(b1_kernel<kWPR>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     int(cudaSharedmemCarveoutMaxShared)));
        attr = true;
    }
    BD_CUDA(launch_pdl(b1_kernel<kWPR>, dim3(p.grid), dim3(kB1Threads), 0, stream, p,
                       static_cast<const uint16_t*>(X), out));
}

void b1_launch(const LutParams& p, const void* X, float* out, cudaStream_t stream) {
    switch (p.cols) {
        case 4096: b1_launch_t<128>(p, X, out, stream); break;
        case 8192: b1_launch_t<256>(p, X, out, stream); break;
        case 11008: b1_launch_t<344>(p, X, out, stream); break;
        case 14336: b1_launch_t<448>(p, X, out, stream); break;
        case 28672: b1_launch_t<896>(p, X, out, stream); break;
        default: b1_launch_t<0>(p, X, out, stream); break;
    }
    note_launch();
    BD_CUDA(cudaGetLastError());
}

}  // namespace bd
