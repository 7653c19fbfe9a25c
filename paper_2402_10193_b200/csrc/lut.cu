// K3 (few requests per tenant) — byte-LUT signed accumulation on the CUDA cores.
//
// Replaces per request r of tenant t (P:src/serve.cpp:250-254):
//   apply_delta_correction -> packed_signed_accumulate (P:src/delta.cpp:80-103)
//   y_r[m] += alpha_t * sum_j s_t[m][j] x_r[j]
// reading every plane row with fully coalesced 128-byte warp loads straight from
// the reference layout (flat row-major bits, LSB first), no re-tiling.
//
// Work = (unit = request x 1024-column slice) x (stacked output rows). The grid
// is persistent (<= one CTA per SM): CTA c owns a contiguous range of the
// flattened (unit, row) space, so it rebuilds its tables only when it crosses
// into a new unit and every SM gets the same amount of work (no wave tail).
// For a unit the CTA builds 128 byte tables for the slice's x values
//   T[k][e][l] = sum_{i<8} (bit_i(e) ? +x : -x)[32 l + 8 k + i]   (128 KB smem)
// laid out so that lane l always reads bank l (conflict-free); then for every
// row each lane loads its 32-bit word of the row slice and adds 4 entries.
// 32 rows are accumulated per warp and reduced with a transposing butterfly
// (31 shuffles per 32 rows). Cost per 8 bits: 2 ALU + 1 LDS + 1 FADD.
// Output: one f32 partial per (slice, request, row), scaled by alpha; the
// consumer sums the slices in a fixed order (deterministic).
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace bd {

void note_launch();

namespace {

#ifndef BD_LUT_THREADS
#define BD_LUT_THREADS 512
#endif
#ifndef BD_LUT_REGS
#define BD_LUT_REGS 96
#endif
constexpr int kLutThreads = BD_LUT_THREADS;
// <= 96 registers so a base-GEMM CTA (128 threads) can be co-resident on the SM
constexpr int kLutRegs = BD_LUT_REGS;
constexpr int kSliceCols = 1024;
constexpr size_t kTableBytes = 4 * 256 * 32 * sizeof(float);  // 128 KB
constexpr size_t kLut2Smem = kTableBytes + (kSliceCols + kSliceCols / 128) * sizeof(float);
constexpr int R = 16;                                          // rows per warp batch

// Table layout (bytes): entry (k, e, lane l) at (k>>1)*65536 + e*256 + (k&1)*128 + 4*l,
// so the lookup address of byte k of a word is a single PRMT (byte k of the word
// placed at bit 8, the lane offset in the low byte) plus an immediate.
__device__ __forceinline__ void build_tables(float* T, const float* xs) {
    // thread t -> lane l = t%32, quarter (t/32)%4 of the 256 entries, table k = t/128;
    // a warp covers the 32 lanes of one (k, quarter) -> its stores hit 32 distinct banks.
    // xs is [32][33] (padded) so the per-lane x reads are conflict-free too.
    const int l = threadIdx.x & 31, quarter = (threadIdx.x >> 5) & 3, k = threadIdx.x >> 7;
    const float* xv = xs + 33 * l + 8 * k;
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
    float* Tk = T + (k >> 1) * 16384 + (k & 1) * 32 + l;  // float index
#pragma unroll
    for (int eh = 0; eh < 4; ++eh)
#pragma unroll
        for (int el = 0; el < 16; ++el) Tk[((quarter * 4 + eh) * 16 + el) * 64] = hi[eh] + lo[el];
}

template <int kWPR>  // words per plane row (cols/32); 0 = runtime value
__global__ void __maxnreg__(kLutRegs)
    lut_kernel(const __grid_constant__ LutParams p, const uint16_t* __restrict__ X,
               float* __restrict__ out) {
    extern __shared__ float T[];
    __shared__ float xs[32 * 33];  // x of the slice, [lane][32 columns] padded to 33
    const unsigned long long t_entry = gtimer();
    griddep_wait();  // PDL: X comes from the previous kernel; D is still read by it
    const unsigned long long t_wait = gtimer();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int kWarps = kLutThreads / 32;
    const uint32_t lb0 = 4u * lane, lb1 = 4u * lane + 128u;  // low byte of the entry offset
    const char* Tc = reinterpret_cast<const char*>(T);
    const int wpr = kWPR ? kWPR : p.cols / 32;
    const long long total = static_cast<long long>(p.n_jobs) * p.slices * p.M;
    const long long g0 = total * blockIdx.x / gridDim.x;
    const long long g1 = total * (blockIdx.x + 1) / gridDim.x;
    int cur = -1;
    // rows [ga, gb) of the flattened (unit, row) space; CTA-uniform (tables are rebuilt
    // with block barriers when the range enters a new unit)
    auto run_range = [&](long long ga, long long gb) {
    for (long long g = ga; g < gb;) {
        const int u = static_cast<int>(g / p.M);
        const int ra = static_cast<int>(g % p.M);
        const int rb = static_cast<int>(std::min<long long>(p.M, ra + (gb - g)));
        const int job_i = u / p.slices, slice = u % p.slices;
        const LutJob& job = p.jobs[job_i];
        const int c0 = slice * kSliceCols;
        if (u != cur) {
            __syncthreads();  // previous unit's lookups done
            const uint16_t* xr = X + static_cast<size_t>(job.req) * p.ldx;
            for (int i = threadIdx.x; i < kSliceCols; i += kLutThreads)
                xs[(i >> 5) * 33 + (i & 31)] = (c0 + i < p.cols) ? bf16_to_f32(xr[c0 + i]) : 0.0f;
            __syncthreads();
            if (threadIdx.x < 512) build_tables(T, xs);  // 512 builders: 128 tables x 4 quarters
            __syncthreads();
            cur = u;
        }
        const bool lane_on = c0 + 32 * lane < p.cols;
        float* out_u = out + (static_cast<size_t>(slice) * p.batch + job.req) * p.M;
        for (int s = 0; s < p.n_segs; ++s) {
            const int s0 = p.seg_row0[s], s1 = p.seg_row0[s + 1];
            const int la = std::max(ra, s0) - s0, lb = std::min(rb, s1) - s0;
            if (la >= lb) continue;
            const int n_planes = job.n_planes[s];
            // software pipeline: the words of the warp's next batch are in flight
            // while the current batch is looked up (one plane at a time)
            for (int pl = 0; pl < n_planes; ++pl) {
                const uint32_t* plane = reinterpret_cast<const uint32_t*>(job.bits[s][pl]) + slice * 32 + lane;
                const float a = job.alpha[s][pl];
                auto load = [&](int r0, uint32_t (&w)[R]) {
                    const uint32_t* rowp = plane + static_cast<size_t>(r0) * wpr;
                    if (lane_on && r0 + R <= lb) {
#pragma unroll
                        for (int j = 0; j < R; ++j) w[j] = __ldcs(rowp + j * wpr);
                    } else {
#pragma unroll
                        for (int j = 0; j < R; ++j) w[j] = (lane_on && r0 + j < lb) ? __ldcs(rowp + j * wpr) : 0u;
                    }
                };
                uint32_t wn[R];
                int r0 = la + warp * R;
                if (r0 < lb) load(r0, wn);
                for (; r0 < lb; r0 += kWarps * R) {
                    uint32_t w[R];
#pragma unroll
                    for (int j = 0; j < R; ++j) w[j] = wn[j];
                    if (r0 + kWarps * R < lb) load(r0 + kWarps * R, wn);
                    float acc[R];
#pragma unroll
                    for (int j = 0; j < R; ++j) {
                        const uint32_t v = w[j];
                        const float t0 = *reinterpret_cast<const float*>(Tc + __byte_perm(v, lb0, 0x5504));
                        const float t1 = *reinterpret_cast<const float*>(Tc + __byte_perm(v, lb1, 0x5514));
                        const float t2 = *reinterpret_cast<const float*>(Tc + 65536 + __byte_perm(v, lb0, 0x5524));
                        const float t3 = *reinterpret_cast<const float*>(Tc + 65536 + __byte_perm(v, lb1, 0x5534));
                        acc[j] = a * ((t0 + t1) + (t2 + t3));
                    }
                    // transposing butterfly over lane bits 4..1, then a pair sum:
                    // lanes 2i and 2i+1 end with the total of row r0 + i
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
                    const int r = r0 + ((lane >> 1) & 15);
                    if ((lane & 1) == 0 && r < lb) {
                        if (pl == 0) out_u[s0 + r] = tot;
                        else out_u[s0 + r] += tot;  // same thread wrote it for plane 0
                    }
                }
            }
        }
        g += rb - ra;
    }
    };
    run_range(g0, g1);
    if (tracing()) {
        __syncthreads();
        if (threadIdx.x == 0) trace_rec(TR_LUT, t_entry, t_wait);
    }
}

// ---------------------------------------------------------------------------------------
// v2 (cols % 128 == 0, 16-byte aligned planes — every BASELINE shape): fewer MIO operations
// per 32-bit row word than v1's 6 (1 LDG.32 + 4 LDS + 1 SHFL):
//   * lane l = (chunk c = l & 7, row group g = l >> 3) loads 16 bytes (128 columns) of a row
//     with one LDG.128 — a warp instruction covers 4 whole 128-byte row slices;
//   * the 4 rows of a lane are reduced over the 8 chunk lanes with a 3-level transposing
//     butterfly: 4 SHFL per 16 words (v1: 16);
//   * lookups stay conflict-free although 4 lanes (one per row group) read each table at
//     once: row group g reads byte (b + g) & 3 of a word in lookup slot b, and table
//     (c, w, b') lives in bank 4c + b' — a runtime PRMT selector does the rotation for free.
// Per word: 4 PRMT + 4 LDS + 4 FADD, 1/4 LDG, 1/4 SHFL.
// Table entry (chunk c, word w, byte b', value e) at byte
//   65536 (w >> 1) + 256 e + 128 (w & 1) + 4 (4c + b')   (128 KB, same footprint as v1).
// plane words: read once, never reused by this SM
__device__ __forceinline__ uint4 ld_plane(const uint4* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}

// lut2 keeps no static shared memory, so its dynamic buffer (tables first) starts right after
// the CTA's 1 KB reserved shared memory: the table base is an immediate of every lookup
// (checked at kernel entry)
constexpr uint32_t kTableShared = 0x400;
template <uint32_t kOff>
__device__ __forceinline__ float lds_imm(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(addr), "n"(kOff));
    return v;
}

__device__ __forceinline__ void build_tables_v2(float* T, const float* xs, int t) {
    // builder t < 512 -> bank t & 31 (c = bank >> 2, b' = bank & 3), word w = (t >> 5) & 3,
    // quarter (t >> 7) of the 256 entries; a warp stores one 128-byte row per entry.
    const int bank = t & 31, w = (t >> 5) & 3, quarter = t >> 7;
    const int col = 128 * (bank >> 2) + 32 * w + 8 * (bank & 3);
    float xv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) xv[i] = xs[col + i + ((col + i) >> 7)];
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
    float* Tw = T + (w >> 1) * 16384 + (w & 1) * 32 + bank;  // float index
#pragma unroll
    for (int eh = 0; eh < 4; ++eh)
#pragma unroll
        for (int el = 0; el < 16; ++el) Tw[((quarter * 4 + eh) * 16 + el) * 64] = hi[eh] + lo[el];
}

template <int kWPR, int kLdU4 = kWPR / 4>  // words per plane row (cols/32), row stride in 16-B words; 0 = runtime
__global__ void __maxnreg__(kLutRegs)
    lut2_kernel(const __grid_constant__ LutParams p, const uint16_t* __restrict__ X,
                float* __restrict__ out) {
    extern __shared__ float T[];   // [128 KB tables][x of the slice, padded every 128]
    float* xs = T + kTableBytes / 4;
    const unsigned long long t_entry = gtimer();
    griddep_wait();  // PDL: X comes from the previous kernel; D is still read by it
    const unsigned long long t_wait = gtimer();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int chunk = lane & 7, grp = lane >> 3;
    constexpr int kWarps = kLutThreads / 32;
    constexpr int kRows = 16;  // rows per warp batch (4 per lane)
    // per lookup slot b: PRMT selector (result byte 0 = L byte b = low byte 4*bank,
    // byte 1 = word byte (b + grp) & 3, bytes 2-3 = sign of L byte 0 = 0)
    uint32_t L = 0, sel[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const uint32_t bp = (b + grp) & 3;
        L |= (16u * chunk + 4u * bp) << (8 * b);
        sel[b] = 0xCC00u | (bp << 4) | (4u + b);
    }
    if (threadIdx.x == 0 && static_cast<uint32_t>(__cvta_generic_to_shared(T)) != kTableShared) __trap();
    const int wpr = kWPR ? kWPR : p.cols / 32;
    const long long total = static_cast<long long>(p.n_jobs) * p.slices * p.M;
    const long long g0 = total * blockIdx.x / gridDim.x;
    const long long g1 = total * (blockIdx.x + 1) / gridDim.x;
    int cur = -1;
    // x of a unit (request, slice): kXPer values per thread. The next unit's are loaded into
    // registers right after the current unit's tables are built, so a unit switch does not
    // wait on global memory.
    constexpr int kXPer = (kSliceCols + kLutThreads - 1) / kLutThreads;
    uint16_t xnext[kXPer];
    int pre = -1;
    auto load_x = [&](int unit, uint16_t (&v)[kXPer]) {
        const LutJob& jb = p.jobs[unit / p.slices];
        const int cb = (unit % p.slices) * kSliceCols;
        const uint16_t* xr = X + static_cast<size_t>(jb.req) * p.ldx;
#pragma unroll
        for (int k = 0; k < kXPer; ++k) {
            const int i = threadIdx.x + k * kLutThreads;
            v[k] = (i < kSliceCols && cb + i < p.cols) ? xr[cb + i] : uint16_t(0);
        }
    };
    for (long long g = g0; g < g1;) {
        const int u = static_cast<int>(g / p.M);
        const int ra = static_cast<int>(g % p.M);
        const int rb = static_cast<int>(std::min<long long>(p.M, ra + (g1 - g)));
        const int job_i = u / p.slices, slice = u % p.slices;
        const LutJob& job = p.jobs[job_i];
        const int c0 = slice * kSliceCols;
        if (u != cur) {
            if (pre != u) load_x(u, xnext);
            __syncthreads();  // previous unit's lookups done
#pragma unroll
            for (int k = 0; k < kXPer; ++k) {
                const int i = threadIdx.x + k * kLutThreads;
                if (i < kSliceCols) xs[i + (i >> 7)] = bf16_to_f32(xnext[k]);
            }
            __syncthreads();
            // 512 builders: 128 tables x 4 quarters
            for (int t = threadIdx.x; t < 512; t += kLutThreads) build_tables_v2(T, xs, t);
            __syncthreads();
            cur = u;
            if (g - ra + p.M < g1) {  // this CTA's range continues into unit u + 1
                load_x(u + 1, xnext);
                pre = u + 1;
            }
        }
        const bool lane_on = c0 + 128 * chunk < p.cols;
        float* out_u = out + (static_cast<size_t>(slice) * p.batch + job.req) * p.M;
        for (int s = 0; s < p.n_segs; ++s) {
            const int s0 = p.seg_row0[s], s1 = p.seg_row0[s + 1];
            const int la = std::max(ra, s0) - s0, lb = std::min(rb, s1) - s0;
            if (la >= lb) continue;
            const int n_planes = job.n_planes[s];
            for (int pl = 0; pl < n_planes; ++pl) {
                // lanes past the matrix's last column read chunk 0 (their table entries are 0)
                const uint4* plane = reinterpret_cast<const uint4*>(job.bits[s][pl]) + slice * 8 +
                                     (lane_on ? chunk : 0);
                const float a = job.alpha[s][pl];
                // lane rows r0 + 4 grp + i, i < 4 (each LDG.128 instruction: 4 rows x 128 B); rows
                // past lb re-read row lb - 1 (never stored), so no load is predicated
                auto load = [&](int r0, uint4 (&w)[4]) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int r = min(r0 + 4 * grp + i, lb - 1);
                        w[i] = ld_plane(plane + static_cast<size_t>(r) * (kLdU4 ? kLdU4 : p.ld_u4));
                    }
                };
                auto consume = [&](int r0, const uint4 (&wc)[4]) {
                    float acc[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const uint32_t v[4] = {wc[i].x, wc[i].y, wc[i].z, wc[i].w};
                        float sw[4];
#pragma unroll
                        // every lookup is one PRMT + one LDS [reg + imm]
                        auto word = [&](uint32_t vw, auto off) {
                            constexpr uint32_t o = decltype(off)::value;
                            const float t0 = lds_imm<o>(prmt(vw, L, sel[0]));
                            const float t1 = lds_imm<o>(prmt(vw, L, sel[1]));
                            const float t2 = lds_imm<o>(prmt(vw, L, sel[2]));
                            const float t3 = lds_imm<o>(prmt(vw, L, sel[3]));
                            return (t0 + t1) + (t2 + t3);
                        };
                        sw[0] = word(v[0], std::integral_constant<uint32_t, kTableShared>{});
                        sw[1] = word(v[1], std::integral_constant<uint32_t, kTableShared + 128>{});
                        sw[2] = word(v[2], std::integral_constant<uint32_t, kTableShared + 65536>{});
                        sw[3] = word(v[3], std::integral_constant<uint32_t, kTableShared + 65536 + 128>{});
                        acc[i] = a * ((sw[0] + sw[1]) + (sw[2] + sw[3]));
                    }
                    // transposing butterfly over the chunk bits (lane bits 2, 1), then a pair sum:
                    // lane ends with row 2 * bit2 + bit1 of its group
#pragma unroll
                    for (int o = 4, n = 2; o >= 2; o >>= 1, n >>= 1) {
                        const bool upper = (lane & o) != 0;
#pragma unroll
                        for (int j = 0; j < n; ++j) {
                            const float send = upper ? acc[j] : acc[j + n];
                            const float keep = upper ? acc[j + n] : acc[j];
                            acc[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                        }
                    }
                    const float tot = acc[0] + __shfl_xor_sync(0xffffffffu, acc[0], 1);
                    const int r = r0 + 4 * grp + 2 * ((lane >> 2) & 1) + ((lane >> 1) & 1);
                    if ((lane & 1) == 0 && r < lb) {
                        if (pl == 0) out_u[s0 + r] = tot;
                        else out_u[s0 + r] += tot;  // same thread wrote it for plane 0
                    }
                };
                // ping-pong register buffers: the next batch's words are in flight while the
                // current one is looked up (no register moves between iterations)
                constexpr int kStep = kWarps * kRows;
                int r0 = la + warp * kRows;
                uint4 wa[4], wb[4];
                if (r0 < lb) load(r0, wa);
                while (r0 < lb) {
                    if (r0 + kStep < lb) load(r0 + kStep, wb);
                    consume(r0, wa);
                    r0 += kStep;
                    if (r0 >= lb) break;
                    if (r0 + kStep < lb) load(r0 + kStep, wa);
                    consume(r0, wb);
                    r0 += kStep;
                }
            }
        }
        g += rb - ra;
    }
    if (tracing()) {
        __syncthreads();
        if (threadIdx.x == 0) trace_rec(TR_LUT, t_entry, t_wait);
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
    p.ld_u4 = cols / 128;  // flat reference layout (v2 needs cols % 128 == 0)
    p.n_segs = n_segs;
    int total = 0;
    for (int s = 0; s < n_segs; ++s) {
        p.seg_row0[s] = total;
        total += seg_rows[s];
    }
    p.seg_row0[n_segs] = total;
    p.M = total;
    // persistent: one CTA per SM, but keep >= 512 rows of work per CTA
    const long long work = static_cast<long long>(p.n_jobs) * p.slices * p.M;
    p.grid = static_cast<int>(std::max<long long>(1, std::min<long long>(kNumSMs, work / 512)));
    return true;
}

template <int kWPR>
void lut_launch_t(const LutParams& p, const void* X, float* out, cudaStream_t stream) {
    static bool attr = false;
    if (!attr) {
        BD_CUDA(cudaFuncSetAttribute(lut_kernel<kWPR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(kTableBytes)));
        // Max carveout lets the K2 GEMM CTA co-reside on every SM. Measured on B200 it
        // helps when plane rows are 128-B aligned (qkv/o/gu: -0.34 ms/step) and hurts
        // the down projection (1376-B rows, every warp load spans two lines: +0.35 ms),
        // where the default carveout keeps the two kernels on mostly disjoint SMs.
        if (kWPR % 32 == 0 && kWPR > 0)
            BD_CUDA(cudaFuncSetAttribute(lut_kernel<kWPR>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                         int(cudaSharedmemCarveoutMaxShared)));
        attr = true;
    }
    BD_CUDA(launch_pdl(lut_kernel<kWPR>, dim3(p.grid), dim3(kLutThreads), kTableBytes, stream, p,
                       static_cast<const uint16_t*>(X), out));
}

template <int kWPR, int kLdU4 = kWPR / 4>
void lut2_launch_t(const LutParams& p, const void* X, float* out, cudaStream_t stream) {
    static bool attr = false;
    if (!attr) {
        BD_CUDA(cudaFuncSetAttribute(lut2_kernel<kWPR, kLdU4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(kLut2Smem)));
        // max carveout (K2 co-resident on every SM) where the plane rows are 128-B aligned,
        // which includes the pool's padded down-projection rows (1 408 B: down phase 1.49 ->
        // 1.30 ms/step, profiles/r02_exp_lut_down_padded_rows_ab.txt); unaligned rows (the
        // reference's 1 376 B) ran faster on the default carveout with K2 after the LUT
        // (profiles/r02_exp_down_carveout.txt)
        if (kLdU4 % 8 == 0 && kLdU4 > 0)
            BD_CUDA(cudaFuncSetAttribute(lut2_kernel<kWPR, kLdU4>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                         int(cudaSharedmemCarveoutMaxShared)));
        attr = true;
    }
    BD_CUDA(launch_pdl(lut2_kernel<kWPR, kLdU4>, dim3(p.grid), dim3(kLutThreads), kLut2Smem, stream, p,
                       static_cast<const uint16_t*>(X), out));
}

static bool lut2_ok(const LutParams& p) {
    if (p.cols % 128 != 0) return false;
    for (int j = 0; j < p.n_jobs; ++j)
        for (int s = 0; s < p.n_segs; ++s)
            for (int k = 0; k < p.jobs[j].n_planes[s]; ++k)
                if (reinterpret_cast<uintptr_t>(p.jobs[j].bits[s][k]) % 16) return false;
    return true;
}

void lut_launch(const LutParams& p, const void* X, float* out, cudaStream_t stream) {
    if (lut2_ok(p)) {
        // the row stride is a compile-time constant on the hot shapes (an immediate in every
        // plane address; a runtime stride costs the issue-bound loop ~15 %)
        const bool flat = p.ld_u4 == p.cols / 128;
        switch (flat ? p.cols : (p.cols == 11008 && p.ld_u4 == 88 ? -11008 : 0)) {
            case 4096: lut2_launch_t<128>(p, X, out, stream); break;
            case 8192: lut2_launch_t<256>(p, X, out, stream); break;
            case 11008: lut2_launch_t<344>(p, X, out, stream); break;
            case -11008: lut2_launch_t<344, 88>(p, X, out, stream); break;  // pool: 1 408-B padded rows
            case 14336: lut2_launch_t<448>(p, X, out, stream); break;
            case 28672: lut2_launch_t<896>(p, X, out, stream); break;
            default: lut2_launch_t<0, 0>(p, X, out, stream); break;
        }
        note_launch();
        BD_CUDA(cudaGetLastError());
        return;
    }
    // v1 (cols % 32 == 0 but not % 128: no published shape) with a runtime row stride
    lut_launch_t<0>(p, X, out, stream);
    note_launch();
    BD_CUDA(cudaGetLastError());
}

}  // namespace bd
