// K3m — tenant deltas on the FP4 tensor cores, beside K2 (one request per job; the byte
// LUT's job list, K2 unchanged on the side stream).
//
// Replaces, per request r of tenant t (P:src/serve.cpp:250-254):
//   apply_delta_correction -> packed_signed_accumulate (P:src/delta.cpp:80-103)
//   D[r][m] = alpha_t * sum_k s_t[m][k] x_r[k]      (full K: one partial, dsplits = 1)
//
// Why: the byte LUT does 4 PRMT + 4 LDS + 4 FADD per 32-bit plane word on the CUDA cores and
// its row loads sit in the LSU path, so beside K2's TMA stream it is memory-latency-bound
// (DESIGN.md §7.0). Here plane bytes arrive by TMA into a deep smem ring (like K2's weights)
// and a word costs 8 ALU ops (expand4: shift + LOP3 per 8 elements) + a tcgen05.st; the
// products run on the tensor pipe, which K2 at batch 16 leaves idle:
//   * a task = (job, 128-row tile); its stages are the K/1024 column chunks: a [128 rows x
//     128 B] plane box (TMA, 128-byte swizzle, the reference layout) and the request's FP4
//     activation pieces for the chunk (xp_prep, mt4.cu: 8 pieces, x to 2^-24 of each
//     32-column block maximum, one 4352-byte bulk copy);
//   * one expander warpgroup (thread = tile row = TMEM lane) turns each half stage (K = 512)
//     into e2m1 +-1.0 in one of two TMEM A buffers, meets on a named barrier, and its first
//     warp issues the 8 kind::mxf4 MMAs (M = 128, N = 8 pieces, K = 64) warp-wide; the MMAs'
//     commit frees the A buffer (and, after the second half, the smem stage);
//   * the task's 4..11 stages accumulate in one of two f32 TMEM accumulators (8 columns); the
//     epilogue sums the 8 piece columns, applies alpha and writes D once per (request, row).
// Warp roles (160 threads, <= 112 KB smem, 256 TMEM columns: a K2 CTA stays co-resident):
//   warp 0 TMA producer (one elected lane), warps 1-4 expanders / MMA issue (warp 1) /
//   epilogue. Persistent grid: CTA c takes a contiguous range of tasks.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace bd {

void note_launch();

namespace {

constexpr int kMxThreads = 160;
constexpr int kRing = 5;                                 // smem stages in flight
constexpr uint32_t kPlaneBytes = 16384;                  // [128 rows x 128 B]
constexpr uint32_t kStageBytes = kPlaneBytes + 5120;     // + pieces (kXpBlock padded to 1 KB)
constexpr uint32_t kSmem = 1024 + kRing * kStageBytes + 256;
// TMEM (256 columns): A scales 1.0 at [0, 8); A buffer h at 8 + 80 h: two K = 256 entries of
// 40 columns (B scales at +0/+2, A at +8..+39, K23's entry layout); accumulators at 168 + 8 d
constexpr uint32_t kColSfa = 0, kColA = 8, kEntry = 40, kColAcc = 168;

struct Task {
    int job, seg, m0, row;  // row: first row inside the segment's plane
};
__device__ __forceinline__ Task task_of(const MxdParams& p, int t) {
    Task k;
    k.job = t / p.tiles;
    k.m0 = (t - k.job * p.tiles) * 128;
    int sg = 0;
    while (sg + 1 < p.n_segs && k.m0 >= p.seg_row0[sg + 1]) ++sg;
    k.seg = sg;
    k.row = k.m0 - p.seg_row0[sg];
    return k;
}

__device__ __forceinline__ void named_sync(uint32_t id, uint32_t n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__global__ void __launch_bounds__(kMxThreads, 1) mxd_kernel(const __grid_constant__ MxdParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kRing * kStageBytes);
    uint64_t* empty = full + kRing;
    uint64_t* a_free = empty + kRing;   // [2] MMAs of A buffer h complete
    uint64_t* acc_full = a_free + 2;    // [2] a task's MMAs complete
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 2);
    const uint32_t warp = warp_id(), lane = lane_id();
    const int t0 = static_cast<int>(static_cast<long long>(p.n_tasks) * blockIdx.x / gridDim.x);
    const int t1 = static_cast<int>(static_cast<long long>(p.n_tasks) * (blockIdx.x + 1) / gridDim.x);
    const unsigned long long t_entry = gtimer();
    if (warp == 0) {
        if (lane == 0) {
            for (int s = 0; s < kRing; ++s) {
                mbar_init(&full[s], 1);
                mbar_init(&empty[s], 1);  // the stage's last MMAs (commit)
            }
            for (int h = 0; h < 2; ++h) {
                mbar_init(&a_free[h], 1);
                mbar_init(&acc_full[h], 1);
            }
            fence_mbar_init();
        }
        __syncwarp();
        tmem_alloc<256>(tmem_slot);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;

    if (warp == 0) {
        // ---- TMA producer: plane boxes do not depend on the predecessor, the pieces do ----
        const uint64_t pol_stream = policy_evict_first();
        const uint64_t pol_keep = policy_evict_last();
        griddep_wait();  // PDL: the pieces (xp_prep) come from the previous kernel
        int s = 0;
        uint32_t ph = 0;
        for (int t = t0; t < t1; ++t) {
            const Task k = task_of(p, t);
            const CUtensorMap* map = p.maps + k.job * kLutMaxSegs + k.seg;
            const uint8_t* xp = p.xpk + static_cast<size_t>(p.req[k.job]) * p.n_chunks * kXpBlock;
            for (int c = 0; c < p.n_chunks; ++c) {
                mbar_wait_w(&empty[s], ph ^ 1);
                uint8_t* sp = smem + s * kStageBytes;
                mbar_arrive_expect_tx_w(&full[s], kPlaneBytes + kXpBlock);
                tma_load_2d_w(sp, map, &full[s], c * 128, k.row, pol_stream);
                bulk_load_w(sp + kPlaneBytes, xp + static_cast<size_t>(c) * kXpBlock, kXpBlock, &full[s], pol_keep);
                if (++s == kRing) {
                    s = 0;
                    ph ^= 1;
                }
            }
        }
    } else {
        // ---- expander warpgroup: thread = tile row = TMEM lane ----
        const uint32_t q4 = warp & 3;
        const uint32_t trow = q4 * 32 + lane;
        const uint32_t lane_base = (q4 * 32) << 16;
        {
            uint32_t one[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) one[j] = 0x7F7F7F7Fu;  // A block scales 1.0
            tmem_st8(tbase + lane_base + kColSfa, one);
            tmem_st_wait();
        }
        griddep_wait();  // D is still read by the previous kernel's consumer
        const uint32_t idesc = idesc_mxf4(128, 8);
        const uint32_t sw = trow & 7;
        int s = 0;
        uint32_t ph = 0, use[2] = {0, 0}, acc_ph[2] = {0, 0};
        int d = 0;
        for (int t = t0; t < t1; ++t) {
            const Task k = task_of(p, t);
            for (int c = 0; c < p.n_chunks; ++c) {
                mbar_wait(&full[s], ph);
                const uint8_t* sp = smem + s * kStageBytes;
                const uint8_t* rowp = sp + trow * 128;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (use[h]) mbar_wait(&a_free[h], (use[h] - 1) & 1);  // buffer h's last MMAs done
                    ++use[h];
                    tc_fence_after();
#pragma unroll
                    for (int jj = 0; jj < 2; ++jj) {
                        const int j = 2 * h + jj;  // quarter of the stage (256 columns)
                        const uint32_t ent = tbase + lane_base + kColA + (2 * h + jj) * kEntry;
                        uint32_t sc[4] = {0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu};
                        if (lane < 8) {  // B block scales: piece `lane`, blocks 8j..8j+7
                            const uint2 v = *reinterpret_cast<const uint2*>(sp + kPlaneBytes + 4096 + lane * 32 + 8 * j);
                            sc[0] = v.x;
                            sc[2] = v.y;
                        }
                        tmem_st4(ent, sc);
                        const uint4 v0 = *reinterpret_cast<const uint4*>(rowp + (((2 * j) ^ sw) << 4));
                        const uint4 v1 = *reinterpret_cast<const uint4*>(rowp + (((2 * j + 1) ^ sw) << 4));
                        const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
                        uint32_t a[32];
#pragma unroll
                        for (int u = 0; u < 8; ++u)
#pragma unroll
                            for (int cc = 0; cc < 4; ++cc) a[4 * u + cc] = expand4(w[u], cc);
                        tmem_st32(ent + 8, a);
                    }
                    tmem_st_wait();
                    tc_fence_before();
                    named_sync(1, 128);
                    if (warp == 1) {
                        tc_fence_after();
                        const uint64_t db = sdesc_sw128(sp + kPlaneBytes, 5120);
                        const uint32_t dacc = tbase + kColAcc + 8 * d;
#pragma unroll
                        for (int jj = 0; jj < 2; ++jj) {
                            const int j = 2 * h + jj;
                            const uint32_t ent = tbase + kColA + (2 * h + jj) * kEntry;
                            const uint64_t db0 = db + j * (1024u >> 4);
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk)
                                mma_mxf4_ts_w(dacc, ent + 8 + 8 * kk, db0 + 2 * kk,
                                              idesc | (uint32_t(2 * (kk & 1)) << 4), tbase + kColSfa,
                                              ent + 2 * (kk >> 1), (c == 0 && j == 0 && kk == 0) ? 0u : 1u);
                        }
                        tc_commit_w(&a_free[h]);
                        if (h == 1) tc_commit_w(&empty[s]);
                        if (h == 1 && c == p.n_chunks - 1) tc_commit_w(&acc_full[d]);
                    }
                }
                if (++s == kRing) {
                    s = 0;
                    ph ^= 1;
                }
            }
            // ---- epilogue of the task: 8 piece columns -> one f32 per (request, row) ----
            mbar_wait(&acc_full[d], acc_ph[d]);
            acc_ph[d] ^= 1;
            tc_fence_after();
            uint32_t v[8];
            tmem_ld8(tbase + lane_base + kColAcc + 8 * d, v);
            tmem_ld_wait();
            const float sum = ((__uint_as_float(v[0]) + __uint_as_float(v[1])) +
                               (__uint_as_float(v[2]) + __uint_as_float(v[3]))) +
                              ((__uint_as_float(v[4]) + __uint_as_float(v[5])) +
                               (__uint_as_float(v[6]) + __uint_as_float(v[7])));
            p.out[static_cast<size_t>(p.req[k.job]) * p.M + k.m0 + trow] = p.alpha[k.job][k.seg] * sum;
            tc_fence_before();
            d ^= 1;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<256>(tbase);
    if (threadIdx.x == 32) trace_rec(TR_LUT, t_entry, t_entry);
}

}  // namespace

bool plan_mxd(MxdParams& p, const LutParams& lp, const std::vector<int>& seg_rows, std::vector<CUtensorMap>& maps) {
    if (lp.cols % 128 != 0 || lp.n_jobs < 1 || lp.n_jobs > kLutMaxJobs) return false;
    p = MxdParams{};
    p.n_jobs = lp.n_jobs;
    p.n_segs = lp.n_segs;
    p.M = lp.M;
    p.K = lp.cols;
    p.n_chunks = xp_chunks(lp.cols);
    for (int s = 0; s <= lp.n_segs; ++s) p.seg_row0[s] = lp.seg_row0[s];
    for (int s = 0; s < lp.n_segs; ++s)
        if (seg_rows[s] % 128) return false;
    p.tiles = p.M / 128;
    p.n_tasks = p.n_jobs * p.tiles;
    maps.assign(size_t(p.n_jobs) * kLutMaxSegs, CUtensorMap{});
    for (int j = 0; j < p.n_jobs; ++j) {
        const LutJob& jb = lp.jobs[j];
        p.req[j] = jb.req;
        for (int s = 0; s < lp.n_segs; ++s) {
            if (jb.n_planes[s] != 1) return false;  // one plane per projection (alpha per plane)
            if (reinterpret_cast<uintptr_t>(jb.bits[s][0]) % 16) return false;
            p.alpha[j][s] = jb.alpha[s][0];
            maps[size_t(j) * kLutMaxSegs + s] = tmap_bits4(jb.bits[s][0], uint64_t(seg_rows[s]), uint64_t(lp.cols));
        }
    }
    p.grid = std::min(kNumSMs, p.n_tasks);
    return true;
}

void mxd_launch(const MxdParams& p, cudaStream_t stream) {
    static bool attr = false;
    if (!attr) {
        BD_CUDA(cudaFuncSetAttribute(mxd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmem)));
        BD_CUDA(cudaFuncSetAttribute(mxd_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     int(cudaSharedmemCarveoutMaxShared)));
        attr = true;
    }
    BD_CUDA(launch_pdl(mxd_kernel, dim3(p.grid), dim3(kMxThreads), size_t(kSmem), stream, p));
    note_launch();
    BD_CUDA(cudaGetLastError());
}

}  // namespace bd
