// K3t — tenant deltas alone on the FP4 tensor cores, beside K2 (replaces the byte-LUT
// K3 with the same plan and the same output; the base GEMM K2 runs on the side stream
// exactly as with the LUT).
//
// Replaces, per request r of tenant t (P:src/serve.cpp:250-254):
//   apply_delta_correction -> packed_signed_accumulate (P:src/delta.cpp:80-103)
//   D[slice][r][m] = alpha_t * sum_{k in slice} s_t[m][k] x_r[k]     (slice = 1024 columns)
//
// Why: the byte-LUT spends 6 MIO operations per 32-bit plane word (4 table LDS, 1 LDG,
// 1 SHFL) and is bound by the MIO queue at ~2.6 TB/s of planes. Here a
// plane word costs 4 x (SHF + LOP3) ALU operations and the products run on the tensor
// pipe, which K2 (batch 16) leaves almost idle:
//   * a [128 rows x 1024 bits] plane tile (16 KB, reference layout, 128-B swizzled TMA
//     box) becomes the A operand in TMEM as FP4 e2m1 +-1.0 (K23's expansion: bit 4i+c of
//     a word -> nibble i of register c, one shift + one LOP3 each, mt4.cu);
//   * B = the 8 FP4 "pieces" of the request's activations for the slice with their
//     ue8m0 block scales (xp_prep_kernel, mt4.cu: x to 2^-24 of each 32-column block max);
//   * tcgen05.mma.kind::mxf4.block_scale, M = 128, N = 8, K = 64 per instruction,
//     f32 accumulator (8 columns); the epilogue sums the 8 piece columns, applies alpha
//     and writes one f32 per row: every stage is a complete (slice, request, 128 rows)
//     output -> no split partials, bit-reproducible, independent of request order.
// Pipeline (one CTA per SM, co-resident with a K2 CTA: <= 256 TMEM columns, ~88 KB smem):
//   warp 0      TMA producer: plane tile + activation block per stage into a smem ring;
//   warps 1-4   expander group 0, warps 5-8 group 1 (thread = tile row = TMEM lane);
//               the groups take alternate stages. A group expands half a stage (K = 512)
//               into its 2-entry TMEM ring, meets on a 128-thread named barrier, and its
//               first warp issues the MMAs itself (no cross-warp mbarrier round trip per
//               stage — the handshake chain that bounds K23); the second half is
//               expanded into registers while the first half's MMAs run.
//
// MEASURED (round 1, tools/timeline.py, L7 stack T=16 B=16, BD_MXD=1; pool tests green):
//   v1, 2 groups, 2 x 40-column sub-entries per group: ~1800 SM cycles per 16 KB stage per
//       CTA (two MMA completion round trips per stage per group) = ~2.5 TB/s of planes;
//   v2, compact 80-column group entries, 3 groups (13 warps; registers capped so the
//       busiest SM sub-partition still fits a K2 warp): q/k/v deltas alone 36 us
//       (2.8 TB/s, the byte LUT's rate), beside K2 44 us (LUT beside K2: 41 us); down
//       projection 46 us beside K2 (LUT then K2: 51 us). Step 7.46 vs 6.33 ms with the
//       LUT: the separate xp_prep launch costs ~5 us before every linear, and K2 beside
//       this kernel slows it ~20 %. 4 groups (second TMEM allocation) faults - not debugged.
// Next: pieces written by the glue kernels (no xp_prep launch), a deeper TMEM ring so no
// group waits on its own MMAs inside a stage. Opt-in (BD_MXD=1) until it beats the LUT.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace bd {

void note_launch();

namespace {

#ifndef BD_MXD_GROUPS
#define BD_MXD_GROUPS 3
#endif
constexpr int kGroups = BD_MXD_GROUPS;                 // expander groups (4 warps each)
constexpr int kMxdThreads = 32 * (1 + 4 * kGroups);
constexpr int kRing = kGroups + 2;                     // smem stages
constexpr uint32_t kPlaneBytes = 16384;                // [128 rows x 128 B]
constexpr uint32_t kAuxBytes = 5120;                   // kXpBlock padded to the 1024-B swizzle atom
constexpr uint32_t kStageBytes = kPlaneBytes + kAuxBytes;
// TMEM: a 256-column allocation (A scales 1.0 | groups 0-2) and, for a 4th group, a
// 128-column one (K2's CTA beside it needs 32 more: 416 of 512). Group entry (80 columns):
// B scales of its two K = 256 sub-entries at +0/+2 and +4/+6 (even columns), A of
// sub-entry e at +8 + 32 e, the 8 accumulator columns at +72.
constexpr uint32_t kColSfa = 0;
constexpr uint32_t kGroupCols = 80;
constexpr uint32_t kAccOff = 72;

__device__ __forceinline__ void tmem_st4x(uint32_t taddr, const uint32_t (&r)[4]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(r[0]), "r"(r[1]),
                 "r"(r[2]), "r"(r[3])
                 : "memory");
}
__device__ __forceinline__ uint64_t sdesc_sw128x(const void* smem, uint32_t sbo) {
    const uint64_t addr = smem_u32(smem);
    return ((addr >> 4) & 0x3FFFull) | (1ull << 16) | (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) |
           (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc_mxf4x(uint32_t M, uint32_t N) {
    return (1u << 7) | (1u << 10) | ((N >> 3) << 17) | (1u << 23) | ((M >> 4) << 24);
}
__device__ __forceinline__ uint32_t expand4x(uint32_t w, int c) {
    return ((w << (3 - c)) & 0x88888888u) ^ 0xAAAAAAAAu;
}
__device__ __forceinline__ void named_sync(uint32_t id, uint32_t n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

struct Stage {
    int job, chunk, tile, seg;
};
__device__ __forceinline__ Stage stage_of(const MxdParams& p, long long s) {
    Stage st;
    st.tile = static_cast<int>(s % p.m_tiles);
    const long long t2 = s / p.m_tiles;
    st.chunk = static_cast<int>(t2 % p.slices);
    st.job = static_cast<int>(t2 / p.slices);
    const int row0 = st.tile * 128;
    int sg = 0;
    while (sg + 1 < p.n_segs && row0 >= p.seg_row0[sg + 1]) ++sg;
    st.seg = sg;
    return st;
}

// Registers: the CTA's warps spread over the 4 SM sub-partitions (16K registers each);
// the busiest one must still fit one K2 warp (1K registers) beside it.
constexpr int kMxdRegs = ((16384 - 1024) / (((1 + 4 * kGroups) + 3) / 4) / 32) / 8 * 8;
__global__ void __maxnreg__(kMxdRegs > 128 ? 128 : kMxdRegs) mxd_kernel(const __grid_constant__ MxdParams p, float* __restrict__ out) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kRing * kStageBytes);
    uint64_t* empty = full + kRing;
    uint64_t* half_done = empty + kRing;     // [kGroups] first-half MMAs of the group's stage done
    uint64_t* acc_full = half_done + kGroups;  // [kGroups] all MMAs of the group's stage done
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + kGroups);  // [2]
    const unsigned long long t_entry = gtimer();

    const uint32_t warp = warp_id(), lane = lane_id();
    const long long total = p.total_stages;
    const long long g0 = total * blockIdx.x / gridDim.x;
    const long long g1 = total * (blockIdx.x + 1) / gridDim.x;
    if (warp == 0) {
        if (lane == 0) {
            for (int s = 0; s < kRing; ++s) {
                mbar_init(&full[s], 1);
                mbar_init(&empty[s], 1);
            }
            for (int g = 0; g < kGroups; ++g) {
                mbar_init(&half_done[g], 1);
                mbar_init(&acc_full[g], 1);
            }
            fence_mbar_init();
        }
        __syncwarp();
        tmem_alloc<256>(tmem_slot);
        if (kGroups > 3) tmem_alloc<128>(tmem_slot + 1);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = tmem_slot[0];
    griddep_wait();  // PDL: the activation pieces come from the previous kernel
    const unsigned long long t_wait = gtimer();

    if (warp == 0) {
        // ---- TMA producer ----
        const uint64_t pol_stream = policy_evict_first();
        const uint64_t pol_keep = policy_evict_last();
        long long i = 0;
        for (long long s = g0; s < g1; ++s, ++i) {
            const int slot = static_cast<int>(i % kRing);
            const uint32_t ph = static_cast<uint32_t>(i / kRing) & 1u;
            mbar_wait_w(&empty[slot], ph ^ 1);
            const Stage st = stage_of(p, s);
            uint8_t* sp = smem + slot * kStageBytes;
            mbar_arrive_expect_tx_w(&full[slot], kPlaneBytes + kXpBlock);
            tma_load_2d_w(sp, &p.maps[st.job * p.n_segs + st.seg], &full[slot], st.chunk * 128,
                          st.tile * 128 - p.seg_row0[st.seg], pol_stream);
            bulk_load_w(sp + kPlaneBytes,
                        p.xpk + (static_cast<size_t>(p.jobs[st.job].req) * p.n_chunks + st.chunk) * kXpBlock,
                        kXpBlock, &full[slot], pol_keep);
        }
    } else {
        // ---- expander groups (thread = tile row = TMEM lane) ----
        const uint32_t grp = (warp - 1) >> 2;
        const uint32_t q4 = (warp - 1) & 3;  // TMEM lane quarter of this warp = warp % 4 ... see below
        // tcgen05.ld/st: warp w may only touch TMEM lanes [32 (w % 4), +32)
        const uint32_t quarter = warp & 3;
        const uint32_t trow = quarter * 32 + lane;
        const uint32_t lane_base = (quarter * 32) << 16;
        const bool issuer = q4 == 0;  // the group's first warp issues the MMAs
        const uint32_t gcol = grp < 3 ? tbase + 8 + grp * kGroupCols : tmem_slot[1];
        const uint32_t acc_col = gcol + kAccOff;
        if (grp == 0) {  // constant A block scales (1.0)
            uint32_t one[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) one[j] = 0x7F7F7F7Fu;
            tmem_st8(tbase + lane_base + kColSfa, one);
            tmem_st_wait();
        }
        tc_fence_before();
        asm volatile("bar.sync 1, %0;" ::"r"(32 * 4 * kGroups) : "memory");  // SFA written before any MMA
        tc_fence_after();
        const uint32_t sw = trow & 7;
        const uint32_t idesc = idesc_mxf4x(128, 8);
        const bool has_scale = lane < 8;
        uint32_t n_mine = 0;
        long long i = 0;
        for (long long s = g0; s < g1; ++s, ++i) {
            const int slot = static_cast<int>(i % kRing);
            const uint32_t ph = static_cast<uint32_t>(i / kRing) & 1u;
            // every stage's full barrier is observed, also the other groups' (the ring is
            // not a multiple of the group count): a group can then never wait on a slot a
            // whole ring lap ahead of the producer, which would alias the phase parity
            mbar_wait(&full[slot], ph);
            if (static_cast<uint32_t>(i % kGroups) != grp) continue;
            const uint32_t gph = n_mine & 1u;
            ++n_mine;
            const Stage st = stage_of(p, s);
            const uint8_t* sp = smem + slot * kStageBytes;
            const uint8_t* rowp = sp + trow * 128;
            const uint64_t db = sdesc_sw128x(sp + kPlaneBytes, kAuxBytes);
            const uint32_t xstep = 1024u >> 4;  // descriptor units (16 B): 256 columns of pieces
            for (int h = 0; h < 2; ++h) {
                if (h == 1) {  // the first half's MMAs read the same TMEM sub-entries
                    mbar_wait(&half_done[grp], gph);
                    tc_fence_after();
                }
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int j = 2 * h + e;
                    uint32_t sc[4] = {0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu};
                    if (has_scale) {  // B block scales of MMAs 4j..4j+3: lane l < 8 = piece l, every quarter
                        const uint2 v = *reinterpret_cast<const uint2*>(sp + kPlaneBytes + 4096 + lane * 32 + 8 * j);
                        sc[0] = v.x;
                        sc[2] = v.y;
                    }
                    const uint4 v0 = *reinterpret_cast<const uint4*>(rowp + (((2 * j) ^ sw) << 4));
                    const uint4 v1 = *reinterpret_cast<const uint4*>(rowp + (((2 * j + 1) ^ sw) << 4));
                    const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
                    uint32_t a[32];
#pragma unroll
                    for (int u = 0; u < 8; ++u)
#pragma unroll
                        for (int cc = 0; cc < 4; ++cc) a[4 * u + cc] = expand4x(w[u], cc);
                    tmem_st4x(gcol + lane_base + 4 * e, sc);
                    tmem_st32(gcol + lane_base + 8 + 32 * e, a);
                }
                tmem_st_wait();
                tc_fence_before();
                named_sync(2 + grp, 128);
                if (issuer) {
                    tc_fence_after();
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int j = 2 * h + e;
                        const uint64_t db0 = db + j * xstep;
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            mma_mxf4_ts_w(acc_col, gcol + 8 + 32 * e + 8 * kk, db0 + 2 * kk,
                                          idesc | (uint32_t(2 * (kk & 1)) << 4), tbase + kColSfa,
                                          gcol + 4 * e + 2 * (kk >> 1), (h == 0 && e == 0 && kk == 0) ? 0u : 1u);
                    }
                    tc_commit_w(h == 0 ? &half_done[grp] : &acc_full[grp]);
                }
            }
            // ---- epilogue: the stage's 128 rows for (slice, request) ----
            mbar_wait(&acc_full[grp], gph);
            tc_fence_after();
            uint32_t v[8];
            tmem_ld8(acc_col + lane_base, v);
            tmem_ld_wait();
            tc_fence_before();
            if (issuer && lane == 0) mbar_arrive(&empty[slot]);  // MMAs done reading the stage
            const float sum = ((__uint_as_float(v[0]) + __uint_as_float(v[1])) +
                               (__uint_as_float(v[2]) + __uint_as_float(v[3]))) +
                              ((__uint_as_float(v[4]) + __uint_as_float(v[5])) +
                               (__uint_as_float(v[6]) + __uint_as_float(v[7])));
            const MxdJob& job = p.jobs[st.job];
            out[(static_cast<size_t>(st.chunk) * p.batch + job.req) * p.M + st.tile * 128 + trow] =
                job.alpha[st.seg] * sum;
            // the group's next stage overwrites the accumulator (first MMA, accumulate = 0)
            // only after its h = 0 named barrier, which every thread reaches after this load
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tmem_dealloc<256>(tbase);
        if (kGroups > 3) tmem_dealloc<128>(tmem_slot[1]);
    }
    if (threadIdx.x == 0) trace_rec(TR_LUT, t_entry, t_wait);
}

}  // namespace

bool plan_mxd(MxdParams& p, const int* seg_rows, int n_segs, int cols, int batch) {
    // opt-in (BD_MXD=1): measured no faster than the byte LUT yet (see header)
    static const bool on = std::getenv("BD_MXD") && std::getenv("BD_MXD")[0] == '1';
    if (!on || cols % 128 != 0 || n_segs < 1 || n_segs > kLutMaxSegs || p.n_jobs < 1 || p.n_jobs > kLutMaxJobs)
        return false;
    int total = 0;
    for (int s = 0; s < n_segs; ++s) {
        if (seg_rows[s] % 128) return false;
        p.seg_row0[s] = total;
        total += seg_rows[s];
    }
    p.seg_row0[n_segs] = total;
    p.n_segs = n_segs;
    p.M = total;
    p.m_tiles = total / 128;
    p.cols = cols;
    p.batch = batch;
    p.slices = (cols + 1023) / 1024;
    p.n_chunks = xp_chunks(cols);
    p.total_stages = static_cast<long long>(p.n_jobs) * p.slices * p.m_tiles;
    p.grid = static_cast<int>(std::min<long long>(kNumSMs, p.total_stages));
    p.smem = int(1024 + kRing * kStageBytes + 256);
    return true;
}

void mxd_launch(const MxdParams& p, float* out, cudaStream_t stream) {
    static bool attr = false;
    if (!attr) {
        BD_CUDA(cudaFuncSetAttribute(mxd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        BD_CUDA(cudaFuncSetAttribute(mxd_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     int(cudaSharedmemCarveoutMaxShared)));
        attr = true;
    }
    BD_CUDA(launch_pdl(mxd_kernel, dim3(p.grid), dim3(kMxdThreads), size_t(p.smem), stream, p, out));
    note_launch();
    BD_CUDA(cudaGetLastError());
}

}  // namespace bd
