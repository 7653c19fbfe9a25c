// K23 — the multi-tenant linear in ONE persistent tensor-core kernel:
//
//   P[b][m] = sum_k W[m][k] x_b[k]                                (tcgen05 kind::f16)
//           + alpha_t(b) * sum_k s_t(b)[m][k] x_b[k]              (tcgen05 kind::mxf4)
//
// i.e. the shared base contraction (matmul_nt, P:src/matrix.cpp:26-41, via
// ServingPool::backbone_linear_nt, P:src/serve.cpp:120-127) and every tenant's
// 1-bit delta (apply_delta_correction -> packed_signed_accumulate,
// P:src/serve.cpp:19-36 / P:src/delta.cpp:80-103), each byte of the backbone
// and of every tenant's plane read from HBM exactly once per launch.
//
// Sign planes on the tensor cores. A 32-bit word of the reference layout
// (flat row-major, LSB first, 1 = +1) becomes four registers of packed FP4
// (e2m1) +-1.0 with one shift and one LOP3 each:
//     reg_c = ((w << (3 - c)) & 0x88888888) ^ 0xAAAAAAAA      (c = 0..3)
// (bit 4i+c of w -> nibble i: 0x2 = +1.0, 0xA = -1.0). The registers are
// written to TMEM as the A operand of tcgen05.mma kind::mxf4 (A in TMEM, M =
// 128 plane rows = 128 TMEM lanes). The K order inside each 32-column chunk
// is permuted (TMEM element 8c+i <-> column 4i+c) and the activation operand
// is stored with the same permutation, so the product is unchanged.
//
// Activations in FP4. Each request's bf16 row is split (xp_prep_kernel) into
// 8 FP4 "pieces" per 32-column block with a per-(piece, block) power-of-two
// ue8m0 block scale: piece p of block u has scale 2^(E_u - 3p), E_u =
// ceil(log2 max|x_u|) - 2, and magnitudes in {0,.5,1,1.5,2,3,4}; every piece
// removes 3 bits of the residual, so 8 pieces represent x to 2^-24 of its
// block maximum (bf16's 8-bit significands exactly, except far below the
// block maximum). The pieces are the MMA's N rows (N = 8 per request): the
// hardware applies the block scales and accumulates in f32, and the epilogue
// sums the 8 piece columns and applies alpha.
//
// Work = a flat sequence of 16 KB "stages" per 128-row tile: K/64 backbone
// stages (W [128 x 64] bf16) then, per tenant slot, ceil(K/1024) plane stages
// ([128 rows x 1024 bits]). The grid is persistent (one CTA per SM) and CTA c
// owns a contiguous range of the sequence, so every SM streams the same number
// of HBM bytes. A tile's output is written as split partials P[split][b][m]
// (split = rank of the CTA among those covering the tile; the tile's last CTA
// zero-fills unused splits): bit-reproducible and independent of request order.
//
// Warp roles (384 threads): w0 TMA producer, w1 MMA issuer, w2 TMEM owner,
// w4-7 plane expanders (thread = tile row = TMEM lane), w8-11 epilogue.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace bd {

void note_launch();

namespace {

constexpr int kThreads = 384;
constexpr int kMaxStages = 12;
constexpr int kStageMain = 16384;     // W box or plane box
constexpr int kPlaneCols = 1024;      // plane columns per stage (128 B per row)
constexpr int kBaseCols = 64;         // backbone columns per stage
constexpr int kRing = 2;              // TMEM A-operand entries (one plane stage each)
// TMEM columns
constexpr uint32_t kColBase = 0;      // base accumulator (bn <= 64)
constexpr uint32_t kColAcc = 64;      // 2 x 32 slot accumulators
constexpr uint32_t kColSfa = 128;     // A block scales (constant 1.0)
constexpr uint32_t kColRing = 136;    // entries: 16 B-scale columns + 128 A columns
constexpr uint32_t kEntryCols = 144;  // (scale-factor TMEM addresses must be even columns)

struct Layout {
    uint32_t aux_off, xs_off, stage, ys_off, bar_off, total;
};

__host__ __device__ inline Layout mt4_layout(int bn, int nr_max, int stages) {
    Layout L;
    L.aux_off = kStageMain;
    const uint32_t aux = uint32_t(std::max(4 * nr_max * 1024, bn * 128));
    L.xs_off = L.aux_off + aux;
    L.stage = (L.xs_off + nr_max * 256 + 1023) & ~1023u;
    L.ys_off = stages * L.stage;
    L.bar_off = L.ys_off + bn * 128 * 4;
    L.total = 1024 + L.bar_off + 512;
    return L;
}

__device__ __forceinline__ void mma_mxf4_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc,
                                            uint32_t sfa, uint32_t sfb, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%4], [%5], p;\n\t}" ::"r"(d),
        "r"(a), "l"(bdesc), "r"(idesc), "r"(sfa), "r"(sfb), "r"(acc)
        : "memory");
}

// kind::mxf4 instruction descriptor: A = B = E2M1 (1), scale type UE8M0, K = 64
__host__ __device__ constexpr uint32_t idesc_mxf4(uint32_t M, uint32_t N) {
    return (1u << 7) | (1u << 10) | ((N >> 3) << 17) | (1u << 23) | ((M >> 4) << 24);
}

struct Stage {
    int tile, r, kind, slot, chunk;  // kind 0 = backbone, 1 = plane
};

__device__ __forceinline__ Stage decode(const Mt4Params& p, long long g) {
    Stage s;
    s.tile = static_cast<int>(g / p.stages_per_tile);
    s.r = static_cast<int>(g - static_cast<long long>(s.tile) * p.stages_per_tile);
    if (s.r < p.kb_base) {
        s.kind = 0;
        s.slot = 0;
        s.chunk = s.r;
    } else {
        const int q = s.r - p.kb_base;
        s.kind = 1;
        s.slot = q / p.kc_plane;
        s.chunk = q - s.slot * p.kc_plane;
    }
    return s;
}

__device__ __forceinline__ int cta_of(long long s, long long total, int grid) {
    return static_cast<int>(((s + 1) * grid + total - 1) / total) - 1;
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}

__device__ __forceinline__ uint32_t expand4(uint32_t w, int c) {
    return ((w << (3 - c)) & 0x88888888u) ^ 0xAAAAAAAAu;
}

__global__ void __launch_bounds__(kThreads, 1) mt4_kernel(const __grid_constant__ Mt4Params p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    const Layout L = mt4_layout(p.bn, p.nr_max, p.stages);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bar_off);
    uint64_t* empty = full + kMaxStages;
    uint64_t* a_full = empty + kMaxStages;
    uint64_t* a_empty = a_full + kRing;
    uint64_t* acc_full = a_empty + kRing;
    uint64_t* acc_empty = acc_full + 2;
    uint64_t* base_full = acc_empty + 2;
    uint64_t* base_empty = base_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(base_empty + 1);
    float* ys = reinterpret_cast<float*>(smem + L.ys_off);

    const uint32_t warp = warp_id(), lane = lane_id();
    const long long total = p.total_stages;
    const long long g0 = total * blockIdx.x / gridDim.x;
    const long long g1 = total * (blockIdx.x + 1) / gridDim.x;

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&p.map_w);
        prefetch_tmap(&p.map_x);
        prefetch_tmap(&p.map_xp);
        prefetch_tmap(&p.map_xs);
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1 + 128);  // MMA commit + every expander thread
        }
        for (int e = 0; e < kRing; ++e) {
            mbar_init(&a_full[e], 128);
            mbar_init(&a_empty[e], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 128);
        }
        mbar_init(base_full, 1);
        mbar_init(base_empty, 128);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---- TMA producer ----
            const uint64_t pol_stream = policy_evict_first();
            const uint64_t pol_keep = policy_evict_last();
            int i = 0;
            for (long long g = g0; g < g1; ++g, ++i) {
                const Stage st = decode(p, g);
                const int s = i % p.stages;
                mbar_wait(&empty[s], ((i / p.stages) & 1) ^ 1);
                uint8_t* sp = smem + s * L.stage;
                const int m0 = st.tile * 128;
                if (st.kind == 0) {
                    mbar_arrive_expect_tx(&full[s], kStageMain + p.bn * 128);
                    const int kc = st.chunk * kBaseCols;
                    tma_load_2d_hint(sp, &p.map_w, &full[s], kc, m0, pol_stream);
                    tma_load_2d_hint(sp + L.aux_off, &p.map_x, &full[s], kc, 0, pol_keep);
                } else {
                    const Mt4Slot& sl = p.slots[st.slot];
                    int sub = 0;
                    while (sub + 1 < p.n_subs && m0 >= p.sub_row0[sub + 1]) ++sub;
                    mbar_arrive_expect_tx(&full[s], kStageMain + sl.n_req * (4 * 1024 + 256));
                    tma_load_2d_hint(sp, &p.bits_maps[sl.map_idx[sub]], &full[s], st.chunk * 128,
                                     m0 - p.sub_row0[sub], pol_stream);
                    for (int q = 0; q < sl.n_req; ++q) {
                        const int row = 8 * sl.req[q];
#pragma unroll
                        for (int t = 0; t < 4; ++t)
                            tma_load_2d_hint(sp + L.aux_off + (t * p.nr_max + q) * 1024, &p.map_xp, &full[s],
                                             st.chunk * 512 + t * 128, row, pol_keep);
                        tma_load_2d_hint(sp + L.xs_off + q * 256, &p.map_xs, &full[s], st.chunk * 32, row,
                                         pol_keep);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---- MMA issuer ----
            const uint32_t id_base = idesc_bf16_f32(128, p.bn);
            int i = 0, pe = 0, n_slot = 0, n_base = 0;
            for (long long g = g0; g < g1; ++g, ++i) {
                const Stage st = decode(p, g);
                const int s = i % p.stages;
                mbar_wait(&full[s], (i / p.stages) & 1);
                tc_fence_after();
                uint8_t* sp = smem + s * L.stage;
                if (st.kind == 0) {
                    const bool first = st.chunk == 0 || g == g0;
                    const bool last = st.chunk == p.kb_base - 1 || g == g1 - 1;
                    if (first) {
                        mbar_wait(base_empty, (n_base & 1) ^ 1);
                        tc_fence_after();
                    }
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint64_t da = sdesc_k128(sp) + 2 * k;
                        const uint64_t db = sdesc_k128(sp + L.aux_off) + 2 * k;
                        mma_bf16_ss(tbase + kColBase, da, db, id_base, (first && k == 0) ? 0u : 1u);
                    }
                    tc_commit(&empty[s]);
                    if (last) {
                        tc_commit(base_full);
                        ++n_base;
                    }
                } else {
                    const Mt4Slot& sl = p.slots[st.slot];
                    const bool first = st.chunk == 0 || g == g0;
                    const bool last = st.chunk == p.kc_plane - 1 || g == g1 - 1;
                    const int buf = n_slot & 1;
                    const int e = pe % kRing;
                    mbar_wait(&a_full[e], (pe / kRing) & 1);
                    if (first) mbar_wait(&acc_empty[buf], ((n_slot >> 1) & 1) ^ 1);
                    tc_fence_after();
                    const uint32_t idesc = idesc_mxf4(128, 8 * sl.n_req);
                    const uint32_t ent = tbase + kColRing + e * kEntryCols;
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        const uint64_t db = sdesc_k128(sp + L.aux_off + (k >> 2) * p.nr_max * 1024) + 2 * (k & 3);
                        mma_mxf4_ts(tbase + kColAcc + 32 * buf, ent + 16 + 8 * k, db,
                                    idesc | (uint32_t(2 * (k & 1)) << 4), tbase + kColSfa, ent + 2 * (k >> 1),
                                    (first && k == 0) ? 0u : 1u);
                    }
                    tc_commit(&a_empty[e]);
                    tc_commit(&empty[s]);
                    ++pe;
                    if (last) {
                        tc_commit(&acc_full[buf]);
                        ++n_slot;
                    }
                }
            }
        }
    } else if (warp >= 4 && warp < 8) {
        // ---- plane expanders: thread = tile row = TMEM lane ----
        const uint32_t q4 = warp - 4;
        const uint32_t trow = q4 * 32 + lane;
        const uint32_t lane_base = (q4 * 32) << 16;
        {   // constant A block scales (1.0)
            uint32_t one[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) one[j] = 0x7F7F7F7Fu;
            tmem_st8(tbase + lane_base + kColSfa, one);
            tmem_st_wait();
        }
        int i = 0, pe = 0;
        for (long long g = g0; g < g1; ++g, ++i) {
            const Stage st = decode(p, g);
            const int s = i % p.stages;
            mbar_wait(&full[s], (i / p.stages) & 1);
            if (st.kind == 1) {
                const Mt4Slot& sl = p.slots[st.slot];
                const uint8_t* sp = smem + s * L.stage;
                const int e = pe % kRing;
                mbar_wait(&a_empty[e], ((pe / kRing) & 1) ^ 1);
                const uint32_t ent = tbase + lane_base + kColRing + e * kEntryCols;
                // B block scales for this stage: lane l < N holds row l (32 bytes = 32 blocks),
                // in every lane quarter; word j (blocks 4j..4j+3, MMAs 2j and 2j+1) -> column 2j
                {
                    uint32_t sc[8];
                    if (lane < uint32_t(8 * sl.n_req)) {
                        const uint4 v0 = *reinterpret_cast<const uint4*>(sp + L.xs_off + lane * 32);
                        const uint4 v1 = *reinterpret_cast<const uint4*>(sp + L.xs_off + lane * 32 + 16);
                        sc[0] = v0.x; sc[1] = v0.y; sc[2] = v0.z; sc[3] = v0.w;
                        sc[4] = v1.x; sc[5] = v1.y; sc[6] = v1.z; sc[7] = v1.w;
                    } else {
#pragma unroll
                        for (int j = 0; j < 8; ++j) sc[j] = 0x7F7F7F7Fu;
                    }
                    uint32_t sc2[16];
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        sc2[2 * j] = sc[j];
                        sc2[2 * j + 1] = 0x7F7F7F7Fu;
                    }
                    tmem_st16(ent, sc2);
                }
                const uint8_t* rowp = sp + trow * 128;
                const uint32_t sw = trow & 7;
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const uint4 v0 = *reinterpret_cast<const uint4*>(rowp + (((2 * h) ^ sw) << 4));
                    const uint4 v1 = *reinterpret_cast<const uint4*>(rowp + (((2 * h + 1) ^ sw) << 4));
                    const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
                    uint32_t a[32];
#pragma unroll
                    for (int u = 0; u < 8; ++u)
#pragma unroll
                        for (int c = 0; c < 4; ++c) a[4 * u + c] = expand4(w[u], c);
                    tmem_st32(ent + 16 + 32 * h, a);
                }
                tmem_st_wait();
                tc_fence_before();
                mbar_arrive(&a_full[e]);
                ++pe;
            }
            mbar_arrive(&empty[s]);
        }
    } else if (warp >= 8) {
        // ---- epilogue: thread = tile row ----
        const uint32_t q4 = warp - 8;
        const uint32_t trow = q4 * 32 + lane;
        const uint32_t lane_base = (q4 * 32) << 16;
        for (int b = 0; b < p.batch; ++b) ys[b * 128 + trow] = 0.0f;
        int n_slot = 0, n_base = 0;
        for (long long g = g0; g < g1; ++g) {
            const Stage st = decode(p, g);
            const int m0 = st.tile * 128;
            if (st.kind == 0 && (st.chunk == p.kb_base - 1 || g == g1 - 1)) {
                mbar_wait(base_full, n_base & 1);
                tc_fence_after();
                for (int c0 = 0; c0 < p.batch; c0 += 16) {
                    uint32_t v[16];
                    tmem_ld16(tbase + lane_base + kColBase + c0, v);
                    tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (c0 + j < p.batch) ys[(c0 + j) * 128 + trow] += __uint_as_float(v[j]);
                }
                tc_fence_before();
                mbar_arrive(base_empty);
                ++n_base;
            }
            if (st.kind == 1 && (st.chunk == p.kc_plane - 1 || g == g1 - 1)) {
                const Mt4Slot& sl = p.slots[st.slot];
                int sub = 0;
                while (sub + 1 < p.n_subs && m0 >= p.sub_row0[sub + 1]) ++sub;
                const float alpha = sl.alpha[sub];
                const int buf = n_slot & 1;
                mbar_wait(&acc_full[buf], (n_slot >> 1) & 1);
                tc_fence_after();
                for (int q = 0; q < sl.n_req; ++q) {
                    uint32_t v[8];
                    tmem_ld8(tbase + lane_base + kColAcc + 32 * buf + 8 * q, v);
                    tmem_ld_wait();
                    const float sum = ((__uint_as_float(v[0]) + __uint_as_float(v[1])) +
                                       (__uint_as_float(v[2]) + __uint_as_float(v[3]))) +
                                      ((__uint_as_float(v[4]) + __uint_as_float(v[5])) +
                                       (__uint_as_float(v[6]) + __uint_as_float(v[7])));
                    ys[sl.req[q] * 128 + trow] += alpha * sum;
                }
                tc_fence_before();
                mbar_arrive(&acc_empty[buf]);
                ++n_slot;
            }
            if (st.r == p.stages_per_tile - 1 || g == g1 - 1) {
                const long long first_stage = static_cast<long long>(st.tile) * p.stages_per_tile;
                const int split = static_cast<int>(blockIdx.x) - cta_of(first_stage, total, gridDim.x);
                const size_t pstride = static_cast<size_t>(p.batch) * p.M;
                float* out = p.partial + split * pstride + m0 + trow;
                for (int b = 0; b < p.batch; ++b) {
                    out[static_cast<size_t>(b) * p.M] = ys[b * 128 + trow];
                    ys[b * 128 + trow] = 0.0f;
                }
                if (st.r == p.stages_per_tile - 1)
                    for (int s2 = split + 1; s2 < p.splits; ++s2)
                        for (int b = 0; b < p.batch; ++b)
                            p.partial[s2 * pstride + static_cast<size_t>(b) * p.M + m0 + trow] = 0.0f;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) tmem_dealloc<512>(tbase);
}

// FP4 pieces of the activations: grid (K_pad/256, batch), 8 warps, warp = one
// 32-column block. Xp row 8b+p = piece p of request b (packed e2m1, K permuted
// inside each 32-column chunk: element 8c+i <-> column 4i+c); Xs row 8b+p =
// ue8m0 block scales (one byte per 32 columns).
__device__ __forceinline__ uint32_t e2m1_code(float a) {  // a in [0, 4]: nearest of {0,.5,1,1.5,2,3,4}
    if (a < 2.0f) return static_cast<uint32_t>(rintf(a * 2.0f));           // 0..4 -> codes 0..4
    return static_cast<uint32_t>(rintf(a)) + 2u;                           // 2,3,4 -> codes 4,5,6
}
__device__ __forceinline__ float e2m1_value(uint32_t c) {
    return c < 4 ? 0.5f * c : static_cast<float>(c - 2);
}

__global__ void __launch_bounds__(256) xp_prep_kernel(const uint16_t* __restrict__ X, int ldx, int K,
                                                       uint8_t* __restrict__ Xp, int ldxp,
                                                       uint8_t* __restrict__ Xs, int ldxs) {
    __shared__ uint32_t nib[8][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.y;
    const int u = blockIdx.x * 8 + warp;  // 32-column block
    const int col = 32 * u + lane;
    const float x = col < K ? bf16_to_f32(X[static_cast<size_t>(b) * ldx + col]) : 0.0f;
    float amax = fabsf(x);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    int E = -127;
    if (amax > 0.0f) {
        int e;
        frexpf(amax, &e);  // amax <= 2^e
        E = e - 2;         // amax / 2^E <= 4
    }
    uint32_t packed = 0;
    double r = x;
    uint32_t sbyte[8];
#pragma unroll
    for (int pc = 0; pc < 8; ++pc) {
        const int s = E - 3 * pc;
        uint32_t code = 0;
        if (amax > 0.0f && s >= -127) {
            const double v = ldexp(r, -s);
            code = e2m1_code(static_cast<float>(fabs(v)));
            const double qv = (v < 0 ? -1.0 : 1.0) * e2m1_value(code);
            r -= ldexp(qv, s);
            if (v < 0 && code) code |= 8u;
        }
        packed |= code << (4 * pc);
        sbyte[pc] = static_cast<uint32_t>(s >= -127 ? s + 127 : 0);
    }
    nib[warp][lane] = packed;
    __syncwarp();
    // lane L -> piece p = L/4, word c = L%4: nibble t of the word = column c + 4t
    const int pc = lane >> 2, c = lane & 3;
    uint32_t word = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) word |= ((nib[warp][c + 4 * t] >> (4 * pc)) & 0xFu) << (4 * t);
    const size_t row = static_cast<size_t>(8 * b + pc);
    *reinterpret_cast<uint32_t*>(Xp + row * ldxp + 16 * u + 4 * c) = word;
    if (lane < 8) Xs[static_cast<size_t>(8 * b + lane) * ldxs + u] = static_cast<uint8_t>(sbyte[lane]);
}

}  // namespace

bool plan_mt4(Mt4Params& p, uint64_t M, uint64_t K, int batch) {
    p.M = int(M);
    p.K = int(K);
    p.batch = batch;
    p.bn = std::max(16, ((batch + 15) / 16) * 16);
    if (p.bn > 64 || p.n_slots < 1 || p.n_slots > kMt4MaxSlots || M % 128 || K % 128) return false;
    p.nr_max = 1;
    for (int j = 0; j < p.n_slots; ++j) {
        if (p.slots[j].n_req < 1 || p.slots[j].n_req > kMt4MaxReq) return false;
        p.nr_max = std::max(p.nr_max, p.slots[j].n_req);
    }
    for (int s = 0; s < p.n_subs; ++s)
        if ((p.sub_row0[s + 1] - p.sub_row0[s]) % 128) return false;
    p.kb_base = int(K / kBaseCols);
    p.kc_plane = int((K + kPlaneCols - 1) / kPlaneCols);
    p.stages_per_tile = p.kb_base + p.n_slots * p.kc_plane;
    const int m_tiles = int(M / 128);
    p.total_stages = static_cast<long long>(m_tiles) * p.stages_per_tile;
    p.grid = int(std::min<long long>(kNumSMs, p.total_stages));
    int stages = kMaxStages;
    while (stages > 2 && mt4_layout(p.bn, p.nr_max, stages).total > 227 * 1024) --stages;
    if (mt4_layout(p.bn, p.nr_max, stages).total > 227 * 1024) return false;
    p.stages = stages;
    p.smem = int(mt4_layout(p.bn, p.nr_max, stages).total);
    // splits = most CTAs covering one tile
    auto cta_of_h = [&](long long s) {
        return int(((s + 1) * p.grid + p.total_stages - 1) / p.total_stages) - 1;
    };
    int splits = 1;
    for (int t = 0; t < m_tiles; ++t) {
        const long long a = static_cast<long long>(t) * p.stages_per_tile;
        splits = std::max(splits, cta_of_h(a + p.stages_per_tile - 1) - cta_of_h(a) + 1);
    }
    p.splits = splits;
    return true;
}

void mt4_launch(const Mt4Params& p, cudaStream_t stream) {
    static bool attr = false;
    if (!attr) {
        BD_CUDA(cudaFuncSetAttribute(mt4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        attr = true;
    }
    mt4_kernel<<<p.grid, kThreads, p.smem, stream>>>(p);
    note_launch();
    BD_CUDA(cudaGetLastError());
}

int xp_k_pad(int K) { return ((K + kPlaneCols - 1) / kPlaneCols) * kPlaneCols; }

void xp_prep_launch(const void* X, int ldx, int K, int batch, uint8_t* Xp, int ldxp, uint8_t* Xs, int ldxs,
                    cudaStream_t stream) {
    const int kpad = xp_k_pad(K);
    xp_prep_kernel<<<dim3(kpad / 256, batch), 256, 0, stream>>>(static_cast<const uint16_t*>(X), ldx, K, Xp, ldxp,
                                                               Xs, ldxs);
    note_launch();
    BD_CUDA(cudaGetLastError());
}

CUtensorMap tmap_bits4(const uint8_t* bits, uint64_t rows, uint64_t cols) {
    return make_tmap_2d(bits, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, rows, cols / 8, cols / 8, 128, 128, true);
}
CUtensorMap tmap_xp(const uint8_t* Xp, int rows, int ldxp) {
    return make_tmap_2d(Xp, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, uint64_t(rows), uint64_t(ldxp), uint64_t(ldxp), 8,
                        128, true);
}
CUtensorMap tmap_xs(const uint8_t* Xs, int rows, int ldxs) {
    return make_tmap_2d(Xs, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, uint64_t(rows), uint64_t(ldxs), uint64_t(ldxs), 8,
                        32, false);
}

}  // namespace bd
