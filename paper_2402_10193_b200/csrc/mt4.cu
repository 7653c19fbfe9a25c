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
// stages (W [128 x 64] bf16) spread evenly among the plane stages (per tenant
// slot, ceil(K/1024) stages of [128 rows x 1024 bits]). The grid is persistent (one CTA per SM) and CTA c
// owns a contiguous range of the sequence, so every SM streams the same number
// of HBM bytes. A tile's output is written as split partials P[split][b][m]
// (split = rank of the CTA among those covering the tile; the tile's last CTA
// zero-fills unused splits): bit-reproducible and independent of request order.
//
// Warp roles (512 threads): w0 TMA producer, w1 MMA issuer (whole warps, one
// elected lane issues), w2 TMEM owner, w4-7 and w8-11 plane expanders taking
// alternate plane stages (thread = tile row = TMEM lane), w12-15 epilogue.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace bd {

void note_launch();

namespace {

constexpr int kThreads = 544;  // 17 warps
constexpr int kMaxRingB = 12;        // smem stage ring for backbone stages
constexpr int kMaxRingP = 12;        // ... and for plane stages
constexpr int kStageMain = 16384;     // W box or plane box
constexpr int kPlaneCols = 1024;      // plane columns per stage (128 B per row)
constexpr int kBaseCols = 64;         // backbone columns per stage
constexpr int kMaxRing = 16;          // TMEM A-operand entries (a quarter plane stage, K = 256, each)
constexpr int kMaxAcc = 4;            // slot accumulators in flight
constexpr uint32_t kProducers = 3;  // ring slots >= producers (phase-parity safety)
constexpr int kMaxSched = 1024;       // stages per tile
// TMEM ring entry: B-scale columns 0 and 2 (scale-factor addresses must be even), A in 8..39
constexpr uint32_t kEntryCols = 40;
constexpr uint32_t kStageCols = 4 * kEntryCols;  // one plane stage = 4 sub-entries (K = 1024)

constexpr uint32_t kAuxReq = 5120;     // smem per request: kXpBlock padded to the 1024-B swizzle atom

struct Layout {
    uint32_t aux_off, bstage, pstage, pring_off, ys_off, sched_off, bar_off, total;
};

__host__ __device__ inline Layout mt4_layout(int bn, int nr_max, int ring_b, int ring_p) {
    Layout L;
    L.aux_off = kStageMain;
    L.bstage = (kStageMain + bn * 128 + 1023) & ~1023u;
    L.pstage = (kStageMain + kAuxReq * nr_max + 1023) & ~1023u;
    L.pring_off = ring_b * L.bstage;
    L.ys_off = L.pring_off + ring_p * L.pstage;
    L.sched_off = L.ys_off + bn * 128 * 4;
    L.bar_off = L.sched_off + kMaxSched * 4;
    L.total = 1024 + L.bar_off + 1024;
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

__device__ __forceinline__ int cta_of(long long s, long long total, int grid) {
    return static_cast<int>(((s + 1) * grid + total - 1) / total) - 1;
}

__device__ __forceinline__ uint64_t sdesc_sw128(const void* smem, uint32_t sbo) {
    const uint64_t addr = smem_u32(smem);
    return ((addr >> 4) & 0x3FFFull) | (1ull << 16) | (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) |
           (2ull << 61);
}

__device__ __forceinline__ void tmem_st4(uint32_t taddr, const uint32_t (&r)[4]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(r[0]), "r"(r[1]),
                 "r"(r[2]), "r"(r[3])
                 : "memory");
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


// Stage cursor over a per-tile schedule table (built on the host, kept in smem).
// Inside a tile the backbone stages are spread evenly among the plane stages
// (Bresenham: stage r is a backbone stage iff floor((r+1)KB/S) > floor(rKB/S)),
// so every stretch of the sequence mixes cheap backbone MMAs with the plane
// stages' expansion + FP4 MMAs and the HBM stream never waits on either.
// Entry: bit 0 backbone | 1-10 chunk | 11-17 slot | 18-24 distance to the
// previous stage of the same segment (0: first) | 25-31 to the next (0: last).
// first/last mark a segment's (tile backbone / one slot's plane) first/last
// stage inside this CTA's range [g0, g1).
struct Cursor {
    long long g, g0, g1;
    int tile, r;
    int chunk, slot;
    bool base, first, last, tile_last;
    __device__ __forceinline__ void compute(const Mt4Params& p, const uint32_t* sched) {
        const uint32_t e = sched[r];
        base = e & 1u;
        chunk = (e >> 1) & 1023u;
        slot = (e >> 11) & 127u;
        const int dp = (e >> 18) & 127u, dn = e >> 25;
        first = dp == 0 || g - dp < g0;
        last = dn == 0 || g + dn >= g1;
        tile_last = r == p.stages_per_tile - 1 || g == g1 - 1;
    }
    __device__ __forceinline__ void init(const Mt4Params& p, const uint32_t* sched, long long a, long long b) {
        g0 = a;
        g1 = b;
        g = a;
        tile = static_cast<int>(a / p.stages_per_tile);
        r = static_cast<int>(a - static_cast<long long>(tile) * p.stages_per_tile);
        compute(p, sched);
    }
    __device__ __forceinline__ void next(const Mt4Params& p, const uint32_t* sched) {
        ++g;
        if (++r == p.stages_per_tile) {
            r = 0;
            ++tile;
        }
        compute(p, sched);
    }
};

// ring position with its mbarrier phase
struct Ring {
    int i = 0;
    uint32_t ph = 0;
    __device__ __forceinline__ void next(int n) {
        if (++i == n) {
            i = 0;
            ph ^= 1;
        }
    }
};

__global__ void __launch_bounds__(kThreads, 1) mt4_kernel(const __grid_constant__ Mt4Params p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    const Layout L = mt4_layout(p.bn, p.nr_max, p.ring_b, p.ring_p);
    uint64_t* full_b = reinterpret_cast<uint64_t*>(smem + L.bar_off);
    uint64_t* empty_b = full_b + kMaxRingB;
    uint64_t* full_p = empty_b + kMaxRingB;
    uint64_t* empty_p = full_p + kMaxRingP;
    uint64_t* a_full = empty_p + kMaxRingP;
    uint64_t* a_empty = a_full + kMaxRing;
    uint64_t* acc_full = a_empty + kMaxRing;
    uint64_t* acc_empty = acc_full + kMaxAcc;
    uint64_t* base_full = acc_empty + kMaxAcc;
    uint64_t* base_empty = base_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(base_empty + 1);
    // fills issued so far per ring slot (backbone slots, then plane slots): a producer arms a
    // slot only after the slot's previous fill was issued, so no slot's barriers run a lap
    // ahead (with a plane ring as short as the producer count the empty-barrier parity
    // otherwise aliases: seen with 2-request slots on Llama-2-7B shapes)
    volatile uint32_t* slot_fills = tmem_slot + 1;
    float* ys = reinterpret_cast<float*>(smem + L.ys_off);
    uint32_t* sched = reinterpret_cast<uint32_t*>(smem + L.sched_off);
    for (int i = threadIdx.x; i < p.stages_per_tile; i += blockDim.x) sched[i] = p.sched[i];

    const uint32_t warp = warp_id(), lane = lane_id();
    const long long total = p.total_stages;
    const long long g0 = total * blockIdx.x / gridDim.x;
    const long long g1 = total * (blockIdx.x + 1) / gridDim.x;

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&p.map_w);
        prefetch_tmap(&p.map_x);
        for (int s = 0; s < p.ring_b; ++s) {
            mbar_init(&full_b[s], 1);
            mbar_init(&empty_b[s], 1);      // backbone MMA commit
        }
        for (int s = 0; s < p.ring_p; ++s) {
            mbar_init(&full_p[s], 1);
            mbar_init(&empty_p[s], 1 + 4);  // plane MMA commit + the expander group's 4 warps
        }
        for (int e = 0; e < p.n_ring; ++e) {
            mbar_init(&a_full[e], 4);  // one per expander warp of the group (lane 0 after __syncwarp)
            mbar_init(&a_empty[e], 1);
        }
        for (int b = 0; b < p.n_acc; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 4);
        }
        mbar_init(base_full, 1);
        mbar_init(base_empty, 4);
        for (int i = 0; i < kMaxRingB + kMaxRingP; ++i) slot_fills[i] = 0;
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;
    griddep_wait();  // PDL: activations come from the previous kernels

    if (warp == 0 || warp == 2 || warp == 3) {
        // ---- TMA producers: three warps take stages round-robin (the copies one
        // thread issues complete about one at a time, so independent issuers are
        // what keeps enough bytes in flight); one elected lane issues. Backbone
        // and plane stages cycle through separate smem rings. ----
        const uint32_t prod = warp == 0 ? 0 : warp - 1;
        const uint64_t pol_stream = policy_evict_first();
        const uint64_t pol_keep = policy_evict_last();
        Cursor c;
        c.init(p, sched, g0, g1);
        Ring rb, rp;
        uint32_t k = 0, nfill[2] = {0, 0};
        for (; c.g < g1; c.next(p, sched), k = (k == kProducers - 1) ? 0 : k + 1) {
            Ring& rr = c.base ? rb : rp;
            const int s = rr.i;
            const uint32_t ph = rr.ph;
            rr.next(c.base ? p.ring_b : p.ring_p);
            const int ri = c.base ? 0 : 1;
            const uint32_t lap = nfill[ri]++ / uint32_t(c.base ? p.ring_b : p.ring_p);
            const int si = (c.base ? 0 : kMaxRingB) + s;
            if (k != prod) continue;
            if (lane == 0) {
                // acquire: the previous fill of this slot (another producer warp) was issued
                uint32_t spins = 0;
                while (ld_acquire_cta(&slot_fills[si]) != lap)
                    if (++spins == (1u << 30)) __trap();  // schedule bug: fault instead of hanging
            }
            __syncwarp();
            const int m0 = c.tile * 128;
            if (c.base) {
                mbar_wait_w(&empty_b[s], ph ^ 1);
                uint8_t* sp = smem + s * L.bstage;
                mbar_arrive_expect_tx_w(&full_b[s], kStageMain + p.bn * 128);
                const int kc = c.chunk * kBaseCols;
                tma_load_2d_w(sp, &p.map_w, &full_b[s], kc, m0, pol_stream);
                tma_load_2d_w(sp + L.aux_off, &p.map_x, &full_b[s], kc, 0, pol_keep);
            } else {
                mbar_wait_w(&empty_p[s], ph ^ 1);
                uint8_t* sp = smem + L.pring_off + s * L.pstage;
                const Mt4Slot& sl = p.slots[c.slot];
                int sub = 0;
                while (sub + 1 < p.n_subs && m0 >= p.sub_row0[sub + 1]) ++sub;
                mbar_arrive_expect_tx_w(&full_p[s], kStageMain + sl.n_req * kXpBlock);
                tma_load_2d_w(sp, &p.bits_maps[sl.map_idx[sub]], &full_p[s], c.chunk * 128, m0 - p.sub_row0[sub],
                              pol_stream);
                for (int q = 0; q < sl.n_req; ++q)
                    bulk_load_w(sp + L.aux_off + q * kAuxReq,
                                p.xpk + (static_cast<size_t>(sl.req[q]) * p.n_chunks + c.chunk) * kXpBlock, kXpBlock,
                                &full_p[s], pol_keep);
            }
            __syncwarp();
            if (lane == 0) st_release_cta(&slot_fills[si], lap + 1);  // the slot's next fill may now be armed
        }
    } else if (warp == 16) {
        // ---- backbone MMA issuer (whole warp, one elected lane issues) ----
        const uint32_t id_base = idesc_bf16_f32(128, p.bn);
        Cursor c;
        c.init(p, sched, g0, g1);
        Ring rb;
        uint32_t base_ph = 0;
        for (; c.g < g1; c.next(p, sched)) {
            if (!c.base) continue;
            const int s = rb.i;
            mbar_wait_w(&full_b[s], rb.ph);
            tc_fence_after();
            uint8_t* sp = smem + s * L.bstage;
            if (c.first) {
                mbar_wait_w(base_empty, base_ph ^ 1);
                tc_fence_after();
            }
            const uint64_t da = sdesc_k128(sp), db = sdesc_k128(sp + L.aux_off);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
                mma_bf16_ss_w(tbase + p.col_base, da + 2 * kk, db + 2 * kk, id_base,
                              (c.first && kk == 0) ? 0u : 1u);
            tc_commit_w(&empty_b[s]);
            if (c.last) {
                tc_commit_w(base_full);
                base_ph ^= 1;
            }
            rb.next(p.ring_b);
        }
    } else if (warp == 1) {
        // ---- plane MMA issuer (FP4, A in TMEM) ----
        Cursor c;
        c.init(p, sched, g0, g1);
        Ring rp, ring, acc;
        for (; c.g < g1; c.next(p, sched)) {
            if (c.base) continue;
            const int s = rp.i;
            mbar_wait_w(&full_p[s], rp.ph);
            uint8_t* sp = smem + L.pring_off + s * L.pstage;
            const Mt4Slot& sl = p.slots[c.slot];
            if (c.first) mbar_wait_w(&acc_empty[acc.i], acc.ph ^ 1);
            const uint32_t idesc = idesc_mxf4(128, 8 * sl.n_req);
            const uint32_t d = tbase + p.col_acc + acc.i * p.acc_stride;
            // B = pieces: 8-row groups (requests) kAuxReq apart, sub-chunk j at +1024 j
            const uint64_t db = sdesc_sw128(sp + L.aux_off, kAuxReq);
            const uint32_t xstep = 1024u >> 4;  // descriptor units (16 B)
            mbar_wait_w(&a_full[ring.i], ring.ph);
            tc_fence_after();
            const uint32_t ent0 = tbase + p.col_ring + ring.i * kStageCols;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t ent = ent0 + j * kEntryCols;
                const uint64_t db0 = db + j * xstep;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    mma_mxf4_ts_w(d, ent + 8 + 8 * kk, db0 + 2 * kk, idesc | (uint32_t(2 * (kk & 1)) << 4),
                                  tbase + p.col_sfa, ent + 2 * (kk >> 1), (c.first && j == 0 && kk == 0) ? 0u : 1u);
            }
            tc_commit_w(&a_empty[ring.i]);
            ring.next(p.n_ring);
            tc_commit_w(&empty_p[s]);
            if (c.last) {
                tc_commit_w(&acc_full[acc.i]);
                acc.next(p.n_acc);
            }
            rp.next(p.ring_p);
        }
    } else if (warp >= 4 && warp < 12) {
        // ---- plane expanders: two groups of 4 warps take alternate plane stages;
        // thread = tile row = TMEM lane ----
        const uint32_t grp = (warp - 4) >> 2;
        const uint32_t q4 = warp & 3;
        const uint32_t trow = q4 * 32 + lane;
        const uint32_t lane_base = (q4 * 32) << 16;
        if (grp == 0) {  // constant A block scales (1.0)
            uint32_t one[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) one[j] = 0x7F7F7F7Fu;
            tmem_st8(tbase + lane_base + p.col_sfa, one);
            tmem_st_wait();
        }
        Cursor c;
        c.init(p, sched, g0, g1);
        Ring rp, ring;
        uint32_t n_plane = 0;
        const uint32_t sw = trow & 7;
        for (; c.g < g1; c.next(p, sched)) {
            if (c.base) continue;
            // every plane stage's full barrier is observed (also the other group's):
            // a group may then never run a ring lap ahead of the producers, which
            // would alias the mbarrier phase parity
            const int s = rp.i;
            mbar_wait(&full_p[s], rp.ph);
            rp.next(p.ring_p);
            const uint32_t mine = (n_plane++ & 1) == grp;
            if (!mine) {
                ring.next(p.n_ring);
                continue;
            }
            const Mt4Slot& sl = p.slots[c.slot];
            const uint8_t* sp = smem + L.pring_off + s * L.pstage;
            const uint8_t* rowp = sp + trow * 128;
            const bool has_scale = lane < uint32_t(8 * sl.n_req);
            mbar_wait(&a_empty[ring.i], ring.ph ^ 1);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t ent = tbase + lane_base + p.col_ring + ring.i * kStageCols + j * kEntryCols;
                // B block scales of MMAs 4j..4j+3 (blocks 8j..8j+7): lane l < N = row l, every quarter
                uint32_t sc[4] = {0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu, 0x7F7F7F7Fu};
                if (has_scale) {
                    const uint2 v = *reinterpret_cast<const uint2*>(sp + L.aux_off + (lane >> 3) * kAuxReq + 4096 +
                                                                    (lane & 7) * 32 + 8 * j);
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
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&a_full[ring.i]);
                mbar_arrive(&empty_p[s]);
            }
            ring.next(p.n_ring);
        }
    } else if (warp >= 12 && warp < 16) {
        // ---- epilogue: thread = tile row ----
        const uint32_t q4 = warp - 12;
        const uint32_t trow = q4 * 32 + lane;
        const uint32_t lane_base = (q4 * 32) << 16;
        for (int b = 0; b < p.batch; ++b) ys[b * 128 + trow] = 0.0f;
        Cursor c;
        c.init(p, sched, g0, g1);
        Ring acc;
        uint32_t base_ph = 0;
        for (; c.g < g1; c.next(p, sched)) {
            const int m0 = c.tile * 128;
            if (c.base && c.last) {
                mbar_wait(base_full, base_ph);
                base_ph ^= 1;
                tc_fence_after();
                for (int c0 = 0; c0 < p.batch; c0 += 16) {
                    uint32_t v[16];
                    tmem_ld16(tbase + lane_base + p.col_base + c0, v);
                    tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (c0 + j < p.batch) ys[(c0 + j) * 128 + trow] += __uint_as_float(v[j]);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(base_empty);
            }
            if (!c.base && c.last) {
                const Mt4Slot& sl = p.slots[c.slot];
                int sub = 0;
                while (sub + 1 < p.n_subs && m0 >= p.sub_row0[sub + 1]) ++sub;
                const float alpha = sl.alpha[sub];
                mbar_wait(&acc_full[acc.i], acc.ph);
                tc_fence_after();
                for (int q = 0; q < sl.n_req; ++q) {
                    uint32_t v[8];
                    tmem_ld8(tbase + lane_base + p.col_acc + acc.i * p.acc_stride + 8 * q, v);
                    tmem_ld_wait();
                    const float sum = ((__uint_as_float(v[0]) + __uint_as_float(v[1])) +
                                       (__uint_as_float(v[2]) + __uint_as_float(v[3]))) +
                                      ((__uint_as_float(v[4]) + __uint_as_float(v[5])) +
                                       (__uint_as_float(v[6]) + __uint_as_float(v[7])));
                    ys[sl.req[q] * 128 + trow] += alpha * sum;
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&acc_empty[acc.i]);
                acc.next(p.n_acc);
            }
            if (c.tile_last) {
                const long long first_stage = static_cast<long long>(c.tile) * p.stages_per_tile;
                const int split = static_cast<int>(blockIdx.x) - cta_of(first_stage, total, gridDim.x);
                const size_t pstride = static_cast<size_t>(p.batch) * p.M;
                float* out = p.partial + split * pstride + m0 + trow;
                for (int b = 0; b < p.batch; ++b) {
                    out[static_cast<size_t>(b) * p.M] = ys[b * 128 + trow];
                    ys[b * 128 + trow] = 0.0f;
                }
                if (c.r == p.stages_per_tile - 1)
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

// FP4 pieces of the activations: grid (chunks * 4, batch), 8 warps, warp = one
// 32-column block u. Output block of (request b, 1024-column chunk c), kXpBlock
// bytes: sub-chunk t (256 columns) at t*1024: row p = piece p (128 B, 16-byte
// groups swizzled by p as TMA SWIZZLE_128B would), element order inside each
// 32-column block permuted (element 8c+i <-> column 4i+c); then at 4096 the
// ue8m0 scales, row p = 32 bytes (one per 32-column block of the chunk).
__device__ __forceinline__ uint32_t e2m1_code(float a) {  // a in [0, 4]: nearest of {0,.5,1,1.5,2,3,4}
    if (a < 2.0f) return static_cast<uint32_t>(rintf(a * 2.0f));           // 0..4 -> codes 0..4
    return static_cast<uint32_t>(rintf(a)) + 2u;                           // 2,3,4 -> codes 4,5,6
}
__device__ __forceinline__ float e2m1_value(uint32_t c) {
    return c < 4 ? 0.5f * c : static_cast<float>(c - 2);
}

// v * 2^k, exact (a multiply by a constructed power of two in the normal exponent range)
__device__ __forceinline__ float mul_pow2(float v, int k) {
    if (k >= -126 && k <= 127) return v * __int_as_float((k + 127) << 23);
    return ldexpf(v, k);
}

__global__ void __launch_bounds__(256) xp_prep_kernel(const uint16_t* __restrict__ X, int ldx, int K, int n_chunks,
                                                       uint8_t* __restrict__ xpk) {
    __shared__ uint32_t nib[8][32];
    griddep_wait();
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
    // f32 is exact here: x is bf16 (8 significant bits), every piece value has <= 2 and the
    // scalings are powers of two, so r keeps <= 8 significant bits (no rounding anywhere)
    uint32_t packed = 0;
    float r = x;
    uint32_t sbyte[8];
#pragma unroll
    for (int pc = 0; pc < 8; ++pc) {
        const int s = E - 3 * pc;
        uint32_t code = 0;
        if (amax > 0.0f && s >= -127) {
            const float v = mul_pow2(r, -s);
            code = e2m1_code(fabsf(v));
            const float qv = v < 0.0f ? -e2m1_value(code) : e2m1_value(code);
            r -= mul_pow2(qv, s);
            if (v < 0.0f && code) code |= 8u;
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
    const int chunk = u >> 5, sub = (u >> 3) & 3, w16 = u & 7;
    uint8_t* blk = xpk + (static_cast<size_t>(b) * n_chunks + chunk) * kXpBlock;
    *reinterpret_cast<uint32_t*>(blk + sub * 1024 + pc * 128 + ((w16 ^ pc) << 4) + 4 * c) = word;
    if (lane < 8) blk[4096 + lane * 32 + (u & 31)] = static_cast<uint8_t>(sbyte[lane]);
}

}  // namespace

std::vector<uint32_t> mt4_schedule(const Mt4Params& p) {
    const int S = p.stages_per_tile, KB = p.kb_base;
    std::vector<uint32_t> e(S);
    std::vector<int> seg(S), chunk(S);
    for (int r = 0; r < S; ++r) {
        const int b_r = int((int64_t(r) * KB) / S);
        const bool base = (int64_t(r + 1) * KB) / S > b_r;
        int slot = 0, ch = b_r;
        if (!base) {
            const int pidx = r - b_r;
            slot = pidx / p.kc_plane;
            ch = pidx - slot * p.kc_plane;
        }
        seg[r] = base ? -1 : slot;
        chunk[r] = ch;
        e[r] = uint32_t(base) | (uint32_t(ch) << 1) | (uint32_t(slot) << 11);
    }
    std::vector<int> last_of(p.n_slots + 1, -1);  // last stage seen per segment (index 0 = backbone)
    for (int r = 0; r < S; ++r) {
        int& prev = last_of[seg[r] + 1];
        if (prev >= 0) {
            const uint32_t d = uint32_t(r - prev);
            e[r] |= d << 18;
            e[prev] |= d << 25;
        }
        prev = r;
    }
    return e;
}

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
    p.n_chunks = xp_chunks(int(K));
    p.stages_per_tile = p.kb_base + p.n_slots * p.kc_plane;
    if (p.stages_per_tile > kMaxSched || p.n_slots > 127 || p.kb_base > 1023) return false;
    {   // schedule distances must fit the 7-bit fields
        const std::vector<uint32_t> e = mt4_schedule(p);
        for (int r = 0; r < p.stages_per_tile; ++r) {
            const int base = e[r] & 1, ch = (e[r] >> 1) & 1023;
            const int n_seg = base ? p.kb_base : p.kc_plane;
            if ((ch > 0 && ((e[r] >> 18) & 127) == 0) || (ch < n_seg - 1 && (e[r] >> 25) == 0)) return false;
        }
    }
    const int m_tiles = int(M / 128);
    p.total_stages = static_cast<long long>(m_tiles) * p.stages_per_tile;
    p.grid = int(std::min<long long>(kNumSMs, p.total_stages));
    // smem rings: split the stage budget between backbone and plane stages in
    // proportion to their share of the schedule, at least kProducers each
    const double fb = double(p.kb_base) / p.stages_per_tile;
    int rb = 0, rp = 0;
    for (int n = kMaxRingB + kMaxRingP; n >= 2 * int(kProducers); --n) {
        rb = std::min(kMaxRingB, std::max(int(kProducers), int(std::lround(n * fb))));
        rp = std::min(kMaxRingP, std::max(int(kProducers), n - rb));
        if (mt4_layout(p.bn, p.nr_max, rb, rp).total <= 227 * 1024) break;
    }
    if (mt4_layout(p.bn, p.nr_max, rb, rp).total > 227 * 1024) return false;
    // TMEM: base accumulator | n_acc slot accumulators | A scales (1.0) | ring of entries
    const int n_max = 8 * p.nr_max;
    p.col_base = 0;
    p.col_acc = (p.bn + 7) & ~7;
    p.acc_stride = n_max;
    p.n_acc = n_max <= 16 ? kMaxAcc : 2;
    p.col_sfa = (p.col_acc + p.n_acc * p.acc_stride + 7) & ~7;
    p.col_ring = p.col_sfa + 8;
    p.n_ring = std::min(kMaxRing, int((512 - p.col_ring) / kStageCols));
    if (p.n_ring < 2) return false;
    p.ring_b = rb;
    p.ring_p = rp;
    p.smem = int(mt4_layout(p.bn, p.nr_max, rb, rp).total);
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
    BD_CUDA(launch_pdl(mt4_kernel, dim3(p.grid), dim3(kThreads), size_t(p.smem), stream, p));
    note_launch();
    BD_CUDA(cudaGetLastError());
}

void xp_prep_launch(const void* X, int ldx, int K, int batch, uint8_t* xpk, cudaStream_t stream) {
    const int n_chunks = xp_chunks(K);
    BD_CUDA(launch_pdl(xp_prep_kernel, dim3(n_chunks * 4, batch), dim3(256), 0, stream,
                       static_cast<const uint16_t*>(X), ldx, K, n_chunks, xpk));
    note_launch();
    BD_CUDA(cudaGetLastError());
}

CUtensorMap tmap_bits4(const uint8_t* bits, uint64_t rows, uint64_t cols) {
    return make_tmap_2d(bits, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, rows, cols / 8, cols / 8, 128, 128, true);
}

}  // namespace bd
