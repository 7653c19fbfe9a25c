// K2+K3 fused — one kernel per projection group computes, for a 128-row tile
// of the (stacked) backbone weight and a K range,
//
//   P[b][m] = sum_k W[m][k] x_b[k]                          (tcgen05 kind::f16)
//           + alpha_t(b) * sum_k s_t(b)[m][k] x_b[k]         (tcgen05 kind::i8)
//
// i.e. the shared base contraction (matmul_nt, P:src/matrix.cpp:26-41) fused
// with every tenant's packed delta (packed_signed_accumulate,
// P:src/delta.cpp:80-103, applied per request at P:src/serve.cpp:250-254),
// reading the backbone tile and each tenant's plane from HBM exactly once.
//
// Delta numerics. The reference identity y = 2*sum_{bit=1} x - sum x
// (delta.hpp:64-66) is evaluated in exact integer arithmetic:
//   * each request's activation row is split into two int8 fixed-point pieces,
//     x ~= S_b (q0 + q1/254) with |q| <= 127 (error <= S_b/508, ~2^-16 of
//     max|x_b|: below the bf16 rounding already present in x);
//   * a 32-bit word of sign bits becomes 8 registers of u8 {0,128} with one
//     shift + one mask each ((w << (7-c)) & 0x80808080), written to TMEM as the
//     MMA's A operand; the K order inside each 32-column chunk is permuted
//     (register c, byte i <-> column 8i+c) and the activations are stored with
//     the same permutation, so the product is unchanged;
//   * tcgen05.mma kind::i8 accumulates 128 * sum_{bit=1} q in s32 (exact);
//     sum q over the tile's K range comes from per-block prefix sums;
//   * epilogue: delta = alpha * S_b * ((D0/64 - Q0) + (D1/64 - Q1)/254).
//
// Warp roles (256 threads): w0 TMA producer, w1 MMA issuer, w2 TMEM owner,
// w4-7 expand sign planes into TMEM, then run the epilogue. Pipelines:
// smem stages (TMA -> MMA/expanders, full/empty), TMEM A-ring
// (expanders -> MMA, a_full/a_empty), accumulators (MMA -> epilogue, done).
// Split-K partials are written (not atomically added): bit-reproducible.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace bd {

void note_launch();

namespace {

constexpr int kThreads = 256;
constexpr int kMaxRing = 12;    // TMEM A slots (runtime p.ring <= kMaxRing)
constexpr int kMaxStages = 4;
constexpr int kBitsBox = 16;    // bytes of one plane row per stage (128 bits)

struct Layout {
    uint32_t w_off, x_off, q_off, bits_off, stage, total;
};

__host__ __device__ inline Layout fused_layout(int bn, int xq_rows, int n_slots, int stages) {
    Layout L;
    L.w_off = 0;                                   // 2 x [128 x 64] bf16 (SW128)
    L.x_off = 2 * 128 * 128;                       // 2 x [bn x 64] bf16 (SW128)
    L.q_off = L.x_off + 2 * bn * 128;              // [xq_rows x 128] int8 (SW128)
    L.bits_off = L.q_off + ((xq_rows * 128 + 1023) & ~1023);
    L.stage = (L.bits_off + n_slots * 128 * kBitsBox + 1023) & ~1023u;
    L.total = 1024 + stages * L.stage + 512;
    return L;
}

__global__ void __launch_bounds__(kThreads, 1) fused_kernel(const __grid_constant__ FusedParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    const Layout L = fused_layout(p.bn, p.xq_rows, p.n_slots, p.stages);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.stages * L.stage);
    uint64_t* empty = full + kMaxStages;
    uint64_t* a_full = empty + kMaxStages;
    uint64_t* a_empty = a_full + kMaxRing;
    uint64_t* done = a_empty + kMaxRing;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
    float* ys = reinterpret_cast<float*>(smem);  // epilogue staging (reuses stage 0)

    const uint32_t warp = warp_id(), lane = lane_id();
    const int m0 = blockIdx.x * 128;
    const int split = blockIdx.y;
    const int kb0 = split * p.kb_per_split;
    const int kb1 = min(p.kb_total, kb0 + p.kb_per_split);
    const int nkb = max(0, kb1 - kb0);
    int sub = 0;
    while (sub + 1 < p.n_subs && m0 >= p.sub_row0[sub + 1]) ++sub;
    const int row_in_sub = m0 - p.sub_row0[sub];

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&p.map_w);
        prefetch_tmap(&p.map_x);
        prefetch_tmap(&p.map_xq);
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int r = 0; r < p.ring; ++r) {
            mbar_init(&a_full[r], 128);
            mbar_init(&a_empty[r], 1);
        }
        mbar_init(done, 1);
        fence_mbar_init();
    }
    if (warp == 2) {
        if (p.tmem_cols == 128) tmem_alloc<128>(tmem_slot);
        else if (p.tmem_cols == 256) tmem_alloc<256>(tmem_slot);
        else tmem_alloc<512>(tmem_slot);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---- TMA producer ----
            const uint64_t pol_stream = policy_evict_first();
            const uint32_t bytes = 2 * 128 * 128 + 2 * p.bn * 128 + p.xq_rows * 128 +
                                   p.n_slots * 128 * kBitsBox;
            for (int i = 0; i < nkb; ++i) {
                const int s = i % p.stages;
                mbar_wait(&empty[s], ((i / p.stages) & 1) ^ 1);
                uint8_t* st = smem + s * L.stage;
                mbar_arrive_expect_tx(&full[s], bytes);
                const int kb = kb0 + i;
                const int kc = kb * kFusedBK;
                tma_load_2d_hint(st + L.w_off, &p.map_w, &full[s], kc, m0, pol_stream);
                tma_load_2d_hint(st + L.w_off + 128 * 128, &p.map_w, &full[s], kc + 64, m0, pol_stream);
                tma_load_2d(st + L.x_off, &p.map_x, &full[s], kc, 0);
                tma_load_2d(st + L.x_off + p.bn * 128, &p.map_x, &full[s], kc + 64, 0);
                tma_load_2d(st + L.q_off, &p.map_xq, &full[s], kc, 0);
                for (int j = 0; j < p.n_slots; ++j)
                    tma_load_2d_hint(st + L.bits_off + j * 128 * kBitsBox,
                                     &p.bits_maps[p.slots[j].map_idx[sub]], &full[s],
                                     kb * kBitsBox, row_in_sub, pol_stream);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---- MMA issuer ----
            const uint32_t id_base = idesc_bf16_f32(128, p.bn);
            uint32_t g = 0;
            for (int i = 0; i < nkb; ++i) {
                const int s = i % p.stages;
                mbar_wait(&full[s], (i / p.stages) & 1);
                tc_fence_after();
                uint8_t* st = smem + s * L.stage;
                if (!(p.debug & 8))
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint64_t da = sdesc_k128(st + L.w_off + (k >> 2) * 128 * 128) + 2 * (k & 3);
                    const uint64_t db = sdesc_k128(st + L.x_off + (k >> 2) * p.bn * 128) + 2 * (k & 3);
                    mma_bf16_ss(tbase, da, db, id_base, (i > 0 || k > 0) ? 1u : 0u);
                }
                for (int j = 0; j < p.n_slots; ++j, ++g) {
                    const int r = g % p.ring;
                    mbar_wait(&a_full[r], (g / p.ring) & 1);
                    tc_fence_after();
                    const FusedSlot& sl = p.slots[j];
                    const uint32_t id_q = idesc_u8s8_s32(128, sl.n);
                    const uint64_t dq = sdesc_k128(st + L.q_off + sl.xrow * 128);
                    if (!(p.debug & 4))
#pragma unroll
                    for (int k = 0; k < 4; ++k)  // K = 32 bytes per MMA
                        mma_i8_ts(tbase + sl.dcol, tbase + p.a_col0 + r * 32 + 8 * k, dq + 2 * k, id_q,
                                  (i > 0 || k > 0) ? 1u : 0u);
                    tc_commit(&a_empty[r]);
                }
                tc_commit(&empty[s]);
            }
            tc_commit(done);
        }
    } else if (warp >= 4) {
        // ---- sign-plane expanders: thread = tile row = TMEM lane ----
        const uint32_t trow = (warp - 4) * 32 + lane;
        const uint32_t lane_base = ((warp - 4) * 32) << 16;
        uint32_t g = 0;
        for (int i = 0; i < nkb; ++i) {
            const int s = i % p.stages;
            mbar_wait(&full[s], (i / p.stages) & 1);
            const uint8_t* bits = smem + s * L.stage + L.bits_off;
            for (int j = 0; j < p.n_slots; ++j, ++g) {
                const int r = g % p.ring;
                mbar_wait(&a_empty[r], ((g / p.ring) & 1) ^ 1);
                const uint4 w = *reinterpret_cast<const uint4*>(bits + j * 128 * kBitsBox + trow * kBitsBox);
                const uint32_t wq[4] = {w.x, w.y, w.z, w.w};
                uint32_t a[32];
#pragma unroll
                for (int q = 0; q < 4; ++q)
#pragma unroll
                    for (int c = 0; c < 8; ++c) a[8 * q + c] = (wq[q] << (7 - c)) & 0x80808080u;
                if (p.debug & 1)
#pragma unroll
                    for (int c = 0; c < 32; ++c) a[c] = 0;
                if (!(p.debug & 2)) {
                    tmem_st32(tbase + lane_base + p.a_col0 + r * 32, a);
                    tmem_st_wait();
                }
                tc_fence_before();
                mbar_arrive(&a_full[r]);
            }
        }
        // ---- epilogue ----
        mbar_wait(done, 0);
        tc_fence_after();
        __syncwarp();
        // base accumulator -> ys[b][trow]
        for (int c0 = 0; c0 < p.bn; c0 += 16) {
            uint32_t v[16];
            tmem_ld16(tbase + lane_base + c0, v);
            tmem_ld_wait();
#pragma unroll
            for (int jj = 0; jj < 16; ++jj)
                if (c0 + jj < p.batch) ys[(c0 + jj) * 128 + trow] = nkb > 0 ? __uint_as_float(v[jj]) : 0.0f;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        for (int j = 0; j < p.n_slots; ++j) {
            const FusedSlot& sl = p.slots[j];
            const float alpha = sl.alpha[sub];
            for (int c0 = 0; c0 < 2 * sl.n_req; c0 += 8) {
                uint32_t v[8];
                tmem_ld8(tbase + lane_base + sl.dcol + c0, v);
                tmem_ld_wait();
#pragma unroll
                for (int jj = 0; jj < 8; jj += 2) {
                    const int q = (c0 + jj) >> 1;
                    if (q < sl.n_req && nkb > 0) {
                        const int b = sl.req[q];
                        const int* qs = p.qsum + static_cast<size_t>(b) * 2 * (p.kb_total + 1);
                        const long long Q0 = qs[kb1] - qs[kb0];
                        const long long Q1 = qs[p.kb_total + 1 + kb1] - qs[p.kb_total + 1 + kb0];
                        const long long t0 = static_cast<long long>(static_cast<int>(v[jj])) / 64 - Q0;
                        const long long t1 = static_cast<long long>(static_cast<int>(v[jj + 1])) / 64 - Q1;
                        const double d = static_cast<double>(alpha) * p.xscale[b] *
                                         (static_cast<double>(t0) + static_cast<double>(t1) / 254.0);
                        ys[b * 128 + trow] += static_cast<float>(d);
                    }
                }
            }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        // coalesced store of the partial tile
        float* out = p.partial + static_cast<size_t>(split) * p.batch * p.M;
        for (int idx = trow; idx < p.batch * 128; idx += 128) {
            const int b = idx / 128, rr = idx % 128;
            if (m0 + rr < p.M) out[static_cast<size_t>(b) * p.M + m0 + rr] = ys[idx];
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        if (p.tmem_cols == 128) tmem_dealloc<128>(tbase);
        else if (p.tmem_cols == 256) tmem_dealloc<256>(tbase);
        else tmem_dealloc<512>(tbase);
    }
}

// One block per request: fixed-point split of the bf16 activation row into two
// int8 pieces (permuted K, see header) + per-K-block prefix sums of the pieces.
__global__ void xq_prep_kernel(const uint16_t* __restrict__ X, int ldx, int K,
                               const int* __restrict__ xq_row, int8_t* __restrict__ Xq, int ldq,
                               float* __restrict__ xscale, int* __restrict__ qsum, int kb_total) {
    __shared__ float red[32];
    __shared__ int blk[2][128];
    const int b = blockIdx.x;
    const uint16_t* x = X + static_cast<size_t>(b) * ldx;
    float amax = 0.0f;
    for (int k = threadIdx.x; k < K; k += blockDim.x) amax = fmaxf(amax, fabsf(bf16_to_f32(x[k])));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = amax;
    __syncthreads();
    if (threadIdx.x == 0) {
        float m = 0.0f;
        for (int i = 0; i < int(blockDim.x >> 5); ++i) m = fmaxf(m, red[i]);
        red[0] = m > 0.0f ? m / 127.0f : 1.0f;
    }
    __syncthreads();
    const float S = red[0];
    if (threadIdx.x == 0) xscale[b] = S;
    int8_t* q0row = Xq + static_cast<size_t>(xq_row[b]) * ldq;
    int8_t* q1row = q0row + ldq;
    const int kpad = kb_total * kFusedBK;
    for (int kb = 0; kb < kb_total; kb += 128) {  // process up to 128 K-blocks per round
        const int nb = min(128, kb_total - kb);
        for (int i = threadIdx.x; i < 2 * 128; i += blockDim.x) blk[i >> 7][i & 127] = 0;
        __syncthreads();
        for (int d = threadIdx.x; d < nb * kFusedBK; d += blockDim.x) {
            const int dest = kb * kFusedBK + d;  // destination (permuted) index
            const int chunk = dest & ~31, pidx = dest & 31;
            const int src = chunk + 8 * (pidx & 3) + (pidx >> 2);
            int q0 = 0, q1 = 0;
            if (src < K) {
                const float v = bf16_to_f32(x[src]) / S;
                const float r0 = rintf(v);
                q0 = static_cast<int>(r0);
                q1 = static_cast<int>(rintf((v - r0) * 254.0f));
                q0 = max(-127, min(127, q0));
                q1 = max(-127, min(127, q1));
            }
            if (dest < kpad) {
                q0row[dest] = static_cast<int8_t>(q0);
                q1row[dest] = static_cast<int8_t>(q1);
            }
            atomicAdd(&blk[0][d / kFusedBK], q0);
            atomicAdd(&blk[1][d / kFusedBK], q1);
        }
        __syncthreads();
        if (threadIdx.x < 2) {
            int* qs = qsum + (static_cast<size_t>(b) * 2 + threadIdx.x) * (kb_total + 1);
            int acc = kb == 0 ? 0 : qs[kb];
            if (kb == 0) qs[0] = 0;
            for (int i = 0; i < nb; ++i) {
                acc += blk[threadIdx.x][i];
                qs[kb + i + 1] = acc;
            }
        }
        __syncthreads();
    }
}

}  // namespace

bool plan_fused(FusedParams& p, uint64_t M, uint64_t K, int batch) {
    p.M = int(M);
    p.batch = batch;
    p.bn = std::max(16, ((batch + 15) / 16) * 16);
    if (p.bn > 256 || p.n_slots > kFusedMaxSlots || p.n_slots < 1) return false;
    // TMEM: base accumulator, slot accumulators, A ring
    int col = p.bn;
    int xrow = 0;
    for (int j = 0; j < p.n_slots; ++j) {
        FusedSlot& s = p.slots[j];
        if (s.n_req < 1 || s.n_req > kFusedMaxReq) return false;
        s.n = 2 * s.n_req <= 8 ? 8 : ((2 * s.n_req + 15) / 16) * 16;
        col = (col + 7) & ~7;
        if (s.n >= 16) col = (col + 15) & ~15;
        s.dcol = col;
        col += s.n;
        (void)xrow;
    }
    col = (col + 31) & ~31;
    p.a_col0 = col;
    p.ring = std::min(kMaxRing, (512 - col) / 32);
    if (const char* e = std::getenv("BD_FUSED_RING")) p.ring = std::max(1, std::min(p.ring, atoi(e)));
    if (p.ring < 2) return false;
    col += p.ring * 32;
    p.debug = std::getenv("BD_FUSED_DEBUG") ? atoi(std::getenv("BD_FUSED_DEBUG")) : 0;
    if (col > 512) return false;
    p.tmem_cols = col <= 128 ? 128 : (col <= 256 ? 256 : 512);
    // Xq rows: each slot reads n rows from its xrow (which the caller set, multiple of 8)
    int rows = 0;
    for (int j = 0; j < p.n_slots; ++j) rows = std::max(rows, p.slots[j].xrow + p.slots[j].n);
    p.xq_rows = ((rows + 7) / 8) * 8;
    if (p.xq_rows > 256) return false;
    // stages within the smem budget
    int stages = kMaxStages;
    while (stages > 2 && fused_layout(p.bn, p.xq_rows, p.n_slots, stages).total > 225 * 1024) --stages;
    const Layout Lt = fused_layout(p.bn, p.xq_rows, p.n_slots, stages);
    if (Lt.total > 225 * 1024) return false;
    // epilogue staging (batch x 128 floats) must fit in one stage
    if (uint32_t(batch) * 128 * 4 > Lt.stage) return false;
    p.stages = stages;
    p.smem = int(Lt.total);
    p.m_tiles = int((M + 127) / 128);
    p.kb_total = int((K + kFusedBK - 1) / kFusedBK);
    // split-K to fill 148 SMs (1 CTA / SM): minimise ceil(tiles*s/148) * (kb/s + overhead)
    int best = 1;
    double best_cost = 1e30;
    for (int s = 1; s <= std::min(p.kb_total, 16); ++s) {
        const int per = (p.kb_total + s - 1) / s;
        const int se = (p.kb_total + per - 1) / per;
        const double cost = std::ceil(double(p.m_tiles) * se / kNumSMs) * (per + 1.5);
        if (cost < best_cost - 1e-9) {
            best_cost = cost;
            best = se;
        }
    }
    p.kb_per_split = (p.kb_total + best - 1) / best;
    p.splits = (p.kb_total + p.kb_per_split - 1) / p.kb_per_split;
    return true;
}

void fused_launch(const FusedParams& p, cudaStream_t stream) {
    static bool attr = false;
    if (!attr) {
        BD_CUDA(cudaFuncSetAttribute(fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
        attr = true;
    }
    fused_kernel<<<dim3(p.m_tiles, p.splits), kThreads, p.smem, stream>>>(p);
    note_launch();
    BD_CUDA(cudaGetLastError());
}

void xq_prep_launch(const void* X, int ldx, int K, int batch, const int* xq_row_dev, int8_t* Xq,
                    int ldq, float* xscale, int* qsum, int kb_total, cudaStream_t stream) {
    xq_prep_kernel<<<batch, 256, 0, stream>>>(static_cast<const uint16_t*>(X), ldx, K, xq_row_dev, Xq,
                                              ldq, xscale, qsum, kb_total);
    note_launch();
    BD_CUDA(cudaGetLastError());
}

CUtensorMap tmap_bits(const uint8_t* bits, uint64_t rows, uint64_t cols) {
    return make_tmap_2d(bits, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, rows, cols / 8, cols / 8, 128,
                        kBitsBox, false);
}
CUtensorMap tmap_xq(const int8_t* Xq, int rows, uint64_t K, uint64_t ldq) {
    return make_tmap_2d(Xq, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, uint64_t(rows), K, ldq,
                        uint32_t(rows), 128, true);
}

}  // namespace bd
