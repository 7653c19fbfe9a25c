// K2 — shared base contraction on the 5th-gen tensor cores (replaces
// deltakit::matmul_nt, P:src/matrix.cpp:26-41, as called by
// ServingPool::backbone_linear_nt, P:src/serve.cpp:120-127).
//
//   P[split][n][m] = sum_{k in split} W[m][k] * X[n][k]     (bf16 in, f32 out)
//
// Swap-AB: the weight rows are the MMA M dimension (128 per CTA tile) and the
// decode batch is N (16..256), so a batch of 16 costs one 128x16 MMA per
// 16-wide K step. Operands are staged by TMA (128-byte swizzle) through an
// mbarrier ring; one elected thread issues tcgen05.mma into a TMEM
// accumulator; all four warps drain TMEM with tcgen05.ld. Split-K partials are
// written, not atomically added, so results are bit-reproducible and
// independent of the order of requests in the batch (test_serve.cpp:169-190).
//
// Roofline: HBM — 2 bytes per weight element; at batch B the intensity is B
// flop/byte, far below the tensor pipe's ridge point.
//
// Persistent: one CTA per resident slot walks its work units (row tile, K split) through
// ONE continuous stage ring, with two TMEM accumulators so unit i + 1 accumulates while
// four epilogue warps drain unit i: no per-unit pipeline refill or CTA launch. Measured
// (ncu, M7 B=64 gate/up, 1120 units): 54 -> 43 us.
#include <cstdlib>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <mutex>

#include "common.cuh"
#include "kernels.h"

namespace bd {

namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;  // bf16 elements = 128 bytes = one swizzle row
constexpr int kMaxStages = 8;
constexpr int kGemmThreads = 256;  // producer, issuer, TMEM allocator, idle, 4 epilogue warps

struct GemmSmemLayout {
    uint32_t a_bytes, b_bytes, stage_bytes, stages, total;
};

__host__ __device__ inline GemmSmemLayout gemm_layout(int bn, int stages) {
    GemmSmemLayout L;
    L.a_bytes = kBM * kBK * 2;
    L.b_bytes = bn * kBK * 2;
    L.stage_bytes = L.a_bytes + L.b_bytes;
    L.stages = stages;
    L.total = 1024 /*align slack*/ + stages * L.stage_bytes + 256 /*barriers*/;
    return L;
}

// kI8 (the INT8 RTN backbone of P:src/int8.cpp:67-81): W is the int8
// RTN tensor, X holds kPieces int8 pieces per request (quant_pieces_kernel), the MMA is
// kind::i8 (s8 x s8 -> exact s32) with K = 128 per 128-byte stage row, and the epilogue
// recombines y = row_scale[m] * float(sum_p acc_p * piece_scale_p).
template <bool kI8>
__global__ void __launch_bounds__(kGemmThreads, 1)
    base_gemm_kernel(const __grid_constant__ CUtensorMap map_w,
                     const __grid_constant__ CUtensorMap map_x, float* __restrict__ partial,
                     int M, int N_valid, int bn, int kb_total, int kb_per_split, int splits, int n_units,
                     int stages, const float* __restrict__ row_scale, const float* __restrict__ piece_scale) {
    extern __shared__ uint8_t smem_raw[];
    const unsigned long long t_entry = gtimer();
    unsigned long long t_wait = 0;
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    const GemmSmemLayout L = gemm_layout(bn, stages);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * L.stage_bytes);
    uint64_t* empty = full + kMaxStages;
    uint64_t* done = empty + kMaxStages;  // [2]: accumulator a complete
    uint64_t* acc_free = done + 2;        // [2]: accumulator a drained by the epilogue
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_free + 2);

    const uint32_t warp = warp_id(), lane = lane_id();
    const uint32_t acc_cols = bn <= 32 ? 32 : (bn <= 64 ? 64 : (bn <= 128 ? 128 : 256));
    constexpr int kbk = kI8 ? 128 : kBK;  // K elements per 128-byte stage row
    // work unit u = (row tile u / splits, K split u % splits); CTA b takes b, b + grid, ...
    auto unit = [&](int u, int& m0, int& split, int& kb0, int& nkb) {
        m0 = (u / splits) * kBM;
        split = u % splits;
        kb0 = split * kb_per_split;
        nkb = min(kb_total, kb0 + kb_per_split) - kb0;
    };

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&map_w);
        prefetch_tmap(&map_x);
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&done[a], 1);
            mbar_init(&acc_free[a], 4);
        }
        fence_mbar_init();
    }
    if (warp == 2) {
        // two accumulators (unit i + 1 accumulates while unit i drains); the allocation
        // size must be a compile-time immediate
        if (acc_cols == 32) tmem_alloc<64>(tmem_slot);
        else if (acc_cols == 64) tmem_alloc<128>(tmem_slot);
        else if (acc_cols == 128) tmem_alloc<256>(tmem_slot);
        else tmem_alloc<512>(tmem_slot);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t taddr = *tmem_slot;

    if (warp == 0 && lane == 0) {
        // ---- TMA producer: one continuous ring over all of the CTA's units ----
        // The weights do not depend on the predecessor kernel: the first ring's worth is
        // requested before waiting for it (PDL), the activations only after.
        const uint64_t pol_w = policy_evict_first();  // weights stream once per step
        int m0, split, kb0, nkb;
        unit(blockIdx.x, m0, split, kb0, nkb);
        const int npre = min(nkb, stages);
        for (int i = 0; i < npre; ++i) {
            mbar_arrive_expect_tx(&full[i], L.stage_bytes);
            tma_load_2d_hint(smem + i * L.stage_bytes, &map_w, &full[i], (kb0 + i) * kbk, m0, pol_w);
        }
        griddep_wait();  // PDL: the activations come from the previous kernel
        t_wait = gtimer();
        int it = 0;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
            unit(u, m0, split, kb0, nkb);
            for (int i = 0; i < nkb; ++i, ++it) {
                const int s = it % stages;
                const uint32_t round = it / stages;
                uint8_t* a = smem + s * L.stage_bytes;
                uint8_t* b = a + L.a_bytes;
                const int kc = (kb0 + i) * kbk;
                if (it >= npre) {
                    mbar_wait(&empty[s], (round & 1) ^ 1);
                    mbar_arrive_expect_tx(&full[s], L.stage_bytes);
                    tma_load_2d_hint(a, &map_w, &full[s], kc, m0, pol_w);
                }
                tma_load_2d(b, &map_x, &full[s], kc, 0);
            }
        }
    } else if (warp == 1 && lane == 0) {
        // ---- MMA issuer ---- (consumes only what the producer's barriers release)
        const uint32_t idesc = kI8 ? idesc_s8s8_s32(kBM, bn) : idesc_bf16_f32(kBM, bn);
        int it = 0, lu = 0;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++lu) {
            int m0, split, kb0, nkb;
            unit(u, m0, split, kb0, nkb);
            const int acc = lu & 1;
            if (lu >= 2) mbar_wait(&acc_free[acc], ((lu >> 1) - 1) & 1);
            tc_fence_after();
            const uint32_t tacc = taddr + acc * acc_cols;
            for (int i = 0; i < nkb; ++i, ++it) {
                const int s = it % stages;
                const uint32_t round = it / stages;
                mbar_wait(&full[s], round & 1);
                tc_fence_after();
                uint8_t* a = smem + s * L.stage_bytes;
                uint8_t* b = a + L.a_bytes;
                const uint64_t da = sdesc_k128(a), db = sdesc_k128(b);
#pragma unroll
                for (int k = 0; k < 4; ++k) {  // +32 bytes per K step (16 bf16 / 32 int8)
                    if (kI8) mma_i8_ss(tacc, da + 2 * k, db + 2 * k, idesc, (i > 0 || k > 0) ? 1u : 0u);
                    else mma_bf16_ss(tacc, da + 2 * k, db + 2 * k, idesc, (i > 0 || k > 0) ? 1u : 0u);
                }
                tc_commit(&empty[s]);
            }
            tc_commit(&done[acc]);
        }
    } else if (warp >= 4) {
        // ---- epilogue: warps 4-7 drain their 32 TMEM lanes (lane quadrant = warp % 4) ----
        const uint32_t q = warp & 3;
        int lu = 0;
        for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++lu) {
            int m0, split, kb0, nkb;
            unit(u, m0, split, kb0, nkb);
            const int acc = lu & 1;
            mbar_wait(&done[acc], (lu >> 1) & 1);
            tc_fence_after();
            const int row = m0 + q * 32 + lane;
            float* out = partial + static_cast<size_t>(split) * N_valid * M;
            for (int c0 = 0; c0 < bn; c0 += 16) {
                uint32_t r[16];
                tmem_ld16(taddr + ((q * 32) << 16) + acc * acc_cols + c0, r);
                tmem_ld_wait();
                if (nkb <= 0) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) r[j] = 0;
                }
                if (row < M) {
                    if (kI8) {
                        // 16 columns = 4 requests x kPieces (4) int32 accumulators
                        const float rs = row_scale[row];
#pragma unroll
                        for (int g = 0; g < 4; ++g) {
                            const int n = c0 / kPieces + g;
                            if (n >= N_valid) break;
                            double sum = 0.0;  // exact: |acc_p| < 2^31, piece scales are powers of two
#pragma unroll
                            for (int pc = 0; pc < kPieces; ++pc)
                                sum += static_cast<double>(static_cast<int32_t>(r[g * kPieces + pc])) *
                                       static_cast<double>(piece_scale[n * kPieces + pc]);
                            out[static_cast<size_t>(n) * M + row] = static_cast<float>(sum) * rs;
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            const int n = c0 + j;
                            if (n < N_valid) out[static_cast<size_t>(n) * M + row] = __uint_as_float(r[j]);
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_free[acc]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        if (acc_cols == 32) tmem_dealloc<64>(taddr);
        else if (acc_cols == 64) tmem_dealloc<128>(taddr);
        else if (acc_cols == 128) tmem_dealloc<256>(taddr);
        else tmem_dealloc<512>(taddr);
    }
    if (warp == 0 && lane == 0) trace_rec(TR_GEMM, t_entry, t_wait);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        BD_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        require(p != nullptr && q == cudaDriverEntryPointSuccess, BD_ERR_CUDA,
                "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

}  // namespace

void note_launch();

// 2-D row-major [rows x cols] tensor, box {box_cols, box_rows}, 128B swizzle.
CUtensorMap make_tmap_2d(const void* ptr, CUtensorMapDataType dt, uint32_t elem_bytes,
                         uint64_t rows, uint64_t cols, uint64_t row_stride_elems,
                         uint32_t box_rows, uint32_t box_cols, bool swizzle128) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {row_stride_elems * elem_bytes};
    const cuuint32_t box[2] = {box_cols, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    require((strides[0] % 16) == 0, BD_ERR_BAD_ARGUMENT,
            "TMA: row stride must be a multiple of 16 bytes");
    require((reinterpret_cast<uintptr_t>(ptr) % 16) == 0, BD_ERR_BAD_ARGUMENT,
            "TMA: base pointer must be 16-byte aligned");
    const CUresult r = encode_fn()(&m, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                              : CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    require(r == CUDA_SUCCESS, BD_ERR_CUDA,
            "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
    return m;
}

GemmPlan plan_base_gemm(uint64_t M, uint64_t K, int batch, int smem_cap) {
    return plan_gemm(M, K, batch, smem_cap, false);
}
GemmPlan plan_i8_gemm(uint64_t M, uint64_t K, int batch, int smem_cap) {
    return plan_gemm(M, K, batch, smem_cap, true);
}

GemmPlan plan_gemm(uint64_t M, uint64_t K, int batch, int smem_cap, bool i8) {
    GemmPlan p;
    p.M = M;
    p.K = K;
    p.batch = batch;
    p.i8 = i8;
    const int n_cols = i8 ? kPieces * batch : batch;  // int8: kPieces MMA columns per request
    p.bn = std::max(16, ((n_cols + 15) / 16) * 16);
    require(p.bn <= 256, BD_ERR_BAD_ARGUMENT,
            i8 ? "int8 gemm: batch chunk must be <= 64" : "base gemm: batch chunk must be <= 256");
    const GemmSmemLayout L0 = gemm_layout(p.bn, 1);
    int slots;
    if (smem_cap > 0) {
        // co-resident with another kernel on every SM (the K3 LUT): one CTA per SM
        // within the shared-memory left over
        p.stages = std::max(2, std::min(kMaxStages, int((smem_cap - 1280) / L0.stage_bytes)));
        slots = kNumSMs;
    } else {
        // as many stages as fit in ~200 KB (2 CTAs/SM when the stage is small)
        int stages = std::min(kMaxStages, int((200 * 1024 - 1024 - 256) / L0.stage_bytes));
        const bool two_per_sm = (gemm_layout(p.bn, 4).total * 2 <= 227 * 1024);
        if (two_per_sm) stages = std::min(stages, int((110 * 1024 - 1280) / L0.stage_bytes));
        p.stages = std::max(2, stages);
        slots = kNumSMs * (two_per_sm ? 2 : 1);
    }
    p.smem = gemm_layout(p.bn, p.stages).total;
    const int m_tiles = int((M + kBM - 1) / kBM);
    const int kbk = i8 ? 128 : kBK;  // K elements per 128-byte stage row
    const int kb = int((K + kbk - 1) / kbk);
    // split-K to fill the machine: minimise ceil(tiles*s/slots) * ceil(kb/s)
    int best_s = 1;
    double best_cost = 1e30;
    for (int s = 1; s <= std::min(kb, 32); ++s) {
        const int per = (kb + s - 1) / s;
        const int s_eff = (kb + per - 1) / per;
        const double waves = std::ceil(double(m_tiles) * s_eff / slots);
        const double cost = waves * (per + 2.0 /*fixed per-CTA overhead in k-blocks*/);
        if (cost < best_cost - 1e-9) {
            best_cost = cost;
            best_s = s_eff;
        }
    }
    p.kb_total = kb;
    p.kb_per_split = (kb + best_s - 1) / best_s;
    p.splits = (kb + p.kb_per_split - 1) / p.kb_per_split;
    p.m_tiles = m_tiles;
    p.grid = slots;  // persistent: at most one CTA per slot, each walking its units
    return p;
}

template <bool kI8>
static void gemm_launch_t(const GemmPlan& p, const CUtensorMap& map_w, const CUtensorMap& map_x,
                          float* partial, const float* row_scale, const float* piece_scale, cudaStream_t stream) {
    static bool attr_set = false;
    if (!attr_set) {
        BD_CUDA(cudaFuncSetAttribute(base_gemm_kernel<kI8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     227 * 1024));
        // full carveout: an SM first configured for the co-resident K3 LUT must still
        // have room for a GEMM CTA (the default picks the smallest fitting carveout)
        BD_CUDA(cudaFuncSetAttribute(base_gemm_kernel<kI8>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     int(cudaSharedmemCarveoutMaxShared)));
        attr_set = true;
    }
    const int n_units = p.m_tiles * p.splits;
    BD_CUDA(launch_pdl(base_gemm_kernel<kI8>, dim3(std::min(n_units, p.grid)), dim3(kGemmThreads), size_t(p.smem),
                       stream, map_w, map_x, partial, int(p.M), p.batch, p.bn, p.kb_total, p.kb_per_split, p.splits,
                       n_units, p.stages, row_scale, piece_scale));
    note_launch();
    BD_CUDA(cudaGetLastError());
}

void base_gemm_launch(const GemmPlan& p, const CUtensorMap& map_w, const CUtensorMap& map_x,
                      float* partial, cudaStream_t stream) {
    require(!p.i8, BD_ERR_BAD_ARGUMENT, "base gemm: int8 plan on the bf16 kernel");
    gemm_launch_t<false>(p, map_w, map_x, partial, nullptr, nullptr, stream);
}

void i8_gemm_launch(const GemmPlan& p, const CUtensorMap& map_wq, const CUtensorMap& map_xq,
                    const float* row_scale, const float* piece_scale, float* partial, cudaStream_t stream) {
    require(p.i8, BD_ERR_BAD_ARGUMENT, "int8 gemm: bf16 plan");
    gemm_launch_t<true>(p, map_wq, map_xq, partial, row_scale, piece_scale, stream);
}

CUtensorMap tmap_weights(const void* W, uint64_t M, uint64_t K, uint64_t ld) {
    return make_tmap_2d(W, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, M, K, ld, kBM, kBK, true);
}
CUtensorMap tmap_weights_i8(const void* Wq, uint64_t M, uint64_t K, uint64_t ld) {
    return make_tmap_2d(Wq, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, M, K, ld, kBM, 128, true);
}
CUtensorMap tmap_pieces(const void* Xq, int batch, uint64_t K, uint64_t ld, int bn) {
    return make_tmap_2d(Xq, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, uint64_t(kPieces) * batch, K, ld,
                        uint32_t(bn), 128, true);
}
CUtensorMap tmap_acts(const void* X, int batch, uint64_t K, uint64_t ld, int bn) {
    return make_tmap_2d(X, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, uint64_t(batch), K, ld,
                        uint32_t(bn), kBK, true);
}

}  // namespace bd
