// Host-side interface of the kernels (K1..K4) shared by the C-ABI and engine.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <vector>

#include "../../include/bitdelta/capi.h"

namespace bd {

// ---- K2 base GEMM ----
struct GemmPlan {
    uint64_t M = 0, K = 0;
    int batch = 0, bn = 16, stages = 4, smem = 0;
    int m_tiles = 0, kb_total = 0, kb_per_split = 0, splits = 1;
    int grid = 1;  // persistent CTAs (resident slots); units = m_tiles x splits
    bool i8 = false;  // INT8 RTN backbone (kind::i8 against kPieces int8 pieces of X)
};
// int8 pieces per activation row (quant_pieces_launch): x = sum_p piece_scale_p * q_p with
// |q_p| <= 64 and 7 bits per piece, i.e. x to 2^-27 of its row maximum (f32 has 24 bits)
constexpr int kPieces = 4;
// smem_cap > 0: plan one CTA per SM within smem_cap bytes (co-resident with the K3 LUT)
GemmPlan plan_base_gemm(uint64_t M, uint64_t K, int batch, int smem_cap = 0);
GemmPlan plan_i8_gemm(uint64_t M, uint64_t K, int batch, int smem_cap = 0);
GemmPlan plan_gemm(uint64_t M, uint64_t K, int batch, int smem_cap, bool i8);
CUtensorMap make_tmap_2d(const void* ptr, CUtensorMapDataType dt, uint32_t elem_bytes,
                         uint64_t rows, uint64_t cols, uint64_t row_stride_elems,
                         uint32_t box_rows, uint32_t box_cols, bool swizzle128);
CUtensorMap tmap_weights(const void* W, uint64_t M, uint64_t K, uint64_t ld);
CUtensorMap tmap_acts(const void* X, int batch, uint64_t K, uint64_t ld, int bn);
// partial: [splits][batch][M] f32
void base_gemm_launch(const GemmPlan& p, const CUtensorMap& map_w, const CUtensorMap& map_x,
                      float* partial, cudaStream_t stream);
// ---- K2 int8 (int8_matmul_nt, P:src/int8.cpp:67-81) ----
// Wq: int8 [M x K] (row stride ld bytes, % 16 == 0); Xq: kPieces rows per request
CUtensorMap tmap_weights_i8(const void* Wq, uint64_t M, uint64_t K, uint64_t ld);
CUtensorMap tmap_pieces(const void* Xq, int batch, uint64_t K, uint64_t ld, int bn);
// partial[s][b][m] = row_scale[m] * float(sum_p piece_scale[b*kPieces+p] * (Wq[m] . Xq[b*kPieces+p]))
void i8_gemm_launch(const GemmPlan& p, const CUtensorMap& map_wq, const CUtensorMap& map_xq,
                    const float* row_scale, const float* piece_scale, float* partial, cudaStream_t stream);
// X (bf16 or f32 [batch x ldx], K valid columns) -> Xq int8 [batch*kPieces x ldq] (columns
// >= K zeroed up to ldq) and piece_scale [batch*kPieces] (powers of two)
void quant_pieces_launch(const void* X, bool x_f32, int ldx, int K, int batch, int8_t* Xq, int ldq,
                         float* piece_scale, cudaStream_t stream);
// RTN quantize (P:src/int8.cpp:15-42): per row s = amax/127, q = clamp(nearbyint(double(w)/s))
void rtn_quantize_launch(const float* W, uint64_t rows, uint64_t cols, int8_t* q, uint64_t ldq,
                         float* row_scales, cudaStream_t stream);

// ---- K1 compressor ----
void compress_launch(const bd_compress_job* jobs, int n_jobs, bd_dtype dtype, cudaStream_t s);
void compress_stack_launch(const void* base, const void* fine, bd_dtype dtype, uint64_t rows,
                           uint64_t cols, uint64_t planes, uint8_t* bits, float* alphas,
                           cudaStream_t stream);

// ---- K3 drop-in (a7/a8) ----
void packed_accumulate_launch(const uint8_t* bits, uint64_t rows, uint64_t cols, const float* x,
                              uint64_t n_vec, float* out, float scale, bool overwrite,
                              cudaStream_t stream);

// ---- K6 distill backward (backward.cu) ----
// out[v][j] (overwrite ? = : +=) scale * float(sum_i s_ij y[v][i])  (P:src/delta.cpp:105-131)
void packed_transpose_launch(const uint8_t* bits, uint64_t rows, uint64_t cols, const float* y,
                             uint64_t n_vec, float* out, float scale, bool overwrite, cudaStream_t s);
// acc[0] += sum_i double(a[i]) * double(b[i])  (P:src/model.cpp:92-95)
void dot_f64_launch(const float* a, const float* b, uint64_t n, double* acc, cudaStream_t s);

// ---- K3 multi-tenant delta ----
// One delta "unit" = one sign plane of one tenant applied to the rows
// [row0, row0+rows) of a (possibly stacked) projection output, for the
// requests req[0..n_req). Output d[b][row] = sum over units of alpha * S x_b.
constexpr int kMaxReqPerUnit = 4;
constexpr int kMaxPlanesPerUnit = 4;
constexpr int kMaxPlanesPerTensor = 32;  // pool: planes beyond 4 run as accumulate passes
struct DeltaUnit {
    const uint8_t* bits[kMaxPlanesPerUnit];  // reference layout of one [rows x cols] plane each
    float alpha[kMaxPlanesPerUnit];
    int32_t n_planes;
    int32_t row0, rows;  // output rows [row0, row0+rows) of the stacked projection
    int32_t n_req;
    int32_t req[kMaxReqPerUnit];
};
// X: bf16 [batch x ldx] activations; D: f32 [batch x out_rows] (zeroed here, or added to with
// accumulate: a projection's planes beyond the first kMaxPlanesPerUnit, in a later launch)
void delta_units_launch(const DeltaUnit* units_host, int n_units, const void* X, int ldx,
                        int cols, int batch, float* D, int out_rows, cudaStream_t stream,
                        bool accumulate = false);

// ---- raw (unquantised f32) projection deltas, P:src/serve.cpp:27-35 (packed.cu) ----
// D[req][row0 + r] += sum_k W[r][k] x_req[k] for the job's requests (after the units pass,
// which zeroes D and leaves the rows of raw projections at 0)
constexpr int kRawMaxReq = 16;
struct RawJob {
    const float* W;  // [rows x cols] f32, this rank's rows
    int32_t row0, rows, n_req;
    int32_t req[kRawMaxReq];
};
void raw_delta_launch(const RawJob* jobs, int n_jobs, const void* X, int ldx, int cols, float* D, int out_rows,
                      cudaStream_t stream);

// ---- K23: base GEMM + tenant deltas as FP4 (kind::mxf4) MMAs in one persistent kernel (mt4.cu) ----
constexpr int kMt4MaxSlots = 64;
constexpr int kMt4MaxReq = 4;   // requests per slot (MMA N = 8 pieces x n_req <= 32)
constexpr int kMt4MaxSubs = 3;
struct Mt4Slot {
    int n_req;
    int req[kMt4MaxReq];          // batch indices (activation piece blocks of request req[q])
    float alpha[kMt4MaxSubs];     // per stacked sub-matrix
    int map_idx[kMt4MaxSubs];     // index into the bits tensor-map table
};
struct Mt4Params {
    CUtensorMap map_w, map_x;
    const CUtensorMap* bits_maps;  // device table (tmap_bits4)
    const uint8_t* xpk;            // FP4 activation pieces + scales, [batch][n_chunks][kXpBlock]
    const uint32_t* sched;         // per-tile stage schedule (mt4_schedule), device memory
    float* partial;                // [splits][batch][M]
    long long total_stages;
    int M, K, batch, bn, nr_max, n_subs, n_slots;
    int sub_row0[kMt4MaxSubs + 1];
    int kb_base, kc_plane, stages_per_tile, grid, splits, ring_b, ring_p, smem, n_chunks;
    int col_base, col_acc, acc_stride, n_acc, col_sfa, col_ring, n_ring;  // TMEM layout
    Mt4Slot slots[kMt4MaxSlots];
};
// mean requests per tenant from which the auto policy uses K23: 4, or 2 at batch >= 64.
// Measured at 2 requests/tenant (K23 vs byte LUT): Mistral-7B B=64 +8 %, Llama-2-7B B=64
// +3 %, Mistral-7B B=32 +1 %, Llama-2-7B B=32 -2 %, Llama-2-7B B=16 -22 %.
inline int k23_min_requests(int batch = 0) { return batch >= 64 ? 2 : 4; }
// requests in the next K23 slot of a tenant with `remaining` requests left (slots of 4, then
// the remainder)
inline int mt4_slot_requests(size_t remaining) {
    return remaining >= size_t(kMt4MaxReq) ? kMt4MaxReq : int(remaining);
}
// Fills the schedule (stages per tile, persistent grid, splits, smem ring); false if unsupported.
bool plan_mt4(Mt4Params& p, uint64_t M, uint64_t K, int batch);
// Host copy of the per-tile stage schedule for p (upload it and set p.sched).
std::vector<uint32_t> mt4_schedule(const Mt4Params& p);
void mt4_launch(const Mt4Params& p, cudaStream_t stream);
// Activation pieces, one contiguous block per (request, 1024-column chunk): 4 x [8 pieces x 128 B]
// packed e2m1 (128-byte swizzled, K permuted inside 32-column blocks) + [8 x 32 B] ue8m0 scales.
constexpr int kXpBlock = 4096 + 256;
inline int xp_chunks(int K) { return (K + 1023) / 1024; }
// X bf16 [batch x ldx] -> xpk [batch][xp_chunks(K)][kXpBlock]
void xp_prep_launch(const void* X, int ldx, int K, int batch, uint8_t* xpk, cudaStream_t stream);
// 2-D map of a sign plane (reference layout), box [128 rows x 128 B], 128-byte swizzle
CUtensorMap tmap_bits4(const uint8_t* bits, uint64_t rows, uint64_t cols);

// ---- K3 byte-LUT (few requests per tenant; lut.cu) ----
constexpr int kLutMaxSegs = 3;
constexpr int kLutMaxChunks = 48;
constexpr int kLutMaxJobs = 64;
struct LutJob {
    int req;                                              // batch index
    int n_planes[kLutMaxSegs];
    const uint8_t* bits[kLutMaxSegs][kMaxPlanesPerUnit];  // reference layout, cols % 32 == 0
    float alpha[kLutMaxSegs][kMaxPlanesPerUnit];
};
struct LutParams {
    int n_jobs, slices, cols, ldx, batch, M, n_segs, grid;
    int ld_u4;  // plane row stride in 16-byte words (v2 kernel): cols / 128, or the pool's padded rows
    int seg_row0[kLutMaxSegs + 1];  // stacked row offsets of the sub-matrices
    LutJob jobs[kLutMaxJobs];
};
// Fills the geometry (slices, persistent grid) for the stacked rows; false if unsupported.
bool plan_lut(LutParams& p, const int* seg_rows, int n_segs, int cols, int ldx, int batch);
// out: [slices][batch][M] f32, alpha already applied; every (slice, req, row) of a job written
void lut_launch(const LutParams& p, const void* X, float* out, cudaStream_t stream);

// ---- K3d: tenants with many requests, dense tensor-core delta (mtd.cu) ----
constexpr int kMtdMaxTenants = 8;
constexpr int kMtdMaxN = 64;  // requests per tenant (MMA N, padded to 16)
// the auto policy takes K3d from 8 requests per tenant at batch >= 64. Measured (tok/s, M7 B=64,
// round-2 build with grouped-query attention and K3d inputs written by their producers):
// T=8 (8/tenant) K3d 5 280 vs K23 5 183-5 232; T=16 (4/tenant) K3d 4 763 vs K23 5 168; earlier:
// T=1 K3d 7 963 vs K23 5 089, T=4 6 272 vs 5 072; L7 B=16 T=1 (16/tenant) K3d 2 807 vs the byte
// LUT 3 129 (its 16 jobs read one plane, mostly from L2, and it runs beside K2 while K3d runs
// after it)
constexpr double kMtdMinRequests = 8.0;
constexpr int kMtdMinBatch = 64;
struct MtdTenant {
    std::vector<int> reqs;  // batch indices
    int n_planes[kLutMaxSegs];
    const uint8_t* bits[kLutMaxSegs];
    float alpha[kLutMaxSegs];
};
struct MtdGather {
    int rows;
    int n_req[kMtdMaxTenants], n_pad[kMtdMaxTenants], row0[kMtdMaxTenants];
    int req[kMtdMaxTenants][kMtdMaxN];
};
struct MtdParams {
    int n_tasks, tiles, M, K, n_segs, n_ten, x_rows, grid;
    int n_chunks, ksplit, chunks_per_split;  // 256-column chunks; K splits (delta partials)
    int ring, stage_bytes;                   // stage ring sized for the launch's largest N_t
    size_t dstride;                          // elements between delta partials (batch x M)
    int seg_row0[kLutMaxSegs + 1];
    const CUtensorMap* plane_maps;  // device [tenant][seg]: box [128 rows x 32 B]
    const CUtensorMap* x_maps;      // device [tenant]: gathered X rows, box [n_pad rows x 64 cols]
    float* out;                     // D [batch][M]
    int n_req[kMtdMaxTenants], n_pad[kMtdMaxTenants], x_row0[kMtdMaxTenants];
    int req[kMtdMaxTenants][kMtdMaxN];
    float alpha[kMtdMaxTenants][kLutMaxSegs];
};
// false if unsupported (K % 256, tenant / request counts, one plane per projection)
bool plan_mtd(MtdParams& p, MtdGather& g, const std::vector<MtdTenant>& tens, const int* seg_rows, int n_segs,
              int K, int ldx, int max_splits, std::vector<CUtensorMap>& plane_maps);
std::vector<CUtensorMap> mtd_x_maps(const MtdParams& p, const void* Xp, int ldp);
void mtd_gather_launch(const void* X, int ldx, int K, const MtdGather& g, int n_ten, void* Xp, int ldp,
                       cudaStream_t stream);
void mtd_launch(const MtdParams& p, cudaStream_t stream);

// ---- K5: fp32 multi-tenant linear (SIMT, fp64 accumulation; packed.cu) ----
// Y[b] = W x_b + alpha_b S_b x_b for every b < batch (req_bits[b] == null: base only);
// W f32 [rows x cols], X f32 [batch x cols], Y f32 [batch x rows]
void f32_linear_launch(const float* W, uint64_t rows, uint64_t cols, const uint8_t* const* req_bits,
                       const float* req_alpha, int batch, const float* X, float* Y, cudaStream_t stream);

// Y[b][m] = sum_s P[s][b][m] (+ D[b][m])
void combine_launch(const float* P, int splits, const float* D, int batch, int M, float* Y,
                    cudaStream_t stream, int dsplits = 1);

}  // namespace bd
