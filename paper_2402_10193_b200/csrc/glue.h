// Host interface of the decode glue kernels (K4).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace bd {

// A projection's output as produced by K2/K3: value(b, m) =
//   sum_{s < splits} P[s*pstride + b*M + m] + D[b*M + m]   (D may be null).
struct ProjOut {
    const float* P = nullptr;
    int splits = 0;
    size_t pstride = 0;
    const float* D = nullptr;  // delta partials: sum_{k < dsplits} D[k*pstride_d + b*M + m]
    int dsplits = 1;
    size_t dstride = 0;
    int M = 0;
    int col0 = 0;  // column offset used by resid_norm (o / down outputs)
    // all-gathered row shards (world > 1): value(b, m) = G[(m / g_cols) * g_batch + b][m % g_cols]
    const float* G = nullptr;
    int g_cols = 0, g_batch = 0;
};

// Fused step epilogues (fuse.cuh): the residual + RMSNorm after the o / down projections and
// the SiLU after gate/up run inside the projection kernels instead of their own launches.
// Every producer CTA (K2, the K3 LUT) arrives on the group's counter after its partial
// stores; the K2 CTAs (the waiter) wait for all arrivals, then run the
// 128-row output tiles (tile t: rows [128 t, 128 t + 128), gate/up: and the same rows of up
// at + fold) for every request, spread over all of their warps:
//   kind 1 (residual + norm, serve.cpp:283-293): x += proj; xn = bf16(x * w_b);
//          msq_out[b][t] = sum over the tile of double(x)^2
//   kind 2 (SiLU, serve.cpp:301-302): act = bf16(silu(r_b g) * (r_b u)) with r_b from msq_in
// RMSNorm's scale r_b = 1 / sqrt(mean x^2 + 1e-12) is a per-request scalar, so it moves to the
// consumers of the following projection (W (r x) = r (W x)): attention scales q / k / v by
// r_b (AttnArgs::msq), kind 2 scales gate / up.
struct TileFuse {
    int kind = 0;  // 0 = none
    unsigned* cnt = nullptr;  // [0] arrivals, [32] departures (0 between phases)
    unsigned arrivals = 0;    // producer CTAs of the group (K2 + every LUT launch)
    int waiter = 0;           // this launch waits for every producer and runs the tiles (K2)
    int tiles = 0, fold = 0, B = 0;
    ProjOut src;  // the projection's partials
    // kind 1
    float* x = nullptr;
    int dim = 0;
    const float* const* norm_w = nullptr;  // [B] per-request norm rows (base + tenant delta)
    uint16_t* xn = nullptr;
    int ldxn = 0;
    double* msq_out = nullptr;  // [B][tiles]
    // kind 2
    const double* msq_in = nullptr;  // [B][msq_tiles] from the kind-1 tiles of the norm
    int msq_tiles = 0, msq_dim = 0;
    uint16_t* act = nullptr;
    int ld_act = 0;
};
struct LutParams;
bool lut_fusable(const LutParams& p);
size_t lut2_smem_bytes();
// kind-1 tiles as a launch of their own (the first layer's norm1: no producer kernel)
void fuse_norm_launch(const TileFuse& f, cudaStream_t s);

// [world][batch][n_l] f32 partial sums of a row-sharded projection -> dst [batch][n_l]
void shard_reduce_launch(const ProjOut& p, int batch, int n_l, float* dst, cudaStream_t s);
// all-gathered [world][batch][n_l] bf16 -> [batch][ld] (columns r*n_l + i)
void gather_transpose_launch(const uint16_t* src, int world, int batch, int n_l, uint16_t* dst, int ld,
                             cudaStream_t s);

struct AttnArgs {
    int dim, kv_dim, n_heads, n_kv_heads, hd, max_seq, layer;
    uint16_t* const* kcache;  // per request: [n_layers][max_seq][kv_dim] bf16
    uint16_t* const* vcache;
    const float2* rope;       // [max_seq][hd/2] (cos, sin)
    const double* msq = nullptr;  // fused norm1 (TileFuse kind 1): q/k/v *= r_b
    int msq_tiles = 0, msq_dim = 0;
};

// ws: norm_ws_bytes(batch, dim) bytes, zeroed once at allocation (arrival counters
// + chunk sums of squares); launches using one ws must be stream-ordered
int norm_chunks(int dim);
size_t norm_ws_bytes(int batch, int dim);
void resid_norm_launch(float* x, int batch, int dim, const ProjOut& proj, const float* const* norm_w,
                       uint16_t* xn, int ldxn, float* xn_f32, void* ws, cudaStream_t s);
void attn_launch(const ProjOut& qkv, const AttnArgs& a, const int* pos_dev, int batch,
                 uint16_t* ctx, int ld_ctx, cudaStream_t s);
void silu_launch(const ProjOut& gu, int batch, int inter, uint16_t* act, int ld_act, cudaStream_t s);
void embed_launch(const float* embed, const int* tokens, const float* const* embed_delta, int batch,
                  int dim, float* x, cudaStream_t s);
void logits_launch(const ProjOut& lm, const float* const* raw_delta, const float* xn_f32, int batch,
                   int dim, int vocab, float* logits, cudaStream_t s);

}  // namespace bd
