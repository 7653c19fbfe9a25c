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

// [world][batch][n_l] f32 partial sums of a row-sharded projection -> dst [batch][n_l]
void shard_reduce_launch(const ProjOut& p, int batch, int n_l, float* dst, cudaStream_t s);
// all-gathered [world][batch][n_l] bf16 -> [batch][ld] (columns r*n_l + i)
void gather_transpose_launch(const uint16_t* src, int world, int batch, int n_l, uint16_t* dst, int ld,
                             cudaStream_t s);

// K3d's gathered activations written directly by the kernel producing a projection's input
// (instead of mtd_gather_kernel): request b's row goes to row[b] of xg, each 32-column block in
// the MMA's column order (2 i <- i, 2 i + 1 <- i + 16); padding rows stay zero
struct XgOut {
    uint16_t* xg = nullptr;
    int ld = 0;
    const int* row = nullptr;  // [batch]
};

struct AttnArgs {
    int dim, kv_dim, n_heads, n_kv_heads, hd, max_seq, layer;
    uint16_t* const* kcache;  // per request: [n_layers][max_seq][kv_dim] bf16
    uint16_t* const* vcache;
    const float2* rope;       // [max_seq][hd/2] (cos, sin)
    XgOut xo{};               // optional K3d copy of ctx (hd 128 kernels)
};

// ws: norm_ws_bytes(batch, dim) bytes, zeroed once at allocation (arrival counters
// + chunk sums of squares); launches using one ws must be stream-ordered
int norm_chunks(int dim);
size_t norm_ws_bytes(int batch, int dim);
// the launchers write an XgOut copy on their one-launch / head_dim-128 paths and return whether
// they did (false: the caller gathers)
bool resid_norm_launch(float* x, int batch, int dim, const ProjOut& proj, const float* const* norm_w,
                       uint16_t* xn, int ldxn, float* xn_f32, void* ws, cudaStream_t s, const XgOut& xo = XgOut{});
bool attn_launch(const ProjOut& qkv, const AttnArgs& a, const int* pos_dev, int batch,
                 uint16_t* ctx, int ld_ctx, cudaStream_t s);
bool silu_launch(const ProjOut& gu, int batch, int inter, uint16_t* act, int ld_act, cudaStream_t s,
                 const XgOut& xo = XgOut{});
void embed_launch(const float* embed, const int* tokens, const float* const* embed_delta, int batch,
                  int dim, float* x, cudaStream_t s);
void logits_launch(const ProjOut& lm, const float* const* raw_delta, const float* xn_f32, int batch,
                   int dim, int vocab, float* logits, cudaStream_t s);

}  // namespace bd
