// K4 — decode-layer glue of ServingPool::decode_shared (P:src/serve.cpp:224-321)
// with the reference's numerics (P:include/deltakit/nn_ops.hpp:15-59):
//   * RMSNorm with double statistics and eps 1e-12 (nn_ops.hpp:15-25), the
//     per-tenant weight being backbone row + raw delta row (serve.cpp:224-228);
//   * interleaved-pair RoPE (nn_ops.hpp:29-45) from a host-built table whose
//     cos/sin come from the same double pow/cos/sin the reference evaluates;
//   * f32 softmax (nn_ops.hpp:48-57) and SiLU (nn_ops.hpp:59).
// Each glue kernel also folds in the split-K reduction of the projection that
// produced its input (sum of base partials + tenant delta partials), so the
// linears never make an extra pass over their outputs. All reductions use a
// fixed order (no atomics): outputs are bit-reproducible and independent of a
// request's position in the batch.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "glue.h"

namespace bd {

void note_launch();

namespace {

#ifndef BD_PDL_EARLY
#define BD_PDL_EARLY 1  // glue kernels let the next (PDL) kernel start its prologue at once
#endif

constexpr int kNormChunk = 256;  // elements per block in the residual/norm kernels

// k-th partial of output (b, m): base split-K partials first, then delta partials
__device__ __forceinline__ const float* proj_ptr(const ProjOut& p, int k, int b, int m) {
    return k < p.splits ? p.P + static_cast<size_t>(k) * p.pstride + size_t(b) * p.M + m
                        : p.D + static_cast<size_t>(k - p.splits) * p.dstride + size_t(b) * p.M + m;
}
__device__ __forceinline__ int proj_parts(const ProjOut& p) { return p.splits + (p.D ? p.dsplits : 0); }

// All partial loads are issued before the (fixed-order) additions: the reduction
// costs one memory latency per group of partials instead of one per partial.
constexpr int kPartGroup = 16;  // float4 paths (norm: 128 threads, one float4 each)
__device__ __forceinline__ float proj_val(const ProjOut& p, int b, int m) {
    if (p.G) {
        const int r = m / p.g_cols, i = m - r * p.g_cols;
        return p.G[(static_cast<size_t>(r) * p.g_batch + b) * p.g_cols + i];
    }
    const int n = proj_parts(p);
    float s = 0.0f;
    for (int k0 = 0; k0 < n; k0 += 8) {  // 8: register budget of the 4-CTA/SM attention kernel
        float t[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) t[j] = (k0 + j < n) ? *proj_ptr(p, k0 + j, b, m) : 0.0f;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (k0 + j < n) s += t[j];
    }
    return s;
}
__device__ __forceinline__ uint16_t f32_to_bf16(float v) {
    return __bfloat16_as_ushort(__float2bfloat16_rn(v));
}

// K3d gathered copy (XgOut): column c of request b
__device__ __forceinline__ void xg_store(const XgOut& xo, int b, int c, uint16_t v) {
    const int j = c & 31;
    xo.xg[static_cast<size_t>(xo.row[b]) * xo.ld + (c & ~31) + (j < 16 ? 2 * j : 2 * (j - 16) + 1)] = v;
}
__device__ __forceinline__ void xg_store4(const XgOut& xo, int b, int c, uint2 pk) {
    xg_store(xo, b, c, uint16_t(pk.x & 0xFFFFu));
    xg_store(xo, b, c + 1, uint16_t(pk.x >> 16));
    xg_store(xo, b, c + 2, uint16_t(pk.y & 0xFFFFu));
    xg_store(xo, b, c + 3, uint16_t(pk.y >> 16));
}

template <typename T>
__device__ T block_sum(T v, T* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    T t = 0;
    for (int i = 0; i < nw; ++i) t += red[i];
    return t;
}
__device__ float block_max(float v, float* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    float t = red[0];
    for (int i = 1; i < nw; ++i) t = fmaxf(t, red[i]);
    return t;
}

// phase 1, grid (chunks, batch): x += proj (optional); per-chunk sum of squares (double)
__global__ void __launch_bounds__(kNormChunk)
    resid_kernel(float* __restrict__ x, int dim, ProjOut proj, double* __restrict__ msq_part) {
    __shared__ double red_d[32];
    const int b = blockIdx.y;
    const int i = blockIdx.x * kNormChunk + threadIdx.x;
    double sq = 0.0;
    if (i < dim) {
        float v = x[size_t(b) * dim + i];
        if (proj.P) {
            v = v + proj_val(proj, b, proj.col0 + i);
            x[size_t(b) * dim + i] = v;
        }
        sq = static_cast<double>(v) * v;
    }
    if (!msq_part) return;
    sq = block_sum(sq, red_d);
    if (threadIdx.x == 0) msq_part[size_t(b) * gridDim.x + blockIdx.x] = sq;
}

// phase 2, grid (chunks, batch): xn = rmsnorm(x) * w_b  (every block re-sums the
// chunk partials of its request in index order -> deterministic)
__global__ void __launch_bounds__(kNormChunk)
    norm_kernel(const float* __restrict__ x, int dim, const double* __restrict__ msq_part,
                const float* const* __restrict__ norm_w, uint16_t* __restrict__ xn, int ldxn,
                float* __restrict__ xn_f32) {
    const int b = blockIdx.y;
    const int i = blockIdx.x * kNormChunk + threadIdx.x;
    double msq = 0.0;
    for (int k = 0; k < int(gridDim.x); ++k) msq += msq_part[size_t(b) * gridDim.x + k];
    const double inv = 1.0 / sqrt(msq / static_cast<double>(dim) + 1e-12);
    if (i >= dim) return;
    const float y = static_cast<float>(static_cast<double>(x[size_t(b) * dim + i]) * inv) * norm_w[b][i];
    if (xn) xn[size_t(b) * ldxn + i] = f32_to_bf16(y);
    if (xn_f32) xn_f32[size_t(b) * dim + i] = y;
}

// ---- default residual + RMSNorm: one launch, chunk partials joined in-kernel ----
// grid (chunks of kRnChunk, batch) = 128 CTAs at dim 4096 / batch 16, all co-resident.
// Every CTA adds the projection partials into its chunk of x (float4), writes its
// double sum of squares, then the CTAs of a request meet on an arrival counter and
// each re-sums the chunk partials in index order (deterministic, no float atomics).
constexpr int kRnThreads = 128, kRnChunk = 4 * kRnThreads;

__device__ __forceinline__ float4 f4_add(float4 a, float4 b) {
    return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
// proj_val for 4 consecutive outputs (same addition order as proj_val -> same bits)
__device__ __forceinline__ float4 proj_val4(const ProjOut& p, int b, int m) {
    if (p.G) {
        const int r = m / p.g_cols, i = m - r * p.g_cols;
        return *reinterpret_cast<const float4*>(p.G + (static_cast<size_t>(r) * p.g_batch + b) * p.g_cols + i);
    }
    const int n = proj_parts(p);
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k0 = 0; k0 < n; k0 += kPartGroup) {
        float4 t[kPartGroup];
#pragma unroll
        for (int j = 0; j < kPartGroup; ++j)
            t[j] = (k0 + j < n) ? *reinterpret_cast<const float4*>(proj_ptr(p, k0 + j, b, m))
                                : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int j = 0; j < kPartGroup; ++j)
            if (k0 + j < n) s = f4_add(s, t[j]);
    }
    return s;
}
// gate and up (same projection, columns m and m + off) with both load sets in flight
__device__ __forceinline__ void proj_val4_pair(const ProjOut& p, int b, int m, int off, float4& g, float4& u) {
    if (p.G) {
        g = proj_val4(p, b, m);
        u = proj_val4(p, b, m + off);
        return;
    }
    constexpr int kG = kPartGroup / 2;
    const int n = proj_parts(p);
    g = make_float4(0.f, 0.f, 0.f, 0.f);
    u = g;
    for (int k0 = 0; k0 < n; k0 += kG) {
        float4 tg[kG], tu[kG];
#pragma unroll
        for (int j = 0; j < kG; ++j) {
            const bool on = k0 + j < n;
            tg[j] = on ? *reinterpret_cast<const float4*>(proj_ptr(p, k0 + j, b, m)) : make_float4(0.f, 0.f, 0.f, 0.f);
            tu[j] = on ? *reinterpret_cast<const float4*>(proj_ptr(p, k0 + j, b, m + off))
                       : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int j = 0; j < kG; ++j)
            if (k0 + j < n) {
                g = f4_add(g, tg[j]);
                u = f4_add(u, tu[j]);
            }
    }
}

__global__ void __launch_bounds__(kRnThreads)
    resid_norm_kernel(float* __restrict__ x, int dim, ProjOut proj, const float* const* __restrict__ norm_w,
                      uint16_t* __restrict__ xn, int ldxn, float* __restrict__ xn_f32,
                      unsigned* __restrict__ arrive, double* __restrict__ msq_part, XgOut xo) {
    __shared__ double red_d[32];
    __shared__ double inv_s;
    const unsigned long long t_entry = gtimer();
    if (BD_PDL_EARLY) griddep_launch_dependents();  // next linear's prologue may start
    griddep_wait();  // PDL: the projection partials come from the previous kernel
    const unsigned long long t_wait = gtimer();
    const int b = blockIdx.y, nc = gridDim.x;
    const int i = blockIdx.x * kRnChunk + 4 * threadIdx.x;
    const bool on = i < dim;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    float* xb = x + size_t(b) * dim;
    if (on) {
        v = *reinterpret_cast<const float4*>(xb + i);
        if (proj.P || proj.G) {
            v = f4_add(v, proj_val4(proj, b, proj.col0 + i));
            *reinterpret_cast<float4*>(xb + i) = v;
        }
    }
    if (!norm_w) return;
    // the tenant's norm row does not depend on the arrival: load it before the sync
    const float4 w = on ? *reinterpret_cast<const float4*>(norm_w[b] + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    double sq = static_cast<double>(v.x) * v.x + static_cast<double>(v.y) * v.y +
                static_cast<double>(v.z) * v.z + static_cast<double>(v.w) * v.w;
    sq = block_sum(sq, red_d);
    if (threadIdx.x == 0) {
        msq_part[size_t(b) * nc + blockIdx.x] = sq;
        __threadfence();
        const unsigned old = atomicAdd(arrive + b, 1u);
        const unsigned target = old - old % unsigned(nc) + unsigned(nc);
        while (static_cast<int>(*reinterpret_cast<volatile unsigned*>(arrive + b) - target) < 0) __nanosleep(20);
        __threadfence();
        double msq = 0.0;
        for (int k = 0; k < nc; ++k) msq += __ldcg(msq_part + size_t(b) * nc + k);
        inv_s = 1.0 / sqrt(msq / static_cast<double>(dim) + 1e-12);
    }
    __syncthreads();
    if (!on) return;
    const double inv = inv_s;
    const float y0 = static_cast<float>(static_cast<double>(v.x) * inv) * w.x;
    const float y1 = static_cast<float>(static_cast<double>(v.y) * inv) * w.y;
    const float y2 = static_cast<float>(static_cast<double>(v.z) * inv) * w.z;
    const float y3 = static_cast<float>(static_cast<double>(v.w) * inv) * w.w;
    if (xn) {
        uint2 pk;
        pk.x = uint32_t(f32_to_bf16(y0)) | (uint32_t(f32_to_bf16(y1)) << 16);
        pk.y = uint32_t(f32_to_bf16(y2)) | (uint32_t(f32_to_bf16(y3)) << 16);
        *reinterpret_cast<uint2*>(xn + size_t(b) * ldxn + i) = pk;
        if (xo.xg) xg_store4(xo, b, i, pk);
    }
    if (xn_f32) *reinterpret_cast<float4*>(xn_f32 + size_t(b) * dim + i) = make_float4(y0, y1, y2, y3);
    if (threadIdx.x == 0) trace_rec(TR_NORM, t_entry, t_wait);
}

// The same with the CTAs of a request as one thread-block cluster (dim <= 8 x kRnChunk): the
// chunk sums of squares meet in distributed shared memory behind a cluster barrier instead of
// a global arrival counter (same addition order -> same bits).
__global__ void __launch_bounds__(kRnThreads)
    resid_norm_cluster_kernel(float* __restrict__ x, int dim, ProjOut proj, const float* const* __restrict__ norm_w,
                              uint16_t* __restrict__ xn, int ldxn, float* __restrict__ xn_f32, XgOut xo) {
    __shared__ double red_d[32];
    __shared__ double part_sq[8];  // chunk k's sum of squares, pushed here by CTA k
    __shared__ double inv_s;
    const unsigned long long t_entry = gtimer();
    griddep_wait();  // PDL: the projection partials come from the previous kernel
    const unsigned long long t_wait = gtimer();
    const int b = blockIdx.y, nc = gridDim.x;
    const int i = blockIdx.x * kRnChunk + 4 * threadIdx.x;
    const bool on = i < dim;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    float* xb = x + size_t(b) * dim;
    if (on) {
        v = *reinterpret_cast<const float4*>(xb + i);
        if (proj.P || proj.G) {
            v = f4_add(v, proj_val4(proj, b, proj.col0 + i));
            *reinterpret_cast<float4*>(xb + i) = v;
        }
    }
    const float4 w = on ? *reinterpret_cast<const float4*>(norm_w[b] + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    double sq = static_cast<double>(v.x) * v.x + static_cast<double>(v.y) * v.y +
                static_cast<double>(v.z) * v.z + static_cast<double>(v.w) * v.w;
    sq = block_sum(sq, red_d);
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    if (threadIdx.x < nc) {  // push this chunk's sum into slot `rank` of every CTA of the request
        const uint32_t local = static_cast<uint32_t>(__cvta_generic_to_shared(&part_sq[rank]));
        uint32_t remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(int(threadIdx.x)));
        asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(remote), "d"(sq) : "memory");
    }
    // one cluster barrier: every push has landed, and no CTA touches another's memory after it
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x == 0) {
        double msq = 0.0;
        for (int k = 0; k < nc; ++k) msq += part_sq[k];  // chunk order (same bits as before)
        inv_s = 1.0 / sqrt(msq / static_cast<double>(dim) + 1e-12);
    }
    __syncthreads();
    if (!on) return;
    const double inv = inv_s;
    const float y0 = static_cast<float>(static_cast<double>(v.x) * inv) * w.x;
    const float y1 = static_cast<float>(static_cast<double>(v.y) * inv) * w.y;
    const float y2 = static_cast<float>(static_cast<double>(v.z) * inv) * w.z;
    const float y3 = static_cast<float>(static_cast<double>(v.w) * inv) * w.w;
    if (xn) {
        uint2 pk;
        pk.x = uint32_t(f32_to_bf16(y0)) | (uint32_t(f32_to_bf16(y1)) << 16);
        pk.y = uint32_t(f32_to_bf16(y2)) | (uint32_t(f32_to_bf16(y3)) << 16);
        *reinterpret_cast<uint2*>(xn + size_t(b) * ldxn + i) = pk;
        if (xo.xg) xg_store4(xo, b, i, pk);
    }
    if (xn_f32) *reinterpret_cast<float4*>(xn_f32 + size_t(b) * dim + i) = make_float4(y0, y1, y2, y3);
    if (threadIdx.x == 0) trace_rec(TR_NORM, t_entry, t_wait);
}

// one block per (head, request): RoPE, KV append, scores, softmax, context
__global__ void attn_kernel(ProjOut qkv, AttnArgs a, const int* __restrict__ pos_dev,
                            uint16_t* __restrict__ ctx_out, int ld_ctx) {
    extern __shared__ float sm[];
    float* qs = sm;                 // hd
    float* ks = qs + a.hd;          // hd (this step's key, bf16-rounded)
    float* vs = ks + a.hd;          // hd
    float* scores = vs + a.hd;      // max_seq
    __shared__ float red[32];
    const int h = blockIdx.x, b = blockIdx.y;
    const int hd = a.hd, half = hd / 2;
    const int group = a.n_heads / a.n_kv_heads;
    const int kh = h / group;
    const int pos = pos_dev[b];
    const float2* rope = a.rope + static_cast<size_t>(pos) * half;
    const int n_ctx = pos + 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const bool vec = (hd % 4) == 0 && (a.kv_dim % 4) == 0;
    const bool fast = vec && hd == 128;
    uint16_t* kc = a.kcache[b] + (static_cast<size_t>(a.layer) * a.max_seq) * a.kv_dim + kh * hd;
    uint16_t* vc = a.vcache[b] + (static_cast<size_t>(a.layer) * a.max_seq) * a.kv_dim + kh * hd;

    // q, k, v of this step (split-K reduction + tenant delta): one element per
    // thread over all 3*hd values, then RoPE on the q and k pairs in smem
    for (int i = threadIdx.x; i < 3 * hd; i += blockDim.x) {
        const int which = i / hd, d = i - which * hd;
        const int col = which == 0 ? h * hd + d : (which == 1 ? a.dim + kh * hd + d : a.dim + a.kv_dim + kh * hd + d);
        const float v = proj_val(qkv, b, col);
        (which == 0 ? qs : (which == 1 ? ks : vs))[d] = which == 2 ? bf16_to_f32(f32_to_bf16(v)) : v;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 2 * half; i += blockDim.x) {
        const int pi = i % half;
        float* buf = i < half ? qs : ks;
        const float2 cs = rope[pi];
        const float v0 = buf[2 * pi], v1 = buf[2 * pi + 1];
        const float r0 = v0 * cs.x - v1 * cs.y, r1 = v0 * cs.y + v1 * cs.x;
        if (i < half) {
            buf[2 * pi] = r0;
            buf[2 * pi + 1] = r1;
        } else {
            buf[2 * pi] = bf16_to_f32(f32_to_bf16(r0));
            buf[2 * pi + 1] = bf16_to_f32(f32_to_bf16(r1));
        }
    }
    __syncthreads();
    if (h % group == 0) {  // KV append (serve.cpp:261-264), post-RoPE
        for (int i = threadIdx.x; i < hd; i += blockDim.x) {
            kc[static_cast<size_t>(pos) * a.kv_dim + i] = f32_to_bf16(ks[i]);
            vc[static_cast<size_t>(pos) * a.kv_dim + i] = f32_to_bf16(vs[i]);
        }
    }
    // scores (serve.cpp:267-275): one warp per key, lane l owns dims [4l, 4l+4) (+128k),
    // 8-byte loads -> each key row is one coalesced 256-byte warp access
    const float inv_sqrt_hd = 1.0f / sqrtf(static_cast<float>(hd));
    if (fast) {
        // fast path: 8 keys per warp in flight (all loads issued before the math)
        const float q0 = qs[4 * lane], q1 = qs[4 * lane + 1], q2 = qs[4 * lane + 2], q3 = qs[4 * lane + 3];
        for (int j0 = warp; j0 < n_ctx; j0 += nw * 8) {
            uint2 u[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const int j = j0 + t * nw;
                u[t] = (j < n_ctx && j != pos)
                           ? *reinterpret_cast<const uint2*>(kc + static_cast<size_t>(j) * a.kv_dim + 4 * lane)
                           : make_uint2(0u, 0u);
            }
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const int j = j0 + t * nw;
                float acc;
                if (j == pos)
                    acc = q0 * ks[4 * lane] + q1 * ks[4 * lane + 1] + q2 * ks[4 * lane + 2] + q3 * ks[4 * lane + 3];
                else
                    acc = q0 * __uint_as_float(u[t].x << 16) + q1 * __uint_as_float(u[t].x & 0xFFFF0000u) +
                          q2 * __uint_as_float(u[t].y << 16) + q3 * __uint_as_float(u[t].y & 0xFFFF0000u);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                if (lane == 0 && j < n_ctx) scores[j] = acc * inv_sqrt_hd;
            }
        }
    } else
    for (int j = warp; j < n_ctx; j += nw) {
        float acc = 0.0f;
        if (j == pos) {
            for (int d = lane; d < hd; d += 32) acc += qs[d] * ks[d];
        } else if (vec) {
            const uint16_t* kj = kc + static_cast<size_t>(j) * a.kv_dim;
            for (int d0 = 4 * lane; d0 < hd; d0 += 128) {
                const uint2 u = *reinterpret_cast<const uint2*>(kj + d0);
                acc += qs[d0] * __uint_as_float(u.x << 16) + qs[d0 + 1] * __uint_as_float(u.x & 0xFFFF0000u) +
                       qs[d0 + 2] * __uint_as_float(u.y << 16) + qs[d0 + 3] * __uint_as_float(u.y & 0xFFFF0000u);
            }
        } else {
            const uint16_t* kj = kc + static_cast<size_t>(j) * a.kv_dim;
            for (int d = lane; d < hd; d += 32) acc += qs[d] * bf16_to_f32(kj[d]);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) scores[j] = acc * inv_sqrt_hd;
    }
    __syncthreads();
    // softmax (nn_ops.hpp:48-57)
    float mx = -INFINITY;
    for (int j = threadIdx.x; j < n_ctx; j += blockDim.x) mx = fmaxf(mx, scores[j]);
    mx = block_max(mx, red);
    float sum = 0.0f;
    for (int j = threadIdx.x; j < n_ctx; j += blockDim.x) {
        const float e = expf(scores[j] - mx);
        scores[j] = e;
        sum += e;
    }
    sum = block_sum(sum, red);
    __syncthreads();
    // ctx (serve.cpp:276-281): p_j = e_j / sum as in the reference; warp w sums the
    // positions j = w (mod nw) for dims [4l, 4l+4), then the warps' partials are
    // added in warp order (fixed) through shared memory
    float* part = scores + a.max_seq;  // [nw][hd]
    if (fast) {
        // fast path: 8 value rows per warp in flight
        float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        for (int j0 = warp; j0 < n_ctx; j0 += nw * 8) {
            uint2 u[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const int j = j0 + t * nw;
                u[t] = (j < n_ctx && j != pos)
                           ? *reinterpret_cast<const uint2*>(vc + static_cast<size_t>(j) * a.kv_dim + 4 * lane)
                           : make_uint2(0u, 0u);
            }
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                const int j = j0 + t * nw;
                if (j >= n_ctx) break;
                const float pj = scores[j] / sum;
                float v[4];
                if (j == pos) {
#pragma unroll
                    for (int e = 0; e < 4; ++e) v[e] = vs[4 * lane + e];
                } else {
                    v[0] = __uint_as_float(u[t].x << 16);
                    v[1] = __uint_as_float(u[t].x & 0xFFFF0000u);
                    v[2] = __uint_as_float(u[t].y << 16);
                    v[3] = __uint_as_float(u[t].y & 0xFFFF0000u);
                }
#pragma unroll
                for (int e = 0; e < 4; ++e) acc[e] += pj * v[e];
            }
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) part[warp * hd + 4 * lane + e] = acc[e];
    } else
    for (int d0 = 4 * lane; d0 < hd; d0 += 128) {
        float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        for (int j = warp; j < n_ctx; j += nw) {
            const float pj = scores[j] / sum;
            float v[4];
            if (j == pos) {
#pragma unroll
                for (int e = 0; e < 4; ++e) v[e] = d0 + e < hd ? vs[d0 + e] : 0.0f;
            } else if (vec) {
                const uint2 u = *reinterpret_cast<const uint2*>(vc + static_cast<size_t>(j) * a.kv_dim + d0);
                v[0] = __uint_as_float(u.x << 16);
                v[1] = __uint_as_float(u.x & 0xFFFF0000u);
                v[2] = __uint_as_float(u.y << 16);
                v[3] = __uint_as_float(u.y & 0xFFFF0000u);
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    v[e] = d0 + e < hd ? bf16_to_f32(vc[static_cast<size_t>(j) * a.kv_dim + d0 + e]) : 0.0f;
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[e] += pj * v[e];
        }
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (d0 + e < hd) part[warp * hd + d0 + e] = acc[e];
    }
    __syncthreads();
    for (int d = threadIdx.x; d < hd; d += blockDim.x) {
        float acc = 0.0f;
        for (int w = 0; w < nw; ++w) acc += part[w * hd + d];
        ctx_out[size_t(b) * ld_ctx + h * hd + d] = f32_to_bf16(acc);
    }
}

// head_dim 128 path. The cached K and V rows of the (request, head) are copied
// into shared memory with cp.async at kernel start (they do not depend on this
// step), so the whole context is in flight at once while q/k/v are reduced; a
// context longer than the staging buffer is processed in chunks (K pass, then
// V pass). Thread t owns dims [8 (t%16), +8) of rows t/16 (mod 16). Same math
// as attn_kernel, different f32 summation order.
constexpr int kA2Threads = 256;

__device__ __forceinline__ void bf16x8_to_f32(const uint4 u, float (&f)[8]) {
    f[0] = __uint_as_float(u.x << 16); f[1] = __uint_as_float(u.x & 0xFFFF0000u);
    f[2] = __uint_as_float(u.y << 16); f[3] = __uint_as_float(u.y & 0xFFFF0000u);
    f[4] = __uint_as_float(u.z << 16); f[5] = __uint_as_float(u.z & 0xFFFF0000u);
    f[6] = __uint_as_float(u.w << 16); f[7] = __uint_as_float(u.w & 0xFFFF0000u);
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
                 "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// rows [r0, r0 + n) of one head (256 B each, row stride ld elements) -> dst[n][128]
__device__ __forceinline__ void stage_rows(uint16_t* dst, const uint16_t* src, int r0, int n, int ld) {
    for (int i = threadIdx.x; i < n * 16; i += kA2Threads) {
        const int r = i >> 4, c = i & 15;
        cp_async16(dst + r * 128 + 8 * c, src + static_cast<size_t>(r0 + r) * ld + 8 * c);
    }
}

__global__ void __launch_bounds__(kA2Threads)
    attn128_kernel(ProjOut qkv, AttnArgs a, const int* __restrict__ pos_dev, uint16_t* __restrict__ ctx_out,
                   int ld_ctx, int stage_rows_max) {
    constexpr int hd = 128, half = 64;
    extern __shared__ __align__(16) float sm[];
    float* qs = sm;                  // hd
    float* ks = qs + hd;             // hd (this step's key, bf16-rounded)
    float* vs = ks + hd;             // hd
    uint16_t* st = reinterpret_cast<uint16_t*>(vs + hd);            // [stage_rows_max][hd]: K, then V, then partials
    float* scores = reinterpret_cast<float*>(st + stage_rows_max * hd);  // max_seq
    __shared__ float red[32];
    const unsigned long long t_entry = gtimer();
    if (BD_PDL_EARLY) griddep_launch_dependents();  // next linear's prologue may start
    const int h = blockIdx.x, b = blockIdx.y;
    const int group = a.n_heads / a.n_kv_heads;
    const int kh = h / group;
    const int pos = pos_dev[b];  // uploaded before the step's first kernel
    const int n_ctx = pos + 1;
    const int rs = threadIdx.x >> 4, dg = threadIdx.x & 15;
    uint16_t* kc = a.kcache[b] + (static_cast<size_t>(a.layer) * a.max_seq) * a.kv_dim + kh * hd;
    uint16_t* vc = a.vcache[b] + (static_cast<size_t>(a.layer) * a.max_seq) * a.kv_dim + kh * hd;
    // The cached rows are from earlier steps: staged before waiting for the predecessor.
    // Row `pos` is this step's own key/value (taken from smem below, never read from the cache).
    stage_rows(st, kc, 0, min(n_ctx, stage_rows_max), a.kv_dim);
    griddep_wait();  // PDL: q/k/v partials come from the previous kernel
    const unsigned long long t_wait = gtimer();

    // q, k, v of this step (split-K + tenant delta), RoPE (same as attn_kernel)
    const float2* rope = a.rope + static_cast<size_t>(pos) * half;
    for (int i = threadIdx.x; i < 3 * hd; i += kA2Threads) {
        const int which = i / hd, d = i - which * hd;
        const int col = which == 0 ? h * hd + d : (which == 1 ? a.dim + kh * hd + d : a.dim + a.kv_dim + kh * hd + d);
        const float v = proj_val(qkv, b, col);
        (which == 0 ? qs : (which == 1 ? ks : vs))[d] = which == 2 ? bf16_to_f32(f32_to_bf16(v)) : v;
    }
    __syncthreads();
    if (threadIdx.x < 2 * half) {
        const int i = threadIdx.x, pi = i % half;
        float* buf = i < half ? qs : ks;
        const float2 cs = rope[pi];
        const float v0 = buf[2 * pi], v1 = buf[2 * pi + 1];
        const float r0 = v0 * cs.x - v1 * cs.y, r1 = v0 * cs.y + v1 * cs.x;
        if (i < half) {
            buf[2 * pi] = r0;
            buf[2 * pi + 1] = r1;
        } else {
            buf[2 * pi] = bf16_to_f32(f32_to_bf16(r0));
            buf[2 * pi + 1] = bf16_to_f32(f32_to_bf16(r1));
        }
    }
    cp_async_wait_all();
    __syncthreads();
    if (h % group == 0 && threadIdx.x < hd) {  // KV append (serve.cpp:261-264), post-RoPE
        kc[static_cast<size_t>(pos) * a.kv_dim + threadIdx.x] = f32_to_bf16(ks[threadIdx.x]);
        vc[static_cast<size_t>(pos) * a.kv_dim + threadIdx.x] = f32_to_bf16(vs[threadIdx.x]);
    }
    // scores (serve.cpp:267-275)
    const float inv_sqrt_hd = 1.0f / sqrtf(static_cast<float>(hd));
    float q[8], kn[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        q[e] = qs[8 * dg + e];
        kn[e] = ks[8 * dg + e];
    }
    for (int c0 = 0; c0 < n_ctx; c0 += stage_rows_max) {
        const int nr = min(stage_rows_max, n_ctx - c0);
        if (c0) {
            __syncthreads();  // previous chunk consumed
            stage_rows(st, kc, c0, nr, a.kv_dim);
            cp_async_wait_all();
            __syncthreads();
        }
        for (int rb = 0; rb < nr; rb += 16) {  // warp-uniform trip count (shuffles below)
            const int r = rb + rs, j = c0 + r;
            float k8[8];
            bf16x8_to_f32(r < nr ? *reinterpret_cast<const uint4*>(st + r * hd + 8 * dg) : make_uint4(0u, 0u, 0u, 0u),
                          k8);
            float acc = 0.0f;
#pragma unroll
            for (int e = 0; e < 8; ++e) acc += q[e] * (j == pos ? kn[e] : k8[e]);
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (dg == 0 && r < nr) scores[j] = acc * inv_sqrt_hd;
        }
    }
    __syncthreads();
    // the first V chunk streams in while the softmax runs
    stage_rows(st, vc, 0, min(n_ctx, stage_rows_max), a.kv_dim);
    // softmax (nn_ops.hpp:48-57)
    float mx = -INFINITY;
    for (int j = threadIdx.x; j < n_ctx; j += kA2Threads) mx = fmaxf(mx, scores[j]);
    mx = block_max(mx, red);
    float sum = 0.0f;
    for (int j = threadIdx.x; j < n_ctx; j += kA2Threads) {
        const float e = expf(scores[j] - mx);
        scores[j] = e;
        sum += e;
    }
    sum = block_sum(sum, red);
    // p_j = e_j / sum once per row (not once per row and dims group in the PV loop)
    for (int j = threadIdx.x; j < n_ctx; j += kA2Threads) scores[j] = scores[j] / sum;
    cp_async_wait_all();
    __syncthreads();
    // ctx (serve.cpp:276-281): p_j = e_j / sum; row-slot partials added in slot order
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    float vn[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) vn[e] = vs[8 * dg + e];
    for (int c0 = 0; c0 < n_ctx; c0 += stage_rows_max) {
        const int nr = min(stage_rows_max, n_ctx - c0);
        if (c0) {
            __syncthreads();
            stage_rows(st, vc, c0, nr, a.kv_dim);
            cp_async_wait_all();
            __syncthreads();
        }
        for (int r = rs; r < nr; r += 16) {
            const int j = c0 + r;
            const float pj = scores[j];
            float v8[8];
            bf16x8_to_f32(*reinterpret_cast<const uint4*>(st + r * hd + 8 * dg), v8);
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[e] += pj * (j == pos ? vn[e] : v8[e]);
        }
    }
    __syncthreads();  // staging buffer reused for the row-slot partials [16][hd] f32
    float* part = reinterpret_cast<float*>(st);
#pragma unroll
    for (int e = 0; e < 8; ++e) part[rs * hd + 8 * dg + e] = acc[e];
    __syncthreads();
    if (threadIdx.x < hd) {
        float t = 0.0f;
#pragma unroll
        for (int r = 0; r < 16; ++r) t += part[r * hd + threadIdx.x];
        const uint16_t v = f32_to_bf16(t);
        ctx_out[size_t(b) * ld_ctx + h * hd + threadIdx.x] = v;
        if (a.xo.xg) xg_store(a.xo, b, h * hd + threadIdx.x, v);
    }
    if (threadIdx.x == 0) trace_rec(TR_ATTN, t_entry, t_wait);
}

// block_max (kMax) / block_sum of G values at once, each in their order
template <int G, bool kMax>
__device__ __forceinline__ void block_reduce_g(float (&v)[G], float* red) {
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float w = __shfl_xor_sync(0xffffffffu, v[g], o);
            v[g] = kMax ? fmaxf(v[g], w) : v[g] + w;
        }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
    __syncthreads();
    if (l == 0)
#pragma unroll
        for (int g = 0; g < G; ++g) red[g * 32 + w] = v[g];
    __syncthreads();
#pragma unroll
    for (int g = 0; g < G; ++g) {
        float t = kMax ? red[g * 32] : 0.0f;
        for (int i = kMax ? 1 : 0; i < nw; ++i) t = kMax ? fmaxf(t, red[g * 32 + i]) : t + red[g * 32 + i];
        v[g] = t;
    }
}

// Grouped-query attention (kv_dim < dim, BASELINE configs[3] / [4]): one CTA per (request, KV
// head) runs the G query heads that share it, so each cached K / V row is staged into shared
// memory once instead of once per query head (G x fewer CTAs and K/V transfers). Per head the
// arithmetic and summation order are attn128_kernel's, so the outputs are bit-identical.
// G <= 4: <= 64 registers, so 4 CTAs share an SM and batch 64 x 8 KV heads = 512 CTAs run as
// one wave on 148 SMs (at 80 registers the last 68 CTAs formed a second wave: +15 us per layer)
template <int G>
__global__ void __launch_bounds__(kA2Threads, G <= 4 ? 4 : 2)
    attn128g_kernel(ProjOut qkv, AttnArgs a, const int* __restrict__ pos_dev, uint16_t* __restrict__ ctx_out,
                    int ld_ctx, int stage_rows_max) {
    constexpr int hd = 128, half = 64;
    extern __shared__ __align__(16) float sm[];
    float* qs = sm;                  // [G][hd]
    float* ks = qs + G * hd;         // hd (this step's key, bf16-rounded)
    float* vs = ks + hd;             // hd
    uint16_t* st = reinterpret_cast<uint16_t*>(vs + hd);                 // [stage_rows_max][hd]: K, then V, then partials
    float* scores = reinterpret_cast<float*>(st + stage_rows_max * hd);  // [G][max_seq]
    __shared__ float redg[G * 32];
    const unsigned long long t_entry = gtimer();
    if (BD_PDL_EARLY) griddep_launch_dependents();  // next linear's prologue may start
    const int kh = blockIdx.x, b = blockIdx.y;
    const int pos = pos_dev[b];
    const int n_ctx = pos + 1;
    const int rs = threadIdx.x >> 4, dg = threadIdx.x & 15;
    uint16_t* kc = a.kcache[b] + (static_cast<size_t>(a.layer) * a.max_seq) * a.kv_dim + kh * hd;
    uint16_t* vc = a.vcache[b] + (static_cast<size_t>(a.layer) * a.max_seq) * a.kv_dim + kh * hd;
    stage_rows(st, kc, 0, min(n_ctx, stage_rows_max), a.kv_dim);  // earlier steps' rows: before the wait
    griddep_wait();  // PDL: q/k/v partials come from the previous kernel
    const unsigned long long t_wait = gtimer();

    const float2* rope = a.rope + static_cast<size_t>(pos) * half;
    for (int i = threadIdx.x; i < (G + 2) * hd; i += kA2Threads) {
        const int which = i / hd, d = i - which * hd;  // < G: query head kh G + which; G: key; G + 1: value
        const int col = which < G ? (kh * G + which) * hd + d
                                  : (which == G ? a.dim + kh * hd + d : a.dim + a.kv_dim + kh * hd + d);
        const float v = proj_val(qkv, b, col);
        (which < G ? qs + which * hd : (which == G ? ks : vs))[d] = which == G + 1 ? bf16_to_f32(f32_to_bf16(v)) : v;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < (G + 1) * half; i += kA2Threads) {
        const int which = i / half, pi = i - which * half;
        float* buf = which < G ? qs + which * hd : ks;
        const float2 cs = rope[pi];
        const float v0 = buf[2 * pi], v1 = buf[2 * pi + 1];
        const float r0 = v0 * cs.x - v1 * cs.y, r1 = v0 * cs.y + v1 * cs.x;
        if (which < G) {
            buf[2 * pi] = r0;
            buf[2 * pi + 1] = r1;
        } else {
            buf[2 * pi] = bf16_to_f32(f32_to_bf16(r0));
            buf[2 * pi + 1] = bf16_to_f32(f32_to_bf16(r1));
        }
    }
    cp_async_wait_all();
    __syncthreads();
    if (threadIdx.x < hd) {  // KV append (serve.cpp:261-264), post-RoPE
        kc[static_cast<size_t>(pos) * a.kv_dim + threadIdx.x] = f32_to_bf16(ks[threadIdx.x]);
        vc[static_cast<size_t>(pos) * a.kv_dim + threadIdx.x] = f32_to_bf16(vs[threadIdx.x]);
    }
    const float inv_sqrt_hd = 1.0f / sqrtf(static_cast<float>(hd));
    float q[G][8], kn[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
#pragma unroll
        for (int g = 0; g < G; ++g) q[g][e] = qs[g * hd + 8 * dg + e];
        kn[e] = ks[8 * dg + e];
    }
    for (int c0 = 0; c0 < n_ctx; c0 += stage_rows_max) {
        const int nr = min(stage_rows_max, n_ctx - c0);
        if (c0) {
            __syncthreads();
            stage_rows(st, kc, c0, nr, a.kv_dim);
            cp_async_wait_all();
            __syncthreads();
        }
        for (int rb = 0; rb < nr; rb += 16) {
            const int r = rb + rs, j = c0 + r;
            float k8[8];
            bf16x8_to_f32(r < nr ? *reinterpret_cast<const uint4*>(st + r * hd + 8 * dg) : make_uint4(0u, 0u, 0u, 0u),
                          k8);
#pragma unroll
            if (j == pos)
#pragma unroll
                for (int e = 0; e < 8; ++e) k8[e] = kn[e];
#pragma unroll
            for (int g = 0; g < G; ++g) {
                float acc = 0.0f;
#pragma unroll
                for (int e = 0; e < 8; ++e) acc += q[g][e] * k8[e];
#pragma unroll
                for (int o = 8; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                if (dg == 0 && r < nr) scores[g * a.max_seq + j] = acc * inv_sqrt_hd;
            }
        }
    }
    __syncthreads();
    stage_rows(st, vc, 0, min(n_ctx, stage_rows_max), a.kv_dim);  // streams in during the softmax
    // softmax of the G heads with one pair of block reductions (per head the order of
    // block_max / block_sum)
    float mx[G], sum[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        mx[g] = -INFINITY;
        for (int j = threadIdx.x; j < n_ctx; j += kA2Threads) mx[g] = fmaxf(mx[g], scores[g * a.max_seq + j]);
    }
    block_reduce_g<G, true>(mx, redg);
#pragma unroll
    for (int g = 0; g < G; ++g) {
        float* sc = scores + g * a.max_seq;
        sum[g] = 0.0f;
        for (int j = threadIdx.x; j < n_ctx; j += kA2Threads) {
            const float e = expf(sc[j] - mx[g]);
            sc[j] = e;
            sum[g] += e;
        }
    }
    block_reduce_g<G, false>(sum, redg);
    // p_j = e_j / sum once per row and head (not in the PV loop)
#pragma unroll
    for (int g = 0; g < G; ++g)
        for (int j = threadIdx.x; j < n_ctx; j += kA2Threads) scores[g * a.max_seq + j] = scores[g * a.max_seq + j] / sum[g];
    cp_async_wait_all();
    __syncthreads();
    float acc[G][8];
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[g][e] = 0.0f;
    float vn[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) vn[e] = vs[8 * dg + e];
    for (int c0 = 0; c0 < n_ctx; c0 += stage_rows_max) {
        const int nr = min(stage_rows_max, n_ctx - c0);
        if (c0) {
            __syncthreads();
            stage_rows(st, vc, c0, nr, a.kv_dim);
            cp_async_wait_all();
            __syncthreads();
        }
        for (int r = rs; r < nr; r += 16) {
            const int j = c0 + r;
            float v8[8];
            bf16x8_to_f32(*reinterpret_cast<const uint4*>(st + r * hd + 8 * dg), v8);
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const float pj = scores[g * a.max_seq + j];
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[g][e] += pj * (j == pos ? vn[e] : v8[e]);
            }
        }
    }
    float* part = reinterpret_cast<float*>(st);  // f32 row-slot partials [heads][16][hd]
    if (stage_rows_max * hd * 2 >= G * 16 * hd * 4) {  // all G heads in one pass
        __syncthreads();
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
            for (int e = 0; e < 8; ++e) part[(g * 16 + rs) * hd + 8 * dg + e] = acc[g][e];
        __syncthreads();
        for (int i = threadIdx.x; i < G * hd; i += kA2Threads) {
            const int g = i / hd, d = i - g * hd;
            float t = 0.0f;
#pragma unroll
            for (int r = 0; r < 16; ++r) t += part[(g * 16 + r) * hd + d];
            const uint16_t v = f32_to_bf16(t);
            ctx_out[size_t(b) * ld_ctx + (kh * G + g) * hd + d] = v;
            if (a.xo.xg) xg_store(a.xo, b, (kh * G + g) * hd + d, v);
        }
    } else {
#pragma unroll
        for (int g = 0; g < G; ++g) {
            __syncthreads();
#pragma unroll
            for (int e = 0; e < 8; ++e) part[rs * hd + 8 * dg + e] = acc[g][e];
            __syncthreads();
            if (threadIdx.x < hd) {
                float t = 0.0f;
#pragma unroll
                for (int r = 0; r < 16; ++r) t += part[r * hd + threadIdx.x];
                const uint16_t v = f32_to_bf16(t);
                ctx_out[size_t(b) * ld_ctx + (kh * G + g) * hd + threadIdx.x] = v;
                if (a.xo.xg) xg_store(a.xo, b, (kh * G + g) * hd + threadIdx.x, v);
            }
        }
    }
    if (threadIdx.x == 0) trace_rec(TR_ATTN, t_entry, t_wait);
}

// act = silu(gate) * up (serve.cpp:301-302)
__global__ void silu_kernel(ProjOut gu, int inter, uint16_t* __restrict__ act, int ld_act) {
    const int b = blockIdx.y;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < inter; i += gridDim.x * blockDim.x) {
        const float g = proj_val(gu, b, i);
        const float u = proj_val(gu, b, inter + i);
        const float s = g / (1.0f + expf(-g));
        act[size_t(b) * ld_act + i] = f32_to_bf16(s * u);
    }
}
// 4 outputs per thread (aligned shapes), same per-element arithmetic
__global__ void silu4_kernel(ProjOut gu, int inter, uint16_t* __restrict__ act, int ld_act, XgOut xo) {
    const unsigned long long t_entry = gtimer();
    if (BD_PDL_EARLY) griddep_launch_dependents();  // next linear's prologue may start
    griddep_wait();  // PDL: gate/up partials come from the previous kernel
    const unsigned long long t_wait = gtimer();
    const int b = blockIdx.y;
    for (int i = 4 * (blockIdx.x * blockDim.x + threadIdx.x); i < inter; i += 4 * gridDim.x * blockDim.x) {
        float4 g, u;
        proj_val4_pair(gu, b, i, inter, g, u);
        auto f = [](float gv, float uv) { return f32_to_bf16(gv / (1.0f + expf(-gv)) * uv); };
        uint2 pk;
        pk.x = uint32_t(f(g.x, u.x)) | (uint32_t(f(g.y, u.y)) << 16);
        pk.y = uint32_t(f(g.z, u.z)) | (uint32_t(f(g.w, u.w)) << 16);
        *reinterpret_cast<uint2*>(act + size_t(b) * ld_act + i) = pk;
        if (xo.xg) xg_store4(xo, b, i, pk);
    }
    if (threadIdx.x == 0) trace_rec(TR_SILU, t_entry, t_wait);
}

// x[b] = embed[tok_b] + raw embed delta row (serve.cpp:230-236)
__global__ void embed_kernel(const float* __restrict__ embed, const int* __restrict__ tokens,
                             const float* const* __restrict__ embed_delta, int dim,
                             float* __restrict__ x) {
    const int b = blockIdx.x;
    const size_t tok = static_cast<size_t>(tokens[b]);
    const float* d = embed_delta ? embed_delta[b] : nullptr;
    for (int i = threadIdx.x; i < dim; i += blockDim.x) {
        float v = embed[tok * dim + i];
        if (d) v += d[tok * dim + i];
        x[size_t(b) * dim + i] = v;
    }
}

// logits[b][r] = proj(b, r) + raw lm_head delta row . xn_f32[b]  (serve.cpp:316-320)
__global__ void logits_kernel(ProjOut lm, const float* const* __restrict__ raw_delta,
                              const float* __restrict__ xn_f32, int dim, int vocab,
                              float* __restrict__ logits) {
    const int b = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float* rd = raw_delta ? raw_delta[b] : nullptr;
    for (int r = blockIdx.x * (blockDim.x >> 5) + warp; r < vocab; r += gridDim.x * (blockDim.x >> 5)) {
        float acc = 0.0f;
        if (rd)
            for (int c = lane; c < dim; c += 32) acc += rd[size_t(r) * dim + c] * xn_f32[size_t(b) * dim + c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) logits[size_t(b) * vocab + r] = proj_val(lm, b, r) + acc;
    }
}

__global__ void shard_reduce_kernel(ProjOut p, int batch, int n_l, float* __restrict__ dst) {
    const size_t n = static_cast<size_t>(batch) * n_l;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        dst[i] = proj_val(p, static_cast<int>(i / n_l), static_cast<int>(i % n_l));
}

__global__ void gather_transpose_kernel(const uint16_t* __restrict__ src, int world, int batch, int n_l,
                                        uint16_t* __restrict__ dst, int ld) {
    const size_t n = static_cast<size_t>(world) * batch * n_l;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        const size_t r = i / (static_cast<size_t>(batch) * n_l);
        const size_t rem = i - r * batch * n_l;
        const size_t b = rem / n_l, c = rem % n_l;
        dst[b * ld + r * n_l + c] = src[i];
    }
}

}  // namespace

void shard_reduce_launch(const ProjOut& p, int batch, int n_l, float* dst, cudaStream_t s) {
    const size_t n = static_cast<size_t>(batch) * n_l;
    shard_reduce_kernel<<<static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 1184)), 256, 0, s>>>(p, batch, n_l, dst);
    note_launch();
    BD_CUDA(cudaGetLastError());
}

void gather_transpose_launch(const uint16_t* src, int world, int batch, int n_l, uint16_t* dst, int ld,
                             cudaStream_t s) {
    const size_t n = static_cast<size_t>(world) * batch * n_l;
    gather_transpose_kernel<<<static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 1184)), 256, 0, s>>>(
        src, world, batch, n_l, dst, ld);
    note_launch();
    BD_CUDA(cudaGetLastError());
}

int norm_chunks(int dim) { return (dim + kNormChunk - 1) / kNormChunk; }

namespace {
bool proj_vec4_ok(const ProjOut& p) {
    if (p.G) return p.g_cols % 4 == 0 && reinterpret_cast<uintptr_t>(p.G) % 16 == 0;
    if (!p.P) return true;
    return p.M % 4 == 0 && p.col0 % 4 == 0 && p.pstride % 4 == 0 && reinterpret_cast<uintptr_t>(p.P) % 16 == 0 &&
           (!p.D || (p.dstride % 4 == 0 && reinterpret_cast<uintptr_t>(p.D) % 16 == 0));
}
}  // namespace

size_t norm_ws_bytes(int batch, int dim) {
    const size_t cnt = (size_t(batch) * sizeof(unsigned) + 255) / 256 * 256;
    return cnt + size_t(batch) * std::max(norm_chunks(dim), (dim + kRnChunk - 1) / kRnChunk) * sizeof(double);
}

bool resid_norm_launch(float* x, int batch, int dim, const ProjOut& proj, const float* const* norm_w,
                       uint16_t* xn, int ldxn, float* xn_f32, void* ws, cudaStream_t s, const XgOut& xo) {
    unsigned* arrive = static_cast<unsigned*>(ws);
    double* msq_ws = reinterpret_cast<double*>(static_cast<char*>(ws) +
                                               (size_t(batch) * sizeof(unsigned) + 255) / 256 * 256);
    // one-launch path: the CTAs of a request meet on an arrival counter, so the whole
    // grid must be co-resident (<= 8 CTAs per SM here) -> bounded grid size
    const int nc = (dim + kRnChunk - 1) / kRnChunk;
    if (norm_w && dim % 4 == 0 && ldxn % 4 == 0 && proj_vec4_ok(proj) && nc >= 2 && nc <= 8) {
        BD_CUDA(launch_pdl_cluster(resid_norm_cluster_kernel, dim3(nc, batch), dim3(kRnThreads), 0, s, unsigned(nc),
                                   x, dim, proj, norm_w, xn, ldxn, xn_f32, xo));
        note_launch();
        BD_CUDA(cudaGetLastError());
        return xo.xg != nullptr;
    }
    if (dim % 4 == 0 && ldxn % 4 == 0 && proj_vec4_ok(proj) &&
        size_t(nc) * batch <= size_t(kNumSMs) * 8) {
        BD_CUDA(launch_pdl(resid_norm_kernel, dim3(nc, batch), dim3(kRnThreads), 0, s, x, dim, proj, norm_w, xn,
                           ldxn, xn_f32, arrive, msq_ws, xo));
        note_launch();
        BD_CUDA(cudaGetLastError());
        return xo.xg != nullptr;
    }
    // two-phase fallback (unaligned shapes / grids too wide to be co-resident)
    const dim3 grid(norm_chunks(dim), batch);
    resid_kernel<<<grid, kNormChunk, 0, s>>>(x, dim, proj, norm_w ? msq_ws : nullptr);
    note_launch();
    BD_CUDA(cudaGetLastError());
    if (!norm_w) return false;
    norm_kernel<<<grid, kNormChunk, 0, s>>>(x, dim, msq_ws, norm_w, xn, ldxn, xn_f32);
    note_launch();
    BD_CUDA(cudaGetLastError());
    return false;
}

bool attn_launch(const ProjOut& qkv, const AttnArgs& a, const int* pos_dev, int batch,
                 uint16_t* ctx, int ld_ctx, cudaStream_t s) {
    const int group = a.n_heads / a.n_kv_heads;
    const int g_rows = std::min(192, std::max(32, a.max_seq));
    const size_t g_smem =
        ((group + 2) * 128 + size_t(group) * a.max_seq) * sizeof(float) + size_t(g_rows) * 128 * 2;
    // (score buffers of G heads too large for shared memory: one CTA per query head below)
    if (a.hd == 128 && a.kv_dim % 8 == 0 && a.dim % 8 == 0 && (group == 2 || group == 4 || group == 8) &&
        g_smem <= 220 * 1024) {
        // grouped-query heads: one CTA per (request, KV head), K / V staged once for the group
        const int rows = g_rows;
        const size_t smem = g_smem;
        static bool attr[3] = {false, false, false};
        auto launch = [&](auto kern, int gi) {
            if (!attr[gi]) {
                BD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
                attr[gi] = true;
            }
            BD_CUDA(launch_pdl(kern, dim3(a.n_kv_heads, batch), dim3(kA2Threads), smem, s, qkv, a, pos_dev, ctx, ld_ctx,
                               rows));
        };
        if (group == 2) launch(attn128g_kernel<2>, 0);
        else if (group == 4) launch(attn128g_kernel<4>, 1);
        else launch(attn128g_kernel<8>, 2);
        note_launch();
        BD_CUDA(cudaGetLastError());
        return a.xo.xg != nullptr;
    }
    if (a.hd == 128 && a.kv_dim % 8 == 0 && a.dim % 8 == 0) {
        // one staging buffer of up to 192 rows (48 KB: K, then V): four CTAs per SM,
        // so batch x heads = 512 CTAs run as a single wave on 148 SMs
        const int rows = std::min(192, std::max(32, a.max_seq));
        const size_t smem = (3 * 128 + size_t(a.max_seq)) * sizeof(float) + size_t(rows) * 128 * 2;
        static bool attr2 = false;
        if (!attr2) {
            BD_CUDA(cudaFuncSetAttribute(attn128_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
            attr2 = true;
        }
        require(smem <= 220 * 1024, BD_ERR_BAD_ARGUMENT, "attention: max_seq too large for the score buffer");
        BD_CUDA(launch_pdl(attn128_kernel, dim3(a.n_heads, batch), dim3(kA2Threads), smem, s, qkv, a, pos_dev, ctx,
                           ld_ctx, rows));
        note_launch();
        BD_CUDA(cudaGetLastError());
        return a.xo.xg != nullptr;
    }
    constexpr int kAttnThreads = 256;
    const size_t smem = (3 * a.hd + a.max_seq + (kAttnThreads / 32) * a.hd) * sizeof(float);
    static bool attr = false;
    if (!attr) {
        BD_CUDA(cudaFuncSetAttribute(attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = true;
    }
    attn_kernel<<<dim3(a.n_heads, batch), kAttnThreads, smem, s>>>(qkv, a, pos_dev, ctx, ld_ctx);
    note_launch();
    BD_CUDA(cudaGetLastError());
    return false;
}

bool silu_launch(const ProjOut& gu, int batch, int inter, uint16_t* act, int ld_act, cudaStream_t s,
                 const XgOut& xo) {
    if (inter % 4 == 0 && ld_act % 4 == 0 && proj_vec4_ok(gu)) {
        const int bx = std::max(1, std::min((inter / 4 + 127) / 128, 64));
        BD_CUDA(launch_pdl(silu4_kernel, dim3(bx, batch), dim3(128), 0, s, gu, inter, act, ld_act, xo));
    } else {
        const int bx = std::max(1, std::min((inter + 255) / 256, 64));
        silu_kernel<<<dim3(bx, batch), 256, 0, s>>>(gu, inter, act, ld_act);
    }
    note_launch();
    BD_CUDA(cudaGetLastError());
    return xo.xg != nullptr && inter % 4 == 0 && ld_act % 4 == 0 && proj_vec4_ok(gu);
}

void embed_launch(const float* embed, const int* tokens, const float* const* embed_delta, int batch,
                  int dim, float* x, cudaStream_t s) {
    embed_kernel<<<batch, 256, 0, s>>>(embed, tokens, embed_delta, dim, x);
    note_launch();
    BD_CUDA(cudaGetLastError());
}

void logits_launch(const ProjOut& lm, const float* const* raw_delta, const float* xn_f32, int batch,
                   int dim, int vocab, float* logits, cudaStream_t s) {
    const int bx = std::max(1, std::min((vocab + 7) / 8, 256));
    logits_kernel<<<dim3(bx, batch), 256, 0, s>>>(lm, raw_delta, xn_f32, dim, vocab, logits);
    note_launch();
    BD_CUDA(cudaGetLastError());
}

}  // namespace bd
