// Device side of the fused step epilogues (TileFuse, glue.h): the tile work one warp does for
// one request, the RMS scale, and the producer-side arrival. Included by the producers (K2
// gemm.cu, the K3 LUT lut.cu) and by glue.cu (attention's q/k/v scale, the first layer's
// norm launch).
//
// Ordering: a producer's threads store their partials, fence (gpu scope) and meet at a
// barrier; one thread arrives (atomicAdd) on each tile it wrote. The last arriver fences
// again and reads every partial through L2 (ld.global.cg: other SMs wrote them during this
// kernel, so L1 may not hold them). Partials are summed in the consumers' fixed order.
#pragma once

#include "common.cuh"
#include "glue.h"

namespace bd {

__device__ __forceinline__ float4 fz_ld4(const float* p) { return __ldcg(reinterpret_cast<const float4*>(p)); }

__device__ __forceinline__ const float* fz_part(const ProjOut& p, int k, int b, int m) {
    return k < p.splits ? p.P + static_cast<size_t>(k) * p.pstride + size_t(b) * p.M + m
                        : p.D + static_cast<size_t>(k - p.splits) * p.dstride + size_t(b) * p.M + m;
}

__device__ __forceinline__ float4 fz_add4(float4 a, float4 b) {
    return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
// sum of the partials of outputs m..m+3, partial k = 0, 1, ... in order (the glue kernels'
// order), kG loads in flight
__device__ __forceinline__ float4 fz_val4(const ProjOut& p, int b, int m) {
    const int n = p.splits + (p.D ? p.dsplits : 0);
    float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
    constexpr int kG = 8;
    for (int k0 = 0; k0 < n; k0 += kG) {
        float4 t[kG];
#pragma unroll
        for (int j = 0; j < kG; ++j) t[j] = k0 + j < n ? fz_ld4(fz_part(p, k0 + j, b, m)) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int j = 0; j < kG; ++j)
            if (k0 + j < n) g = fz_add4(g, t[j]);
    }
    return g;
}
// the same for outputs m..m+3 (g) and m+off..m+off+3 (u) with both load sets in flight
__device__ __forceinline__ void fz_val4_pair(const ProjOut& p, int b, int m, int off, float4& g, float4& u) {
    const int n = p.splits + (p.D ? p.dsplits : 0);
    g = make_float4(0.f, 0.f, 0.f, 0.f);
    u = g;
    constexpr int kG = 4;
    for (int k0 = 0; k0 < n; k0 += kG) {
        float4 tg[kG], tu[kG];
#pragma unroll
        for (int j = 0; j < kG; ++j) {
            const bool on = k0 + j < n;
            tg[j] = on ? fz_ld4(fz_part(p, k0 + j, b, m)) : make_float4(0.f, 0.f, 0.f, 0.f);
            tu[j] = on ? fz_ld4(fz_part(p, k0 + j, b, m + off)) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int j = 0; j < kG; ++j)
            if (k0 + j < n) {
                g = fz_add4(g, tg[j]);
                u = fz_add4(u, tu[j]);
            }
    }
}

__device__ __forceinline__ double fz_warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// r_b = 1 / sqrt(mean x^2 + 1e-12) from the per-tile sums (one warp, fixed order: lane sums
// tiles lane, lane + 32, ..., then a fixed butterfly) -> every caller gets the same bits
__device__ __forceinline__ double fz_rinv(const double* msq, int tiles, int dim, int b, int lane) {
    double s = 0.0;
    for (int t = lane; t < tiles; t += 32) s += __ldcg(msq + size_t(b) * tiles + t);
    s = fz_warp_sum(s);
    return 1.0 / sqrt(s / static_cast<double>(dim) + 1e-12);
}

__device__ __forceinline__ uint32_t fz_pack_bf16(float a, float b) {
    return uint32_t(__bfloat16_as_ushort(__float2bfloat16_rn(a))) |
           (uint32_t(__bfloat16_as_ushort(__float2bfloat16_rn(b))) << 16);
}

// tile t of request b, one warp (4 consecutive outputs per lane)
__device__ __forceinline__ void fz_tile_warp_inl(const TileFuse& f, int t, int b, int lane) {
    const int i = 128 * t + 4 * lane;
    if (f.kind == 1) {
        float* xb = f.x + size_t(b) * f.dim;
        float4 v = fz_ld4(xb + i);
        if (f.src.P || f.src.D) {
            v = fz_add4(v, fz_val4(f.src, b, i));
            *reinterpret_cast<float4*>(xb + i) = v;
        }
        const float4 w = __ldg(reinterpret_cast<const float4*>(f.norm_w[b] + i));
        uint2 pk;
        pk.x = fz_pack_bf16(v.x * w.x, v.y * w.y);
        pk.y = fz_pack_bf16(v.z * w.z, v.w * w.w);
        *reinterpret_cast<uint2*>(f.xn + size_t(b) * f.ldxn + i) = pk;
        double sq = static_cast<double>(v.x) * v.x + static_cast<double>(v.y) * v.y +
                    static_cast<double>(v.z) * v.z + static_cast<double>(v.w) * v.w;
        sq = fz_warp_sum(sq);
        if (lane == 0) f.msq_out[size_t(b) * f.tiles + t] = sq;
    } else {
        float4 g, u;
        fz_val4_pair(f.src, b, i, f.fold, g, u);
        const double inv = fz_rinv(f.msq_in, f.msq_tiles, f.msq_dim, b, lane);
        auto sc = [&](float v) { return static_cast<float>(static_cast<double>(v) * inv); };
        auto a = [&](float gv, float uv) {
            const float gs = sc(gv);
            return gs / (1.0f + expf(-gs)) * sc(uv);
        };
        uint2 pk;
        pk.x = fz_pack_bf16(a(g.x, u.x), a(g.y, u.y));
        pk.y = fz_pack_bf16(a(g.z, u.z), a(g.w, u.w));
        *reinterpret_cast<uint2*>(f.act + size_t(b) * f.ld_act + i) = pk;
    }
}

// the same as a call (the LUT's epilogue function keeps it out of the kernel's main loop)
static __device__ __noinline__ void fz_tile_warp(const TileFuse& f, int t, int b, int lane) { fz_tile_warp_inl(f, t, b, lane); }

// Arrive on tile counter c; true for the tile's last arriver (which resets the counter). Call
// from one thread after the producer's stores are fenced and barrier-joined.
// ---- phase barrier ----
// Producers arrive once per CTA after their partial stores (fenced, barrier-joined). The tile
// work needs the partials of EVERY producer, and the last finisher covers most tiles (a LUT
// CTA's rows span ~75 of them), so it is spread over all CTAs of K2 (the waiter): they wait
// for every arrival, take tiles x requests round robin, and the last to leave resets the
// counters for the next phase. The LUT never waits, so it always drains: K2 CTAs spinning
// on an SM cannot starve it (a LUT CTA fits beside one K2 CTA; plan_fuse checks), and
// where the LUT holds an SM first (default carveout) K2 simply lands after it.
__device__ __forceinline__ void fz_producer_arrive(const TileFuse& f) {
    atomicAdd(f.cnt, 1u);
}
__device__ __forceinline__ void fz_wait_all(const TileFuse& f) {
    const unsigned long long t0 = gtimer();
    while (true) {
        unsigned v;
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(f.cnt) : "memory");
        if (v >= f.arrivals) break;
        __nanosleep(64);
        if (gtimer() - t0 > 2000000000ull) __trap();  // 2 s: a schedule bug faults, never hangs
    }
}
// after the tile work; thread 0 of each waiting CTA
__device__ __forceinline__ void fz_depart(const TileFuse& f) {
    unsigned* dep = f.cnt + 32;
    if (atomicAdd(dep, 1u) + 1u == gridDim.x) {
        atomicExch(f.cnt, 0u);
        atomicExch(dep, 0u);
    }
}

}  // namespace bd
