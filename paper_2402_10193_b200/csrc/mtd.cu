// K3d — the delta of a tenant with MANY requests in the batch, as a dense tensor-core GEMM
// (SURVEY.md §8 a9 at batch 64: BASELINE configs[3], T <= 4 tenants).
//
// Replaces, for all n_t requests of tenant t at once (P:src/serve.cpp:250-254 per request):
//   apply_delta_correction -> packed_signed_accumulate (P:src/delta.cpp:80-103)
//   D[r][m] = alpha_t * sum_k s_t[m][k] x_r[k],   r in the tenant's requests
// i.e. Y_t = alpha_t * S_t X_t^T with X_t the tenant's activation rows (bf16, gathered
// tenant by tenant, zero-padded to N_t = 16 ceil(n_t / 16) rows).
//
// The byte LUT repeats its table work per request and K23 re-reads a plane for every slot
// of <= 4 requests; here each plane byte is read and expanded ONCE per step and serves all
// of the tenant's requests as the N dimension of a kind::f16 MMA:
//   * a task = (tenant, 128-row tile); its stages are 256-column chunks: a [128 rows x 32 B]
//     plane box (TMA, reference layout) and the tenant's X rows for the chunk (TMA, 4 boxes
//     of [N_t rows x 64 columns], 128-byte swizzle: K2's B-operand layout);
//   * 8 expander warps (two per TMEM lane quadrant, thread = tile row = TMEM lane, each warp
//     half of the chunk) turn a chunk's 8 plane words into 256 bf16 +-1.0 (two per 32-bit
//     TMEM column, one shift + one LOP3: see expand_bf16x2) in one of three 128-column TMEM
//     entries; a ring of 6 stages (two producer warps) keeps the loads ahead.
//     Measured (ncu, M7 gate/up, 4 tenants): a skeleton with no loads, expansion or MMAs
//     takes ~45 % of the kernel (mbarrier / tcgen05.commit round trips per chunk), the
//     expansion ~45 %, loads and MMAs the rest: 4 -> 8 expanders, 2 -> 3 entries and
//     4 -> 6 stages took gate/up 77 -> 70 us at 4 tenants, 35 -> 29 us at 1;
//   * an issuer warp runs 16 MMAs (M = 128, N = N_t, K = 16, A from TMEM, B from smem) per
//     chunk into one of two f32 accumulators (N_t columns), accumulating over the task's K;
//   * the epilogue (the expander warps, deferred by one chunk) applies alpha and writes
//     D[split][r][m] for the tenant's real requests; K is split so the grid fills the GPU
//     (a single tenant has few row tiles), the consumer sums the split partials in order.
// Exact like K2: +-1 and bf16 x are exact in the MMA, f32 accumulation.
// One CTA per SM (512 TMEM columns): runs after K2, not beside it (a 256-column variant with
// 128-column chunks beside K2 on the side stream measured slower: DESIGN.md §7.0).
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace bd {

void note_launch();

namespace {

constexpr int kExpanders = 8;                     // expander warps 1..8 (4 measured slower)
constexpr int kHalves = kExpanders / 4;           // expander warps per TMEM lane quadrant
constexpr int kIssuer = kExpanders + 1;           // MMA issuer warp
constexpr int kProducer2 = kExpanders + 2;        // second TMA producer warp
constexpr int kThreads = 32 * (kExpanders + 3);
// stage ring: as many stages as fit (6 at N_t = 64, up to kMaxRing at N_t = 16); the
// ring depth hides the per-chunk barrier round trips (4 stages measured slower)
constexpr int kMaxRing = 24;
constexpr uint32_t kPlaneBytes = 128 * 32;                          // [128 rows x 32 B]
constexpr uint32_t kXBytesMax = 4 * kMtdMaxN * 128;                  // 4 x [N rows x 128 B]
constexpr uint32_t kRingBytes = 6 * ((kPlaneBytes + kXBytesMax + 1023) / 1024 * 1024);
constexpr uint32_t kSmem = 1024 + kRingBytes + 512;

// TMEM (512 columns): kEntries A entries of 128 columns (K = 256 bf16), two accumulators of
// kMtdMaxN columns
constexpr int kEntries = 3;
constexpr uint32_t kColA = 0, kEntryCols = 128, kColAcc = kEntries * kEntryCols;
static_assert(kColAcc + 2 * kMtdMaxN <= 512, "TMEM budget");

struct Task {
    int ten, seg, m0, row, c0, c1;  // chunks [c0, c1) of the K split
};
__device__ __forceinline__ Task task_of(const MtdParams& p, int t) {
    Task k;
    const int ks = t % p.ksplit;
    t /= p.ksplit;
    k.ten = t / p.tiles;
    k.m0 = (t - k.ten * p.tiles) * 128;
    k.c0 = ks * p.chunks_per_split;
    k.c1 = min(p.n_chunks, k.c0 + p.chunks_per_split);
    int sg = 0;
    while (sg + 1 < p.n_segs && k.m0 >= p.seg_row0[sg + 1]) ++sg;
    k.seg = sg;
    k.row = k.m0 - p.seg_row0[sg];
    return k;
}

// TMEM column j of a plane word w holds the bf16 pair (bit j, bit j + 16) of w: one shift and
// one LOP3 (bit j -> bit 15, bit j + 16 -> bit 31; 1 -> +1.0 = 0x3F80, 0 -> -1.0 = 0xBF80). The
// MMA therefore sees the columns of each 32-column block in the order j, j+16, j+1, j+17, ...;
// the gathered activations are stored in that order (mtd_gather_kernel), so the product is
// unchanged.
template <int j>
__device__ __forceinline__ uint32_t expand_bf16x2(uint32_t w) {
    return ((w << (15 - j)) & 0x80008000u) ^ 0xBF80BF80u;
}

__global__ void __launch_bounds__(kThreads, 1) mtd_kernel(const __grid_constant__ MtdParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int kRing = p.ring;
    const uint32_t kStageBytes = uint32_t(p.stage_bytes);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kRingBytes);
    uint64_t* empty = full + kMaxRing;
    uint64_t* a_full = empty + kMaxRing;      // [kEntries]
    uint64_t* a_free = a_full + kEntries;     // [kEntries]
    uint64_t* acc_full = a_free + kEntries;   // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 2);
    const uint32_t warp = warp_id(), lane = lane_id();
    const int t0 = static_cast<int>(static_cast<long long>(p.n_tasks) * blockIdx.x / gridDim.x);
    const int t1 = static_cast<int>(static_cast<long long>(p.n_tasks) * (blockIdx.x + 1) / gridDim.x);
    if (warp == 0) {
        if (lane == 0) {
            for (int s = 0; s < kRing; ++s) {
                mbar_init(&full[s], 1);
                mbar_init(&empty[s], 1);
            }
            for (int i = 0; i < kEntries; ++i) {
                mbar_init(&a_full[i], kExpanders);
                mbar_init(&a_free[i], 1);
            }
            for (int i = 0; i < 2; ++i) mbar_init(&acc_full[i], 1);
            fence_mbar_init();
        }
        __syncwarp();
        tmem_alloc<512>(tmem_slot);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;

    if (warp == 0 || warp == kProducer2) {
        // ---- TMA producers: two warps take alternate stages (ring slots {p, p + 2} belong to
        // producer p, so no slot is ever armed out of order); copies issued by one thread
        // complete about one at a time ----
        const int prod = warp == 0 ? 0 : 1;
        const uint64_t pol_stream = policy_evict_first();
        const uint64_t pol_keep = policy_evict_last();
        griddep_wait();  // PDL: X (gathered by the previous kernel)
        int s = 0, gidx = 0;
        uint32_t ph = 0;
        for (int t = t0; t < t1; ++t) {
            const Task k = task_of(p, t);
            const CUtensorMap* pmap = p.plane_maps + k.ten * kLutMaxSegs + k.seg;
            const CUtensorMap* xmap = p.x_maps + k.ten;
            const uint32_t xbytes = uint32_t(p.n_pad[k.ten]) * 128;
            for (int c = k.c0; c < k.c1; ++c, ++gidx) {
                if ((gidx & 1) == prod) {
                    mbar_wait_w(&empty[s], ph ^ 1);
                    uint8_t* sp = smem + s * kStageBytes;
                    mbar_arrive_expect_tx_w(&full[s], kPlaneBytes + 4 * xbytes);
                    tma_load_2d_w(sp, pmap, &full[s], c * 32, k.row, pol_stream);
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        tma_load_2d_w(sp + kPlaneBytes + q * xbytes, xmap, &full[s], c * 256 + q * 64,
                                      p.x_row0[k.ten], pol_keep);
                }
                if (++s == kRing) {
                    s = 0;
                    ph ^= 1;
                }
            }
        }
    } else if (warp == kIssuer) {
        // ---- MMA issuer (whole warp, one elected lane issues) ----
        int s = 0, e = 0, d = 0;
        uint32_t ph = 0, eph = 0;
        for (int t = t0; t < t1; ++t) {
            const Task k = task_of(p, t);
            const uint32_t N = uint32_t(p.n_pad[k.ten]);
            const uint32_t idesc = idesc_bf16_f32(128, N);
            const uint32_t xbytes = N * 128;
            for (int c = k.c0; c < k.c1; ++c) {
                mbar_wait_w(&a_full[e], eph);
                tc_fence_after();
                const uint8_t* xs = smem + s * kStageBytes + kPlaneBytes;
                const uint32_t ent = tbase + kColA + e * kEntryCols;
                const uint32_t dacc = tbase + kColAcc + d * kMtdMaxN;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint64_t db = sdesc_k128(xs + q * xbytes);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)  // K = 16 per MMA: 8 A columns, +32 B of B
                        mma_bf16_ts_w(dacc, ent + (q * 4 + kk) * 8, db + 2 * kk, idesc,
                                      (c == k.c0 && q == 0 && kk == 0) ? 0u : 1u);
                }
                tc_commit_w(&a_free[e]);
                tc_commit_w(&empty[s]);
                if (c == k.c1 - 1) tc_commit_w(&acc_full[d]);
                if (++e == kEntries) {
                    e = 0;
                    eph ^= 1;
                }
                if (++s == kRing) {
                    s = 0;
                    ph ^= 1;
                }
            }
            d ^= 1;
        }
    } else {
        // ---- expanders: thread = tile row = TMEM lane ----
        const uint32_t q4 = warp & 3;  // a warp reaches TMEM lanes 32 (warp % 4) ..
        const uint32_t half = (warp - 1) / 4;  // which part of the chunk (and of the epilogue)
        const uint32_t trow = q4 * 32 + lane;
        const uint32_t lane_base = (q4 * 32) << 16;
        griddep_wait();  // D is still read by the previous kernel's consumer
        int s = 0, e = 0, d = 0;
        uint32_t ph = 0, eph = 0, acc_ph[2] = {0, 0};
        uint32_t n_entries = 0;
        int pend_ten = -1, pend_seg = 0, pend_m0 = 0, pend_d = 0, pend_ks = 0;
        auto epilogue = [&]() {
            mbar_wait(&acc_full[pend_d], acc_ph[pend_d]);
            acc_ph[pend_d] ^= 1;
            tc_fence_after();
            const int n = p.n_req[pend_ten];
            const float alpha = p.alpha[pend_ten][pend_seg];
            for (int c0 = 16 * int(half); c0 < n; c0 += 16 * kHalves) {
                uint32_t v[16];
                tmem_ld16(tbase + lane_base + kColAcc + pend_d * kMtdMaxN + c0, v);
                tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (c0 + j < n)
                        p.out[static_cast<size_t>(pend_ks) * p.dstride +
                              static_cast<size_t>(p.req[pend_ten][c0 + j]) * p.M + pend_m0 + trow] =
                            alpha * __uint_as_float(v[j]);
            }
            tc_fence_before();
            pend_ten = -1;
        };
        for (int t = t0; t < t1; ++t) {
            const Task k = task_of(p, t);
            for (int c = k.c0; c < k.c1; ++c) {
                mbar_wait(&full[s], ph);  // every lane polls (one polling lane measured slower)
                if (n_entries >= kEntries) mbar_wait(&a_free[e], eph ^ 1);  // the entry's previous MMAs done
                tc_fence_after();
                constexpr int kWords = 8 / kHalves;  // plane words of this warp's part of the row
                uint32_t w[kWords];
                const uint32_t rowp = smem_u32(smem + s * kStageBytes + trow * 32 + half * 4 * kWords);
#pragma unroll
                for (int v = 0; v < kWords / 4; ++v) lds128(rowp + 16 * v, w + 4 * v);
                const uint32_t ent = tbase + lane_base + kColA + e * kEntryCols + half * 16 * kWords;
#pragma unroll
                for (int h = 0; h < kWords / 2; ++h) {  // 64 columns (2 words) -> 32 TMEM columns
                    uint32_t a[32];
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const uint32_t x = w[2 * h + u];
                        a[16 * u + 0] = expand_bf16x2<0>(x);   a[16 * u + 1] = expand_bf16x2<1>(x);
                        a[16 * u + 2] = expand_bf16x2<2>(x);   a[16 * u + 3] = expand_bf16x2<3>(x);
                        a[16 * u + 4] = expand_bf16x2<4>(x);   a[16 * u + 5] = expand_bf16x2<5>(x);
                        a[16 * u + 6] = expand_bf16x2<6>(x);   a[16 * u + 7] = expand_bf16x2<7>(x);
                        a[16 * u + 8] = expand_bf16x2<8>(x);   a[16 * u + 9] = expand_bf16x2<9>(x);
                        a[16 * u + 10] = expand_bf16x2<10>(x); a[16 * u + 11] = expand_bf16x2<11>(x);
                        a[16 * u + 12] = expand_bf16x2<12>(x); a[16 * u + 13] = expand_bf16x2<13>(x);
                        a[16 * u + 14] = expand_bf16x2<14>(x); a[16 * u + 15] = expand_bf16x2<15>(x);
                    }
                    tmem_st32(ent + 32 * h, a);
                }
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&a_full[e]);
                ++n_entries;
                if (++e == kEntries) {
                    e = 0;
                    eph ^= 1;
                }
                if (++s == kRing) {
                    s = 0;
                    ph ^= 1;
                }
                if (c == k.c0 && pend_ten >= 0) epilogue();
            }
            pend_ten = k.ten;
            pend_ks = k.c0 / p.chunks_per_split;
            pend_seg = k.seg;
            pend_m0 = k.m0;
            pend_d = d;
            d ^= 1;
        }
        if (pend_ten >= 0) epilogue();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tbase);
}

// Xp[row0_t + i] = X[req_t[i]] (i < n_t; zero rows up to n_pad_t), each 32-column block in
// the MMA's column order (2 i <- i, 2 i + 1 <- i + 16); grid (gathered rows, column chunks),
// thread = one 32-column block (4 x 16-byte loads, the pairs interleaved with PRMT)
__global__ void mtd_gather_kernel(const uint16_t* __restrict__ X, int ldx, int K, const MtdGather g,
                                  uint16_t* __restrict__ Xp, int ldp) {
    griddep_launch_dependents();  // K2's weight prefetch does not depend on the gathered X
    griddep_wait();
    const int row = blockIdx.x;
    int t = 0;
    while (t + 1 < kMtdMaxTenants && row >= g.row0[t] + g.n_pad[t]) ++t;
    const int i = row - g.row0[t];
    const int r = i < g.n_req[t] ? g.req[t][i] : -1;
    uint4* dst = reinterpret_cast<uint4*>(Xp + static_cast<size_t>(row) * ldp);
    const uint4* src = r >= 0 ? reinterpret_cast<const uint4*>(X + static_cast<size_t>(r) * ldx) : nullptr;
    for (int b = blockIdx.y * blockDim.x + threadIdx.x; b * 32 < K; b += gridDim.y * blockDim.x) {
        uint4 lo0 = make_uint4(0, 0, 0, 0), lo1 = lo0, hi0 = lo0, hi1 = lo0;  // columns 0-7, 8-15, 16-23, 24-31
        if (src) {
            lo0 = src[4 * b];
            lo1 = src[4 * b + 1];
            hi0 = src[4 * b + 2];
            hi1 = src[4 * b + 3];
        }
        // output word m = (column m, column m + 16), m < 16
        const uint32_t l[8] = {lo0.x, lo0.y, lo0.z, lo0.w, lo1.x, lo1.y, lo1.z, lo1.w};
        const uint32_t h[8] = {hi0.x, hi0.y, hi0.z, hi0.w, hi1.x, hi1.y, hi1.z, hi1.w};
        uint32_t o[16];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            o[2 * q] = __byte_perm(l[q], h[q], 0x5410);      // (column 2q, column 2q + 16)
            o[2 * q + 1] = __byte_perm(l[q], h[q], 0x7632);  // (column 2q + 1, column 2q + 17)
        }
#pragma unroll
        for (int v = 0; v < 4; ++v) dst[4 * b + v] = make_uint4(o[4 * v], o[4 * v + 1], o[4 * v + 2], o[4 * v + 3]);
    }
}

}  // namespace

bool plan_mtd(MtdParams& p, MtdGather& g, const std::vector<MtdTenant>& tens, const int* seg_rows, int n_segs,
              int K, int ldx, int max_splits, std::vector<CUtensorMap>& plane_maps) {
    if (K % 256 != 0 || tens.empty() || int(tens.size()) > kMtdMaxTenants || n_segs > kLutMaxSegs) return false;
    p = MtdParams{};
    g = MtdGather{};
    p.n_segs = n_segs;
    p.K = K;
    int M = 0;
    for (int s = 0; s < n_segs; ++s) {
        if (seg_rows[s] % 128) return false;
        p.seg_row0[s] = M;
        M += seg_rows[s];
    }
    p.seg_row0[n_segs] = M;
    p.M = M;
    p.tiles = M / 128;
    p.n_ten = int(tens.size());
    p.n_tasks = p.n_ten * p.tiles;
    plane_maps.assign(size_t(p.n_ten) * kLutMaxSegs, CUtensorMap{});
    int row = 0;
    for (int t = 0; t < p.n_ten; ++t) {
        const MtdTenant& mt = tens[t];
        const int n = int(mt.reqs.size());
        if (n < 1 || n > kMtdMaxN) return false;
        p.n_req[t] = g.n_req[t] = n;
        p.n_pad[t] = g.n_pad[t] = (n + 15) / 16 * 16;
        p.x_row0[t] = g.row0[t] = row;
        row += p.n_pad[t];
        for (int i = 0; i < n; ++i) p.req[t][i] = g.req[t][i] = mt.reqs[i];
        for (int s = 0; s < n_segs; ++s) {
            if (mt.n_planes[s] != 1 || reinterpret_cast<uintptr_t>(mt.bits[s]) % 16) return false;
            p.alpha[t][s] = mt.alpha[s];
            plane_maps[size_t(t) * kLutMaxSegs + s] = make_tmap_2d(
                mt.bits[s], CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, uint64_t(seg_rows[s]), uint64_t(K / 8), uint64_t(K / 8),
                128, 32, false);
        }
    }
    p.x_rows = g.rows = row;
    (void)ldx;
    // split K so the grid has ~2 tasks per SM (one tenant's few row tiles would leave most SMs
    // idle); every split writes its own delta partial D[split] (<= max_splits of them)
    p.n_chunks = K / 256;
    const int base_tasks = p.n_ten * p.tiles;
    int ks = std::max(1, std::min({(2 * kNumSMs + base_tasks - 1) / base_tasks, p.n_chunks, max_splits}));
    p.chunks_per_split = (p.n_chunks + ks - 1) / ks;
    p.ksplit = (p.n_chunks + p.chunks_per_split - 1) / p.chunks_per_split;
    p.n_tasks = base_tasks * p.ksplit;
    p.grid = std::min(kNumSMs, p.n_tasks);
    int max_pad = 16;
    for (int t = 0; t < p.n_ten; ++t) max_pad = std::max(max_pad, p.n_pad[t]);
    p.stage_bytes = int((kPlaneBytes + 4 * uint32_t(max_pad) * 128 + 1023) / 1024 * 1024);
    p.ring = std::min(kMaxRing, int(kRingBytes / uint32_t(p.stage_bytes))) & ~1;  // even: two producers
    return true;
}

std::vector<CUtensorMap> mtd_x_maps(const MtdParams& p, const void* Xp, int ldp) {
    std::vector<CUtensorMap> m(p.n_ten);
    for (int t = 0; t < p.n_ten; ++t)
        m[t] = make_tmap_2d(Xp, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, uint64_t(p.x_rows), uint64_t(p.K), uint64_t(ldp),
                            uint32_t(p.n_pad[t]), 64, true);
    return m;
}

void mtd_gather_launch(const void* X, int ldx, int K, const MtdGather& g, int n_ten, void* Xp, int ldp,
                       cudaStream_t stream) {
    (void)n_ten;
    require(K % 32 == 0 && ldx % 8 == 0 && ldp % 8 == 0, BD_ERR_BAD_ARGUMENT, "K3d gather: alignment");
    BD_CUDA(launch_pdl(mtd_gather_kernel, dim3(g.rows, (K / 32 + 31) / 32), dim3(32), 0, stream,
                       static_cast<const uint16_t*>(X), ldx, K, g, static_cast<uint16_t*>(Xp), ldp));
    note_launch();
    BD_CUDA(cudaGetLastError());
}

void mtd_launch(const MtdParams& p, cudaStream_t stream) {
    static bool attr = false;
    if (!attr) {
        BD_CUDA(cudaFuncSetAttribute(mtd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmem)));
        attr = true;
    }
    BD_CUDA(launch_pdl(mtd_kernel, dim3(p.grid), dim3(kThreads), size_t(kSmem), stream, p));
    note_launch();
    BD_CUDA(cudaGetLastError());
}

}  // namespace bd
