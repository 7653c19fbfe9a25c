// extern "C" implementation of include/bitdelta/capi.h. No exception crosses
// the ABI: every entry point maps bd::Failure to its status code and stores the
// message for bd_last_error(); CUDA errors map to BD_ERR_CUDA.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <vector>

#include "bdelta_io.h"
#include "common.cuh"
#include "kernels.h"

struct bd_pool;

namespace bd {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
}  // namespace

void set_error(const std::string& msg) { g_last_error = msg; }
[[noreturn]] void fail(int code, const std::string& msg) { throw Failure{code, msg}; }
void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw Failure{BD_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
}
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

namespace {
std::mutex g_pdl_mu;
std::set<const void*>& pdl_set() {
    static std::set<const void*> s;
    return s;
}
}  // namespace
std::vector<TraceBinder>& trace_binders() {
    static std::vector<TraceBinder> v;
    return v;
}
int trace_register(TraceBinder b) {
    trace_binders().push_back(b);
    return 0;
}
namespace {
TraceRec* g_tr_buf = nullptr;
unsigned* g_tr_cnt = nullptr;
unsigned g_tr_cap = 0;
}  // namespace
void note_pdl_kernel(const void* fn) {
    std::lock_guard<std::mutex> g(g_pdl_mu);
    pdl_set().insert(fn);
}
bool is_pdl_kernel(const void* fn) {
    std::lock_guard<std::mutex> g(g_pdl_mu);
    return pdl_set().count(fn) != 0;
}
uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

// pool.cu
bd_pool* pool_create(const bd_arch& a, int device, int world, int rank);
void pool_destroy(bd_pool* p);
void pool_set_tensor(bd_pool* p, const char* name, const void* data, bd_dtype dt, int is_dev,
                     uint64_t rows, uint64_t cols);
void pool_set_tensor_i8(bd_pool* p, const char* name, const int8_t* q, const float* scales, int is_dev,
                        uint64_t rows, uint64_t cols);
void pool_register(bd_pool* p, const char* id, const bd_delta_entry* e, int n);
void pool_register_file(bd_pool* p, const char* id, const char* path, int resident);
uint64_t pool_open(bd_pool* p, const char* id);
void pool_close(bd_pool* p, uint64_t rid);
void pool_decode(bd_pool* p, const bd_request* r, uint64_t n, int mode, float* logits, void* s);
void pool_decode_layers(bd_pool* p, const bd_request* r, uint64_t n, const float* xin, float* xout,
                        void* s);
void pool_stats(const bd_pool* p, bd_pool_stats* out);
void pool_profile_layers(bd_pool* p, const bd_request* r, uint64_t n, const float* xin,
                         float* xout, double* ms, uint64_t* cnt, void* s, bool serial);
void nccl_unique_id(void* out);
void pool_init_comm(bd_pool* p, const void* id);
void pool_init_loopback(bd_pool* p, const char* group);

template <class F>
int guarded(F&& f) {
    try {
        f();
        return BD_OK;
    } catch (const Failure& e) {
        set_error(e.msg);
        return e.code;
    } catch (const std::exception& e) {
        set_error(e.what());
        return BD_ERR_CUDA;
    }
}

// ---- bd_multitenant_linear: K2 (tcgen05) + K3 (tenant-segmented) + combine ----
struct LinearScratch {
    float* P = nullptr;
    size_t P_cap = 0;
    float* D = nullptr;
    size_t D_cap = 0;
};

void multitenant_linear(const void* W, uint64_t out_dim, uint64_t in_dim, int32_t n_tenants,
                        const uint8_t* const* tenant_bits, const float* tenant_alpha,
                        int32_t batch, const int32_t* req_tenant, const void* X, float* Y,
                        cudaStream_t stream) {
    require(W && X && Y, BD_ERR_BAD_ARGUMENT, "multitenant_linear: null pointer");
    require(batch >= 1 && batch <= 256, BD_ERR_BAD_ARGUMENT, "multitenant_linear: batch must be 1..256");
    require(in_dim % 8 == 0, BD_ERR_BAD_ARGUMENT, "multitenant_linear: in_dim must be a multiple of 8");
    require(out_dim >= 1 && out_dim < (1ull << 31), BD_ERR_BAD_ARGUMENT, "multitenant_linear: bad out_dim");
    for (int b = 0; b < batch; ++b)
        require(req_tenant == nullptr || req_tenant[b] < n_tenants, BD_ERR_UNKNOWN_ID,
                "multitenant_linear: request tenant out of range");
    const GemmPlan g = plan_base_gemm(out_dim, in_dim, batch);
    const CUtensorMap mw = tmap_weights(W, out_dim, in_dim, in_dim);
    const CUtensorMap mx = tmap_acts(X, batch, in_dim, in_dim, g.bn);
    // tenant segmentation: each tenant's plane once for all of its requests
    std::map<int, std::vector<int>> by_t;
    std::vector<int> order;
    for (int b = 0; b < batch; ++b) {
        const int t = req_tenant ? req_tenant[b] : -1;
        if (t < 0) continue;
        require(tenant_bits && tenant_alpha && tenant_bits[t], BD_ERR_BAD_ARGUMENT,
                "multitenant_linear: missing tenant bits");
        if (!by_t.count(t)) order.push_back(t);
        by_t[t].push_back(b);
    }
    static const char* mode_env = std::getenv("BD_DELTA");
    const std::string mode = mode_env ? mode_env : "auto";
    size_t with_delta = 0;
    for (int t : order) with_delta += by_t[t].size();
    const double mean_per_tenant = order.empty() ? 0.0 : double(with_delta) / double(order.size());
    // ---- K23: base GEMM + FP4 tensor-core deltas in one persistent kernel ----
    bool aligned16 = in_dim % 128 == 0 && out_dim % 128 == 0;
    for (int t : order) aligned16 &= (reinterpret_cast<uintptr_t>(tenant_bits[t]) % 16) == 0;
    // K23 when tenants average k23_min_requests(batch) requests or more (a plane is then read
    // once per slot of up to 4 requests instead of once per request; same policy as the pool)
    if ((mode == "mt4" || (mode == "auto" && mean_per_tenant >= k23_min_requests(batch))) && aligned16 &&
        !order.empty() && batch <= 64) {
        Mt4Params prm{};
        prm.n_subs = 1;
        prm.sub_row0[0] = 0;
        prm.sub_row0[1] = int(out_dim);
        std::vector<CUtensorMap> maps;
        bool ok = true;
        // canonical slot order (tenant id): the schedule, and so every output bit, does not
        // depend on the order of the requests in the batch (test_serve.cpp:169-190)
        std::vector<int> sorted_t(order);
        std::sort(sorted_t.begin(), sorted_t.end());
        for (int t : sorted_t) {
            const auto& rq = by_t[t];
            const int mi = int(maps.size());
            maps.push_back(tmap_bits4(tenant_bits[t], out_dim, in_dim));
            for (size_t c = 0, n = 0; c < rq.size(); c += n) {
                if (prm.n_slots >= kMt4MaxSlots) { ok = false; break; }
                Mt4Slot& sl = prm.slots[prm.n_slots++];
                n = size_t(mt4_slot_requests(rq.size() - c));
                sl.n_req = int(n);
                for (int q = 0; q < sl.n_req; ++q) sl.req[q] = rq[c + q];
                sl.alpha[0] = tenant_alpha[t];
                sl.map_idx[0] = mi;
            }
        }
        if (ok && plan_mt4(prm, out_dim, in_dim, batch)) {
            const size_t sz_p = sizeof(float) * prm.splits * batch * out_dim;
            const size_t sz_xp = size_t(batch) * prm.n_chunks * kXpBlock;
            const size_t sz_m = maps.size() * sizeof(CUtensorMap);
            const std::vector<uint32_t> sched = mt4_schedule(prm);
            const size_t sz_s = sched.size() * sizeof(uint32_t);
            char* ws = nullptr;
            BD_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ws), sz_p + sz_xp + sz_m + sz_s + 1024, stream));
            char* cur = ws;
            auto take = [&](size_t n) { char* r = cur; cur += (n + 255) & ~size_t(255); return r; };
            float* P = reinterpret_cast<float*>(take(sz_p));
            uint8_t* xpk = reinterpret_cast<uint8_t*>(take(sz_xp));
            CUtensorMap* dmaps = reinterpret_cast<CUtensorMap*>(take(sz_m));
            uint32_t* dsched = reinterpret_cast<uint32_t*>(take(sz_s));
            BD_CUDA(cudaMemcpyAsync(dmaps, maps.data(), sz_m, cudaMemcpyHostToDevice, stream));
            BD_CUDA(cudaMemcpyAsync(dsched, sched.data(), sz_s, cudaMemcpyHostToDevice, stream));
            BD_CUDA(cudaStreamSynchronize(stream));  // host staging consumed
            prm.map_w = mw;
            prm.map_x = tmap_acts(X, batch, in_dim, in_dim, prm.bn);
            prm.xpk = xpk;
            prm.sched = dsched;
            prm.bits_maps = dmaps;
            prm.partial = P;
            xp_prep_launch(X, int(in_dim), int(in_dim), batch, xpk, stream);
            mt4_launch(prm, stream);
            combine_launch(P, prm.splits, nullptr, batch, int(out_dim), Y, stream);
            BD_CUDA(cudaFreeAsync(ws, stream));
            return;
        }
    }
    // ---- byte-LUT path (few requests per tenant): tcgen05 base GEMM + K3 LUT ----
    // one launch per kLutMaxJobs requests; each writes its own requests' rows of D
    if ((mode == "lut" || mode == "auto") && !order.empty()) {
        std::vector<LutParams> prms;
        bool ok = true;
        const int seg_rows[1] = {int(out_dim)};
        int n_jobs = 0;
        for (int b0 = 0; b0 < batch && ok; b0 += kLutMaxJobs) {
            LutParams prm{};
            for (int b = b0; b < std::min(batch, b0 + kLutMaxJobs); ++b) {
                const int t = req_tenant ? req_tenant[b] : -1;
                if (t < 0) continue;
                LutJob& j = prm.jobs[prm.n_jobs++];
                j.req = b;
                j.n_planes[0] = 1;
                j.bits[0][0] = tenant_bits[t];
                j.alpha[0][0] = tenant_alpha[t];
            }
            n_jobs += prm.n_jobs;
            if (prm.n_jobs == 0) continue;
            ok = plan_lut(prm, seg_rows, 1, int(in_dim), int(in_dim), batch);
            prms.push_back(prm);
        }
        if (ok && !prms.empty()) {
            const int slices = prms[0].slices;
            float* P = nullptr;
            float* D = nullptr;
            BD_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&P), sizeof(float) * g.splits * batch * out_dim, stream));
            BD_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&D), sizeof(float) * slices * batch * out_dim, stream));
            // base-only requests have no job: their delta slices must read as zero
            if (n_jobs < batch)
                BD_CUDA(cudaMemsetAsync(D, 0, sizeof(float) * slices * batch * out_dim, stream));
            base_gemm_launch(g, mw, mx, P, stream);
            for (const LutParams& prm : prms) lut_launch(prm, X, D, stream);
            combine_launch(P, g.splits, D, batch, int(out_dim), Y, stream, slices);
            BD_CUDA(cudaFreeAsync(P, stream));
            BD_CUDA(cudaFreeAsync(D, stream));
            return;
        }
    }
    // ---- SIMT fallback: tcgen05 base GEMM + tenant-segmented delta units ----
    float* P = nullptr;
    float* D = nullptr;
    BD_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&P), sizeof(float) * g.splits * batch * out_dim, stream));
    BD_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&D), sizeof(float) * batch * out_dim, stream));
    base_gemm_launch(g, mw, mx, P, stream);
    std::vector<DeltaUnit> units;
    for (int t : order) {
        const auto& rq = by_t[t];
        for (size_t c = 0; c < rq.size(); c += kMaxReqPerUnit) {
            DeltaUnit u{};
            u.n_planes = 1;
            u.bits[0] = tenant_bits[t];
            u.alpha[0] = tenant_alpha[t];
            u.row0 = 0;
            u.rows = int(out_dim);
            u.n_req = int(std::min<size_t>(kMaxReqPerUnit, rq.size() - c));
            for (int q = 0; q < u.n_req; ++q) u.req[q] = rq[c + q];
            units.push_back(u);
        }
    }
    delta_units_launch(units.data(), int(units.size()), X, int(in_dim), int(in_dim), batch, D,
                       int(out_dim), stream);
    combine_launch(P, g.splits, D, batch, int(out_dim), Y, stream);
    BD_CUDA(cudaFreeAsync(P, stream));
    BD_CUDA(cudaFreeAsync(D, stream));
}

// int8_matmul_nt (P:src/int8.cpp:67-81) on the tensor cores: Y [s x out] = A Wq^T * row_scale
static void int8_matmul_impl(const float* A, uint64_t s, uint64_t in_dim, const int8_t* q,
                             const float* row_scales, uint64_t out_dim, float* Y, cudaStream_t stream) {
    require(A && q && row_scales && Y, BD_ERR_BAD_ARGUMENT, "int8_matmul_nt: null pointer");
    if (s == 0 || out_dim == 0) return;
    if (in_dim == 0) {
        BD_CUDA(cudaMemsetAsync(Y, 0, s * out_dim * sizeof(float), stream));
        return;
    }
    require(out_dim <= 0x7fffffffull && in_dim <= 0x7fffffffull, BD_ERR_BAD_ARGUMENT, "int8_matmul_nt: too large");
    // TMA needs 16-byte row strides: copy Wq into a padded buffer when in_dim % 16 != 0
    const uint64_t ld = (in_dim + 15) / 16 * 16;
    int8_t* wq = const_cast<int8_t*>(q);
    int8_t* wpad = nullptr;
    if (ld != in_dim || reinterpret_cast<uintptr_t>(q) % 16) {
        BD_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&wpad), out_dim * ld, stream));
        BD_CUDA(cudaMemsetAsync(wpad, 0, out_dim * ld, stream));
        BD_CUDA(cudaMemcpy2DAsync(wpad, ld, q, in_dim, in_dim, out_dim, cudaMemcpyDeviceToDevice, stream));
        wq = wpad;
    }
    const CUtensorMap mw = tmap_weights_i8(wq, out_dim, in_dim, ld);
    constexpr int kChunk = 64;  // requests per launch (kPieces x 64 = 256 MMA columns)
    const int bmax = int(std::min<uint64_t>(s, kChunk));
    int8_t* xq = nullptr;
    float* ps = nullptr;
    BD_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&xq), size_t(kPieces) * bmax * ld, stream));
    BD_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ps), sizeof(float) * kPieces * bmax, stream));
    for (uint64_t b0 = 0; b0 < s; b0 += kChunk) {
        const int nb = int(std::min<uint64_t>(kChunk, s - b0));
        const GemmPlan g = plan_i8_gemm(out_dim, in_dim, nb);
        float* P = nullptr;
        BD_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&P), sizeof(float) * g.splits * nb * out_dim, stream));
        quant_pieces_launch(A + b0 * in_dim, true, int(in_dim), int(in_dim), nb, xq, int(ld), ps, stream);
        const CUtensorMap mx = tmap_pieces(xq, nb, in_dim, ld, g.bn);
        i8_gemm_launch(g, mw, mx, row_scales, ps, P, stream);
        combine_launch(P, g.splits, nullptr, nb, int(out_dim), Y + b0 * out_dim, stream);
        BD_CUDA(cudaFreeAsync(P, stream));
    }
    BD_CUDA(cudaFreeAsync(xq, stream));
    BD_CUDA(cudaFreeAsync(ps, stream));
    if (wpad) BD_CUDA(cudaFreeAsync(wpad, stream));
}

}  // namespace bd

using namespace bd;

extern "C" {

int bd_abi_version(void) { return BD_ABI_VERSION; }
const char* bd_last_error(void) { return g_last_error.c_str(); }
uint64_t bd_launch_count(void) { return launch_count(); }

int bd_trace_enable(uint32_t capacity) {
    return guarded([&] {
        if (g_tr_buf) {
            cudaFree(g_tr_buf);
            cudaFree(g_tr_cnt);
            g_tr_buf = nullptr;
            g_tr_cnt = nullptr;
        }
        g_tr_cap = capacity;
        if (capacity) {
            BD_CUDA(cudaMalloc(&g_tr_buf, sizeof(TraceRec) * capacity));
            BD_CUDA(cudaMalloc(&g_tr_cnt, sizeof(unsigned)));
            BD_CUDA(cudaMemset(g_tr_cnt, 0, sizeof(unsigned)));
        }
        for (TraceBinder b : trace_binders()) b(g_tr_buf, g_tr_cnt, g_tr_cap);
        BD_CUDA(cudaDeviceSynchronize());
    });
}

int bd_trace_read(void* out, uint32_t capacity, uint32_t* n_out) {
    return guarded([&] {
        require(g_tr_buf != nullptr, BD_ERR_BAD_ARGUMENT, "trace: not enabled");
        BD_CUDA(cudaDeviceSynchronize());
        unsigned n = 0;
        BD_CUDA(cudaMemcpy(&n, g_tr_cnt, sizeof(n), cudaMemcpyDeviceToHost));
        n = std::min(n, std::min(g_tr_cap, capacity));
        if (n) BD_CUDA(cudaMemcpy(out, g_tr_buf, sizeof(TraceRec) * n, cudaMemcpyDeviceToHost));
        BD_CUDA(cudaMemset(g_tr_cnt, 0, sizeof(unsigned)));
        if (n_out) *n_out = n;
    });
}

int bd_device_check(int device) {
    return guarded([&] {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) fail(BD_ERR_NO_DEVICE, "no CUDA device");
        require(device >= 0 && device < n, BD_ERR_NO_DEVICE, "device index out of range");
        cudaDeviceProp p;
        BD_CUDA(cudaGetDeviceProperties(&p, device));
        require(p.major == 10 && p.minor == 0, BD_ERR_UNSUPPORTED_DEVICE,
                std::string("libbitdelta_b200 is built for sm_100a; device is ") + p.name + " (sm_" +
                    std::to_string(p.major) + std::to_string(p.minor) + ")");
    });
}

uint64_t bd_packed_size(uint64_t rows, uint64_t cols) { return (rows * cols + 7) / 8; }

int bd_compress(const void* base, const void* fine, bd_dtype dtype, uint64_t rows, uint64_t cols,
                uint8_t* bits, float* alpha, void* stream) {
    return guarded([&] {
        bd_compress_job j{base, fine, rows, cols, bits, alpha};
        compress_launch(&j, 1, dtype, static_cast<cudaStream_t>(stream));
    });
}

int bd_compress_batched(const bd_compress_job* jobs, int n_jobs, bd_dtype dtype, void* stream) {
    return guarded([&] {
        require(jobs != nullptr || n_jobs == 0, BD_ERR_BAD_ARGUMENT, "compress_batched: null jobs");
        require(n_jobs >= 0, BD_ERR_BAD_ARGUMENT, "compress_batched: negative job count");
        if (n_jobs) compress_launch(jobs, n_jobs, dtype, static_cast<cudaStream_t>(stream));
    });
}

int bd_compress_stack(const void* base, const void* fine, bd_dtype dtype, uint64_t rows,
                      uint64_t cols, uint64_t planes, uint8_t* bits, float* alphas, void* stream) {
    return guarded([&] {
        require(fine && bits && alphas, BD_ERR_BAD_ARGUMENT, "compress_stack: null pointer");
        compress_stack_launch(base, fine, dtype, rows, cols, planes, bits, alphas,
                              static_cast<cudaStream_t>(stream));
    });
}

int bd_packed_signed_accumulate(const uint8_t* bits, uint64_t rows, uint64_t cols, const float* x,
                                uint64_t n_vec, float* out, void* stream) {
    return guarded([&] {
        packed_accumulate_launch(bits, rows, cols, x, n_vec, out, 1.0f, false,
                                 static_cast<cudaStream_t>(stream));
    });
}

int bd_packed_matvec(const uint8_t* bits, float alpha, uint64_t rows, uint64_t cols,
                     const float* x, uint64_t n_vec, float* y, void* stream) {
    return guarded([&] {
        packed_accumulate_launch(bits, rows, cols, x, n_vec, y, alpha, true,
                                 static_cast<cudaStream_t>(stream));
    });
}

int bd_packed_signed_accumulate_t(const uint8_t* bits, uint64_t rows, uint64_t cols, const float* y,
                                  uint64_t n_vec, float* out, void* stream) {
    return guarded([&] {
        packed_transpose_launch(bits, rows, cols, y, n_vec, out, 1.0f, false, static_cast<cudaStream_t>(stream));
    });
}

int bd_delta_linear_backward(int32_t n_planes, const uint8_t* const* plane_bits, const float* scales,
                             uint64_t rows, uint64_t cols, const float* dy, uint64_t s,
                             const float* const* plane_u, float* dx, double* scale_grad, void* stream) {
    return guarded([&] {
        require(n_planes >= 0, BD_ERR_BAD_ARGUMENT, "delta_linear_backward: negative plane count");
        require(n_planes == 0 || (plane_bits && scales && plane_u && scale_grad), BD_ERR_BAD_ARGUMENT,
                "delta_linear_backward: null pointer");
        require(dy && dx, BD_ERR_BAD_ARGUMENT, "delta_linear_backward: null pointer");
        const cudaStream_t st = static_cast<cudaStream_t>(stream);
        for (int32_t pl = 0; pl < n_planes; ++pl) {
            dot_f64_launch(dy, plane_u[pl], s * rows, scale_grad + pl, st);
            packed_transpose_launch(plane_bits[pl], rows, cols, dy, s, dx, scales[pl], false, st);
        }
    });
}

int bd_rtn_quantize(const float* W, uint64_t rows, uint64_t cols, int8_t* q, float* row_scales, void* stream) {
    return guarded([&] { rtn_quantize_launch(W, rows, cols, q, cols, row_scales, static_cast<cudaStream_t>(stream)); });
}

int bd_int8_matmul_nt(const float* A, uint64_t s, uint64_t in_dim, const int8_t* q, const float* row_scales,
                      uint64_t out_dim, float* Y, void* stream) {
    return guarded([&] {
        int8_matmul_impl(A, s, in_dim, q, row_scales, out_dim, Y, static_cast<cudaStream_t>(stream));
    });
}

int bd_multitenant_linear(const void* W, uint64_t out_dim, uint64_t in_dim, int32_t n_tenants,
                          const uint8_t* const* tenant_bits, const float* tenant_alpha,
                          int32_t batch, const int32_t* req_tenant, const void* X, float* Y,
                          void* stream) {
    return guarded([&] {
        multitenant_linear(W, out_dim, in_dim, n_tenants, tenant_bits, tenant_alpha, batch,
                           req_tenant, X, Y, static_cast<cudaStream_t>(stream));
    });
}

int bd_multitenant_linear_f32(const float* W, uint64_t out_dim, uint64_t in_dim, int32_t n_tenants,
                              const uint8_t* const* tenant_bits, const float* tenant_alpha,
                              int32_t batch, const int32_t* req_tenant, const float* X, float* Y,
                              void* stream) {
    return guarded([&] {
        require(W && X && Y, BD_ERR_BAD_ARGUMENT, "multitenant_linear_f32: null pointer");
        require(batch >= 1 && batch <= 256, BD_ERR_BAD_ARGUMENT, "multitenant_linear_f32: batch must be 1..256");
        require(out_dim >= 1 && in_dim >= 1, BD_ERR_BAD_ARGUMENT, "multitenant_linear_f32: empty matrix");
        std::vector<const uint8_t*> rb(batch, nullptr);
        std::vector<float> ra(batch, 0.0f);
        for (int b = 0; b < batch; ++b) {
            const int t = req_tenant ? req_tenant[b] : -1;
            require(t < n_tenants, BD_ERR_UNKNOWN_ID, "multitenant_linear_f32: request tenant out of range");
            if (t < 0) continue;
            require(tenant_bits && tenant_alpha && tenant_bits[t], BD_ERR_BAD_ARGUMENT,
                    "multitenant_linear_f32: missing tenant bits");
            rb[b] = tenant_bits[t];
            ra[b] = tenant_alpha[t];
        }
        f32_linear_launch(W, out_dim, in_dim, rb.data(), ra.data(), batch, X, Y,
                          static_cast<cudaStream_t>(stream));
    });
}

int bd_pool_create(const bd_arch* arch, int device, int world_size, int rank, bd_pool** out) {
    return guarded([&] {
        require(arch && out, BD_ERR_BAD_ARGUMENT, "pool_create: null argument");
        *out = pool_create(*arch, device, world_size, rank);
    });
}
void bd_pool_destroy(bd_pool* pool) {
    if (pool) pool_destroy(pool);
}
int bd_nccl_unique_id(void* id_out) {
    return guarded([&] {
        require(id_out != nullptr, BD_ERR_BAD_ARGUMENT, "nccl_unique_id: null output");
        nccl_unique_id(id_out);
    });
}
int bd_pool_init_comm(bd_pool* pool, const void* id) {
    return guarded([&] {
        require(pool && id, BD_ERR_BAD_ARGUMENT, "init_comm: null argument");
        pool_init_comm(pool, id);
    });
}

int bd_bdelta_validate(const char* path, uint64_t* n_tensors, uint64_t* n_packed, uint64_t* max_planes) {
    return guarded([&] {
        require(path != nullptr, BD_ERR_BAD_ARGUMENT, "bdelta_validate: null path");
        const DeltaFileHost f = read_bdelta(path);
        uint64_t packed = 0, mp = 0;
        for (const auto& e : f.entries) {
            packed += e.packed ? 1 : 0;
            mp = std::max(mp, e.planes);
        }
        if (n_tensors) *n_tensors = f.entries.size();
        if (n_packed) *n_packed = packed;
        if (max_planes) *max_planes = mp;
    });
}

int bd_pool_init_loopback(bd_pool* pool, const char* group) {
    return guarded([&] {
        require(pool, BD_ERR_BAD_ARGUMENT, "init_loopback: null pool");
        pool_init_loopback(pool, group);
    });
}
int bd_pool_set_tensor(bd_pool* pool, const char* name, const void* data, bd_dtype dtype,
                       int is_device, uint64_t rows, uint64_t cols) {
    return guarded([&] {
        require(pool != nullptr, BD_ERR_BAD_ARGUMENT, "null pool");
        pool_set_tensor(pool, name, data, dtype, is_device, rows, cols);
    });
}
int bd_pool_set_tensor_i8(bd_pool* pool, const char* name, const int8_t* q, const float* row_scales,
                          int is_device, uint64_t rows, uint64_t cols) {
    return guarded([&] {
        require(pool != nullptr, BD_ERR_BAD_ARGUMENT, "null pool");
        pool_set_tensor_i8(pool, name, q, row_scales, is_device, rows, cols);
    });
}
int bd_pool_register_delta(bd_pool* pool, const char* id, const bd_delta_entry* entries,
                           int n_entries) {
    return guarded([&] {
        require(pool != nullptr, BD_ERR_BAD_ARGUMENT, "null pool");
        pool_register(pool, id, entries, n_entries);
    });
}
int bd_pool_register_delta_file(bd_pool* pool, const char* id, const char* path, int resident) {
    return guarded([&] {
        require(pool != nullptr, BD_ERR_BAD_ARGUMENT, "null pool");
        pool_register_file(pool, id, path, resident);
    });
}
int bd_pool_open_request(bd_pool* pool, const char* delta_id, uint64_t* request_id) {
    return guarded([&] {
        require(pool && request_id, BD_ERR_BAD_ARGUMENT, "null argument");
        *request_id = pool_open(pool, delta_id);
    });
}
int bd_pool_close_request(bd_pool* pool, uint64_t request_id) {
    return guarded([&] {
        require(pool != nullptr, BD_ERR_BAD_ARGUMENT, "null pool");
        pool_close(pool, request_id);
    });
}
int bd_pool_decode_step(bd_pool* pool, const bd_request* reqs, uint64_t n, int mode,
                        float* logits, void* stream) {
    return guarded([&] {
        require(pool != nullptr, BD_ERR_BAD_ARGUMENT, "null pool");
        pool_decode(pool, reqs, n, mode, logits, stream);
    });
}
int bd_pool_decode_layers(bd_pool* pool, const bd_request* reqs, uint64_t n, const float* x_in,
                          float* x_out, void* stream) {
    return guarded([&] {
        require(pool != nullptr, BD_ERR_BAD_ARGUMENT, "null pool");
        pool_decode_layers(pool, reqs, n, x_in, x_out, stream);
    });
}
int bd_pool_profile_layers(bd_pool* pool, const bd_request* reqs, uint64_t n, const float* x_in,
                           float* x_out, double* ms_out, uint64_t* count_out, void* stream) {
    return guarded([&] {
        require(pool != nullptr, BD_ERR_BAD_ARGUMENT, "null pool");
        pool_profile_layers(pool, reqs, n, x_in, x_out, ms_out, count_out, stream, false);
    });
}
int bd_pool_profile_layers_serial(bd_pool* pool, const bd_request* reqs, uint64_t n, const float* x_in,
                                  float* x_out, double* ms_out, uint64_t* count_out, void* stream) {
    return guarded([&] {
        require(pool != nullptr, BD_ERR_BAD_ARGUMENT, "null pool");
        pool_profile_layers(pool, reqs, n, x_in, x_out, ms_out, count_out, stream, true);
    });
}
int bd_pool_get_stats(const bd_pool* pool, bd_pool_stats* out) {
    return guarded([&] {
        require(pool && out, BD_ERR_BAD_ARGUMENT, "null argument");
        pool_stats(pool, out);
    });
}

}  // extern "C"
