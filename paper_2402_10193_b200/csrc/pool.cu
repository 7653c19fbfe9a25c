// Device-resident multi-tenant ServingPool — the B200 replacement of
// deltakit::ServingPool (P:include/deltakit/serve.hpp:59-125,
// P:src/serve.cpp:93-342).
//
// Layout in HBM (one process per GPU, rank r of world W holds rows
// [r*R/W, (r+1)*R/W) of every projection; W = 1 on one GPU):
//   * per layer, bf16 backbone linears stacked so one GEMM serves a group:
//       Wqkv [q_l + 2 kv_l, dim]   Wo [dim_l, dim]   Wgu [2 inter_l, dim]
//       Wdown [dim_l, inter]       (row stride padded to 8 elements for TMA)
//   * per tenant, per layer and projection: the sign planes in the reference
//     byte layout (one device buffer per plane, 16-byte aligned) + f32 alpha;
//     effective norm rows (backbone + raw delta, serve.cpp:224-228) in f32;
//   * per request: a bf16 KV cache [n_layers][max_seq][kv_dim] for k and v.
// A decode step runs, per layer, K4 norm -> K2+K3 qkv -> K4 attention ->
// K2+K3 o -> K4 residual+norm -> K2+K3 gate|up -> K4 silu -> K2+K3 down, with
// the split-K/delta reduction folded into the next glue kernel. Requests are
// segmented by tenant so each tenant's planes are streamed once per step.
// Steps for a fixed batch composition are captured once into a CUDA graph
// and replayed; only positions/tokens are re-uploaded per step.
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <map>
#include <mutex>
#include <memory>
#include <string>
#include <vector>

#include "bdelta_io.h"
#include "common.cuh"
#include "glue.h"
#include "kernels.h"

#include <nccl.h>

#define BD_NCCL(x)                                                                            \
    do {                                                                                      \
        const ncclResult_t r_ = (x);                                                          \
        if (r_ != ncclSuccess) ::bd::fail(BD_ERR_CUDA, std::string(#x) + ": " + ncclGetErrorString(r_)); \
    } while (0)

#ifndef BD_K2_CAP_KB
#define BD_K2_CAP_KB 88  // K2 beside the LUT: shared memory for its stage ring (KB)
#endif

namespace bd {

void note_launch();
uint64_t launch_count();

namespace {

enum Proj { P_Q, P_K, P_V, P_O, P_GATE, P_UP, P_DOWN, P_COUNT };
const char* kProjNames[P_COUNT] = {"attn_q", "attn_k", "attn_v", "attn_o",
                                   "mlp_gate", "mlp_up", "mlp_down"};

__global__ void f32_to_bf16_2d(const float* __restrict__ src, uint64_t rows, uint64_t cols,
                               uint64_t lds, uint16_t* __restrict__ dst, uint64_t ldd) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < rows * cols;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t r = i / cols, c = i % cols;
        dst[r * ldd + c] = __bfloat16_as_ushort(__float2bfloat16_rn(src[r * lds + c]));
    }
}

uint64_t round_up(uint64_t v, uint64_t m) { return (v + m - 1) / m * m; }

// Test hook (bd_pool_init_loopback): the row-sharded pools of one process on ONE device,
// each driven from its own host thread, exchange through device copies instead of NCCL
// (NCCL refuses two ranks on one GPU). Every other part of the tensor-parallel path (rank
// row slices, head-local attention, shard_reduce, gather_transpose) runs as with NCCL.
struct LoopbackGroup {
    int world = 0;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    std::vector<void*> recv;
    std::vector<cudaEvent_t> ready, done;
    void barrier() {
        std::unique_lock<std::mutex> lk(m);
        const uint64_t g = gen;
        if (++arrived == world) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};
std::mutex g_loop_m;
std::map<std::string, std::shared_ptr<LoopbackGroup>> g_loop_groups;

template <typename T>
T* dmalloc(size_t n, std::vector<void*>* owner = nullptr) {
    void* p = nullptr;
    BD_CUDA(cudaMalloc(&p, std::max<size_t>(n * sizeof(T), 16)));
    if (owner) owner->push_back(p);
    return static_cast<T*>(p);
}

struct Plane {
    const uint8_t* bits;
    float alpha;
    // the same rows padded to a multiple of 128 bytes for the byte-LUT (rows of 11 008 columns
    // are 1 376 B: 3 of 4 row slices would straddle two L2 lines); null where rows are aligned
    const uint8_t* bits_lut = nullptr;
    int ld_lut = 0;  // bytes per padded row
};
// LUT row padding: 128-B multiples where the rows are long and not already aligned
inline uint64_t lut_row_bytes(uint64_t cols) {
    const uint64_t b = cols / 8;
    return (cols % 128 == 0 && b > 128 && b % 128 != 0) ? (b + 127) / 128 * 128 : 0;
}

struct Tenant {
    std::string id, path;
    bool resident = false, loaded = false;
    // [layer][proj] -> planes (this rank's row slice)
    std::vector<std::array<std::vector<Plane>, P_COUNT>> proj;
    // [layer][proj] -> raw (unquantised) f32 delta, this rank's rows; null if packed / all-zero
    std::vector<std::array<float*, P_COUNT>> raw;
    std::vector<float*> norm1, norm2;  // device, effective
    float* final_norm = nullptr;
    float* embed_raw = nullptr;        // device [vocab x dim] or null
    float* lm_raw = nullptr;           // device [vocab x dim] or null
    std::vector<Plane> lm_planes;      // packed lm_head (rank-local rows)
    std::vector<void*> allocs;
    uint64_t bytes = 0;                // payload bytes as accounted by the reference
};

struct Request {
    int tenant = -1;
    bool open = false;
    uint64_t pos = 0;
    uint16_t* kc = nullptr;
    uint16_t* vc = nullptr;
};

struct LayerW {
    uint16_t *qkv = nullptr, *o = nullptr, *gu = nullptr, *down = nullptr;  // bf16 backbone
    CUtensorMap m_qkv, m_o, m_gu, m_down;
    // INT8 RTN backbone (ServingPool(QuantizedCheckpoint), P:src/serve.cpp:99-108): per
    // projection group (qkv, o, gu, down) stacked int8 rows + f32 row scales
    int8_t* q8[4] = {nullptr, nullptr, nullptr, nullptr};
    float* s8[4] = {nullptr, nullptr, nullptr, nullptr};
    CUtensorMap m8[4];
};

struct Plan {
    int B = 0;
    std::vector<int> reqs;  // pool request indices
    // device pointer tables
    float** d_norm = nullptr;       // [(2L+1) * B]
    uint16_t** d_kc = nullptr;      // [B]
    uint16_t** d_vc = nullptr;
    float** d_embed = nullptr;      // [B] or null
    float** d_lmraw = nullptr;      // [B] or null
    int* d_pos = nullptr;
    int* d_tok = nullptr;
    // pinned staging of positions / tokens, two slots: a slot is rewritten only after the
    // copy that last read it has run (event), not after the whole previous step, so the host
    // enqueues step N+1 while step N executes
    int* h_pos[2] = {nullptr, nullptr};
    int* h_tok[2] = {nullptr, nullptr};
    cudaEvent_t staged[2] = {nullptr, nullptr};
    int slot = 0;
    std::vector<void*> allocs;
    // per layer & group: delta units
    std::vector<std::array<std::vector<DeltaUnit>, 4>> units;  // qkv, o, gu, down
    // raw projection deltas (serve.cpp:27-35) and planes beyond kMaxPlanesPerUnit: groups with
    // any take the units path + these extra passes
    std::vector<std::array<std::vector<RawJob>, 4>> raw;
    std::vector<std::array<std::vector<DeltaUnit>, 4>> units_x;  // planes 5, 6, ... (D +=)
    bool raw_group[4] = {false, false, false, false};
    std::vector<DeltaUnit> lm_units;
    GemmPlan g_qkv, g_o, g_gu, g_down, g_lm;
    CUtensorMap x_xn, x_ctx, x_act;  // B-operand maps for this batch size
    CUtensorMap xq_dim, xq_inter;    // int8 backbone: activation pieces (quant_pieces_launch)
    // byte-LUT deltas (few requests per tenant) per layer & group; one launch per
    // kLutMaxJobs requests (each launch writes its own requests' rows of D)
    struct Lut {
        bool ok = false;
        std::vector<LutParams> prm;
    };
    std::vector<std::array<Lut, 4>> lut;
    // K23 (base + FP4 tensor-core deltas in one kernel) per layer & group
    struct M4 {
        bool ok = false;
        Mt4Params prm;
    };
    std::vector<std::array<M4, 4>> mt4;
    // K3d (tenants with many requests: one dense tensor-core delta per tenant) per layer & group
    struct Md {
        bool ok = false;
        MtdParams prm;
        MtdGather gat;
    };
    std::vector<std::array<Md, 4>> mtd;
    uint16_t* xg = nullptr;  // gathered activations (tenant-major, padded), K3d only
    int xg_ld = 0;
    // every K3d group gathers the same way: the glue kernel producing a K3d group's input writes
    // its gathered copy (XgOut, row d_xrow[b] for request b) and the gather launch is skipped
    bool xg_direct = false;
    int* d_xrow = nullptr;
    uint8_t* xpk = nullptr;  // FP4 activation pieces + scales [B][chunks][kXpBlock]
    cudaGraphExec_t graph_layers = nullptr, graph_full = nullptr;
    uint64_t kernels_layers = 0, kernels_full = 0;
};

}  // namespace

struct PoolImpl {
    bd_arch a{};
    int device = 0, world = 1, rank = 0;
    uint64_t hd = 0, n_kv_heads = 0;
    uint64_t q_l = 0, kv_l = 0, dim_l = 0, inter_l = 0;  // rank-local rows
    uint64_t q_r0 = 0, kv_r0 = 0, dim_r0 = 0, inter_r0 = 0;
    uint64_t ld_dim = 0, ld_inter = 0;  // padded strides (elements)
    std::vector<LayerW> L;
    int base_kind = 0;                  // projections: 0 = none set yet, 1 = bf16, 2 = int8 RTN
    uint64_t ld8_dim = 0, ld8_inter = 0;  // int8 row strides (TMA: multiples of 16 bytes)
    int8_t* xq = nullptr;                 // int8 activation pieces [kPieces * ws_B][ld8 max]
    float* xps = nullptr;                 // their scales [kPieces * ws_B]
    std::vector<std::vector<float>> base_norm1, base_norm2;  // host copies (full)
    std::vector<float> base_final_norm;
    float* embed = nullptr;
    uint16_t* lm_head = nullptr;
    CUtensorMap m_lm;
    std::vector<bool> have;  // tensor set flags (tensor_shapes order)
    std::vector<void*> allocs;
    float2* rope = nullptr;
    uint64_t backbone_bytes = 0;

    std::vector<Tenant> tenants;
    std::map<std::string, int> tenant_idx;
    std::vector<Request> requests;
    bd_pool_stats stats{};

    // workspaces (sized for ws_B)
    int ws_B = 0;
    float *x = nullptr, *xn_f32 = nullptr, *P = nullptr, *D = nullptr, *logits = nullptr;
    void* msq = nullptr;  // RMSNorm workspace (norm_ws_bytes: arrival counters + chunk sums)
    // tensor parallel (world > 1)
    ncclComm_t comm = nullptr;
    std::shared_ptr<LoopbackGroup> loop;  // test hook instead of comm (bd_pool_init_loopback)
    cudaEvent_t lb_ready = nullptr, lb_done = nullptr;
    uint16_t *ctx_loc = nullptr, *act_loc = nullptr, *gath16 = nullptr;
    float *red_loc = nullptr, *gath32 = nullptr;
    uint16_t *xn = nullptr, *ctx = nullptr, *act = nullptr;
    size_t P_elems = 0, D_elems = 0;
    std::vector<void*> ws_allocs;

    std::map<std::string, std::unique_ptr<Plan>> plans;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    cudaStream_t stream2 = nullptr;  // side stream: K2 beside K3
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    bool concurrent_k23 = true;      // K2 beside the LUT (false only inside a serial profile)
    bool use_graphs = true;
    // auto | lut | mt4 | units; BD_DELTA forces one K3 variant (test hook: every variant is
    // checked against the oracle on the same inputs)
    std::string delta_mode = "auto";
    bool xg_done = false;  // the next K3d linear's gathered input was written by its producer

    ~PoolImpl() {
        cudaSetDevice(device);
        if (stream) cudaStreamSynchronize(stream);
        clear_plans();
        free_ws();
        for (auto& t : tenants) for (void* p : t.allocs) cudaFree(p);
        for (auto& r : requests) { if (r.kc) cudaFree(r.kc); if (r.vc) cudaFree(r.vc); }
        for (void* p : allocs) cudaFree(p);
        if (ev_in) cudaEventDestroy(ev_in);
        if (ev_out) cudaEventDestroy(ev_out);
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_join) cudaEventDestroy(ev_join);
        if (stream2) cudaStreamDestroy(stream2);
        if (comm) ncclCommDestroy(comm);
        if (lb_ready) cudaEventDestroy(lb_ready);
        if (lb_done) cudaEventDestroy(lb_done);
        if (stream) cudaStreamDestroy(stream);
    }

    void clear_plans() {
        for (auto& kv : plans) {
            Plan& p = *kv.second;
            if (p.graph_layers) cudaGraphExecDestroy(p.graph_layers);
            if (p.graph_full) cudaGraphExecDestroy(p.graph_full);
            for (void* q : p.allocs) cudaFree(q);
            for (int k = 0; k < 2; ++k) {
                if (p.h_pos[k]) cudaFreeHost(p.h_pos[k]);
                if (p.h_tok[k]) cudaFreeHost(p.h_tok[k]);
                if (p.staged[k]) cudaEventDestroy(p.staged[k]);
            }
        }
        plans.clear();
    }
    void free_ws() {
        for (void* p : ws_allocs) cudaFree(p);
        ws_allocs.clear();
        ws_B = 0;
    }

    // ------------------------------------------------------------ setup --
    void init(const bd_arch& arch, int dev, int w, int r) {
        a = arch;
        device = dev;
        world = w;
        rank = r;
        require(a.vocab >= 1 && a.dim >= 1 && a.n_layers >= 1 && a.n_heads >= 1 &&
                    a.intermediate >= 1 && a.max_seq >= 1 && a.kv_dim >= 1,
                BD_ERR_BAD_ARGUMENT, "config: all counts must be >= 1");
        require(a.dim % a.n_heads == 0, BD_ERR_BAD_ARGUMENT, "config: dim must be divisible by n_heads");
        hd = a.dim / a.n_heads;
        require(hd % 2 == 0, BD_ERR_BAD_ARGUMENT, "config: head dimension must be even for rotary embeddings");
        require(a.kv_dim % hd == 0 && a.dim % a.kv_dim == 0, BD_ERR_BAD_ARGUMENT,
                "config: kv_dim must be a whole number of heads dividing dim");
        n_kv_heads = a.kv_dim / hd;
        require(w >= 1 && r >= 0 && r < w, BD_ERR_BAD_ARGUMENT, "pool: bad world/rank");
        require(n_kv_heads % w == 0 && a.intermediate % w == 0, BD_ERR_BAD_ARGUMENT,
                "pool: kv heads and intermediate must divide by world size");
        require(hd * 2 + a.max_seq <= 48000, BD_ERR_BAD_ARGUMENT, "pool: max_seq too large");
        q_l = a.dim / w;   q_r0 = q_l * r;
        kv_l = a.kv_dim / w; kv_r0 = kv_l * r;
        dim_l = a.dim / w; dim_r0 = dim_l * r;
        inter_l = a.intermediate / w; inter_r0 = inter_l * r;
        ld_dim = round_up(a.dim, 8);
        ld_inter = round_up(a.intermediate, 8);
        BD_CUDA(cudaSetDevice(device));
        BD_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
        BD_CUDA(cudaStreamCreateWithFlags(&stream2, cudaStreamNonBlocking));
        BD_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
        BD_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
        BD_CUDA(cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming));
        BD_CUDA(cudaEventCreateWithFlags(&ev_out, cudaEventDisableTiming));
        if (const char* e = std::getenv("BD_DELTA")) delta_mode = e;

        ld8_dim = round_up(a.dim, 16);
        ld8_inter = round_up(a.intermediate, 16);
        // layer buffers are allocated with the first projection tensor: bf16 or int8
        L.resize(a.n_layers);
        embed = dmalloc<float>(a.vocab * a.dim, &allocs);
        lm_head = dmalloc<uint16_t>(a.vocab * ld_dim, &allocs);
        BD_CUDA(cudaMemset(lm_head, 0, a.vocab * ld_dim * 2));
        m_lm = tmap_weights(lm_head, a.vocab, a.dim, ld_dim);
        base_norm1.assign(a.n_layers, std::vector<float>(a.dim, 0.0f));
        base_norm2.assign(a.n_layers, std::vector<float>(a.dim, 0.0f));
        base_final_norm.assign(a.dim, 0.0f);
        have.assign(1 + 9 * a.n_layers + 2, false);

        // RoPE table: the reference's double pow/cos/sin (nn_ops.hpp:33-40), rounded to f32
        std::vector<float2> tab(a.max_seq * (hd / 2));
        for (uint64_t p = 0; p < a.max_seq; ++p)
            for (uint64_t i = 0; i < hd / 2; ++i) {
                const double freq = std::pow(static_cast<double>(a.rope_theta),
                                             -2.0 * static_cast<double>(i) / static_cast<double>(hd));
                const double ang = static_cast<double>(p) * freq;
                tab[p * (hd / 2) + i] = make_float2(static_cast<float>(std::cos(ang)),
                                                    static_cast<float>(std::sin(ang)));
            }
        rope = dmalloc<float2>(tab.size(), &allocs);
        BD_CUDA(cudaMemcpy(rope, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice));
        backbone_bytes = 0;
        for (size_t i = 0; i < have.size(); ++i) {
            uint64_t rr, cc;
            shape(i, rr, cc);
            backbone_bytes += 4ull * rr * cc;  // reference accounting: f32 residency (serve.cpp:361)
        }
    }

    // tensor_shapes order (P:src/arch.cpp:51-69), kv_dim for k/v (arch.cpp:98-99)
    void shape(size_t i, uint64_t& rows, uint64_t& cols) const {
        const size_t last = 1 + 9 * a.n_layers;
        if (i == 0 || i == last + 1) { rows = a.vocab; cols = a.dim; return; }
        if (i == last) { rows = 1; cols = a.dim; return; }
        switch ((i - 1) % 9) {
            case 0: case 3: rows = a.dim; cols = a.dim; return;
            case 1: case 2: rows = a.kv_dim; cols = a.dim; return;
            case 4: case 5: rows = a.intermediate; cols = a.dim; return;
            case 6: rows = a.dim; cols = a.intermediate; return;
            default: rows = 1; cols = a.dim; return;
        }
    }
    std::string tname(size_t i) const {
        const size_t last = 1 + 9 * a.n_layers;
        if (i == 0) return "embed";
        if (i == last) return "final_norm";
        if (i == last + 1) return "lm_head";
        static const char* roles[9] = {"attn_q", "attn_k", "attn_v", "attn_o", "mlp_gate",
                                       "mlp_up", "mlp_down", "norm1", "norm2"};
        return "layers." + std::to_string((i - 1) / 9) + "." + roles[(i - 1) % 9];
    }
    int tindex(const std::string& name) const {
        for (size_t i = 0; i < have.size(); ++i)
            if (tname(i) == name) return int(i);
        return -1;
    }

    // rank-local row range of a projection within its (unsharded) matrix, and
    // its destination (buffer, row offset in the stacked buffer, ld)
    void local_rows(int proj, uint64_t& r0, uint64_t& nr) const {
        switch (proj) {
            case P_Q: r0 = q_r0; nr = q_l; return;
            case P_K: case P_V: r0 = kv_r0; nr = kv_l; return;
            case P_O: case P_DOWN: r0 = dim_r0; nr = dim_l; return;
            default: r0 = inter_r0; nr = inter_l; return;
        }
    }
    uint64_t stack_offset(int proj) const {
        switch (proj) {
            case P_K: return q_l;
            case P_V: return q_l + kv_l;
            case P_UP: return inter_l;
            default: return 0;
        }
    }

    void ensure_dense(LayerW& l) {
        if (l.qkv) return;
        l.qkv = dmalloc<uint16_t>((q_l + 2 * kv_l) * ld_dim, &allocs);
        l.o = dmalloc<uint16_t>(dim_l * ld_dim, &allocs);
        l.gu = dmalloc<uint16_t>(2 * inter_l * ld_dim, &allocs);
        l.down = dmalloc<uint16_t>(dim_l * ld_inter, &allocs);
        BD_CUDA(cudaMemset(l.qkv, 0, (q_l + 2 * kv_l) * ld_dim * 2));
        BD_CUDA(cudaMemset(l.o, 0, dim_l * ld_dim * 2));
        BD_CUDA(cudaMemset(l.gu, 0, 2 * inter_l * ld_dim * 2));
        BD_CUDA(cudaMemset(l.down, 0, dim_l * ld_inter * 2));
        l.m_qkv = tmap_weights(l.qkv, q_l + 2 * kv_l, a.dim, ld_dim);
        l.m_o = tmap_weights(l.o, dim_l, a.dim, ld_dim);
        l.m_gu = tmap_weights(l.gu, 2 * inter_l, a.dim, ld_dim);
        l.m_down = tmap_weights(l.down, dim_l, a.intermediate, ld_inter);
    }
    // rows of group g (qkv, o, gu, down) and its K
    uint64_t group_rows(int g) const {
        return g == 0 ? q_l + 2 * kv_l : g == 2 ? 2 * inter_l : dim_l;
    }
    uint64_t group_k(int g) const { return g == 3 ? a.intermediate : a.dim; }
    void ensure_i8(LayerW& l) {
        if (l.q8[0]) return;
        for (int g = 0; g < 4; ++g) {
            const uint64_t rows = group_rows(g), ld8 = g == 3 ? ld8_inter : ld8_dim;
            l.q8[g] = dmalloc<int8_t>(rows * ld8, &allocs);
            l.s8[g] = dmalloc<float>(rows, &allocs);
            BD_CUDA(cudaMemset(l.q8[g], 0, rows * ld8));
            BD_CUDA(cudaMemset(l.s8[g], 0, rows * 4));
            l.m8[g] = tmap_weights_i8(l.q8[g], rows, group_k(g), ld8);
        }
    }
    static int proj_group(int role) {
        return role <= P_V ? 0 : role == P_O ? 1 : role <= P_UP ? 2 : 3;
    }
    void set_base_kind(int kind, const std::string& name) {
        require(base_kind == 0 || base_kind == kind, BD_ERR_UNSUPPORTED_DTYPE,
                "tensor '" + name + "': a pool's projections are all int8 or all dense");
        base_kind = kind;
    }

    // INT8 RTN projection (Int8Tensor, P:include/deltakit/int8.hpp: values + row scales),
    // the backbone of ServingPool(QuantizedCheckpoint) (serve.cpp:99-108, 120-125)
    void set_tensor_i8(const std::string& name, const int8_t* q, const float* scales, bool is_dev,
                       uint64_t rows, uint64_t cols) {
        const int idx = tindex(name);
        require(idx >= 0, BD_ERR_NAME_MISMATCH, "backbone: unknown tensor '" + name + "'");
        uint64_t er, ec;
        shape(idx, er, ec);
        require(rows == er && cols == ec, BD_ERR_SHAPE_MISMATCH,
                "backbone: tensor '" + name + "' has shape " + std::to_string(rows) + "x" +
                    std::to_string(cols) + ", config expects " + std::to_string(er) + "x" +
                    std::to_string(ec));
        const size_t last = 1 + 9 * a.n_layers;
        const int role = (idx >= 1 && size_t(idx) < last) ? (idx - 1) % 9 : -1;
        require(role >= 0 && role < 7, BD_ERR_UNSUPPORTED_DTYPE,
                "tensor '" + name + "': only the 7 layer projections may be int8 on the device");
        set_base_kind(2, name);
        BD_CUDA(cudaSetDevice(device));
        const int l = (idx - 1) / 9, g = proj_group(role);
        ensure_i8(L[l]);
        uint64_t r0, nr;
        local_rows(role, r0, nr);
        const uint64_t ld8 = g == 3 ? ld8_inter : ld8_dim;
        const cudaMemcpyKind k = is_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
        BD_CUDA(cudaMemcpy2D(L[l].q8[g] + stack_offset(role) * ld8, ld8, q + r0 * cols, cols, cols, nr, k));
        BD_CUDA(cudaMemcpy(L[l].s8[g] + stack_offset(role), scales + r0, nr * 4, k));
        if (!have[idx]) backbone_bytes = backbone_bytes - 4ull * rows * cols + rows * cols + 4ull * rows;
        have[idx] = true;
    }

    void upload_bf16(uint16_t* dst, uint64_t ldd, const void* src, bd_dtype dt, bool is_dev,
                     uint64_t rows, uint64_t cols, uint64_t src_row0) {
        const size_t es = dt == BD_BF16 ? 2 : 4;
        const char* s = static_cast<const char*>(src) + src_row0 * cols * es;
        if (dt == BD_BF16) {
            BD_CUDA(cudaMemcpy2D(dst, ldd * 2, s, cols * 2, cols * 2, rows,
                                 is_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
            return;
        }
        const float* dsrc = reinterpret_cast<const float*>(s);
        float* tmp = nullptr;
        if (!is_dev) {
            tmp = dmalloc<float>(rows * cols);
            BD_CUDA(cudaMemcpy(tmp, s, rows * cols * 4, cudaMemcpyHostToDevice));
            dsrc = tmp;
        }
        f32_to_bf16_2d<<<std::min<uint64_t>((rows * cols + 255) / 256, 4096), 256>>>(
            dsrc, rows, cols, cols, dst, ldd);
        note_launch();
        BD_CUDA(cudaGetLastError());
        BD_CUDA(cudaDeviceSynchronize());
        if (tmp) cudaFree(tmp);
    }

    std::vector<float> to_host_f32(const void* src, bd_dtype dt, bool is_dev, uint64_t n) {
        std::vector<float> out(n);
        if (dt == BD_F32) {
            BD_CUDA(cudaMemcpy(out.data(), src, n * 4, is_dev ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost));
        } else {
            std::vector<uint16_t> h(n);
            BD_CUDA(cudaMemcpy(h.data(), src, n * 2, is_dev ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost));
            for (uint64_t i = 0; i < n; ++i) {
                const uint32_t u = uint32_t(h[i]) << 16;
                std::memcpy(&out[i], &u, 4);
            }
        }
        return out;
    }

    void set_tensor(const std::string& name, const void* data, bd_dtype dt, bool is_dev,
                    uint64_t rows, uint64_t cols) {
        require(dt == BD_F32 || dt == BD_BF16, BD_ERR_UNSUPPORTED_DTYPE,
                "tensor '" + name + "': unsupported dtype");
        const int idx = tindex(name);
        require(idx >= 0, BD_ERR_NAME_MISMATCH, "backbone: unknown tensor '" + name + "'");
        uint64_t er, ec;
        shape(idx, er, ec);
        require(rows == er && cols == ec, BD_ERR_SHAPE_MISMATCH,
                "backbone: tensor '" + name + "' has shape " + std::to_string(rows) + "x" +
                    std::to_string(cols) + ", config expects " + std::to_string(er) + "x" +
                    std::to_string(ec));
        BD_CUDA(cudaSetDevice(device));
        const size_t last = 1 + 9 * a.n_layers;
        if (idx == 0) {
            const std::vector<float> h = to_host_f32(data, dt, is_dev, rows * cols);
            BD_CUDA(cudaMemcpy(embed, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
        } else if (size_t(idx) == last) {
            base_final_norm = to_host_f32(data, dt, is_dev, cols);
        } else if (size_t(idx) == last + 1) {
            upload_bf16(lm_head, ld_dim, data, dt, is_dev, rows, cols, 0);
        } else {
            const int l = (idx - 1) / 9, role = (idx - 1) % 9;
            if (role == 7) base_norm1[l] = to_host_f32(data, dt, is_dev, cols);
            else if (role == 8) base_norm2[l] = to_host_f32(data, dt, is_dev, cols);
            else {
                set_base_kind(1, name);
                ensure_dense(L[l]);
                uint64_t r0, nr;
                local_rows(role, r0, nr);
                uint16_t* buf;
                uint64_t ld;
                switch (role) {
                    case P_Q: case P_K: case P_V: buf = L[l].qkv; ld = ld_dim; break;
                    case P_O: buf = L[l].o; ld = ld_dim; break;
                    case P_GATE: case P_UP: buf = L[l].gu; ld = ld_dim; break;
                    default: buf = L[l].down; ld = ld_inter; break;
                }
                upload_bf16(buf + stack_offset(role) * ld, ld, data, dt, is_dev, nr, cols, r0);
            }
        }
        have[idx] = true;
    }

    // ---------------------------------------------------------- tenants --
    struct EntryView {
        bool packed;
        uint64_t rows, cols, planes;
        const uint8_t* bits;
        const float* scales;
        const float* raw;
        bool is_dev;
    };

    void check_complete() {
        for (size_t i = 0; i < have.size(); ++i)
            require(have[i], BD_ERR_NAME_MISMATCH, "backbone: tensor '" + tname(i) + "' not set");
    }

    // validate coverage & shapes like register_delta (serve.cpp:134-149)
    std::vector<EntryView> resolve(const std::string& id, const std::map<std::string, EntryView>& ents) {
        std::vector<EntryView> out;
        for (size_t i = 0; i < have.size(); ++i) {
            const std::string n = tname(i);
            auto it = ents.find(n);
            require(it != ents.end(), BD_ERR_NAME_MISMATCH,
                    "delta '" + id + "': missing tensor '" + n + "'");
            uint64_t er, ec;
            shape(i, er, ec);
            require(it->second.rows == er && it->second.cols == ec, BD_ERR_SHAPE_MISMATCH,
                    "delta '" + id + "': tensor '" + n + "' has shape " +
                        std::to_string(it->second.rows) + "x" + std::to_string(it->second.cols) +
                        ", backbone expects " + std::to_string(er) + "x" + std::to_string(ec));
            out.push_back(it->second);
        }
        return out;
    }

    // host copy of row r of the reconstructed delta (add_delta_row, serve.cpp:39-48)
    std::vector<float> delta_row(const EntryView& e, uint64_t r) {
        std::vector<float> row(e.cols, 0.0f);
        if (e.packed) {
            const uint64_t nb = (e.rows * e.cols + 7) / 8;
            for (uint64_t k = 0; k < e.planes; ++k) {
                // fetch the bytes covering row r
                const uint64_t b0 = (r * e.cols) >> 3, b1 = ((r + 1) * e.cols + 7) >> 3;
                std::vector<uint8_t> bytes(b1 - b0);
                BD_CUDA(cudaMemcpy(bytes.data(), e.bits + k * nb + b0, b1 - b0,
                                   e.is_dev ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost));
                for (uint64_t c = 0; c < e.cols; ++c) {
                    const uint64_t idx = r * e.cols + c - b0 * 8;
                    row[c] += ((bytes[idx >> 3] >> (idx & 7)) & 1u) ? e.scales[k] : -e.scales[k];
                }
            }
        } else if (e.raw) {  // raw == null encodes an all-zero raw delta
            BD_CUDA(cudaMemcpy(row.data(), e.raw + r * e.cols, e.cols * 4,
                               e.is_dev ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost));
        }
        return row;
    }

    float* upload_f32(Tenant& t, const std::vector<float>& v) {
        float* d = dmalloc<float>(v.size(), &t.allocs);
        BD_CUDA(cudaMemcpy(d, v.data(), v.size() * 4, cudaMemcpyHostToDevice));
        return d;
    }

    std::vector<Plane> upload_planes(Tenant& t, const EntryView& e, uint64_t r0, uint64_t nr) {
        std::vector<Plane> out;
        const uint64_t nb = (e.rows * e.cols + 7) / 8;
        require((r0 * e.cols) % 8 == 0 || nr == e.rows, BD_ERR_BAD_ARGUMENT,
                "row shard does not start on a byte of the packed plane");
        const uint64_t b0 = (r0 * e.cols) / 8;
        const uint64_t len = nr == e.rows ? nb : (nr * e.cols + 7) / 8;
        for (uint64_t k = 0; k < e.planes; ++k) {
            uint8_t* d = dmalloc<uint8_t>(round_up(len, 16), &t.allocs);
            BD_CUDA(cudaMemset(d, 0, round_up(len, 16)));
            BD_CUDA(cudaMemcpy(d, e.bits + k * nb + b0, len,
                               e.is_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
            Plane pl{d, e.scales[k]};
            if (const uint64_t ld = lut_row_bytes(e.cols)) {  // padded copy for the LUT (+2.3 % at 11 008)
                uint8_t* q = dmalloc<uint8_t>(nr * ld, &t.allocs);
                BD_CUDA(cudaMemset(q, 0, nr * ld));
                BD_CUDA(cudaMemcpy2D(q, ld, d, e.cols / 8, e.cols / 8, nr, cudaMemcpyDeviceToDevice));
                pl.bits_lut = q;
                pl.ld_lut = int(ld);
            }
            out.push_back(pl);
        }
        return out;
    }

    float* upload_raw(Tenant& t, const EntryView& e) {
        if (!e.raw) return nullptr;  // all-zero raw delta: nothing resident
        float* d = dmalloc<float>(e.rows * e.cols, &t.allocs);
        BD_CUDA(cudaMemcpy(d, e.raw, e.rows * e.cols * 4,
                           e.is_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
        return d;
    }

    void load_tenant(Tenant& t, const std::vector<EntryView>& ev) {
        BD_CUDA(cudaSetDevice(device));
        t.proj.assign(a.n_layers, {});
        t.raw.assign(a.n_layers, {});
        t.norm1.assign(a.n_layers, nullptr);
        t.norm2.assign(a.n_layers, nullptr);
        t.bytes = 0;
        for (const auto& e : ev)
            t.bytes += e.packed ? e.planes * ((e.rows * e.cols + 7) / 8 + 4) : 4ull * e.rows * e.cols;
        const size_t last = 1 + 9 * a.n_layers;
        // embedding delta
        {
            const EntryView& e = ev[0];
            if (e.packed) {
                std::vector<float> full(e.rows * e.cols);
                for (uint64_t r = 0; r < e.rows; ++r) {
                    const auto row = delta_row(e, r);
                    std::copy(row.begin(), row.end(), full.begin() + r * e.cols);
                }
                t.embed_raw = upload_f32(t, full);
            } else {
                t.embed_raw = upload_raw(t, e);
            }
        }
        for (uint64_t l = 0; l < a.n_layers; ++l) {
            for (int p = 0; p < P_COUNT; ++p) {
                const EntryView& e = ev[1 + 9 * l + p];
                uint64_t r0, nr;
                local_rows(p, r0, nr);
                t.raw[l][p] = nullptr;
                if (!e.packed) {  // raw projection delta: resident in f32 (memory_report's 4 B/param)
                    if (e.raw) {
                        float* d = dmalloc<float>(nr * e.cols, &t.allocs);
                        BD_CUDA(cudaMemcpy(d, e.raw + r0 * e.cols, nr * e.cols * 4,
                                           e.is_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice));
                        t.raw[l][p] = d;
                    }
                    continue;
                }
                require(e.planes >= 1 && e.planes <= kMaxPlanesPerTensor, BD_ERR_BAD_ARGUMENT,
                        "delta '" + t.id + "': tensor '" + tname(1 + 9 * l + p) + "' has too many planes");
                t.proj[l][p] = upload_planes(t, e, r0, nr);
            }
            std::vector<float> n1 = base_norm1[l], n2 = base_norm2[l];
            const auto d1 = delta_row(ev[1 + 9 * l + 7], 0), d2 = delta_row(ev[1 + 9 * l + 8], 0);
            for (uint64_t i = 0; i < a.dim; ++i) { n1[i] += d1[i]; n2[i] += d2[i]; }
            t.norm1[l] = upload_f32(t, n1);
            t.norm2[l] = upload_f32(t, n2);
        }
        {
            std::vector<float> fn = base_final_norm;
            const auto d = delta_row(ev[last], 0);
            for (uint64_t i = 0; i < a.dim; ++i) fn[i] += d[i];
            t.final_norm = upload_f32(t, fn);
        }
        {
            const EntryView& e = ev[last + 1];
            if (e.packed) {
                require(e.planes <= kMaxPlanesPerUnit, BD_ERR_BAD_ARGUMENT, "lm_head: too many planes");
                t.lm_planes = upload_planes(t, e, 0, e.rows);
            } else {
                t.lm_raw = upload_raw(t, e);
            }
        }
        t.loaded = true;
        t.resident = true;
    }

    void register_entries(const std::string& id, const bd_delta_entry* ents, int n) {
        require(tenant_idx.count(id) == 0, BD_ERR_DUPLICATE_ID, "delta id already registered: " + id);
        check_complete();
        std::map<std::string, EntryView> m;
        for (int i = 0; i < n; ++i) {
            const bd_delta_entry& e = ents[i];
            require(e.name != nullptr, BD_ERR_BAD_ARGUMENT, "delta entry without a name");
            m[e.name] = EntryView{e.kind == 1, e.rows, e.cols, e.planes, e.bits, e.scales, e.raw,
                                  e.is_device != 0};
        }
        const auto ev = resolve(id, m);
        Tenant t;
        t.id = id;
        load_tenant(t, ev);
        tenant_idx[id] = int(tenants.size());
        tenants.push_back(std::move(t));
    }

    static std::map<std::string, EntryView> views(const DeltaFileHost& f) {
        std::map<std::string, EntryView> m;
        for (const auto& e : f.entries)
            m[e.name] = EntryView{e.packed, e.rows, e.cols, e.planes, e.bits.data(),
                                  e.scales.data(), e.raw.data(), false};
        return m;
    }

    void register_file(const std::string& id, const std::string& path, bool resident) {
        require(tenant_idx.count(id) == 0, BD_ERR_DUPLICATE_ID, "delta id already registered: " + id);
        check_complete();
        const DeltaFileHost f = read_bdelta(path);  // validate even when cold (serve.cpp:132)
        const auto ev = resolve(id, views(f));
        Tenant t;
        t.id = id;
        t.path = path;
        if (resident) load_tenant(t, ev);
        tenant_idx[id] = int(tenants.size());
        tenants.push_back(std::move(t));
    }

    // delta_for (serve.cpp:154-166): cold tenants are hot-swapped in on first use
    void ensure_loaded(int ti) {
        Tenant& t = tenants[ti];
        if (t.loaded) return;
        const auto t0 = std::chrono::steady_clock::now();
        const DeltaFileHost f = read_bdelta(t.path);
        load_tenant(t, resolve(t.id, views(f)));
        BD_CUDA(cudaDeviceSynchronize());
        const auto t1 = std::chrono::steady_clock::now();
        stats.cold_loads += 1;
        stats.last_cold_load_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        clear_plans();
    }

    uint64_t open_request(const std::string& id) {
        auto it = tenant_idx.find(id);
        require(it != tenant_idx.end(), BD_ERR_UNKNOWN_ID, "unknown delta id: " + id);
        Request r;
        r.tenant = it->second;
        r.open = true;
        const size_t n = a.n_layers * a.max_seq * kv_l;
        r.kc = dmalloc<uint16_t>(n);
        r.vc = dmalloc<uint16_t>(n);
        requests.push_back(r);
        return requests.size() - 1;
    }

    void close_request(uint64_t rid) {
        require(rid < requests.size() && requests[rid].open, BD_ERR_UNKNOWN_ID, "close_request: unknown request");
        Request& r = requests[rid];
        r.open = false;
        cudaFree(r.kc);
        cudaFree(r.vc);
        r.kc = r.vc = nullptr;
        clear_plans();
    }

    // ------------------------------------------------------------ decode --
    void ensure_ws(int B) {
        if (B <= ws_B) return;
        BD_CUDA(cudaStreamSynchronize(stream));
        clear_plans();
        free_ws();
        ws_B = std::max(B, 16);
        const uint64_t Mmax = std::max<uint64_t>({q_l + 2 * kv_l, a.dim, 2 * inter_l, a.vocab});
        x = dmalloc<float>(ws_B * a.dim, &ws_allocs);
        xn_f32 = dmalloc<float>(ws_B * a.dim, &ws_allocs);
        xn = dmalloc<uint16_t>(ws_B * ld_dim, &ws_allocs);
        ctx = dmalloc<uint16_t>(ws_B * ld_dim, &ws_allocs);
        act = dmalloc<uint16_t>(ws_B * ld_inter, &ws_allocs);
        BD_CUDA(cudaMemset(xn, 0, ws_B * ld_dim * 2));
        BD_CUDA(cudaMemset(ctx, 0, ws_B * ld_dim * 2));
        BD_CUDA(cudaMemset(act, 0, ws_B * ld_inter * 2));
        // delta partials: up to one per 1024-column slice (LUT path)
        D_elems = ws_B * Mmax * ((std::max(a.dim, a.intermediate) + 1023) / 1024);
        D = dmalloc<float>(D_elems, &ws_allocs);
        // split-K partials: bound by the planner's worst case (<= 32 splits)
        P_elems = 33ull * ws_B * Mmax;
        P = dmalloc<float>(P_elems, &ws_allocs);
        logits = dmalloc<float>(ws_B * a.vocab, &ws_allocs);
        msq = dmalloc<char>(norm_ws_bytes(int(ws_B), int(a.dim)), &ws_allocs);
        if (base_kind == 2) {
            xq = dmalloc<int8_t>(size_t(kPieces) * ws_B * std::max(ld8_dim, ld8_inter), &ws_allocs);
            xps = dmalloc<float>(size_t(kPieces) * ws_B, &ws_allocs);
            BD_CUDA(cudaMemset(xq, 0, size_t(kPieces) * ws_B * std::max(ld8_dim, ld8_inter)));
        }
        BD_CUDA(cudaMemset(msq, 0, norm_ws_bytes(int(ws_B), int(a.dim))));
        if (world > 1) {
            ctx_loc = dmalloc<uint16_t>(size_t(ws_B) * q_l, &ws_allocs);
            act_loc = dmalloc<uint16_t>(size_t(ws_B) * inter_l, &ws_allocs);
            gath16 = dmalloc<uint16_t>(size_t(world) * ws_B * std::max(q_l, inter_l), &ws_allocs);
            red_loc = dmalloc<float>(size_t(ws_B) * dim_l, &ws_allocs);
            gath32 = dmalloc<float>(size_t(world) * ws_B * dim_l, &ws_allocs);
        }
    }

    // Byte-LUT delta path (lut.cu): one job per request, planes read in the
    // reference layout with coalesced row loads. Used when tenants have few
    // requests each (the tensor-core path amortises expansion over many).
    void plan_lut_groups(Plan& p) {
        const int B = p.B;
        const uint64_t nL = a.n_layers;
        p.lut.assign(nL, {});
        struct GroupDef {
            std::vector<int> projs;
            uint64_t cols, ldx;
        };
        const GroupDef defs[4] = {{{P_Q, P_K, P_V}, a.dim, ld_dim},
                                  {{P_O}, a.dim, ld_dim},
                                  {{P_GATE, P_UP}, a.dim, ld_dim},
                                  {{P_DOWN}, a.intermediate, ld_inter}};
        for (int gi = 0; gi < 4; ++gi) {
            const GroupDef& gd = defs[gi];
            if (p.raw_group[gi]) continue;  // raw projection deltas: units path
            int seg_rows[kLutMaxSegs];
            for (size_t s = 0; s < gd.projs.size(); ++s) {
                uint64_t r0, nr;
                local_rows(gd.projs[s], r0, nr);
                seg_rows[s] = int(nr);
            }
            bool ok = true;
            const uint64_t lut_ld = lut_row_bytes(gd.cols);
            for (uint64_t l = 0; l < nL && ok; ++l) {
                for (int b0 = 0; b0 < B && ok; b0 += kLutMaxJobs) {
                    LutParams prm{};
                    prm.n_jobs = std::min(kLutMaxJobs, B - b0);
                    for (int q = 0; q < prm.n_jobs; ++q) {
                        LutJob& j = prm.jobs[q];
                        j.req = b0 + q;
                        const Tenant& t = tenants[requests[p.reqs[b0 + q]].tenant];
                        for (size_t s = 0; s < gd.projs.size(); ++s) {
                            const auto& planes = t.proj[l][gd.projs[s]];
                            j.n_planes[s] = int(planes.size());
                            for (size_t k = 0; k < planes.size(); ++k) {
                                // the padded rows where the pool keeps them (lut_row_bytes)
                                j.bits[s][k] = lut_ld ? planes[k].bits_lut : planes[k].bits;
                                j.alpha[s][k] = planes[k].alpha;
                            }
                        }
                    }
                    ok = plan_lut(prm, seg_rows, int(gd.projs.size()), int(gd.cols), int(gd.ldx), B);
                    if (ok && lut_ld) prm.ld_u4 = int(lut_ld / 16);
                    if (ok && size_t(prm.slices) * B * prm.M > D_elems) ok = false;
                    if (ok) p.lut[l][gi].prm.push_back(prm);
                }
                p.lut[l][gi].ok = ok;
            }
            if (!ok)
                for (uint64_t l = 0; l < nL; ++l) p.lut[l][gi] = Plan::Lut{};
        }
    }

    // K3d (mtd.cu): per tenant Y_t = alpha_t S_t X_t^T on the tensor cores, the tenant's
    // requests as the MMA's N (ascending pool request id inside a tenant, tenants by id)
    void plan_mtd_groups(Plan& p, std::map<int, std::vector<int>>& by_t) {
        const uint64_t nL = a.n_layers;
        p.mtd.assign(nL, {});
        struct GroupDef {
            std::vector<int> projs;
            uint64_t cols, ldx;
        };
        const GroupDef defs[4] = {{{P_Q, P_K, P_V}, a.dim, ld_dim},
                                  {{P_O}, a.dim, ld_dim},
                                  {{P_GATE, P_UP}, a.dim, ld_dim},
                                  {{P_DOWN}, a.intermediate, ld_inter}};
        for (int gi = 0; gi < 4; ++gi) {
            const GroupDef& gd = defs[gi];
            if (p.raw_group[gi]) continue;  // raw projection deltas: units path
            int seg_rows[kLutMaxSegs];
            for (size_t s2 = 0; s2 < gd.projs.size(); ++s2) {
                uint64_t r0, nr;
                local_rows(gd.projs[s2], r0, nr);
                seg_rows[s2] = int(nr);
            }
            bool ok = true;
            for (uint64_t l = 0; l < nL && ok; ++l) {
                std::vector<MtdTenant> tens;
                for (auto& kv : by_t) {
                    MtdTenant mt{};
                    mt.reqs = kv.second;
                    std::sort(mt.reqs.begin(), mt.reqs.end(), [&](int x, int y) { return p.reqs[x] < p.reqs[y]; });
                    for (size_t s2 = 0; s2 < gd.projs.size(); ++s2) {
                        const auto& planes = tenants[kv.first].proj[l][gd.projs[s2]];
                        mt.n_planes[s2] = int(planes.size());
                        mt.bits[s2] = planes.empty() ? nullptr : planes[0].bits;
                        mt.alpha[s2] = planes.empty() ? 0.0f : planes[0].alpha;
                    }
                    tens.push_back(mt);
                }
                std::vector<CUtensorMap> pmaps;
                Plan::Md md;
                int M = 0;
                for (size_t s2 = 0; s2 < gd.projs.size(); ++s2) M += seg_rows[s2];
                const int max_splits = int(D_elems / (size_t(p.B) * size_t(M)));
                if (!plan_mtd(md.prm, md.gat, tens, seg_rows, int(gd.projs.size()), int(gd.cols), int(gd.ldx),
                              max_splits, pmaps)) {
                    ok = false;
                    break;
                }
                md.prm.dstride = size_t(p.B) * size_t(M);
                if (!p.xg) {
                    p.xg_ld = int(std::max(ld_dim, ld_inter));
                    p.xg = dmalloc<uint16_t>(size_t(md.prm.x_rows) * p.xg_ld, &p.allocs);
                    BD_CUDA(cudaMemset(p.xg, 0, size_t(md.prm.x_rows) * p.xg_ld * 2));
                }
                const std::vector<CUtensorMap> xmaps = mtd_x_maps(md.prm, p.xg, p.xg_ld);
                CUtensorMap* dp = dmalloc<CUtensorMap>(pmaps.size(), &p.allocs);
                CUtensorMap* dx = dmalloc<CUtensorMap>(xmaps.size(), &p.allocs);
                BD_CUDA(cudaMemcpy(dp, pmaps.data(), pmaps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
                BD_CUDA(cudaMemcpy(dx, xmaps.data(), xmaps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
                md.prm.plane_maps = dp;
                md.prm.x_maps = dx;
                md.prm.out = D;
                md.ok = true;
                p.mtd[l][gi] = md;
            }
            if (!ok)
                for (uint64_t l = 0; l < nL; ++l) p.mtd[l][gi].ok = false;
        }
        // one gather map for every K3d group (the same tenant / request lists): the producers
        // of their inputs write the gathered rows themselves (XgOut)
        const MtdGather* g0 = nullptr;
        bool same = world == 1;
        for (uint64_t l = 0; l < nL; ++l)
            for (int gi = 0; gi < 4; ++gi)
                if (p.mtd[l][gi].ok) {
                    if (!g0) g0 = &p.mtd[l][gi].gat;
                    else same = same && std::memcmp(g0, &p.mtd[l][gi].gat, sizeof(MtdGather)) == 0;
                }
        if (g0 && same) {
            std::vector<int> row(p.B, -1);
            for (int t = 0; t < kMtdMaxTenants; ++t)
                for (int i = 0; i < g0->n_req[t]; ++i) row[g0->req[t][i]] = g0->row0[t] + i;
            if (std::find(row.begin(), row.end(), -1) == row.end()) {
                p.d_xrow = dmalloc<int>(row.size(), &p.allocs);
                BD_CUDA(cudaMemcpy(p.d_xrow, row.data(), row.size() * sizeof(int), cudaMemcpyHostToDevice));
                p.xg_direct = true;
            }
        }
    }
    // XgOut for the input of group gi of layer l (empty unless that group runs K3d)
    XgOut xg_out(const Plan& p, uint64_t l, int gi) const {
        XgOut o;
        if (p.xg_direct && mtd_ok(p, l, gi)) {
            o.xg = p.xg;
            o.ld = p.xg_ld;
            o.row = p.d_xrow;
        }
        return o;
    }

    // K23 (mt4.cu): base GEMM + every tenant plane as FP4 MMAs in one persistent
    // kernel. Slots are ordered by tenant id and, within a tenant, by request id,
    // so the schedule (and every output bit) is independent of the batch order.
    void plan_mt4_groups(Plan& p, std::map<int, std::vector<int>>& by_t) {
        const int B = p.B;
        const uint64_t nL = a.n_layers;
        if (B > 64) return;
        const int max_chunks = xp_chunks(int(std::max(a.dim, a.intermediate)));
        std::vector<int> tids;
        for (auto& kv : by_t) tids.push_back(kv.first);  // std::map: ascending tenant id
        std::map<int, std::vector<int>> rq_sorted;
        for (int t : tids) {
            std::vector<int> rq = by_t[t];
            std::sort(rq.begin(), rq.end(), [&](int x, int y) { return p.reqs[x] < p.reqs[y]; });
            rq_sorted[t] = rq;
        }
        struct GroupDef {
            std::vector<int> projs;
            uint64_t cols;
            const CUtensorMap* mx;
        };
        const GroupDef defs[4] = {{{P_Q, P_K, P_V}, a.dim, &p.x_xn},
                                  {{P_O}, a.dim, &p.x_ctx},
                                  {{P_GATE, P_UP}, a.dim, &p.x_xn},
                                  {{P_DOWN}, a.intermediate, &p.x_act}};
        bool any = false;
        p.mt4.assign(nL, {});
        for (int gi = 0; gi < 4; ++gi) {
            const GroupDef& gd = defs[gi];
            if (gd.cols % 128 || p.raw_group[gi]) continue;
            bool ok = true;
            uint64_t M = 0;
            std::vector<int> sub_row0;
            for (int pj : gd.projs) {
                uint64_t r0, nr;
                local_rows(pj, r0, nr);
                if (nr % 128) ok = false;
                sub_row0.push_back(int(M));
                M += nr;
            }
            sub_row0.push_back(int(M));
            if (!ok) continue;
            for (uint64_t l = 0; l < nL && ok; ++l) {
                Mt4Params prm{};
                prm.n_subs = int(gd.projs.size());
                for (size_t s2 = 0; s2 < sub_row0.size(); ++s2) prm.sub_row0[s2] = sub_row0[s2];
                std::vector<CUtensorMap> maps;
                for (int t : tids) {
                    const auto& rq = rq_sorted[t];
                    const size_t n_planes = tenants[t].proj[l][gd.projs[0]].size();
                    for (size_t k = 0; k < n_planes && ok; ++k) {
                        int midx[kMt4MaxSubs];
                        for (size_t s2 = 0; s2 < gd.projs.size(); ++s2) {
                            const int pj = gd.projs[s2];
                            const auto& planes = tenants[t].proj[l][pj];
                            if (planes.size() != n_planes ||
                                reinterpret_cast<uintptr_t>(planes[k].bits) % 16) { ok = false; break; }
                            uint64_t r0, nr;
                            local_rows(pj, r0, nr);
                            midx[s2] = int(maps.size());
                            maps.push_back(tmap_bits4(planes[k].bits, nr, gd.cols));
                        }
                        for (size_t c = 0, n = 0; c < rq.size() && ok; c += n) {
                            if (prm.n_slots >= kMt4MaxSlots) { ok = false; break; }
                            Mt4Slot& sl = prm.slots[prm.n_slots++];
                            n = size_t(mt4_slot_requests(rq.size() - c));
                            sl.n_req = int(n);
                            for (int q = 0; q < sl.n_req; ++q) sl.req[q] = rq[c + q];
                            for (size_t s2 = 0; s2 < gd.projs.size(); ++s2) {
                                sl.alpha[s2] = tenants[t].proj[l][gd.projs[s2]][k].alpha;
                                sl.map_idx[s2] = midx[s2];
                            }
                        }
                    }
                }
                if (!ok || !plan_mt4(prm, M, gd.cols, B)) { ok = false; break; }
                if (uint64_t(prm.splits) * B * M > P_elems) { ok = false; break; }
                if (!p.xpk) {
                    p.xpk = dmalloc<uint8_t>(size_t(B) * max_chunks * kXpBlock, &p.allocs);
                    BD_CUDA(cudaMemset(p.xpk, 0, size_t(B) * max_chunks * kXpBlock));
                }
                CUtensorMap* dm = dmalloc<CUtensorMap>(maps.size(), &p.allocs);
                BD_CUDA(cudaMemcpy(dm, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
                prm.bits_maps = dm;
                const std::vector<uint32_t> sched = mt4_schedule(prm);
                uint32_t* dsch = dmalloc<uint32_t>(sched.size(), &p.allocs);
                BD_CUDA(cudaMemcpy(dsch, sched.data(), sched.size() * 4, cudaMemcpyHostToDevice));
                prm.sched = dsch;
                const LayerW& W = L[l];
                prm.map_w = gi == 0 ? W.m_qkv : gi == 1 ? W.m_o : gi == 2 ? W.m_gu : W.m_down;
                const uint64_t ldx = gi == 3 ? ld_inter : ld_dim;
                const uint16_t* X = gi == 1 ? ctx : gi == 3 ? act : xn;
                prm.map_x = tmap_acts(X, B, gd.cols, ldx, prm.bn);
                prm.xpk = p.xpk;
                prm.partial = P;
                p.mt4[l][gi].prm = prm;
                p.mt4[l][gi].ok = true;
                any = true;
            }
            if (!ok)
                for (uint64_t l = 0; l < nL; ++l) p.mt4[l][gi].ok = false;
        }
        (void)any;
    }

    Plan& plan_for(const std::vector<int>& reqs) {
        std::string key;
        for (int r : reqs) key += std::to_string(r) + ",";
        auto it = plans.find(key);
        if (it != plans.end()) return *it->second;
        const int B = int(reqs.size());
        ensure_ws(B);
        auto p = std::make_unique<Plan>();
        p->B = B;
        p->reqs = reqs;
        const uint64_t nL = a.n_layers;
        std::vector<float*> norms((2 * nL + 1) * B);
        std::vector<uint16_t*> kc(B), vc(B);
        std::vector<float*> emb(B), lmr(B);
        bool any_lmraw = false;
        for (int b = 0; b < B; ++b) {
            const Request& r = requests[reqs[b]];
            const Tenant& t = tenants[r.tenant];
            for (uint64_t l = 0; l < nL; ++l) {
                norms[(2 * l) * B + b] = t.norm1[l];
                norms[(2 * l + 1) * B + b] = t.norm2[l];
            }
            norms[(2 * nL) * B + b] = t.final_norm;
            kc[b] = r.kc;
            vc[b] = r.vc;
            emb[b] = t.embed_raw;
            lmr[b] = t.lm_raw;
            any_lmraw |= t.lm_raw != nullptr;
        }
        auto upload_ptrs = [&](auto& vec) {
            using T = typename std::remove_reference<decltype(vec)>::type::value_type;
            T* d = dmalloc<T>(vec.size(), &p->allocs);
            BD_CUDA(cudaMemcpy(d, vec.data(), vec.size() * sizeof(T), cudaMemcpyHostToDevice));
            return d;
        };
        p->d_norm = upload_ptrs(norms);
        p->d_kc = upload_ptrs(kc);
        p->d_vc = upload_ptrs(vc);
        p->d_embed = upload_ptrs(emb);
        p->d_lmraw = any_lmraw ? upload_ptrs(lmr) : nullptr;
        p->d_pos = dmalloc<int>(B, &p->allocs);
        p->d_tok = dmalloc<int>(B, &p->allocs);
        for (int k = 0; k < 2; ++k) {
            BD_CUDA(cudaMallocHost(&p->h_pos[k], B * sizeof(int)));
            BD_CUDA(cudaMallocHost(&p->h_tok[k], B * sizeof(int)));
            BD_CUDA(cudaEventCreateWithFlags(&p->staged[k], cudaEventDisableTiming));
        }

        // tenant segmentation
        std::vector<int> order;
        std::map<int, std::vector<int>> by_t;
        for (int b = 0; b < B; ++b) {
            const int t = requests[reqs[b]].tenant;
            if (!by_t.count(t)) order.push_back(t);
            by_t[t].push_back(b);
        }
        // chunk c of a projection's planes (kMaxPlanesPerUnit each): c = 0 the main units,
        // c >= 1 the accumulate passes
        auto units_for = [&](std::initializer_list<int> projs, uint64_t l, int chunk = 0) {
            std::vector<DeltaUnit> out;
            for (int t : order) {
                const auto& rq = by_t[t];
                for (size_t c = 0; c < rq.size(); c += kMaxReqPerUnit) {
                    for (int pj : projs) {
                        DeltaUnit u{};
                        const auto& planes = tenants[t].proj[l][pj];
                        if (planes.empty()) continue;  // raw projection delta (raw pass)
                        const int k0 = chunk * kMaxPlanesPerUnit;
                        if (int(planes.size()) <= k0) continue;
                        u.n_planes = std::min(kMaxPlanesPerUnit, int(planes.size()) - k0);
                        for (int k = 0; k < u.n_planes; ++k) {
                            u.bits[k] = planes[k0 + k].bits;
                            u.alpha[k] = planes[k0 + k].alpha;
                        }
                        uint64_t r0, nr;
                        local_rows(pj, r0, nr);
                        u.row0 = int(stack_offset(pj));
                        u.rows = int(nr);
                        u.n_req = int(std::min<size_t>(kMaxReqPerUnit, rq.size() - c));
                        for (int q = 0; q < u.n_req; ++q) u.req[q] = rq[c + q];
                        out.push_back(u);
                    }
                }
            }
            return out;
        };
        p->units.resize(nL);
        for (uint64_t l = 0; l < nL; ++l) {
            p->units[l][0] = units_for({P_Q, P_K, P_V}, l);
            p->units[l][1] = units_for({P_O}, l);
            p->units[l][2] = units_for({P_GATE, P_UP}, l);
            p->units[l][3] = units_for({P_DOWN}, l);
        }
        // planes beyond kMaxPlanesPerUnit: accumulate passes, the group on the units path
        p->units_x.assign(nL, {});
        {
            const std::vector<int> gp[4] = {{P_Q, P_K, P_V}, {P_O}, {P_GATE, P_UP}, {P_DOWN}};
            for (uint64_t l = 0; l < nL; ++l)
                for (int gi = 0; gi < 4; ++gi) {
                    int max_planes = 0;
                    for (int t : order)
                        for (int pj : gp[gi]) max_planes = std::max(max_planes, int(tenants[t].proj[l][pj].size()));
                    if (max_planes <= kMaxPlanesPerUnit) continue;
                    p->raw_group[gi] = true;
                    for (int c = 1; c * kMaxPlanesPerUnit < max_planes; ++c) {
                        auto more = gi == 0 ? units_for({P_Q, P_K, P_V}, l, c)
                                    : gi == 1 ? units_for({P_O}, l, c)
                                    : gi == 2 ? units_for({P_GATE, P_UP}, l, c)
                                              : units_for({P_DOWN}, l, c);
                        p->units_x[l][gi].insert(p->units_x[l][gi].end(), more.begin(), more.end());
                    }
                }
        }
        // raw projection deltas: one job per (tenant, projection, <= kRawMaxReq requests)
        {
            const std::vector<int> gp[4] = {{P_Q, P_K, P_V}, {P_O}, {P_GATE, P_UP}, {P_DOWN}};
            p->raw.assign(nL, {});
            for (uint64_t l = 0; l < nL; ++l)
                for (int gi = 0; gi < 4; ++gi)
                    for (int pj : gp[gi])
                        for (int t : order) {
                            const Tenant& tn = tenants[t];
                            if (!tn.proj[l][pj].empty()) continue;
                            p->raw_group[gi] = true;  // raw entry (null: all zero, no job)
                            if (!tn.raw[l][pj]) continue;
                            const auto& rq = by_t[t];
                            uint64_t r0, nr;
                            local_rows(pj, r0, nr);
                            for (size_t c = 0; c < rq.size(); c += kRawMaxReq) {
                                RawJob j{};
                                j.W = tn.raw[l][pj];
                                j.row0 = int(stack_offset(pj));
                                j.rows = int(nr);
                                j.n_req = int(std::min<size_t>(kRawMaxReq, rq.size() - c));
                                for (int q = 0; q < j.n_req; ++q) j.req[q] = rq[c + q];
                                p->raw[l][gi].push_back(j);
                            }
                        }
        }
        for (int t : order) {
            const auto& rq = by_t[t];
            const auto& planes = tenants[t].lm_planes;
            if (planes.empty()) continue;
            for (size_t c = 0; c < rq.size(); c += kMaxReqPerUnit) {
                DeltaUnit u{};
                u.n_planes = int(planes.size());
                for (size_t k = 0; k < planes.size(); ++k) {
                    u.bits[k] = planes[k].bits;
                    u.alpha[k] = planes[k].alpha;
                }
                u.row0 = 0;
                u.rows = int(a.vocab);
                u.n_req = int(std::min<size_t>(kMaxReqPerUnit, rq.size() - c));
                for (int q = 0; q < u.n_req; ++q) u.req[q] = rq[c + q];
                p->lm_units.push_back(u);
            }
        }
        const bool i8 = base_kind == 2;
        require(!i8 || B <= 64, BD_ERR_BAD_ARGUMENT, "decode: an int8 backbone serves batches of <= 64");
        p->g_qkv = plan_gemm(q_l + 2 * kv_l, a.dim, B, 0, i8);
        p->g_o = plan_gemm(dim_l, a.dim, B, 0, i8);
        p->g_gu = plan_gemm(2 * inter_l, a.dim, B, 0, i8);
        p->g_down = plan_gemm(dim_l, a.intermediate, B, 0, i8);
        p->g_lm = plan_base_gemm(a.vocab, a.dim, B);
        for (const GemmPlan* g : {&p->g_qkv, &p->g_o, &p->g_gu, &p->g_down, &p->g_lm})
            require(uint64_t(g->splits) * B * g->M <= P_elems, BD_ERR_CUDA, "split-K workspace too small");
        const int bn = p->g_lm.bn;  // bf16 B operand (lm_head is always bf16)
        p->x_xn = tmap_acts(xn, B, a.dim, ld_dim, bn);
        p->x_ctx = tmap_acts(ctx, B, a.dim, ld_dim, bn);
        p->x_act = tmap_acts(act, B, a.intermediate, ld_inter, bn);
        if (i8) {
            p->xq_dim = tmap_pieces(xq, B, a.dim, ld8_dim, p->g_qkv.bn);
            p->xq_inter = tmap_pieces(xq, B, a.intermediate, ld8_inter, p->g_qkv.bn);
        }
        // K3 variant for the whole batch (one backend, chosen by requests per tenant): K3d when
        // tenants average kMtdMinRequests or more at batch >= kMtdMinBatch (a plane expanded once serves all of its
        // tenant's requests as MMA columns), else K23 from k23_min_requests(B) (each plane read
        // once per slot of up to 4 requests), else the byte LUT beside K2 (one job per request);
        // the mean, not the maximum, so one busy tenant does not move a batch of single-request
        // tenants off the LUT (measured slower there). Groups a variant cannot
        // plan fall through to the next one.
        const double mean_per_tenant = order.empty() ? 0.0 : double(B) / double(order.size());
        if (delta_mode == "mtd" ||
            (delta_mode == "auto" && mean_per_tenant >= kMtdMinRequests && B >= kMtdMinBatch))
            plan_mtd_groups(*p, by_t);
        // K23 fuses the bf16 base GEMM: not for an int8 backbone
        if (!i8 && (delta_mode == "mt4" || (delta_mode == "auto" && mean_per_tenant >= k23_min_requests(B))))
            plan_mt4_groups(*p, by_t);
        // forced K3d: groups it cannot plan (> kMtdMaxTenants tenants, ...) take the LUT
        if (delta_mode == "lut" || delta_mode == "auto" || delta_mode == "mtd") plan_lut_groups(*p);
        // groups already served by K3d keep no K23 / LUT plan, groups served by K23 no LUT plan
        for (uint64_t l = 0; l < p->mtd.size(); ++l)
            for (int gi = 0; gi < 4; ++gi)
                if (p->mtd[l][gi].ok) {
                    if (p->mt4.size() > l) p->mt4[l][gi].ok = false;
                    if (p->lut.size() > l) p->lut[l][gi] = Plan::Lut{};
                }
        for (uint64_t l = 0; l < p->mt4.size(); ++l)
            for (int gi = 0; gi < 4; ++gi)
                if (p->mt4[l][gi].ok && !p->lut.empty()) p->lut[l][gi] = Plan::Lut{};
        if (!p->lut.empty()) {
            // K2 runs beside the K3 LUT on every SM: one GEMM CTA per SM within the
            // shared memory the LUT leaves (LUT: 132 KB + 512 threads x 96 regs)
            GemmPlan* gs[4] = {&p->g_qkv, &p->g_o, &p->g_gu, &p->g_down};
            for (int gi = 0; gi < 4; ++gi)
                if (p->lut[0][gi].ok) {
                    *gs[gi] = plan_gemm(gs[gi]->M, gs[gi]->K, B, BD_K2_CAP_KB * 1024, i8);
                    require(uint64_t(gs[gi]->splits) * B * gs[gi]->M <= P_elems, BD_ERR_CUDA,
                            "split-K workspace too small");
                }
        }
        auto& slot = plans[key];
        slot = std::move(p);
        return *slot;
    }

    ProjOut proj_out(const GemmPlan& g, bool with_delta) const {
        ProjOut o;
        o.P = P;
        o.splits = g.splits;
        o.pstride = size_t(g.batch) * g.M;
        o.D = with_delta ? D : nullptr;
        o.dsplits = 1;
        o.dstride = size_t(g.batch) * g.M;
        o.M = int(g.M);
        return o;
    }

    // ---- optional per-kernel profiling (eager mode only) ----
    bool profiling = false;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> prof_events;
    template <class F>
    void prof(int kind, cudaStream_t s, F&& f) {
        if (!profiling) {
            f();
            return;
        }
        // external event-record nodes when captured: the graph is timed as it replays
        cudaEvent_t e0, e1;
        BD_CUDA(cudaEventCreate(&e0));
        BD_CUDA(cudaEventCreate(&e1));
        BD_CUDA(cudaEventRecordWithFlags(e0, s, cudaEventRecordExternal));
        f();
        BD_CUDA(cudaEventRecordWithFlags(e1, s, cudaEventRecordExternal));
        prof_events.push_back({kind, {e0, e1}});
    }

    bool lut_ok(const Plan& p, uint64_t l, int gi) const { return p.lut.size() > l && p.lut[l][gi].ok; }
    bool mt4_ok(const Plan& p, uint64_t l, int gi) const { return p.mt4.size() > l && p.mt4[l][gi].ok; }
    bool mtd_ok(const Plan& p, uint64_t l, int gi) const { return p.mtd.size() > l && p.mtd[l][gi].ok; }
    ProjOut group_out(const Plan& p, uint64_t l, int gi, const GemmPlan& g) const {
        if (mt4_ok(p, l, gi)) {
            const Mt4Params& f = p.mt4[l][gi].prm;
            ProjOut o;
            o.P = P;
            o.splits = f.splits;
            o.pstride = size_t(p.B) * f.M;
            o.D = nullptr;
            o.M = f.M;
            return o;
        }
        if (mtd_ok(p, l, gi)) {  // one delta partial per K split
            ProjOut o = proj_out(g, true);
            o.dsplits = p.mtd[l][gi].prm.ksplit;
            return o;
        }
        if (lut_ok(p, l, gi)) {
            ProjOut o = proj_out(g, true);
            o.dsplits = p.lut[l][gi].prm[0].slices;
            return o;
        }
        return proj_out(g, true);
    }

    // K2 for one projection group: the bf16 tcgen05 GEMM, or (int8 backbone) the kind::i8
    // GEMM against the pieces quant_pieces_launch wrote for this linear's input
    void base_gemm(const GemmPlan& g, uint64_t l, int group, const CUtensorMap& mw, const CUtensorMap& mx,
                   cudaStream_t st) {
        if (g.i8) i8_gemm_launch(g, mw, mx, L[l].s8[group], xps, P, st);
        else base_gemm_launch(g, mw, mx, P, st);
    }

    void linear(Plan& p, uint64_t l, int group, const GemmPlan& g, const CUtensorMap& mw,
                const CUtensorMap& mx, const std::vector<DeltaUnit>& units, const uint16_t* X,
                int ldx, int cols, int B, cudaStream_t s) {
        if (g.i8) {
            // the pieces buffer is free: the previous linear's K2 joined stream s before its
            // consumer ran
            prof(BD_PROF_XQ_PREP, s, [&] {
                quant_pieces_launch(X, false, ldx, cols, B, xq, int(group == 3 ? ld8_inter : ld8_dim), xps, s);
            });
        }
        if (mt4_ok(p, l, group)) {
            prof(BD_PROF_XQ_PREP, s, [&] { xp_prep_launch(X, ldx, cols, B, p.xpk, s); });
            prof(BD_PROF_FUSED_QKV + group, s, [&] { mt4_launch(p.mt4[l][group].prm, s); });
            return;
        }
        if (mtd_ok(p, l, group)) {
            // K2 and K3d both hold the SM's tensor memory: one after the other
            const Plan::Md& md = p.mtd[l][group];
            if (!xg_done)
                prof(BD_PROF_XQ_PREP, s, [&] { mtd_gather_launch(X, ldx, cols, md.gat, md.prm.n_ten, p.xg, p.xg_ld, s); });
            xg_done = false;
            prof(BD_PROF_GEMM_QKV + group, s, [&] { base_gemm(g, l, group, mw, mx, s); });
            prof(BD_PROF_DELTA_QKV + group, s, [&] { mtd_launch(md.prm, s); });
            return;
        }
        if (lut_ok(p, l, group)) {
            const auto& luts = p.lut[l][group].prm;
            if (concurrent_k23) {
                // K3 (CUDA cores / LSU) and K2 (TMA + tensor pipe) share every SM:
                // fork the GEMM onto the side stream, join before the consumer.
                // Profiled as one unit (kind FUSED_*: all of K2+K3 for the group).
                prof(BD_PROF_FUSED_QKV + group, s, [&] {
                    BD_CUDA(cudaEventRecord(ev_fork, s));
                    BD_CUDA(cudaStreamWaitEvent(stream2, ev_fork, 0));
                    for (const LutParams& lp : luts) lut_launch(lp, X, D, s);
                    base_gemm(g, l, group, mw, mx, stream2);
                    BD_CUDA(cudaEventRecord(ev_join, stream2));
                    BD_CUDA(cudaStreamWaitEvent(s, ev_join, 0));
                });
                return;
            }
            // serial (profile_layers_serial): K2 and K3 timed on their own
            prof(BD_PROF_GEMM_QKV + group, s, [&] { base_gemm(g, l, group, mw, mx, s); });
            prof(BD_PROF_DELTA_QKV + group, s, [&] {
                for (const LutParams& lp : luts) lut_launch(lp, X, D, s);
            });
            return;
        }
        prof(BD_PROF_GEMM_QKV + group, s, [&] { base_gemm(g, l, group, mw, mx, s); });
        prof(BD_PROF_DELTA_QKV + group, s, [&] {
            delta_units_launch(units.data(), int(units.size()), X, ldx, cols, B, D, int(g.M), s);
            // one launch per further plane chunk: a unit's rows are never written twice in one launch
            const auto& ux = p.units_x[l][group];
            for (size_t i0 = 0; i0 < ux.size();) {
                size_t i1 = i0 + 1;  // the next run of units with no (request, row) overlap
                auto overlaps = [&](const DeltaUnit& a2, const DeltaUnit& b2) {
                    if (a2.row0 != b2.row0) return false;
                    for (int x = 0; x < a2.n_req; ++x)
                        for (int y = 0; y < b2.n_req; ++y)
                            if (a2.req[x] == b2.req[y]) return true;
                    return false;
                };
                while (i1 < ux.size()) {
                    bool clash = false;
                    for (size_t k = i0; k < i1 && !clash; ++k) clash = overlaps(ux[k], ux[i1]);
                    if (clash) break;
                    ++i1;
                }
                delta_units_launch(ux.data() + i0, int(i1 - i0), X, ldx, cols, B, D, int(g.M), s, true);
                i0 = i1;
            }
            const auto& rj = p.raw[l][group];
            if (!rj.empty()) raw_delta_launch(rj.data(), int(rj.size()), X, ldx, cols, D, int(g.M), s);
        });
    }

    // the layer loop of decode_shared (serve.cpp:240-310); x holds the
    // residual stream entering layer 0 and leaves it after the last layer
    // ---- tensor-parallel exchanges (world > 1): NCCL all-gather over NVLink ----
    // bf16 activation slice [B x n_l] -> every rank's slices -> [B x ld] in column order
    void all_gather(const void* send, void* recv, size_t cnt, ncclDataType_t dt, size_t elem, cudaStream_t s) {
        if (!loop) {
            BD_NCCL(ncclAllGather(send, recv, cnt, dt, comm, s));
            return;
        }
        LoopbackGroup& G = *loop;
        const size_t bytes = cnt * elem;
        G.recv[rank] = recv;
        BD_CUDA(cudaEventRecord(lb_ready, s));  // this rank's earlier readers of recv are done
        G.ready[rank] = lb_ready;
        G.barrier();
        for (int q = 0; q < world; ++q) {
            BD_CUDA(cudaStreamWaitEvent(s, G.ready[q], 0));
            BD_CUDA(cudaMemcpyAsync(static_cast<char*>(G.recv[q]) + rank * bytes, send, bytes,
                                    cudaMemcpyDeviceToDevice, s));
        }
        BD_CUDA(cudaEventRecord(lb_done, s));
        G.done[rank] = lb_done;
        G.barrier();
        for (int q = 0; q < world; ++q) BD_CUDA(cudaStreamWaitEvent(s, G.done[q], 0));
        G.barrier();  // all waits enqueued before any rank re-records its events
    }
    void exchange_bf16(const uint16_t* local, int B, int n_l, uint16_t* full, int ld, cudaStream_t s) {
        const size_t cnt = size_t(B) * n_l;
        all_gather(local, gath16, cnt, ncclBfloat16, 2, s);
        gather_transpose_launch(gath16, world, B, n_l, full, ld, s);
    }
    // row-sharded f32 projection output -> gathered view consumed by the residual kernel
    ProjOut exchange_f32(const ProjOut& part, int B, int n_l, cudaStream_t s) {
        shard_reduce_launch(part, B, n_l, red_loc, s);
        all_gather(red_loc, gath32, size_t(B) * n_l, ncclFloat32, 4, s);
        ProjOut g;
        g.G = gath32;
        g.g_cols = n_l;
        g.g_batch = B;
        return g;
    }

    void run_layers(Plan& p, cudaStream_t s) {
        const int B = p.B;
        const uint64_t nL = a.n_layers;
        const bool tp = world > 1;
        // attention runs on this rank's heads only (q/k/v are sharded by heads)
        AttnArgs aa{int(q_l), int(kv_l), int(a.n_heads / world), int(n_kv_heads / world), int(hd),
                    int(a.max_seq), 0, p.d_kc, p.d_vc, rope};
        ProjOut prev;  // pending residual contribution (previous layer's down)
        for (uint64_t l = 0; l < nL; ++l) {
            const LayerW& W = L[l];
            // x += down(prev); xn = norm1(x)   (x and xn replicated on every rank)
            prof(BD_PROF_NORM, s, [&] {
                xg_done = resid_norm_launch(x, B, int(a.dim), prev, p.d_norm + (2 * l) * B, xn, int(ld_dim),
                                            nullptr, msq, s, xg_out(p, l, 0));
            });
            const bool i8 = base_kind == 2;
            linear(p, l, 0, p.g_qkv, i8 ? W.m8[0] : W.m_qkv, i8 ? p.xq_dim : p.x_xn, p.units[l][0], xn,
                   int(ld_dim), int(a.dim), B, s);
            aa.layer = int(l);
            aa.xo = xg_out(p, l, 1);
            prof(BD_PROF_ATTN, s, [&] {
                xg_done = attn_launch(group_out(p, l, 0, p.g_qkv), aa, p.d_pos, B, tp ? ctx_loc : ctx,
                                      tp ? int(q_l) : int(ld_dim), s);
            });
            if (tp) exchange_bf16(ctx_loc, B, int(q_l), ctx, int(ld_dim), s);
            linear(p, l, 1, p.g_o, i8 ? W.m8[1] : W.m_o, i8 ? p.xq_dim : p.x_ctx, p.units[l][1], ctx,
                   int(ld_dim), int(a.dim), B, s);
            const ProjOut o_out = tp ? exchange_f32(group_out(p, l, 1, p.g_o), B, int(dim_l), s)
                                     : group_out(p, l, 1, p.g_o);
            prof(BD_PROF_NORM, s, [&] {
                xg_done = resid_norm_launch(x, B, int(a.dim), o_out, p.d_norm + (2 * l + 1) * B, xn, int(ld_dim),
                                            nullptr, msq, s, xg_out(p, l, 2));
            });
            linear(p, l, 2, p.g_gu, i8 ? W.m8[2] : W.m_gu, i8 ? p.xq_dim : p.x_xn, p.units[l][2], xn,
                   int(ld_dim), int(a.dim), B, s);
            prof(BD_PROF_SILU, s, [&] {
                xg_done = silu_launch(group_out(p, l, 2, p.g_gu), B, int(inter_l), tp ? act_loc : act,
                                      tp ? int(inter_l) : int(ld_inter), s, xg_out(p, l, 3));
            });
            if (tp) exchange_bf16(act_loc, B, int(inter_l), act, int(ld_inter), s);
            linear(p, l, 3, p.g_down, i8 ? W.m8[3] : W.m_down, i8 ? p.xq_inter : p.x_act, p.units[l][3], act,
                   int(ld_inter), int(a.intermediate), B, s);
            prev = tp ? exchange_f32(group_out(p, l, 3, p.g_down), B, int(dim_l), s)
                      : group_out(p, l, 3, p.g_down);
        }
        prof(BD_PROF_NORM, s, [&] {
            resid_norm_launch(x, B, int(a.dim), prev, nullptr, nullptr, 0, nullptr, msq, s);
        });
    }

    void run_full(Plan& p, cudaStream_t s) {
        const int B = p.B;
        embed_launch(embed, p.d_tok, p.d_embed, B, int(a.dim), x, s);
        run_layers(p, s);
        resid_norm_launch(x, B, int(a.dim), ProjOut{}, p.d_norm + (2 * a.n_layers) * B, xn,
                          int(ld_dim), xn_f32, msq, s);
        base_gemm_launch(p.g_lm, m_lm, p.x_xn, P, s);
        delta_units_launch(p.lm_units.data(), int(p.lm_units.size()), xn, int(ld_dim), int(a.dim),
                           B, D, int(a.vocab), s);
        logits_launch(proj_out(p.g_lm, true), p.d_lmraw, xn_f32, B, int(a.dim), int(a.vocab),
                      logits, s);
    }

    // K3 variant per projection group (q/k/v, o, gate/up, down) of layer 0 of plan p:
    // T = K23 (FP4 tensor cores, fused with K2), L = byte LUT beside K2, U = SIMT units
    void record_paths(const Plan& p) {
        for (int gi = 0; gi < 4; ++gi) {
            char c = 'U';
            if (a.n_layers == 0) c = '-';
            else if (mt4_ok(p, 0, gi)) c = 'T';
            else if (mtd_ok(p, 0, gi)) c = 'D';
            else if (lut_ok(p, 0, gi)) c = 'L';
            stats.delta_paths[gi] = c;
        }
        stats.delta_paths[4] = 0;
    }

    void execute(Plan& p, bool full) {
        record_paths(p);
        cudaGraphExec_t& g = full ? p.graph_full : p.graph_layers;
        uint64_t& kcount = full ? p.kernels_full : p.kernels_layers;
        if (!use_graphs) {
            const uint64_t c0 = launch_count();
            if (full) run_full(p, stream); else run_layers(p, stream);
            stats.kernels_last_step = launch_count() - c0;
            return;
        }
        if (profiling) {
            // a throw-away graph with external event-record nodes around every kernel
            // (or concurrent K2||K3 pair), replayed once: device times as in production
            cudaGraph_t graph;
            cudaGraphExec_t ge;
            BD_CUDA(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
            try {
                if (full) run_full(p, stream); else run_layers(p, stream);
            } catch (...) {
                cudaStreamEndCapture(stream, &graph);
                throw;
            }
            BD_CUDA(cudaStreamEndCapture(stream, &graph));
            BD_CUDA(cudaGraphInstantiate(&ge, graph, 0));
            BD_CUDA(cudaGraphLaunch(ge, stream));
            BD_CUDA(cudaStreamSynchronize(stream));
            BD_CUDA(cudaGraphExecDestroy(ge));
            BD_CUDA(cudaGraphDestroy(graph));
            return;
        }
        if (!g) {
            cudaGraph_t graph;
            const uint64_t c0 = launch_count();
            BD_CUDA(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
            try {
                if (full) run_full(p, stream); else run_layers(p, stream);
            } catch (...) {
                cudaStreamEndCapture(stream, &graph);
                throw;
            }
            BD_CUDA(cudaStreamEndCapture(stream, &graph));
            kcount = launch_count() - c0;
            promote_programmatic_edges(graph);
            BD_CUDA(cudaGraphInstantiate(&g, graph, 0));
            BD_CUDA(cudaGraphDestroy(graph));
        }
        BD_CUDA(cudaGraphLaunch(g, stream));
        stats.kernels_last_step = kcount;
    }

    // Stream capture turns the fork/join of K2 (side stream) into full dependencies;
    // every kernel-to-kernel edge whose consumer waits in griddep_wait() before touching
    // its inputs becomes programmatic, so K2 (and the glue after a join) is scheduled
    // while its predecessor drains and streams its constant weights meanwhile.
    static void promote_programmatic_edges(cudaGraph_t graph) {
        size_t n = 0;
        BD_CUDA(cudaGraphGetEdges_v2(graph, nullptr, nullptr, nullptr, &n));
        std::vector<cudaGraphNode_t> from(n), to(n);
        std::vector<cudaGraphEdgeData> ed(n);
        BD_CUDA(cudaGraphGetEdges_v2(graph, from.data(), to.data(), ed.data(), &n));
        auto kernel_fn = [](cudaGraphNode_t nd) -> const void* {
            cudaGraphNodeType t;
            BD_CUDA(cudaGraphNodeGetType(nd, &t));
            if (t != cudaGraphNodeTypeKernel) return nullptr;
            cudaKernelNodeParams kp{};
            BD_CUDA(cudaGraphKernelNodeGetParams(nd, &kp));
            return kp.func;
        };
        for (size_t i = 0; i < n; ++i) {
            if (ed[i].type != cudaGraphDependencyTypeDefault) continue;
            if (!kernel_fn(from[i])) continue;
            const void* f = kernel_fn(to[i]);
            if (!f || !is_pdl_kernel(f)) continue;
            BD_CUDA(cudaGraphRemoveDependencies_v2(graph, &from[i], &to[i], &ed[i], 1));
            cudaGraphEdgeData e{};
            e.from_port = cudaGraphKernelNodePortProgrammatic;
            e.type = cudaGraphDependencyTypeProgrammatic;
            BD_CUDA(cudaGraphAddDependencies_v2(graph, &from[i], &to[i], &e, 1));
        }
    }

    void validate(const bd_request* reqs, uint64_t n) {
        for (uint64_t i = 0; i < n; ++i) {
            const bd_request& q = reqs[i];
            require(q.request_id < requests.size() && requests[q.request_id].open, BD_ERR_UNKNOWN_ID,
                    "decode: unknown request id");
            const Request& r = requests[q.request_id];
            require(q.position == r.pos, BD_ERR_BAD_ARGUMENT,
                    "decode: request position does not match cache position");
            require(r.pos < a.max_seq, BD_ERR_BAD_ARGUMENT, "decode: context exceeds max_seq");
            require(q.token >= 0 && uint64_t(q.token) < a.vocab, BD_ERR_BAD_TOKEN,
                    "decode: token id out of range");
            for (uint64_t j = 0; j < i; ++j)
                require(reqs[j].request_id != q.request_id, BD_ERR_BAD_ARGUMENT,
                        "decode: request appears twice in one batch");
        }
    }

    void step(const bd_request* reqs, uint64_t n, bool full, const float* x_in, float* x_out,
              float* host_logits, cudaStream_t user) {
        BD_CUDA(cudaSetDevice(device));
        validate(reqs, n);
        if (n == 0) return;
        require(n <= 256, BD_ERR_BAD_ARGUMENT, "decode: batch must be <= 256");
        require(world == 1 || comm != nullptr || loop != nullptr, BD_ERR_BAD_ARGUMENT,
                "decode: world_size > 1 needs bd_pool_init_comm first");
        std::vector<int> idx(n);
        for (uint64_t i = 0; i < n; ++i) {
            idx[i] = int(reqs[i].request_id);
            ensure_loaded(requests[idx[i]].tenant);
        }
        Plan& p = plan_for(idx);
        // order the pool stream after the caller's stream
        BD_CUDA(cudaEventRecord(ev_in, user));
        BD_CUDA(cudaStreamWaitEvent(stream, ev_in, 0));
        const int k = p.slot;
        p.slot ^= 1;
        BD_CUDA(cudaEventSynchronize(p.staged[k]));  // the copy that last read this slot has run
        for (uint64_t i = 0; i < n; ++i) {
            p.h_pos[k][i] = int(reqs[i].position);
            p.h_tok[k][i] = reqs[i].token;
        }
        BD_CUDA(cudaMemcpyAsync(p.d_pos, p.h_pos[k], n * sizeof(int), cudaMemcpyHostToDevice, stream));
        BD_CUDA(cudaMemcpyAsync(p.d_tok, p.h_tok[k], n * sizeof(int), cudaMemcpyHostToDevice, stream));
        BD_CUDA(cudaEventRecord(p.staged[k], stream));
        if (!full)
            BD_CUDA(cudaMemcpyAsync(x, x_in, n * a.dim * 4, cudaMemcpyDeviceToDevice, stream));
        execute(p, full);
        if (full) {
            if (host_logits)
                BD_CUDA(cudaMemcpyAsync(host_logits, logits, n * a.vocab * 4, cudaMemcpyDeviceToHost,
                                        stream));
        } else {
            BD_CUDA(cudaMemcpyAsync(x_out, x, n * a.dim * 4, cudaMemcpyDeviceToDevice, stream));
        }
        BD_CUDA(cudaEventRecord(ev_out, stream));
        BD_CUDA(cudaStreamWaitEvent(user, ev_out, 0));
        if (full && host_logits) BD_CUDA(cudaStreamSynchronize(stream));
        for (uint64_t i = 0; i < n; ++i) requests[idx[i]].pos += 1;
    }

    void decode(const bd_request* reqs, uint64_t n, int mode, float* logits_host, cudaStream_t user) {
        require(mode == 0 || mode == 1, BD_ERR_BAD_ARGUMENT, "decode: mode must be 0 (shared) or 1 (naive)");
        if (mode == 0) {
            validate(reqs, n);
            stats.backbone_passes += 1;  // serve.cpp:210
            step(reqs, n, true, nullptr, nullptr, logits_host, user);
        } else {
            // naive (serve.cpp:327-342): one backbone pass per request
            validate(reqs, n);
            stats.backbone_passes += n;
            for (uint64_t i = 0; i < n; ++i)
                step(reqs + i, 1, true, nullptr, nullptr, logits_host ? logits_host + i * a.vocab : nullptr,
                     user);
        }
    }

    uint64_t resident_bytes() const {
        uint64_t tot = backbone_bytes;
        for (const auto& t : tenants)
            if (t.loaded) tot += t.bytes;
        for (const auto& r : requests)
            if (r.open) tot += 2ull * 4ull * r.pos * a.kv_dim * a.n_layers;  // KvCache::bytes (f32 accounting)
        return tot;
    }
};

}  // namespace bd

struct bd_pool {
    bd::PoolImpl impl;
};

namespace bd {
bd_pool* pool_create(const bd_arch& a, int device, int world, int rank) {
    auto* p = new bd_pool;
    try {
        p->impl.init(a, device, world, rank);
    } catch (...) {
        delete p;
        throw;
    }
    return p;
}
void pool_destroy(bd_pool* p) { delete p; }
void pool_set_tensor(bd_pool* p, const char* name, const void* data, bd_dtype dt, int is_dev,
                     uint64_t rows, uint64_t cols) {
    require(name && data, BD_ERR_BAD_ARGUMENT, "set_tensor: null argument");
    p->impl.set_tensor(name, data, dt, is_dev != 0, rows, cols);
}
void pool_set_tensor_i8(bd_pool* p, const char* name, const int8_t* q, const float* scales, int is_dev,
                        uint64_t rows, uint64_t cols) {
    require(name && q && scales, BD_ERR_BAD_ARGUMENT, "set_tensor_i8: null argument");
    p->impl.set_tensor_i8(name, q, scales, is_dev != 0, rows, cols);
}
void pool_register(bd_pool* p, const char* id, const bd_delta_entry* e, int n) {
    require(id && (e || n == 0), BD_ERR_BAD_ARGUMENT, "register_delta: null argument");
    p->impl.register_entries(id, e, n);
}
void pool_register_file(bd_pool* p, const char* id, const char* path, int resident) {
    require(id && path, BD_ERR_BAD_ARGUMENT, "register_delta_file: null argument");
    p->impl.register_file(id, path, resident != 0);
}
uint64_t pool_open(bd_pool* p, const char* id) {
    require(id != nullptr, BD_ERR_BAD_ARGUMENT, "open_request: null id");
    return p->impl.open_request(id);
}
void pool_close(bd_pool* p, uint64_t rid) { p->impl.close_request(rid); }
void pool_decode(bd_pool* p, const bd_request* r, uint64_t n, int mode, float* logits, void* s) {
    require(r || n == 0, BD_ERR_BAD_ARGUMENT, "decode: null requests");
    p->impl.decode(r, n, mode, logits, static_cast<cudaStream_t>(s));
}
void pool_decode_layers(bd_pool* p, const bd_request* r, uint64_t n, const float* xin, float* xout,
                        void* s) {
    require((r && xin && xout) || n == 0, BD_ERR_BAD_ARGUMENT, "decode_layers: null argument");
    p->impl.validate(r, n);
    p->impl.stats.backbone_passes += 1;
    p->impl.step(r, n, false, xin, xout, nullptr, static_cast<cudaStream_t>(s));
}
void pool_profile_layers(bd_pool* p, const bd_request* r, uint64_t n, const float* xin,
                         float* xout, double* ms, uint64_t* cnt, void* s, bool serial) {
    require((r && xin && xout && ms && cnt) || n == 0, BD_ERR_BAD_ARGUMENT,
            "profile_layers: null argument");
    PoolImpl& P = p->impl;
    P.validate(r, n);
    P.profiling = true;
    P.concurrent_k23 = !serial;
    P.prof_events.clear();
    try {
        P.stats.backbone_passes += 1;
        P.step(r, n, false, xin, xout, nullptr, static_cast<cudaStream_t>(s));
    } catch (...) {
        P.profiling = false;
        P.concurrent_k23 = true;
        throw;
    }
    P.profiling = false;
    P.concurrent_k23 = true;
    BD_CUDA(cudaStreamSynchronize(P.stream));
    for (int k = 0; k < BD_PROF_KINDS; ++k) {
        ms[k] = 0.0;
        cnt[k] = 0;
    }
    for (auto& ev : P.prof_events) {
        float t = 0.0f;
        BD_CUDA(cudaEventElapsedTime(&t, ev.second.first, ev.second.second));
        ms[ev.first] += t;
        cnt[ev.first] += 1;
        cudaEventDestroy(ev.second.first);
        cudaEventDestroy(ev.second.second);
    }
    P.prof_events.clear();
}
void nccl_unique_id(void* out) {
    ncclUniqueId id;
    BD_NCCL(ncclGetUniqueId(&id));
    std::memcpy(out, &id, sizeof(id));
}
void pool_init_comm(bd_pool* p, const void* idp) {
    PoolImpl& P = p->impl;
    require(P.world > 1, BD_ERR_BAD_ARGUMENT, "init_comm: pool was created with world_size 1");
    require(P.comm == nullptr, BD_ERR_BAD_ARGUMENT, "init_comm: communicator already initialised");
    ncclUniqueId id;
    std::memcpy(&id, idp, sizeof(id));
    BD_CUDA(cudaSetDevice(P.device));
    BD_NCCL(ncclCommInitRank(&P.comm, P.world, id, P.rank));
}
void pool_init_loopback(bd_pool* p, const char* group) {
    PoolImpl& P = p->impl;
    require(P.world > 1, BD_ERR_BAD_ARGUMENT, "init_loopback: pool was created with world_size 1");
    require(P.comm == nullptr && P.loop == nullptr, BD_ERR_BAD_ARGUMENT,
            "init_loopback: communicator already initialised");
    std::shared_ptr<LoopbackGroup> g;
    {
        std::lock_guard<std::mutex> lk(g_loop_m);
        auto& slot = g_loop_groups[group ? group : ""];
        if (!slot || slot->world == 0) {
            slot = std::make_shared<LoopbackGroup>();
            slot->world = P.world;
            slot->recv.assign(P.world, nullptr);
            slot->ready.assign(P.world, nullptr);
            slot->done.assign(P.world, nullptr);
        }
        require(slot->world == P.world, BD_ERR_BAD_ARGUMENT, "init_loopback: world size differs in group");
        g = slot;
    }
    BD_CUDA(cudaSetDevice(P.device));
    BD_CUDA(cudaEventCreateWithFlags(&P.lb_ready, cudaEventDisableTiming));
    BD_CUDA(cudaEventCreateWithFlags(&P.lb_done, cudaEventDisableTiming));
    P.loop = g;
    P.use_graphs = false;  // the exchanges synchronise host threads: run eagerly
    P.clear_plans();
}
void pool_stats(const bd_pool* p, bd_pool_stats* out) {
    *out = p->impl.stats;
    out->resident_bytes = p->impl.resident_bytes();
}
}  // namespace bd
