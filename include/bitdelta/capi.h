/*
 * bitdelta C-ABI — the drop-in boundary between host code written against the
 * reference deltakit API (/root/reference/proj, "P:" below) and the sm_100a
 * kernels in libbitdelta_b200.so.
 *
 * Rules:
 *   - plain C, no exceptions, no torch/CUDA C++ types: pointers + sizes;
 *   - every call returns int: 0 = ok, 1 + deltakit::errc for the reference's
 *     error categories (P:include/deltakit/error.hpp:10-25), 100+ for device
 *     errors; bd_last_error() holds the message (thread-local);
 *   - device buffers are caller-owned; calls are stream-ordered on `stream`
 *     (a cudaStream_t; NULL = legacy default stream);
 *   - the packed layout is the reference's (P:include/deltakit/delta.hpp:20-22):
 *     one bit per element, flat row-major element order, LSB-first within each
 *     byte, 1 = +1, 0 = -1, ceil(rows*cols/8) bytes, unused trailing bits 0.
 *
 * The host-side C++ mirror of the reference API over these calls lives in
 * include/deltakit_gpu/ (namespace deltakit_gpu); INTEGRATION.md shows the
 * binding a deltakit maintainer would add.
 */
#ifndef BITDELTA_CAPI_H
#define BITDELTA_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BD_ABI_VERSION 1

enum bd_status {
    BD_OK = 0,
    /* 1 + deltakit::errc, P:include/deltakit/error.hpp:10-25 */
    BD_ERR_IO = 1,
    BD_ERR_MALFORMED_HEADER = 2,
    BD_ERR_JSON_PARSE = 3,
    BD_ERR_BAD_OFFSETS = 4,
    BD_ERR_UNSUPPORTED_DTYPE = 5,
    BD_ERR_SHAPE_MISMATCH = 6,
    BD_ERR_NAME_MISMATCH = 7,
    BD_ERR_LENGTH_MISMATCH = 8,
    BD_ERR_BAD_ARGUMENT = 9,
    BD_ERR_BAD_TOKEN = 10,
    BD_ERR_NON_FINITE = 11,
    BD_ERR_NO_CONVERGENCE = 12,
    BD_ERR_DUPLICATE_ID = 13,
    BD_ERR_UNKNOWN_ID = 14,
    /* device side */
    BD_ERR_CUDA = 100,
    BD_ERR_NO_DEVICE = 101,
    BD_ERR_UNSUPPORTED_DEVICE = 102
};

typedef enum bd_dtype { BD_F32 = 0, BD_BF16 = 1 } bd_dtype;

int bd_abi_version(void);
const char* bd_last_error(void);
/* Fails with BD_ERR_NO_DEVICE / BD_ERR_UNSUPPORTED_DEVICE unless `device` is a
 * compute-capability 10.0 (B200, sm_100a) GPU. */
int bd_device_check(int device);
/* Number of kernel launches this library issued since load (all streams). */
uint64_t bd_launch_count(void);

/* Diagnostics (no reference counterpart): device timeline of the decode-step kernels.
 * bd_trace_enable(cap) allocates room for cap records (0 disables); every CTA of the
 * K2/K3/glue kernels then appends {kind, cta, smid, pad, t_entry, t_wait, t_end}
 * (u32 x4 + u64 x3, %globaltimer ns). bd_trace_read copies up to cap records and
 * resets the count. */
int bd_trace_enable(uint32_t capacity);
int bd_trace_read(void* out, uint32_t capacity, uint32_t* n_out);

/* ------------------------------------------------------------------ K1 -- */
/* Replaces deltakit::compress_tensor (P:include/deltakit/delta.hpp:48,
 * P:src/delta.cpp:31-34) and, with base == NULL, compress_delta
 * (delta.hpp:47, delta.cpp:16-29):
 *   delta = fine - base in f32 (bf16 inputs widen exactly first);
 *   bit i = delta[i] > 0 (NaN, 0, -0 -> 0);  alpha = float(sum|double(delta)| / n)
 * bits: ceil(rows*cols/8) device bytes; alpha: one device float. */
uint64_t bd_packed_size(uint64_t rows, uint64_t cols);
int bd_compress(const void* base, const void* fine, bd_dtype dtype, uint64_t rows, uint64_t cols,
                uint8_t* bits, float* alpha, void* stream);

/* Many independent matrices in one launch (build_delta_file's per-tensor loop,
 * P:src/delta.cpp:181-196). `jobs` is a HOST array. */
typedef struct bd_compress_job {
    const void* base; /* may be NULL (fine is then the delta) */
    const void* fine;
    uint64_t rows, cols;
    uint8_t* bits;
    float* alpha;
} bd_compress_job;
int bd_compress_batched(const bd_compress_job* jobs, int n_jobs, bd_dtype dtype, void* stream);

/* compress_stack (P:src/delta.cpp:57-70): `planes` sign planes back to back in
 * `bits` (planes * ceil(rows*cols/8) bytes) and `planes` alphas. Plane k fits
 * the residual of planes 0..k-1. */
int bd_compress_stack(const void* base, const void* fine, bd_dtype dtype, uint64_t rows,
                      uint64_t cols, uint64_t planes, uint8_t* bits, float* alphas, void* stream);

/* ------------------------------------------------------------------ K3 -- */
/* Replaces deltakit::packed_signed_accumulate (P:include/deltakit/delta.hpp:69-70,
 * P:src/delta.cpp:80-103) for n_vec vectors at once:
 *   out[v*rows + r] += sum_j s_rj * x[v*cols + j],  s = +1 for bit 1, -1 for bit 0.
 * Any rows/cols (rows need not start on a byte). f32 in/out, device pointers. */
int bd_packed_signed_accumulate(const uint8_t* bits, uint64_t rows, uint64_t cols, const float* x,
                                uint64_t n_vec, float* out, void* stream);
/* packed_matvec (delta.hpp:67, delta.cpp:72-78): y = alpha * (S x), overwrites y. */
int bd_packed_matvec(const uint8_t* bits, float alpha, uint64_t rows, uint64_t cols,
                     const float* x, uint64_t n_vec, float* y, void* stream);

/* ------------------------------------------------ K2 int8: RTN backbone -- */
/* rtn_quantize (P:src/int8.cpp:15-42), bit-exact: per row s = amax/127 (f32), q = clamp(
 * nearbyint(double(w)/double(s)), -127, 127); an all-zero row gets s = 0. W: device f32
 * [rows x cols]; q: device int8 [rows x cols]; row_scales: device f32 [rows]. Fails with
 * BD_ERR_NON_FINITE on NaN/inf entries (synchronises the stream to report it). */
int bd_rtn_quantize(const float* W, uint64_t rows, uint64_t cols, int8_t* q, float* row_scales, void* stream);
/* int8_matmul_nt (P:src/int8.cpp:67-81): Y[i][r] = (A[i] . q[r]) * row_scales[r], A device f32
 * [s x in_dim], q device int8 [out_dim x in_dim], Y device f32 [s x out_dim] (overwritten).
 * tcgen05 kind::i8 against 4 int8 pieces of each A row (exact s32 accumulation; A to 2^-27
 * of its row maximum): within the reference's own f32 rounding (rel-L2 <= 1e-5). */
int bd_int8_matmul_nt(const float* A, uint64_t s, uint64_t in_dim, const int8_t* q, const float* row_scales,
                      uint64_t out_dim, float* Y, void* stream);

/* ------------------------------------------------- K6: distill backward -- */
/* Replaces deltakit::packed_signed_accumulate_t (P:include/deltakit/delta.hpp:71-72,
 * P:src/delta.cpp:105-131) for n_vec vectors at once (accumulates, like the reference):
 *   out[v*cols + j] += sum_i s_ij * y[v*rows + i],  s = +1 for bit 1, -1 for bit 0;
 * column sums in fp64, rounded to f32 once. Any rows/cols. Device pointers. */
int bd_packed_signed_accumulate_t(const uint8_t* bits, uint64_t rows, uint64_t cols, const float* y,
                                  uint64_t n_vec, float* out, void* stream);
/* The packed-plane part of the distillation backward: linear_backward's PackedDelta branch
 * (P:src/model.cpp:87-107) for one linear with n_planes sign planes of [rows x cols]:
 *   dx[t*cols + j] += scales[pl] * float((S_pl^T dy[t])[j])     t < s (accumulated)
 *   scale_grad[pl] += sum_i double(dy[i]) * double(plane_u[pl][i])  (i < s*rows, accumulated)
 * dy: device f32 [s x rows]; plane_u[pl]: device f32 [s x rows], the forward's S_pl x
 * (LinearTape::plane_u); dx: device f32 [s x cols]; scale_grad: device f64 [n_planes].
 * plane_bits / plane_u / scales are HOST arrays of n_planes entries. The branch's dense
 * dy * W_base term is a plain library GEMM (cuBLAS / torch.matmul), left to the caller. */
int bd_delta_linear_backward(int32_t n_planes, const uint8_t* const* plane_bits, const float* scales,
                             uint64_t rows, uint64_t cols, const float* dy, uint64_t s,
                             const float* const* plane_u, float* dx, double* scale_grad, void* stream);

/* --------------------------------------------------------------- K2+K3 -- */
/* One multi-tenant linear (the per-projection body of ServingPool::decode_shared,
 * P:src/serve.cpp:247-254: backbone_linear_nt serve.cpp:120-127 + per-request
 * apply_delta_correction serve.cpp:19-36), with requests segmented by tenant so
 * each tenant's bits are read once:
 *   Y[b, :] = X[b, :] W^T + alpha[t(b)] * S_{t(b)} X[b, :]
 * W: device bf16 [out_dim x in_dim]; X: device bf16 [batch x in_dim];
 * Y: device f32 [batch x out_dim] (overwritten); tenant_bits / tenant_alpha /
 * req_tenant: HOST arrays (device bit pointers); req_tenant[b] < 0 = base only. */
int bd_multitenant_linear(const void* W, uint64_t out_dim, uint64_t in_dim, int32_t n_tenants,
                          const uint8_t* const* tenant_bits, const float* tenant_alpha,
                          int32_t batch, const int32_t* req_tenant, const void* X, float* Y,
                          void* stream);

/* The same linear in f32 (W, X device f32; BASELINE configs[0], the reference's own
 * precision, 1e-5 tolerance): K5, a SIMT kernel with fp64 accumulation — tcgen05 has
 * no f32 kind. Rounds like the reference: Y = float(W x) + alpha * float(S x). */
int bd_multitenant_linear_f32(const float* W, uint64_t out_dim, uint64_t in_dim, int32_t n_tenants,
                              const uint8_t* const* tenant_bits, const float* tenant_alpha,
                              int32_t batch, const int32_t* req_tenant, const float* X, float* Y,
                              void* stream);

/* ------------------------------------------------------------- serving -- */
/* Device-resident ServingPool (P:include/deltakit/serve.hpp:59-100,
 * P:src/serve.cpp:93-325). Backbone linears are held in bf16, norms/embed in
 * f32; tenants' packed planes stay in the reference byte layout. */
typedef struct bd_pool bd_pool;

typedef struct bd_arch {
    uint64_t vocab, dim, kv_dim, n_layers, n_heads, intermediate, max_seq;
    float rope_theta;
} bd_arch; /* P:include/deltakit/arch.hpp:11-24 (+ kv_dim, arch.hpp:36-39) */

/* world_size/rank: output-row sharding of every projection and its packed
 * delta; 1/0 on a single GPU. */
int bd_pool_create(const bd_arch* arch, int device, int world_size, int rank, bd_pool** out);
void bd_pool_destroy(bd_pool* pool);

/* Multi-GPU (world_size > 1): every rank holds its row shard; per layer the
 * pool all-gathers (NCCL over NVLink) the attention context, the o-projection
 * output, the MLP activation and the down-projection output. Rank 0 creates
 * the id (bd_nccl_unique_id), the caller broadcasts the 128 bytes, every rank
 * calls bd_pool_init_comm before registering deltas or decoding. */
int bd_nccl_unique_id(void* id_out /* 128 bytes */);
int bd_pool_init_comm(bd_pool* pool, const void* id /* 128 bytes */);
/* Test hook (no reference counterpart): instead of NCCL, the world_size pools of ONE
 * process on ONE device (each driven from its own host thread) exchange through device
 * copies; every other part of the row-sharded path runs unchanged. Pools joining the
 * same `group` name form one world. Decode then runs eagerly (no CUDA graph). */
int bd_pool_init_loopback(bd_pool* pool, const char* group);

/* Backbone tensor by reference name (arch.cpp:51-69: "embed",
 * "layers.{i}.{attn_q,...,norm2}", "final_norm", "lm_head"), full (unsharded)
 * shape. `data` is host memory unless is_device != 0. */
int bd_pool_set_tensor(bd_pool* pool, const char* name, const void* data, bd_dtype dtype,
                       int is_device, uint64_t rows, uint64_t cols);

/* INT8 RTN backbone (ServingPool(QuantizedCheckpoint), P:src/serve.cpp:99-108, 120-125):
 * one of the 7 layer projections as an Int8Tensor (P:include/deltakit/int8.hpp: int8 values
 * [rows x cols] + f32 row scales, e.g. from bd_rtn_quantize), full (unsharded) shape; host
 * memory unless is_device != 0. A pool's projections are all int8 or all dense (the other
 * tensors stay dense); its K2 runs tcgen05 kind::i8 (half the backbone bytes of bf16) and
 * serves batches of <= 64. */
int bd_pool_set_tensor_i8(bd_pool* pool, const char* name, const int8_t* q, const float* row_scales,
                          int is_device, uint64_t rows, uint64_t cols);

/* One tensor of a tenant's delta (DeltaEntry, delta.hpp:76-86). */
typedef struct bd_delta_entry {
    const char* name;
    int kind;             /* 1 = packed planes, 0 = raw f32 delta */
    uint64_t rows, cols, planes;
    const uint8_t* bits;  /* planes * ceil(rows*cols/8) bytes, reference layout */
    const float* scales;  /* planes alphas (host) */
    const float* raw;     /* rows*cols f32 (kind 0); NULL = all-zero delta */
    int is_device;        /* bits/raw live on the pool's device */
} bd_delta_entry;

/* register_delta (serve.cpp:129-152): every backbone tensor must be covered with
 * the matching shape (errors name the tensor). */
int bd_pool_register_delta(bd_pool* pool, const char* id, const bd_delta_entry* entries,
                           int n_entries);
/* Same, from a .bdelta container on disk (delta.cpp:265-334). resident = 0
 * defers loading to first use (cold-load hot swap, serve.cpp:154-166). */
int bd_pool_register_delta_file(bd_pool* pool, const char* id, const char* path, int resident);

/* Host-only check of a .bdelta container (read_delta_file's validation, delta.cpp:265-334,
 * no device needed): *n_tensors = entries, *n_packed = packed entries, *max_planes = the
 * largest plane count. The pool serves packed projections with 1..32 planes and raw (f32)
 * entries anywhere, projections included (a group with a raw projection delta or more than 4
 * planes takes the generic delta units + extra passes for that step); a packed lm_head has
 * at most 4 planes (BD_ERR_BAD_ARGUMENT otherwise). */
int bd_bdelta_validate(const char* path, uint64_t* n_tensors, uint64_t* n_packed, uint64_t* max_planes);

int bd_pool_open_request(bd_pool* pool, const char* delta_id, uint64_t* request_id);
int bd_pool_close_request(bd_pool* pool, uint64_t request_id);

typedef struct bd_request {
    uint64_t request_id;
    int32_t token;
    uint64_t position; /* must equal the request's cache position */
} bd_request;

/* decode_step (serve.cpp:199-203). mode 0 = Shared (one backbone pass),
 * 1 = Naive (one pass per request). logits: HOST [n x vocab] f32 (may be NULL).
 * Validation as validate_batch (serve.cpp:186-197). */
int bd_pool_decode_step(bd_pool* pool, const bd_request* reqs, uint64_t n, int mode,
                        float* logits, void* stream);

/* The layer stack only (serve.cpp:240-310) on device-resident activations:
 * x_in/x_out device f32 [n x dim]; no embedding / final norm / lm_head.
 * Advances the requests' cache positions like decode_step. */
int bd_pool_decode_layers(bd_pool* pool, const bd_request* reqs, uint64_t n, const float* x_in,
                          float* x_out, void* stream);

/* Profiled layer step: same work as bd_pool_decode_layers (advances positions),
 * run eagerly (no graph) with CUDA events on the launching stream around every
 * kernel; ms_out[k] / count_out[k] receive total device ms and launches per
 * kind k (bd_prof_kind). Used by bench.py for the per-kernel roofline. */
enum bd_prof_kind {
    BD_PROF_GEMM_QKV = 0, BD_PROF_GEMM_O, BD_PROF_GEMM_GU, BD_PROF_GEMM_DOWN,
    BD_PROF_DELTA_QKV, BD_PROF_DELTA_O, BD_PROF_DELTA_GU, BD_PROF_DELTA_DOWN,
    BD_PROF_ATTN, BD_PROF_NORM, BD_PROF_SILU,
    /* fused K2+K3 kernels (base GEMM + all tenant planes, tensor cores) */
    BD_PROF_FUSED_QKV, BD_PROF_FUSED_O, BD_PROF_FUSED_GU, BD_PROF_FUSED_DOWN,
    BD_PROF_XQ_PREP, BD_PROF_KINDS
};
int bd_pool_profile_layers(bd_pool* pool, const bd_request* reqs, uint64_t n, const float* x_in,
                           float* x_out, double* ms_out, uint64_t* count_out, void* stream);
/* Same, with the base GEMM (K2) and the tenant-delta kernel (K3) run one after the other
 * instead of side by side, so each is timed on its own (the delta kernel's own GB/s). */
int bd_pool_profile_layers_serial(bd_pool* pool, const bd_request* reqs, uint64_t n, const float* x_in,
                                  float* x_out, double* ms_out, uint64_t* count_out, void* stream);

typedef struct bd_pool_stats {
    uint64_t backbone_passes; /* serve.hpp:77 */
    uint64_t cold_loads;      /* serve.hpp:78 */
    double last_cold_load_ms; /* serve.hpp:79 */
    uint64_t resident_bytes;  /* device bytes: backbone + resident deltas + KV */
    uint64_t kernels_last_step; /* kernels launched by the last decode step */
    char delta_paths[8];        /* K3 variant per projection group (q/k/v, o, gate/up, down) of
                                   the last step: T = K23, L = byte LUT, X = K3t, F = i8 fused,
                                   U = SIMT units; NUL-terminated */
} bd_pool_stats;
int bd_pool_get_stats(const bd_pool* pool, bd_pool_stats* out);

#ifdef __cplusplus
}
#endif
#endif /* BITDELTA_CAPI_H */
