/* TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
 *
 * Plain-C restatement of the reference (deltakit) hot path, used only as the
 * parity checker by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg. Every function cites the reference file:line it restates
 * (P: = /root/reference/proj/). Parity of this restatement is PINNED against
 * the compiled reference (oracle/_ref/libdeltakit_ref.so) and the golden
 * vectors in tests/golden/ by tests/test_oracle.py.
 */
#ifndef BDORACLE_H
#define BDORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

int bdo_sign_of(float x);                                   /* P:include/deltakit/delta.hpp:18 */
uint64_t bdo_packed_size(uint64_t rows, uint64_t cols);     /* delta.hpp:28-30 */
void bdo_compress_delta(const float* v, uint64_t n, uint8_t* bits, float* scale); /* P:src/delta.cpp:16-29 */
void bdo_compress_tensor(const float* base, const float* fine, uint64_t n, uint8_t* bits,
                         float* scale);                     /* delta.cpp:31-34 + matrix.cpp:72-77 */
void bdo_decompress(const uint8_t* bits, uint64_t n, float scale, float* out); /* delta.cpp:36-42 */
void bdo_compress_stack(const float* base, const float* fine, uint64_t n, uint64_t planes,
                        uint8_t* bits, float* scales);      /* delta.cpp:57-70 */
void bdo_packed_signed_accumulate(const uint8_t* bits, uint64_t rows, uint64_t cols,
                                  const float* x, float* out); /* delta.cpp:80-103 */
void bdo_packed_signed_accumulate_t(const uint8_t* bits, uint64_t rows, uint64_t cols,
                                    const float* y, float* out);   /* delta.cpp:105-131 */
void bdo_rtn_quantize(const float* w, uint64_t rows, uint64_t cols, int8_t* q,
                      float* scales);                                   /* P:src/int8.cpp:15-42 */
void bdo_int8_matmul_nt(const float* a, uint64_t s, const int8_t* q, const float* scales,
                        uint64_t rows, uint64_t cols, float* out);      /* int8.cpp:67-81 */
void bdo_packed_matvec(const uint8_t* bits, uint64_t rows, uint64_t cols, float scale,
                       const float* x, float* y);           /* delta.cpp:72-78 */
void bdo_matmul_nt(const float* a, uint64_t s, uint64_t k, const float* b, uint64_t t,
                   float* out);                             /* P:src/matrix.cpp:26-41 */
double bdo_rmsnorm_row(const float* x, const float* w, uint64_t n, float* out); /* nn_ops.hpp:15-25 */
void bdo_rope_row(float* head, uint64_t n, uint64_t pos, float theta);          /* nn_ops.hpp:29-45 */
void bdo_softmax_row(float* row, uint64_t n);                                   /* nn_ops.hpp:48-57 */
float bdo_silu(float x);                                                        /* nn_ops.hpp:59 */

/* Architecture (P:include/deltakit/arch.hpp:11-24). kv_dim == dim is the
 * reference; kv_dim < dim is the documented GQA extension (arch.hpp:36-39
 * presets carry kv_dim; the reference serving path has no GQA). */
typedef struct bdo_arch {
    uint64_t vocab, dim, kv_dim, n_layers, n_heads, intermediate, max_seq;
    float rope_theta;
} bdo_arch;

/* One tensor's delta entry (delta.hpp:76-86): kind 1 = packed planes, 0 = raw f32. */
typedef struct bdo_entry {
    int kind;
    uint64_t planes;
    const uint8_t* bits;   /* planes * packed_size(rows, cols) bytes */
    const float* scales;   /* planes */
    const float* raw;      /* rows * cols */
} bdo_entry;

/* Tensor order = tensor_shapes (P:src/arch.cpp:51-69): embed, per layer
 * {attn_q, attn_k, attn_v, attn_o, mlp_gate, mlp_up, mlp_down, norm1, norm2},
 * final_norm, lm_head. `base` is all tensors concatenated in that order. */
uint64_t bdo_tensor_count(const bdo_arch* a);
void bdo_tensor_shape(const bdo_arch* a, uint64_t i, uint64_t* rows, uint64_t* cols);

/* ServingPool::decode_shared (P:src/serve.cpp:205-325) for one batch.
 *   entries[r]  : the tensor_count() delta entries of request r's tenant
 *   kcache[r], vcache[r] : [n_layers][max_seq][kv_dim] f32, positions < pos[r] filled
 *   logits      : B x vocab out.  layers_only != 0 skips embed/final-norm/lm_head:
 *                 x_in (B x dim) is the residual stream entering layer 0 and
 *                 x_out (B x dim) the stream leaving the last layer. */
int bdo_decode_shared(const bdo_arch* a, const float* base, const bdo_entry* const* entries,
                      uint64_t B, const int32_t* tokens, const uint64_t* pos, float* const* kcache,
                      float* const* vcache, float* logits);
int bdo_decode_layers(const bdo_arch* a, const float* base, const bdo_entry* const* entries,
                      uint64_t B, const uint64_t* pos, float* const* kcache, float* const* vcache,
                      const float* x_in, float* x_out);

#ifdef __cplusplus
}
#endif
#endif
