/* TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT (see bdoracle.h).
 *
 * Plain-C restatement of the deltakit hot path. Parity status: PINNED — the
 * restatement is checked against the compiled reference library and the
 * golden vectors by tests/test_oracle.py (bit-exact bits/scales/logits).
 * Compile with -ffp-contract=off: the reference is built without FMA.
 */
#include "bdoracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* P:include/deltakit/delta.hpp:18 — +1 iff x > 0; 0, -0 and NaN map to -1 */
int bdo_sign_of(float x) { return x > 0.0f ? 1 : -1; }

/* delta.hpp:28-30 */
uint64_t bdo_packed_size(uint64_t rows, uint64_t cols) { return (rows * cols + 7) / 8; }

/* P:src/delta.cpp:16-29: bit i (LSB-first, flat row-major) = v[i] > 0;
 * scale = float(sequential double sum of |v| / n) */
void bdo_compress_delta(const float* v, uint64_t n, uint8_t* bits, float* scale) {
    memset(bits, 0, (n + 7) / 8);
    double abs_sum = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        if (v[i] > 0.0f) bits[i >> 3] |= (uint8_t)(1u << (i & 7));
        abs_sum += fabs((double)v[i]);
    }
    *scale = n == 0 ? 0.0f : (float)(abs_sum / (double)n);
}

/* delta.cpp:31-34 via sub() matrix.cpp:72-77 (fp32 fine - base materialised) */
void bdo_compress_tensor(const float* base, const float* fine, uint64_t n, uint8_t* bits,
                         float* scale) {
    float* d = (float*)malloc((n ? n : 1) * sizeof(float));
    for (uint64_t i = 0; i < n; ++i) d[i] = fine[i] - base[i];
    bdo_compress_delta(d, n, bits, scale);
    free(d);
}

/* delta.cpp:36-42 */
void bdo_decompress(const uint8_t* bits, uint64_t n, float scale, float* out) {
    for (uint64_t i = 0; i < n; ++i) out[i] = ((bits[i >> 3] >> (i & 7)) & 1u) ? scale : -scale;
}

/* delta.cpp:57-70: plane i fits the residual left by planes 0..i-1 */
void bdo_compress_stack(const float* base, const float* fine, uint64_t n, uint64_t planes,
                        uint8_t* bits, float* scales) {
    float* res = (float*)malloc((n ? n : 1) * sizeof(float));
    float* rec = (float*)malloc((n ? n : 1) * sizeof(float));
    const uint64_t nb = (n + 7) / 8;
    for (uint64_t i = 0; i < n; ++i) res[i] = fine[i] - base[i];
    for (uint64_t k = 0; k < planes; ++k) {
        bdo_compress_delta(res, n, bits + k * nb, scales + k);
        bdo_decompress(bits + k * nb, n, scales[k], rec);
        for (uint64_t i = 0; i < n; ++i) res[i] -= rec[i];
    }
    free(res);
    free(rec);
}

/* delta.cpp:80-103: out[r] += float(2 * sum_{bit=1} x_j - sum_j x_j), double
 * accumulators, byte-serial walk of the flat bit stream */
void bdo_packed_signed_accumulate(const uint8_t* bits, uint64_t rows, uint64_t cols,
                                  const float* x, float* out) {
    double total = 0.0;
    for (uint64_t j = 0; j < cols; ++j) total += x[j];
    for (uint64_t r = 0; r < rows; ++r) {
        double set_sum = 0.0;
        uint64_t idx = r * cols, c = 0;
        while (c < cols) {
            uint8_t byte = (uint8_t)(bits[idx >> 3] >> (idx & 7));
            uint64_t take = 8 - (idx & 7);
            if (take > cols - c) take = cols - c;
            for (uint64_t b = 0; b < take; ++b) {
                if (byte & 1u) set_sum += x[c + b];
                byte >>= 1;
            }
            c += take;
            idx += take;
        }
        out[r] += (float)(2.0 * set_sum - total);
    }
}

/* P:src/delta.cpp:105-131: out[j] += float(2 * sum_{bit(i,j)=1} y_i - sum_i y_i), double sums,
 * rows with y_i == 0 skipped (they add nothing) */
void bdo_packed_signed_accumulate_t(const uint8_t* bits, uint64_t rows, uint64_t cols,
                                    const float* y, float* out) {
    double* acc = (double*)calloc(cols ? cols : 1, sizeof(double));
    double total = 0.0;
    for (uint64_t r = 0; r < rows; ++r) total += y[r];
    for (uint64_t r = 0; r < rows; ++r) {
        const double yr = y[r];
        if (yr == 0.0) continue;
        uint64_t idx = r * cols, c = 0;
        while (c < cols) {
            uint8_t byte = (uint8_t)(bits[idx >> 3] >> (idx & 7));
            uint64_t take = 8 - (idx & 7);
            if (take > cols - c) take = cols - c;
            for (uint64_t b = 0; b < take; ++b) {
                if (byte & 1u) acc[c + b] += yr;
                byte >>= 1;
            }
            c += take;
            idx += take;
        }
    }
    for (uint64_t j = 0; j < cols; ++j) out[j] += (float)(2.0 * acc[j] - total);
    free(acc);
}

/* P:src/int8.cpp:15-42: per row s = amax / 127 (f32); a zero row -> s = 0, q = 0; else
 * q = clamp(nearbyint(double(w) / double(s)), -127, 127) (ties to even) */
void bdo_rtn_quantize(const float* w, uint64_t rows, uint64_t cols, int8_t* q, float* scales) {
    for (uint64_t r = 0; r < rows; ++r) {
        const float* row = w + r * cols;
        float amax = 0.0f;
        for (uint64_t c = 0; c < cols; ++c) amax = fmaxf(amax, fabsf(row[c]));
        const float s = amax / 127.0f;
        scales[r] = s;
        for (uint64_t c = 0; c < cols; ++c) {
            double v = 0.0;
            if (s != 0.0f) {
                v = nearbyint((double)row[c] / (double)s);
                v = v < -127.0 ? -127.0 : (v > 127.0 ? 127.0 : v);
            }
            q[r * cols + c] = (int8_t)v;
        }
    }
}

/* P:src/int8.cpp:67-81: out[i][r] = (sequential f32 sum of float(q) * a) * s_r */
void bdo_int8_matmul_nt(const float* a, uint64_t s, const int8_t* q, const float* scales,
                        uint64_t rows, uint64_t cols, float* out) {
    for (uint64_t i = 0; i < s; ++i)
        for (uint64_t r = 0; r < rows; ++r) {
            float acc = 0.0f;
            for (uint64_t c = 0; c < cols; ++c) acc += (float)q[r * cols + c] * a[i * cols + c];
            out[i * rows + r] = acc * scales[r];
        }
}

/* delta.cpp:72-78 */
void bdo_packed_matvec(const uint8_t* bits, uint64_t rows, uint64_t cols, float scale,
                       const float* x, float* y) {
    for (uint64_t r = 0; r < rows; ++r) y[r] = 0.0f;
    bdo_packed_signed_accumulate(bits, rows, cols, x, y);
    for (uint64_t r = 0; r < rows; ++r) y[r] *= scale;
}

/* P:src/matrix.cpp:26-41: out (s x t) = a (s x k) * b (t x k)^T, f32 sequential dot */
void bdo_matmul_nt(const float* a, uint64_t s, uint64_t k, const float* b, uint64_t t,
                   float* out) {
    for (uint64_t i = 0; i < s; ++i) {
        const float* ar = a + i * k;
        for (uint64_t j = 0; j < t; ++j) {
            const float* br = b + j * k;
            float acc = 0.0f;
            for (uint64_t q = 0; q < k; ++q) acc += ar[q] * br[q];
            out[i * t + j] = acc;
        }
    }
}

/* P:include/deltakit/nn_ops.hpp:15-25 (eps 1e-12, double statistics) */
double bdo_rmsnorm_row(const float* x, const float* w, uint64_t n, float* out) {
    const double eps = 1e-12;
    double msq = 0.0;
    for (uint64_t i = 0; i < n; ++i) msq += (double)x[i] * x[i];
    msq /= (double)n;
    const double inv = 1.0 / sqrt(msq + eps);
    for (uint64_t i = 0; i < n; ++i) out[i] = (float)((double)x[i] * inv) * w[i];
    return inv;
}

/* nn_ops.hpp:29-45: interleaved pairs, freq = theta^(-2i/n) in double */
void bdo_rope_row(float* head, uint64_t n, uint64_t pos, float theta) {
    const uint64_t half = n / 2;
    for (uint64_t i = 0; i < half; ++i) {
        const double freq = pow((double)theta, -2.0 * (double)i / (double)n);
        const double angle = (double)pos * freq;
        const float c = (float)cos(angle);
        const float s = (float)sin(angle);
        const float a = head[2 * i], b = head[2 * i + 1];
        head[2 * i] = a * c - b * s;
        head[2 * i + 1] = a * s + b * c;
    }
}

/* nn_ops.hpp:48-57 */
void bdo_softmax_row(float* row, uint64_t n) {
    float mx = row[0];
    for (uint64_t j = 1; j < n; ++j) mx = row[j] > mx ? row[j] : mx;
    float sum = 0.0f;
    for (uint64_t j = 0; j < n; ++j) {
        row[j] = expf(row[j] - mx);
        sum += row[j];
    }
    for (uint64_t j = 0; j < n; ++j) row[j] /= sum;
}

/* nn_ops.hpp:59 */
float bdo_silu(float x) { return x / (1.0f + expf(-x)); }

/* ---- model layout: tensor_shapes (P:src/arch.cpp:51-69, presets 92-110) ---- */

enum { T_Q, T_K, T_V, T_O, T_GATE, T_UP, T_DOWN, T_NORM1, T_NORM2, T_PER_LAYER };

uint64_t bdo_tensor_count(const bdo_arch* a) { return 1 + a->n_layers * T_PER_LAYER + 2; }

void bdo_tensor_shape(const bdo_arch* a, uint64_t i, uint64_t* rows, uint64_t* cols) {
    const uint64_t last = 1 + a->n_layers * T_PER_LAYER;
    if (i == 0) { *rows = a->vocab; *cols = a->dim; return; }
    if (i == last) { *rows = 1; *cols = a->dim; return; }          /* final_norm */
    if (i == last + 1) { *rows = a->vocab; *cols = a->dim; return; } /* lm_head */
    switch ((i - 1) % T_PER_LAYER) {
        case T_Q: case T_O: *rows = a->dim; *cols = a->dim; return;
        case T_K: case T_V: *rows = a->kv_dim; *cols = a->dim; return;
        case T_GATE: case T_UP: *rows = a->intermediate; *cols = a->dim; return;
        case T_DOWN: *rows = a->dim; *cols = a->intermediate; return;
        default: *rows = 1; *cols = a->dim; return;                 /* norm1, norm2 */
    }
}

static const float* tensor_ptr(const bdo_arch* a, const float* base, uint64_t idx) {
    const float* p = base;
    for (uint64_t i = 0; i < idx; ++i) {
        uint64_t r, c;
        bdo_tensor_shape(a, i, &r, &c);
        p += r * c;
    }
    return p;
}

/* serve.cpp:19-36 apply_delta_correction: y += D x for one request */
static void apply_delta_correction(const bdo_entry* e, uint64_t rows, uint64_t cols,
                                   const float* x, float* y) {
    if (e->kind == 1) {
        float* tmp = (float*)malloc(rows * sizeof(float));
        const uint64_t nb = bdo_packed_size(rows, cols);
        for (uint64_t k = 0; k < e->planes; ++k) {
            for (uint64_t i = 0; i < rows; ++i) tmp[i] = 0.0f;
            bdo_packed_signed_accumulate(e->bits + k * nb, rows, cols, x, tmp);
            for (uint64_t i = 0; i < rows; ++i) y[i] += e->scales[k] * tmp[i];
        }
        free(tmp);
    } else {
        for (uint64_t r = 0; r < rows; ++r) {
            const float* row = e->raw + r * cols;
            float acc = 0.0f;
            for (uint64_t c = 0; c < cols; ++c) acc += row[c] * x[c];
            y[r] += acc;
        }
    }
}

/* serve.cpp:39-48 add_delta_row: out += row r of the reconstructed delta.
 * Packed planes (back to back, packed_size(rows, cols) bytes each) are read
 * through the flat index r*cols + c, like PackedSignMatrix::bit_at. */
static void delta_row(const bdo_entry* e, uint64_t rows, uint64_t r, uint64_t cols, float* out) {
    if (e->kind == 1) {
        const uint64_t nb = bdo_packed_size(rows, cols);
        for (uint64_t k = 0; k < e->planes; ++k) {
            const uint8_t* bits = e->bits + k * nb;
            for (uint64_t c = 0; c < cols; ++c) {
                const uint64_t idx = r * cols + c;
                out[c] += ((bits[idx >> 3] >> (idx & 7)) & 1u) ? e->scales[k] : -e->scales[k];
            }
        }
    } else {
        const float* row = e->raw + r * cols;
        for (uint64_t c = 0; c < cols; ++c) out[c] += row[c];
    }
}

/* effective norm (serve.cpp:224-228): backbone row plus the tenant's delta row */
static void effective_norm(const bdo_arch* a, const float* base, const bdo_entry* ents,
                           uint64_t idx, float* out) {
    const float* w = tensor_ptr(a, base, idx);
    memcpy(out, w, a->dim * sizeof(float));
    delta_row(&ents[idx], 1, 0, a->dim, out);
}

/* one linear for the stacked batch: backbone_linear_nt (serve.cpp:120-127) then
 * per-request apply_delta_correction (serve.cpp:247-254 pattern) */
static void linear(const bdo_arch* a, const float* base, const bdo_entry* const* entries,
                   uint64_t B, uint64_t idx, const float* x, float* y) {
    uint64_t rows, cols;
    bdo_tensor_shape(a, idx, &rows, &cols);
    bdo_matmul_nt(x, B, cols, tensor_ptr(a, base, idx), rows, y);
    for (uint64_t r = 0; r < B; ++r)
        apply_delta_correction(&entries[r][idx], rows, cols, x + r * cols, y + r * rows);
}

/* the layer loop of decode_shared, serve.cpp:240-310 */
static void run_layers(const bdo_arch* a, const float* base, const bdo_entry* const* entries,
                       uint64_t B, const uint64_t* pos, float* const* kcache,
                       float* const* vcache, float* x) {
    const uint64_t dim = a->dim, kvd = a->kv_dim, inter = a->intermediate;
    const uint64_t hd = dim / a->n_heads;
    const uint64_t group = dim / kvd; /* query heads per kv head; 1 for the reference */
    const float inv_sqrt_hd = 1.0f / sqrtf((float)hd);
    float* normed = (float*)calloc(B * dim, sizeof(float));
    float* norm_w = (float*)calloc(dim, sizeof(float));
    float* q = (float*)calloc(B * dim, sizeof(float));
    float* k = (float*)calloc(B * kvd, sizeof(float));
    float* v = (float*)calloc(B * kvd, sizeof(float));
    float* ctx = (float*)calloc(B * dim, sizeof(float));
    float* o = (float*)calloc(B * dim, sizeof(float));
    float* g = (float*)calloc(B * inter, sizeof(float));
    float* u = (float*)calloc(B * inter, sizeof(float));
    float* scores = (float*)calloc(a->max_seq, sizeof(float));

    for (uint64_t l = 0; l < a->n_layers; ++l) {
        const uint64_t t0 = 1 + l * T_PER_LAYER;
        for (uint64_t r = 0; r < B; ++r) {
            effective_norm(a, base, entries[r], t0 + T_NORM1, norm_w);
            bdo_rmsnorm_row(x + r * dim, norm_w, dim, normed + r * dim);
        }
        linear(a, base, entries, B, t0 + T_Q, normed, q);
        linear(a, base, entries, B, t0 + T_K, normed, k);
        linear(a, base, entries, B, t0 + T_V, normed, v);
        memset(ctx, 0, B * dim * sizeof(float));
        for (uint64_t r = 0; r < B; ++r) {
            for (uint64_t h = 0; h < a->n_heads; ++h)
                bdo_rope_row(q + r * dim + h * hd, hd, pos[r], a->rope_theta);
            for (uint64_t h = 0; h < kvd / hd; ++h)
                bdo_rope_row(k + r * kvd + h * hd, hd, pos[r], a->rope_theta);
            float* ck = kcache[r] + l * a->max_seq * kvd;
            float* cv = vcache[r] + l * a->max_seq * kvd;
            memcpy(ck + pos[r] * kvd, k + r * kvd, kvd * sizeof(float));
            memcpy(cv + pos[r] * kvd, v + r * kvd, kvd * sizeof(float));
            const uint64_t n_ctx = pos[r] + 1;
            for (uint64_t h = 0; h < a->n_heads; ++h) {
                const float* qh = q + r * dim + h * hd;
                const uint64_t kh = h / group;
                for (uint64_t j = 0; j < n_ctx; ++j) {
                    const float* kj = ck + j * kvd + kh * hd;
                    float acc = 0.0f;
                    for (uint64_t d = 0; d < hd; ++d) acc += qh[d] * kj[d];
                    scores[j] = acc * inv_sqrt_hd;
                }
                bdo_softmax_row(scores, n_ctx);
                float* ch = ctx + r * dim + h * hd;
                for (uint64_t j = 0; j < n_ctx; ++j) {
                    const float* vj = cv + j * kvd + kh * hd;
                    for (uint64_t d = 0; d < hd; ++d) ch[d] += scores[j] * vj[d];
                }
            }
        }
        linear(a, base, entries, B, t0 + T_O, ctx, o);
        for (uint64_t i = 0; i < B * dim; ++i) x[i] += o[i];

        for (uint64_t r = 0; r < B; ++r) {
            effective_norm(a, base, entries[r], t0 + T_NORM2, norm_w);
            bdo_rmsnorm_row(x + r * dim, norm_w, dim, normed + r * dim);
        }
        linear(a, base, entries, B, t0 + T_GATE, normed, g);
        linear(a, base, entries, B, t0 + T_UP, normed, u);
        for (uint64_t i = 0; i < B * inter; ++i) g[i] = bdo_silu(g[i]) * u[i];
        linear(a, base, entries, B, t0 + T_DOWN, g, o);
        for (uint64_t i = 0; i < B * dim; ++i) x[i] += o[i];
    }
    free(normed); free(norm_w); free(q); free(k); free(v); free(ctx); free(o);
    free(g); free(u); free(scores);
}

int bdo_decode_layers(const bdo_arch* a, const float* base, const bdo_entry* const* entries,
                      uint64_t B, const uint64_t* pos, float* const* kcache, float* const* vcache,
                      const float* x_in, float* x_out) {
    if (a->dim % a->n_heads || a->kv_dim % (a->dim / a->n_heads) || a->dim % a->kv_dim) return 9;
    memcpy(x_out, x_in, B * a->dim * sizeof(float));
    run_layers(a, base, entries, B, pos, kcache, vcache, x_out);
    return 0;
}

/* ServingPool::decode_shared, serve.cpp:205-325 */
int bdo_decode_shared(const bdo_arch* a, const float* base, const bdo_entry* const* entries,
                      uint64_t B, const int32_t* tokens, const uint64_t* pos, float* const* kcache,
                      float* const* vcache, float* logits) {
    const uint64_t dim = a->dim;
    if (a->dim % a->n_heads || a->kv_dim % (a->dim / a->n_heads) || a->dim % a->kv_dim) return 9;
    float* x = (float*)calloc(B * dim, sizeof(float));
    float* normed = (float*)calloc(B * dim, sizeof(float));
    float* norm_w = (float*)calloc(dim, sizeof(float));
    const float* emb = tensor_ptr(a, base, 0);
    for (uint64_t r = 0; r < B; ++r) { /* serve.cpp:230-236 */
        const uint64_t tok = (uint64_t)tokens[r];
        memcpy(x + r * dim, emb + tok * dim, dim * sizeof(float));
        delta_row(&entries[r][0], a->vocab, tok, dim, x + r * dim);
    }
    run_layers(a, base, entries, B, pos, kcache, vcache, x);
    const uint64_t fin = 1 + a->n_layers * T_PER_LAYER;
    for (uint64_t r = 0; r < B; ++r) { /* serve.cpp:312-315 */
        effective_norm(a, base, entries[r], fin, norm_w);
        bdo_rmsnorm_row(x + r * dim, norm_w, dim, normed + r * dim);
    }
    linear(a, base, entries, B, fin + 1, normed, logits); /* serve.cpp:316-321 */
    free(x); free(normed); free(norm_w);
    return 0;
}
