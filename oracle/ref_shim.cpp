// TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
//
// extern "C" wrapper over the UNMODIFIED reference library (deltakit, built
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/). Only
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference leg may load the resulting .so, and only as the checker / the CPU
// baseline. Every function forwards to the reference API named beside it; no
// arithmetic lives here.
//
// Status codes: 0 ok, 1 + deltakit::errc on a deltakit::Error, 99 on any other
// exception. dkref_last_error() returns the message of the last failure.

#include <chrono>
#include <cstdint>
#include <cstring>
#include <filesystem>
#include <map>
#include <memory>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "deltakit/arch.hpp"
#include "deltakit/checkpoint.hpp"
#include "deltakit/delta.hpp"
#include "deltakit/int8.hpp"
#include "deltakit/error.hpp"
#include "deltakit/matrix.hpp"
#include "deltakit/nn_ops.hpp"
#include "deltakit/serve.hpp"
#include "deltakit/synth.hpp"

using namespace deltakit;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const Error& e) {
        g_err = e.what();
        return 1 + static_cast<int>(e.code());
    } catch (const std::exception& e) {
        g_err = e.what();
        return 99;
    }
}

DenseMatrix dense(const float* p, std::size_t rows, std::size_t cols) {
    return DenseMatrix(rows, cols, std::vector<float>(p, p + rows * cols));
}

void export_plane(const PackedSignMatrix& p, std::uint8_t* bits, float* scale) {
    std::memcpy(bits, p.bits.data(), p.bits.size());
    *scale = p.scale;
}

ToyArchConfig cfg_from(const char* json) { return ToyArchConfig::from_json(json); }

struct Pool {
    std::unique_ptr<ServingPool> pool;
};

} // namespace

extern "C" {

const char* dkref_last_error() { return g_err.c_str(); }

// delta.hpp:18
int dkref_sign_of(float x) { return sign_of(x); }

// delta.hpp:28-30
std::uint64_t dkref_packed_size(std::uint64_t rows, std::uint64_t cols) {
    return PackedSignMatrix::packed_size(rows, cols);
}

// delta.cpp:16-29
int dkref_compress_delta(const float* delta, std::uint64_t rows, std::uint64_t cols,
                         std::uint8_t* bits, float* scale) {
    return guard([&] { export_plane(compress_delta(dense(delta, rows, cols)), bits, scale); });
}

// delta.cpp:31-34
int dkref_compress_tensor(const float* base, const float* fine, std::uint64_t rows,
                          std::uint64_t cols, std::uint8_t* bits, float* scale) {
    return guard([&] {
        export_plane(compress_tensor(dense(base, rows, cols), dense(fine, rows, cols)), bits,
                     scale);
    });
}

// delta.cpp:57-70; planes written back to back, ceil(rows*cols/8) bytes each
int dkref_compress_stack(const float* base, const float* fine, std::uint64_t rows,
                         std::uint64_t cols, std::uint64_t planes, std::uint8_t* bits,
                         float* scales) {
    return guard([&] {
        const DeltaStack s = compress_stack(dense(base, rows, cols), dense(fine, rows, cols), planes);
        const std::size_t nb = PackedSignMatrix::packed_size(rows, cols);
        for (std::size_t k = 0; k < s.planes.size(); ++k)
            export_plane(s.planes[k], bits + k * nb, scales + k);
    });
}

// delta.cpp:36-42
int dkref_decompress(const std::uint8_t* bits, std::uint64_t rows, std::uint64_t cols,
                     float scale, float* out) {
    return guard([&] {
        PackedSignMatrix p;
        p.rows = rows;
        p.cols = cols;
        p.scale = scale;
        p.bits.assign(bits, bits + PackedSignMatrix::packed_size(rows, cols));
        const DenseMatrix d = decompress_tensor(p);
        std::memcpy(out, d.values().data(), d.size() * sizeof(float));
    });
}

// delta.cpp:80-103 (accumulates into out, like the reference)
int dkref_packed_signed_accumulate(const std::uint8_t* bits, std::uint64_t rows,
                                   std::uint64_t cols, const float* x, float* out) {
    return guard([&] {
        PackedSignMatrix p;
        p.rows = rows;
        p.cols = cols;
        p.bits.assign(bits, bits + PackedSignMatrix::packed_size(rows, cols));
        packed_signed_accumulate(p, {x, cols}, {out, rows});
    });
}

// delta.cpp:105-131 (accumulates into out, like the reference)
int dkref_packed_signed_accumulate_t(const std::uint8_t* bits, std::uint64_t rows,
                                     std::uint64_t cols, const float* y, float* out) {
    return guard([&] {
        PackedSignMatrix p;
        p.rows = rows;
        p.cols = cols;
        p.bits.assign(bits, bits + PackedSignMatrix::packed_size(rows, cols));
        packed_signed_accumulate_t(p, {y, rows}, {out, cols});
    });
}

// int8.cpp:15-42
int dkref_rtn_quantize(const float* w, std::uint64_t rows, std::uint64_t cols, std::int8_t* q,
                       float* scales) {
    return guard([&] {
        const Int8Tensor t = rtn_quantize(DenseMatrix(rows, cols, std::vector<float>(w, w + rows * cols)));
        std::memcpy(q, t.values.data(), t.values.size());
        std::memcpy(scales, t.row_scales.data(), rows * sizeof(float));
    });
}

// int8.cpp:67-81: out (s x rows) = a (s x cols) * q^T, row scale applied after the f32 sum
int dkref_int8_matmul_nt(const float* a, std::uint64_t s, const std::int8_t* q, const float* scales,
                         std::uint64_t rows, std::uint64_t cols, float* out) {
    return guard([&] {
        Int8Tensor t;
        t.rows = rows;
        t.cols = cols;
        t.values.assign(q, q + rows * cols);
        t.row_scales.assign(scales, scales + rows);
        const DenseMatrix y = int8_matmul_nt(DenseMatrix(s, cols, std::vector<float>(a, a + s * cols)), t);
        std::memcpy(out, y.values().data(), s * rows * sizeof(float));
    });
}

// delta.cpp:72-78
int dkref_packed_matvec(const std::uint8_t* bits, std::uint64_t rows, std::uint64_t cols,
                        float scale, const float* x, float* y) {
    return guard([&] {
        PackedSignMatrix p;
        p.rows = rows;
        p.cols = cols;
        p.scale = scale;
        p.bits.assign(bits, bits + PackedSignMatrix::packed_size(rows, cols));
        const std::vector<float> v = packed_matvec(p, {x, cols});
        std::memcpy(y, v.data(), v.size() * sizeof(float));
    });
}

// matrix.cpp:26-41
int dkref_matmul_nt(const float* a, std::uint64_t s, std::uint64_t k, const float* b,
                    std::uint64_t t, float* out) {
    return guard([&] {
        const DenseMatrix y = matmul_nt(dense(a, s, k), dense(b, t, k));
        std::memcpy(out, y.values().data(), y.size() * sizeof(float));
    });
}

// nn_ops.hpp:15-59 (row glue), exported so the oracle port can be pinned to them
double dkref_rmsnorm_row(const float* x, const float* w, std::uint64_t n, float* out) {
    return rmsnorm_row({x, n}, {w, n}, {out, n});
}
void dkref_rope_row(float* head, std::uint64_t n, std::uint64_t pos, float theta) {
    rope_row({head, n}, pos, theta);
}
void dkref_softmax_row(float* row, std::uint64_t n) { softmax_row({row, n}, n); }
float dkref_silu(float x) { return silu(x); }

// arch.cpp:51-69: number of tensors and their (name, rows, cols) in order
int dkref_tensor_count(const char* cfg_json, std::uint64_t* n) {
    return guard([&] { *n = tensor_shapes(cfg_from(cfg_json)).size(); });
}
int dkref_tensor_spec(const char* cfg_json, std::uint64_t i, char* name, std::uint64_t name_cap,
                      std::uint64_t* rows, std::uint64_t* cols) {
    return guard([&] {
        const auto specs = tensor_shapes(cfg_from(cfg_json));
        check(i < specs.size(), errc::bad_argument, "tensor index out of range");
        std::snprintf(name, name_cap, "%s", specs[i].name.c_str());
        *rows = specs[i].rows;
        *cols = specs[i].cols;
    });
}

// synth.cpp:7-21 / 23-44: write tensors in tensor_shapes order into out
int dkref_synth_base(const char* cfg_json, std::uint64_t seed, float weight_scale, float* out) {
    return guard([&] {
        const ToyArchConfig cfg = cfg_from(cfg_json);
        const ModelCheckpoint c = synth_base(cfg, seed, weight_scale);
        for (const auto& spec : tensor_shapes(cfg)) {
            const auto& v = c.tensor(spec.name).values();
            std::memcpy(out, v.data(), v.size() * sizeof(float));
            out += v.size();
        }
    });
}

namespace {
ModelCheckpoint ckpt_from(const char* cfg_json, const float* data) {
    ModelCheckpoint c;
    c.config = cfg_from(cfg_json);
    for (const auto& spec : tensor_shapes(*c.config)) {
        c.tensors.emplace(spec.name, dense(data, spec.rows, spec.cols));
        data += spec.count();
    }
    return c;
}
} // namespace

int dkref_synth_fine(const char* cfg_json, const float* base, int kind_signed, float magnitude,
                     std::uint64_t seed, float* out) {
    return guard([&] {
        const ModelCheckpoint b = ckpt_from(cfg_json, base);
        const ModelCheckpoint f =
            synth_fine(b, kind_signed ? PerturbKind::Signed : PerturbKind::Sigma, magnitude, seed,
                       default_quantize_policy());
        for (const auto& spec : tensor_shapes(*b.config)) {
            const auto& v = f.tensor(spec.name).values();
            std::memcpy(out, v.data(), v.size() * sizeof(float));
            out += v.size();
        }
    });
}

// delta.cpp:174-198 + 223-263: build_delta_file(base, fine, planes, linear policy) -> .bdelta
int dkref_write_delta_file(const char* cfg_json, const float* base, const float* fine,
                           std::uint64_t planes, const char* path) {
    return guard([&] {
        const DeltaFile d = build_delta_file(ckpt_from(cfg_json, base), ckpt_from(cfg_json, fine),
                                             planes, default_quantize_policy());
        write_delta_file(d, path);
    });
}

// serve.cpp:93-97 ServingPool(ModelCheckpoint)
int dkref_pool_create(const char* cfg_json, const float* base, void** out) {
    return guard([&] {
        auto* p = new Pool;
        p->pool = std::make_unique<ServingPool>(ckpt_from(cfg_json, base));
        *out = p;
    });
}
void dkref_pool_destroy(void* p) { delete static_cast<Pool*>(p); }

// serve.cpp:129-152
int dkref_pool_register(void* p, const char* id, const char* path, int resident) {
    return guard([&] { static_cast<Pool*>(p)->pool->register_delta(id, path, resident != 0); });
}

// serve.cpp:168-177
int dkref_pool_open(void* p, const char* id, std::uint64_t* req) {
    return guard([&] { *req = static_cast<Pool*>(p)->pool->open_request(id); });
}

// serve.cpp:199-203; logits written row by row (B x vocab)
int dkref_pool_decode(void* p, std::uint64_t n, const std::uint64_t* req_ids,
                      const std::int32_t* tokens, const std::uint64_t* positions, int naive,
                      float* logits) {
    return guard([&] {
        DecodeBatch b;
        for (std::size_t i = 0; i < n; ++i) b.requests.push_back({req_ids[i], tokens[i], positions[i]});
        const auto out = static_cast<Pool*>(p)->pool->decode_step(
            b, naive ? ServeMode::Naive : ServeMode::Shared);
        for (const auto& row : out) {
            std::memcpy(logits, row.data(), row.size() * sizeof(float));
            logits += row.size();
        }
    });
}

// serve.hpp:76-81
std::uint64_t dkref_pool_backbone_passes(void* p) {
    return static_cast<Pool*>(p)->pool->stats().backbone_passes;
}

// CPU baseline workload: the linear work decode_shared does per projection
// (serve.cpp:247-254): one matmul_nt over the stacked batch + one
// apply_delta_correction (= packed_signed_accumulate, serve.cpp:22-26) per
// request, sharded over `threads` host threads by output-row range (the
// reference functions are pure, README.md:163-166). Returns wall seconds.
int dkref_time_multitenant_linear(const float* w, std::uint64_t rows, std::uint64_t cols,
                                  const std::uint8_t* const* tenant_bits, const float* alpha,
                                  const std::int32_t* req_tenant, const float* x,
                                  std::uint64_t batch, std::uint64_t threads, float* y,
                                  double* seconds) {
    return guard([&] {
        const std::size_t nt = threads ? threads : 1;
        const std::size_t nb_row = cols / 8; // callers pass cols % 8 == 0 for row slicing
        check(cols % 8 == 0, errc::bad_argument, "timing harness needs cols % 8 == 0");
        const DenseMatrix X = dense(x, batch, cols);
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (std::size_t t = 0; t < nt; ++t) {
            pool.emplace_back([&, t] {
                const std::size_t r0 = rows * t / nt, r1 = rows * (t + 1) / nt;
                if (r1 <= r0) return;
                const DenseMatrix W = dense(w + r0 * cols, r1 - r0, cols);
                const DenseMatrix Y = matmul_nt(X, W); // backbone_linear_nt
                std::vector<float> tmp(r1 - r0);
                for (std::size_t b = 0; b < batch; ++b) {
                    PackedSignMatrix p;
                    p.rows = r1 - r0;
                    p.cols = cols;
                    const std::uint8_t* src = tenant_bits[req_tenant[b]] + r0 * nb_row;
                    p.bits.assign(src, src + (r1 - r0) * nb_row);
                    std::fill(tmp.begin(), tmp.end(), 0.0f);
                    packed_signed_accumulate(p, X.row_span(b), tmp);
                    const float a = alpha[req_tenant[b]];
                    for (std::size_t i = 0; i < r1 - r0; ++i)
                        y[b * rows + r0 + i] = Y(b, i) + a * tmp[i];
                }
            });
        }
        for (auto& th : pool) th.join();
        auto t1 = std::chrono::steady_clock::now();
        *seconds = std::chrono::duration<double>(t1 - t0).count();
    });
}

// compress_tensor over `threads` independent matrices (one per thread slot);
// returns wall seconds for all of them.
int dkref_time_compress(const float* const* base, const float* const* fine, std::uint64_t n,
                        std::uint64_t rows, std::uint64_t cols, std::uint64_t threads,
                        std::uint8_t* const* bits, float* scales, double* seconds) {
    return guard([&] {
        const std::size_t nt = threads ? threads : 1;
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (std::size_t t = 0; t < nt; ++t) {
            pool.emplace_back([&, t] {
                for (std::size_t i = t; i < n; i += nt) {
                    const PackedSignMatrix p =
                        compress_tensor(dense(base[i], rows, cols), dense(fine[i], rows, cols));
                    export_plane(p, bits[i], scales + i);
                }
            });
        }
        for (auto& th : pool) th.join();
        auto t1 = std::chrono::steady_clock::now();
        *seconds = std::chrono::duration<double>(t1 - t0).count();
    });
}

} // extern "C"
