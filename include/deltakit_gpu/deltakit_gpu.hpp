// deltakit_gpu — host C++ mirror of the reference deltakit API for the BitDelta
// hot path, implemented over the C-ABI (include/bitdelta/capi.h) and the
// sm_100a kernels. Same names, argument meaning, value semantics and error
// categories as the reference (P: = /root/reference/proj/):
//
//   sign_of, PackedSignMatrix, compress_delta, compress_tensor,
//   decompress_tensor, DeltaStack, compress_stack, packed_matvec,
//   packed_signed_accumulate           (P:include/deltakit/delta.hpp:17-70)
//   ServingPool, DecodeRequest/Batch, ServeMode   (P:include/deltakit/serve.hpp:18-100)
//   Error / errc                       (P:include/deltakit/error.hpp:10-42)
//
// Host-typed calls copy inputs to the device, run the kernel and copy results
// back (the CPU-typed API cannot avoid this); device-resident users call the
// C-ABI directly. A maintainer switches a deltakit caller by changing the
// namespace.
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace deltakit_gpu {

// P:include/deltakit/error.hpp:10-25 (same order; C-ABI status = errc + 1)
enum class errc {
    io,
    malformed_header,
    json_parse,
    bad_offsets,
    unsupported_dtype,
    shape_mismatch,
    name_mismatch,
    length_mismatch,
    bad_argument,
    bad_token,
    non_finite,
    no_convergence,
    duplicate_id,
    unknown_id,
    device,  // CUDA / no B200 (no reference equivalent)
};

class Error : public std::runtime_error {
public:
    Error(errc code, const std::string& msg) : std::runtime_error(msg), code_(code) {}
    errc code() const noexcept { return code_; }

private:
    errc code_;
};

// Row-major f32 matrix with the reference DenseMatrix accessors (matrix.hpp:15-58).
class DenseMatrix {
public:
    DenseMatrix() = default;
    DenseMatrix(std::size_t rows, std::size_t cols) : rows_(rows), cols_(cols), v_(rows * cols, 0.0f) {}
    DenseMatrix(std::size_t rows, std::size_t cols, std::vector<float> values);
    std::size_t rows() const { return rows_; }
    std::size_t cols() const { return cols_; }
    std::size_t size() const { return v_.size(); }
    float operator()(std::size_t r, std::size_t c) const { return v_[r * cols_ + c]; }
    float& operator()(std::size_t r, std::size_t c) { return v_[r * cols_ + c]; }
    const float* row(std::size_t r) const { return v_.data() + r * cols_; }
    float* row(std::size_t r) { return v_.data() + r * cols_; }
    const std::vector<float>& values() const { return v_; }
    std::vector<float>& values() { return v_; }
    bool same_shape(const DenseMatrix& o) const { return rows_ == o.rows_ && cols_ == o.cols_; }

private:
    std::size_t rows_ = 0, cols_ = 0;
    std::vector<float> v_;
};

// delta.hpp:18
inline int sign_of(float x) { return x > 0.0f ? 1 : -1; }

// delta.hpp:23-43 — identical byte layout (flat row-major, LSB-first, 1 = +1)
struct PackedSignMatrix {
    std::size_t rows = 0, cols = 0;
    float scale = 0.0f;
    std::vector<std::uint8_t> bits;

    static std::size_t packed_size(std::size_t rows, std::size_t cols) { return (rows * cols + 7) / 8; }
    bool bit_at(std::size_t r, std::size_t c) const {
        const std::size_t idx = r * cols + c;
        return (bits[idx >> 3] >> (idx & 7)) & 1u;
    }
    std::uint64_t payload_bytes() const { return bits.size() + 4; }
};

PackedSignMatrix compress_delta(const DenseMatrix& delta);                              // delta.hpp:47
PackedSignMatrix compress_tensor(const DenseMatrix& base, const DenseMatrix& fine);     // delta.hpp:48
DenseMatrix decompress_tensor(const PackedSignMatrix& p);                               // delta.hpp:49

struct DeltaStack {  // delta.hpp:53-60
    std::vector<PackedSignMatrix> planes;
    std::size_t rows() const { return planes.empty() ? 0 : planes.front().rows; }
    std::size_t cols() const { return planes.empty() ? 0 : planes.front().cols; }
    DenseMatrix reconstruct() const;
    std::uint64_t payload_bytes() const;
};
DeltaStack compress_stack(const DenseMatrix& base, const DenseMatrix& fine, std::size_t planes);  // delta.hpp:62

std::vector<float> packed_matvec(const PackedSignMatrix& p, std::span<const float> x);  // delta.hpp:67
void packed_signed_accumulate(const PackedSignMatrix& p, std::span<const float> x,
                              std::span<float> out);                                    // delta.hpp:69-70

// ---- serving (serve.hpp:18-100) ----
enum class ServeMode { Shared, Naive };
struct DecodeRequest {
    std::size_t request_id = 0;
    std::int32_t token = 0;
    std::size_t position = 0;
};
struct DecodeBatch {
    std::vector<DecodeRequest> requests;
};
struct ArchConfig {  // ToyArchConfig (arch.hpp:11-24) + kv_dim (presets, arch.hpp:36-39)
    std::size_t vocab = 256, dim = 64, kv_dim = 0, n_layers = 2, n_heads = 4, intermediate = 172,
                max_seq = 128;
    float rope_theta = 10000.0f;
};

class ServingPool {
public:
    // backbone: tensors in tensor_shapes order (arch.cpp:51-69), f32 host
    ServingPool(const ArchConfig& cfg, const std::vector<std::pair<std::string, DenseMatrix>>& backbone,
                int device = 0);
    ~ServingPool();
    ServingPool(const ServingPool&) = delete;
    ServingPool& operator=(const ServingPool&) = delete;

    void register_delta(const std::string& id, const std::string& path, bool resident);
    std::size_t open_request(const std::string& delta_id);
    void close_request(std::size_t request_id);
    std::vector<std::vector<float>> decode_step(const DecodeBatch& batch, ServeMode mode);

    struct Stats {  // serve.hpp:76-81
        std::uint64_t backbone_passes = 0;
        std::uint64_t cold_loads = 0;
        double last_cold_load_ms = 0.0;
    };
    Stats stats() const;
    std::uint64_t resident_bytes() const;

private:
    struct Impl;
    std::unique_ptr<Impl> impl_;
};

}  // namespace deltakit_gpu
