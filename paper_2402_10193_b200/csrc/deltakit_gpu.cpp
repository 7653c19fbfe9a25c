// deltakit_gpu: reference-API mirror over the C-ABI (include/deltakit_gpu/deltakit_gpu.hpp).
#include "../../include/deltakit_gpu/deltakit_gpu.hpp"

#include <cuda_runtime.h>

#include <cstring>

#include "../../include/bitdelta/capi.h"

namespace deltakit_gpu {

namespace {

[[noreturn]] void raise(int rc) {
    const std::string msg = bd_last_error();
    if (rc >= 1 && rc <= 14) throw Error(static_cast<errc>(rc - 1), msg);
    throw Error(errc::device, msg);
}
void ok(int rc) {
    if (rc != BD_OK) raise(rc);
}
void cu(cudaError_t e) {
    if (e != cudaSuccess) throw Error(errc::device, cudaGetErrorString(e));
}

// device buffer with value semantics restricted to this translation unit
struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(std::size_t bytes) { cu(cudaMalloc(&p, bytes ? bytes : 16)); }
    ~DevBuf() { cudaFree(p); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p) { o.p = nullptr; }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

DevBuf upload(const void* src, std::size_t bytes) {
    DevBuf d(bytes);
    if (bytes) cu(cudaMemcpy(d.p, src, bytes, cudaMemcpyHostToDevice));
    return d;
}

PackedSignMatrix compress_impl(const DenseMatrix* base, const DenseMatrix& fine) {
    PackedSignMatrix p;
    p.rows = fine.rows();
    p.cols = fine.cols();
    const std::size_t n = fine.size(), nb = PackedSignMatrix::packed_size(p.rows, p.cols);
    DevBuf df = upload(fine.values().data(), n * 4);
    DevBuf bits(nb), alpha(4);
    if (base) {
        DevBuf db = upload(base->values().data(), n * 4);
        ok(bd_compress(db.p, df.p, BD_F32, p.rows, p.cols, bits.as<uint8_t>(), alpha.as<float>(), nullptr));
        cu(cudaDeviceSynchronize());
    } else {
        ok(bd_compress(nullptr, df.p, BD_F32, p.rows, p.cols, bits.as<uint8_t>(), alpha.as<float>(), nullptr));
    }
    p.bits.resize(nb);
    if (nb) cu(cudaMemcpy(p.bits.data(), bits.p, nb, cudaMemcpyDeviceToHost));
    cu(cudaMemcpy(&p.scale, alpha.p, 4, cudaMemcpyDeviceToHost));
    return p;
}

}  // namespace

DenseMatrix::DenseMatrix(std::size_t rows, std::size_t cols, std::vector<float> values)
    : rows_(rows), cols_(cols), v_(std::move(values)) {
    if (v_.size() != rows_ * cols_)
        throw Error(errc::length_mismatch, "DenseMatrix: data length does not equal rows*cols");
}

PackedSignMatrix compress_delta(const DenseMatrix& delta) { return compress_impl(nullptr, delta); }

PackedSignMatrix compress_tensor(const DenseMatrix& base, const DenseMatrix& fine) {
    if (!base.same_shape(fine)) throw Error(errc::shape_mismatch, "compress_tensor: shape mismatch");
    return compress_impl(&base, fine);
}

// Format conversion only (delta.cpp:36-42 semantics): +/-scale per bit.
DenseMatrix decompress_tensor(const PackedSignMatrix& p) {
    DenseMatrix out(p.rows, p.cols);
    auto& v = out.values();
    for (std::size_t i = 0; i < v.size(); ++i) v[i] = ((p.bits[i >> 3] >> (i & 7)) & 1u) ? p.scale : -p.scale;
    return out;
}

DenseMatrix DeltaStack::reconstruct() const {
    if (planes.empty()) throw Error(errc::bad_argument, "DeltaStack: no planes");
    DenseMatrix out = decompress_tensor(planes.front());
    for (std::size_t i = 1; i < planes.size(); ++i) {
        const DenseMatrix d = decompress_tensor(planes[i]);
        for (std::size_t j = 0; j < out.size(); ++j) out.values()[j] += d.values()[j];
    }
    return out;
}

std::uint64_t DeltaStack::payload_bytes() const {
    std::uint64_t t = 0;
    for (const auto& p : planes) t += p.payload_bytes();
    return t;
}

DeltaStack compress_stack(const DenseMatrix& base, const DenseMatrix& fine, std::size_t planes) {
    if (planes < 1) throw Error(errc::bad_argument, "compress_stack: plane count must be >= 1");
    if (!base.same_shape(fine)) throw Error(errc::shape_mismatch, "compress_stack: shape mismatch");
    const std::size_t n = fine.size(), nb = PackedSignMatrix::packed_size(fine.rows(), fine.cols());
    DevBuf db = upload(base.values().data(), n * 4), df = upload(fine.values().data(), n * 4);
    DevBuf bits(planes * nb), alphas(planes * 4);
    ok(bd_compress_stack(db.p, df.p, BD_F32, fine.rows(), fine.cols(), planes, bits.as<uint8_t>(),
                         alphas.as<float>(), nullptr));
    std::vector<std::uint8_t> hb(planes * nb);
    std::vector<float> ha(planes);
    if (!hb.empty()) cu(cudaMemcpy(hb.data(), bits.p, hb.size(), cudaMemcpyDeviceToHost));
    cu(cudaMemcpy(ha.data(), alphas.p, planes * 4, cudaMemcpyDeviceToHost));
    DeltaStack s;
    for (std::size_t k = 0; k < planes; ++k) {
        PackedSignMatrix p;
        p.rows = fine.rows();
        p.cols = fine.cols();
        p.scale = ha[k];
        p.bits.assign(hb.begin() + k * nb, hb.begin() + (k + 1) * nb);
        s.planes.push_back(std::move(p));
    }
    return s;
}

void packed_signed_accumulate(const PackedSignMatrix& p, std::span<const float> x, std::span<float> out) {
    if (x.size() != p.cols || out.size() != p.rows)
        throw Error(errc::length_mismatch, "packed_signed_accumulate: length mismatch");
    DevBuf bits = upload(p.bits.data(), p.bits.size());
    DevBuf dx = upload(x.data(), x.size() * 4), dout = upload(out.data(), out.size() * 4);
    ok(bd_packed_signed_accumulate(bits.as<uint8_t>(), p.rows, p.cols, dx.as<float>(), 1,
                                   dout.as<float>(), nullptr));
    if (!out.empty()) cu(cudaMemcpy(out.data(), dout.p, out.size() * 4, cudaMemcpyDeviceToHost));
}

std::vector<float> packed_matvec(const PackedSignMatrix& p, std::span<const float> x) {
    if (x.size() != p.cols) throw Error(errc::length_mismatch, "packed_matvec: length mismatch");
    std::vector<float> y(p.rows, 0.0f);
    DevBuf bits = upload(p.bits.data(), p.bits.size());
    DevBuf dx = upload(x.data(), x.size() * 4), dy(y.size() * 4);
    ok(bd_packed_matvec(bits.as<uint8_t>(), p.scale, p.rows, p.cols, dx.as<float>(), 1, dy.as<float>(),
                        nullptr));
    if (!y.empty()) cu(cudaMemcpy(y.data(), dy.p, y.size() * 4, cudaMemcpyDeviceToHost));
    return y;
}

// ---------------------------------------------------------------- serving --
struct ServingPool::Impl {
    bd_pool* pool = nullptr;
    std::size_t vocab = 0;
};

ServingPool::ServingPool(const ArchConfig& cfg,
                         const std::vector<std::pair<std::string, DenseMatrix>>& backbone, int device)
    : impl_(std::make_unique<Impl>()) {
    ok(bd_device_check(device));
    bd_arch a{cfg.vocab, cfg.dim, cfg.kv_dim ? cfg.kv_dim : cfg.dim, cfg.n_layers, cfg.n_heads,
              cfg.intermediate, cfg.max_seq, cfg.rope_theta};
    ok(bd_pool_create(&a, device, 1, 0, &impl_->pool));
    impl_->vocab = cfg.vocab;
    for (const auto& [name, m] : backbone)
        ok(bd_pool_set_tensor(impl_->pool, name.c_str(), m.values().data(), BD_F32, 0, m.rows(), m.cols()));
}

ServingPool::~ServingPool() {
    if (impl_ && impl_->pool) bd_pool_destroy(impl_->pool);
}

void ServingPool::register_delta(const std::string& id, const std::string& path, bool resident) {
    ok(bd_pool_register_delta_file(impl_->pool, id.c_str(), path.c_str(), resident ? 1 : 0));
}

std::size_t ServingPool::open_request(const std::string& delta_id) {
    uint64_t r = 0;
    ok(bd_pool_open_request(impl_->pool, delta_id.c_str(), &r));
    return r;
}

void ServingPool::close_request(std::size_t request_id) {
    ok(bd_pool_close_request(impl_->pool, request_id));
}

std::vector<std::vector<float>> ServingPool::decode_step(const DecodeBatch& batch, ServeMode mode) {
    std::vector<bd_request> reqs;
    for (const auto& r : batch.requests) reqs.push_back({r.request_id, r.token, r.position});
    std::vector<float> flat(reqs.size() * impl_->vocab);
    ok(bd_pool_decode_step(impl_->pool, reqs.data(), reqs.size(), mode == ServeMode::Shared ? 0 : 1,
                           flat.data(), nullptr));
    std::vector<std::vector<float>> out(reqs.size());
    for (std::size_t i = 0; i < reqs.size(); ++i)
        out[i].assign(flat.begin() + i * impl_->vocab, flat.begin() + (i + 1) * impl_->vocab);
    return out;
}

ServingPool::Stats ServingPool::stats() const {
    bd_pool_stats s{};
    ok(bd_pool_get_stats(impl_->pool, &s));
    return {s.backbone_passes, s.cold_loads, s.last_cold_load_ms};
}

std::uint64_t ServingPool::resident_bytes() const {
    bd_pool_stats s{};
    ok(bd_pool_get_stats(impl_->pool, &s));
    return s.resident_bytes;
}

}  // namespace deltakit_gpu
