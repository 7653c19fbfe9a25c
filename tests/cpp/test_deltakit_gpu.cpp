// Parity checks of the deltakit_gpu C++ mirror (include/deltakit_gpu), written
// against the same behaviours the reference suites pin (P:tests/test_delta.cpp,
// P:tests/test_serve.cpp, P:tests/acceptance.cpp criteria 1-3). Runs on a B200:
//
//   tests/cpp/test_deltakit_gpu <golden_dir>
//
// Prints one line per case and exits non-zero on the first failure.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "deltakit_gpu/deltakit_gpu.hpp"

using namespace deltakit_gpu;

namespace {

int g_fail = 0;
#define CHECK(cond)                                                                  \
    do {                                                                             \
        if (!(cond)) {                                                               \
            std::printf("    CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);  \
            ++g_fail;                                                                \
        }                                                                            \
    } while (0)

DenseMatrix gaussian(std::size_t r, std::size_t c, std::uint64_t seed, float sigma = 1.0f) {
    std::mt19937_64 rng(seed);
    std::normal_distribution<float> d(0.0f, sigma);
    DenseMatrix m(r, c);
    for (float& v : m.values()) v = d(rng);
    return m;
}

double rel_l2(const std::vector<float>& a, const std::vector<float>& b) {
    double num = 0, den = 0;
    for (std::size_t i = 0; i < a.size(); ++i) {
        num += (double(a[i]) - b[i]) * (double(a[i]) - b[i]);
        den += double(b[i]) * b[i];
    }
    return std::sqrt(num) / (den > 0 ? std::sqrt(den) : 1.0);
}

double abs_residual(const DenseMatrix& m, double a) {  // Eq. 3 objective
    double s = 0;
    for (float v : m.values()) s += (std::fabs(double(v)) - a) * (std::fabs(double(v)) - a);
    return s;
}

std::vector<float> dense_matvec(const DenseMatrix& w, const std::vector<float>& x) {
    std::vector<float> y(w.rows());
    for (std::size_t i = 0; i < w.rows(); ++i) {
        double acc = 0;
        for (std::size_t j = 0; j < w.cols(); ++j) acc += double(w(i, j)) * x[j];
        y[i] = float(acc);
    }
    return y;
}

template <class T>
std::vector<T> read_raw(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    std::vector<char> b((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    std::vector<T> v(b.size() / sizeof(T));
    std::memcpy(v.data(), b.data(), v.size() * sizeof(T));
    return v;
}

void run(const char* name, const std::function<void()>& f) {
    const int before = g_fail;
    try {
        f();
    } catch (const std::exception& e) {
        std::printf("    exception: %s\n", e.what());
        ++g_fail;
    }
    std::printf("%s %s\n", g_fail == before ? "PASS" : "FAIL", name);
}

}  // namespace

int main(int argc, char** argv) {
    const std::string golden = argc > 1 ? argv[1] : "tests/golden";

    run("sign convention: zero maps to -1", [] {
        CHECK(sign_of(3.2f) == 1 && sign_of(0.0f) == -1 && sign_of(-0.0f) == -1);
        CHECK(sign_of(-1e-30f) == -1 && sign_of(1e-30f) == 1);
    });
    run("compress: signs and mean-absolute scale", [] {
        const PackedSignMatrix p = compress_tensor(DenseMatrix(2, 2), DenseMatrix(2, 2, {1, -2, 3, -4}));
        CHECK(std::fabs(p.scale - 2.5f) < 1e-7f);
        CHECK(p.bit_at(0, 0) && !p.bit_at(0, 1) && p.bit_at(1, 0) && !p.bit_at(1, 1));
    });
    run("zero delta: zero scale, zero reconstruction", [] {
        const DenseMatrix m = gaussian(6, 5, 3);
        const PackedSignMatrix p = compress_tensor(m, m);
        CHECK(p.scale == 0.0f);
        const DenseMatrix rec = decompress_tensor(p);
        for (float v : rec.values()) CHECK(v == 0.0f);
    });
    run("bit layout: row-major, LSB-first, zero trailing bits", [] {
        const PackedSignMatrix p = compress_delta(DenseMatrix(3, 3, {1, -1, 1, 1, -1, -1, 1, -1, 1}));
        CHECK(p.bits.size() == 2 && p.bits[0] == 0x4D && p.bits[1] == 0x01);
    });
    run("alpha = mean|delta| beats a 1000-point grid", [] {
        const DenseMatrix d = gaussian(64, 64, 42);
        const PackedSignMatrix p = compress_delta(d);
        const double best = abs_residual(d, p.scale);
        float mx = 0;
        for (float v : d.values()) mx = std::max(mx, std::fabs(v));
        for (int i = 0; i < 1000; ++i) CHECK(best <= abs_residual(d, 2.0 * mx * i / 999.0));
    });
    run("round trip keeps signs; compress is idempotent", [] {
        const DenseMatrix d = gaussian(5, 9, 17);
        const PackedSignMatrix p = compress_delta(d);
        const DenseMatrix rec = decompress_tensor(p);
        for (std::size_t i = 0; i < d.size(); ++i)
            if (d.values()[i] != 0.0f) CHECK(sign_of(rec.values()[i]) == sign_of(d.values()[i]));
        const PackedSignMatrix p2 = compress_delta(rec);
        CHECK(p2.bits == p.bits && std::fabs(p2.scale - p.scale) <= 1e-6f * p.scale);
    });
    run("pack/unpack bijection on ragged random patterns", [] {
        std::mt19937_64 rng(99);
        for (int it = 0; it < 300; ++it) {
            const std::size_t r = 1 + rng() % 12, c = 1 + rng() % 23;
            DenseMatrix d(r, c);
            for (float& v : d.values()) v = (rng() & 1) ? 1.0f : -1.0f;
            const PackedSignMatrix p = compress_delta(d);
            const std::size_t tail = (r * c) % 8;
            if (tail) CHECK((p.bits.back() >> tail) == 0);
            const DenseMatrix rec = decompress_tensor(p);
            for (std::size_t i = 0; i < d.size(); ++i) CHECK(sign_of(rec.values()[i]) == sign_of(d.values()[i]));
        }
    });
    run("compress_stack: exact +/-c in one plane; residual decreases; 1-bit error ~ 1-2/pi", [] {
        std::mt19937_64 rng(5);
        DenseMatrix fine(16, 16);
        for (float& v : fine.values()) v = (rng() & 1) ? 0.25f : -0.25f;
        const DenseMatrix r1 = compress_stack(DenseMatrix(16, 16), fine, 1).reconstruct();
        CHECK(rel_l2(r1.values(), fine.values()) <= 1e-6);
        const DenseMatrix g = gaussian(256, 256, 555);
        const DeltaStack s8 = compress_stack(DenseMatrix(256, 256), g, 8);
        std::vector<float> res = g.values();
        double prev = 1e300;
        for (const auto& pl : s8.planes) {
            const DenseMatrix d = decompress_tensor(pl);
            double n = 0;
            for (std::size_t i = 0; i < res.size(); ++i) {
                res[i] -= d.values()[i];
                n += double(res[i]) * res[i];
            }
            CHECK(n < prev);
            prev = n;
        }
        const DeltaStack s1 = compress_stack(DenseMatrix(256, 256), g, 1);
        const double e = rel_l2(s1.reconstruct().values(), g.values());
        CHECK(e * e > 0.33 && e * e < 0.40);
    });
    run("packed_matvec hand examples and dense oracle", [] {
        PackedSignMatrix p1 = compress_delta(DenseMatrix(1, 3, {1, 1, 1}));
        p1.scale = 1.0f;
        CHECK(packed_matvec(p1, std::vector<float>{1, 2, 3})[0] == 6.0f);
        PackedSignMatrix p2 = compress_delta(DenseMatrix(1, 2, {1, -1}));
        p2.scale = 2.0f;
        CHECK(packed_matvec(p2, std::vector<float>{3, 1})[0] == 4.0f);
        const DenseMatrix d = gaussian(256, 256, 777);
        const PackedSignMatrix p = compress_delta(d);
        const DenseMatrix x = gaussian(1, 256, 778);
        CHECK(rel_l2(packed_matvec(p, x.values()), dense_matvec(decompress_tensor(p), x.values())) <= 1e-5);
    });
    run("packed_signed_accumulate accumulates into out; linearity", [] {
        const DenseMatrix d = gaussian(40, 64, 800);
        const PackedSignMatrix p = compress_delta(d);
        const DenseMatrix x = gaussian(1, 64, 801), y = gaussian(1, 64, 802);
        std::vector<float> fx(40, 1.0f), fy(40, 0.0f), fxy(40, 0.0f), xy(64);
        for (int i = 0; i < 64; ++i) xy[i] = x.values()[i] + y.values()[i];
        packed_signed_accumulate(p, x.values(), fx);
        packed_signed_accumulate(p, y.values(), fy);
        packed_signed_accumulate(p, xy, fxy);
        std::vector<float> sum(40);
        for (int i = 0; i < 40; ++i) sum[i] = (fx[i] - 1.0f) + fy[i];
        CHECK(rel_l2(fxy, sum) <= 1e-5);
        bool threw = false;
        try {
            packed_signed_accumulate(p, std::vector<float>(3), fy);
        } catch (const Error& e) {
            threw = e.code() == errc::length_mismatch;
        }
        CHECK(threw);
    });
    run("ServingPool: shared decode vs reference logits, determinism, counters", [&] {
        ArchConfig cfg;
        cfg.vocab = 48;
        cfg.dim = 32;
        cfg.n_layers = 2;
        cfg.n_heads = 4;
        cfg.intermediate = 40;
        cfg.max_seq = 32;
        const std::vector<float> base = read_raw<float>(golden + "/toy_base.f32");
        const std::vector<int> toks = read_raw<int>(golden + "/toy_tokens_B4.i32");
        const std::vector<float> want = read_raw<float>(golden + "/toy_logits_B4.f32");
        std::vector<std::pair<std::string, DenseMatrix>> bb;
        std::size_t off = 0;
        auto add = [&](const std::string& n, std::size_t r, std::size_t c) {
            bb.emplace_back(n, DenseMatrix(r, c, std::vector<float>(base.begin() + off, base.begin() + off + r * c)));
            off += r * c;
        };
        add("embed", 48, 32);
        for (int l = 0; l < 2; ++l) {
            const std::string p = "layers." + std::to_string(l) + ".";
            add(p + "attn_q", 32, 32);
            add(p + "attn_k", 32, 32);
            add(p + "attn_v", 32, 32);
            add(p + "attn_o", 32, 32);
            add(p + "mlp_gate", 40, 32);
            add(p + "mlp_up", 40, 32);
            add(p + "mlp_down", 32, 40);
            add(p + "norm1", 1, 32);
            add(p + "norm2", 1, 32);
        }
        add("final_norm", 1, 32);
        add("lm_head", 48, 32);
        CHECK(off == base.size());
        ServingPool pool(cfg, bb);
        for (int i = 0; i < 4; ++i)
            pool.register_delta("t" + std::to_string(i), golden + "/toy_t" + std::to_string(i) + ".bdelta", true);
        std::vector<std::size_t> rid;
        for (int i = 0; i < 4; ++i) rid.push_back(pool.open_request("t" + std::to_string(i)));
        for (std::size_t pos = 0; pos < toks.size(); ++pos) {
            DecodeBatch b;
            for (int i = 0; i < 4; ++i) b.requests.push_back({rid[i], toks[pos], pos});
            const auto out = pool.decode_step(b, ServeMode::Shared);
            for (int i = 0; i < 4; ++i) {
                const std::vector<float> w(want.begin() + (pos * 4 + i) * 48, want.begin() + (pos * 4 + i + 1) * 48);
                CHECK(rel_l2(out[i], w) <= 1e-2);
            }
        }
        CHECK(pool.stats().backbone_passes == toks.size());
        const std::size_t a = pool.open_request("t0"), c = pool.open_request("t0");
        DecodeBatch same;
        same.requests = {{a, 7, 0}, {c, 7, 0}};
        const auto o = pool.decode_step(same, ServeMode::Shared);
        CHECK(o[0] == o[1]);
        bool threw = false;
        try {
            pool.open_request("nope");
        } catch (const Error& e) {
            threw = e.code() == errc::unknown_id;
        }
        CHECK(threw);
    });
    std::printf("%s: %d failed check(s)\n", g_fail ? "FAILED" : "ALL PASSED", g_fail);
    return g_fail ? 1 : 0;
}
