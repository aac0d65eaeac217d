// ref_shim.cpp -- extern "C" face of the UNMODIFIED reference library, TEST / BASELINE ONLY.
//
// oracle/Makefile compiles this file together with the reference sources where
// they lie (/root/reference/proj/src/*.cpp) into oracle/_ref/libtaco_ref.so.
// It is used (a) to pin the C restatement in taco_oracle.c, (b) to generate the
// golden fixtures in tests/golden/, and (c) as bench.py's `--impl reference`
// arm and cpu_baseline (kind "reference").  The product never links it.
#include <cstdlib>
#include <cstring>
#include <span>
#include <string>
#include <vector>

#include "taco/analysis.hpp"
#include "taco/codec.hpp"
#include "taco/collective.hpp"
#include "taco/error.hpp"
#include "taco/parallel.hpp"
#include "taco/serialize.hpp"

namespace {
thread_local std::string g_msg;

int code_of(const taco::Error& e) { return static_cast<int>(e.code()) + 1; }

taco::CodecConfig make_cfg(uint32_t b, float tau, float eps, int fmt, int kind) {
    taco::CodecConfig c;
    c.block_size = b;
    c.target_energy = tau;
    c.stability_epsilon = eps;
    c.format = fmt ? taco::Fp8Variant::E5M2 : taco::Fp8Variant::E4M3;
    c.kind = static_cast<taco::CodecKind>(kind);
    return c;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const taco::Error& e) {
        g_msg = e.what();
        return code_of(e);
    } catch (const std::exception& e) {
        g_msg = e.what();
        return 99;
    }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_msg.c_str(); }

void ref_set_threads(int t) {
    if (t <= 0)
        unsetenv("TACO_THREADS");
    else
        setenv("TACO_THREADS", std::to_string(t).c_str(), 1);
}

unsigned ref_worker_count() { return taco::worker_count(); }

// taco::compress (codec.hpp:57) flattened: codes[M*B], alpha[M], scale[M]
int ref_compress(const float* x, uint64_t n, uint32_t b, float tau, float eps, int fmt, int kind,
                 uint8_t* codes, float* alpha, float* scale) {
    return guarded([&] {
        auto ct = taco::compress(std::span<const float>(x, n), make_cfg(b, tau, eps, fmt, kind));
        const size_t pay = ct.blocks.empty() ? 0 : ct.blocks[0].payload.size();
        for (size_t k = 0; k < ct.blocks.size(); ++k) {
            std::memcpy(codes + k * pay, ct.blocks[k].payload.data(), pay);
            alpha[k] = ct.blocks[k].alpha;
            scale[k] = ct.blocks[k].scale;
        }
    });
}

// taco::decompress (codec.hpp:62) from the flattened form
int ref_decompress(const uint8_t* codes, const float* alpha, const float* scale, uint64_t n,
                   uint32_t b, int fmt, int kind, float* out) {
    return guarded([&] {
        auto cfg = make_cfg(b, 1.0f, 1e-12f, fmt, kind);
        taco::CompressedTensor ct;
        ct.kind = cfg.kind;
        ct.format = cfg.format;
        ct.block_size = b;
        ct.original_length = n;
        const size_t pay = cfg.kind == taco::CodecKind::Identity ? 4u * b : b;
        ct.blocks.resize((n + b - 1) / b);
        for (size_t k = 0; k < ct.blocks.size(); ++k) {
            ct.blocks[k].payload.assign(codes + k * pay, codes + (k + 1) * pay);
            ct.blocks[k].alpha = alpha[k];
            ct.blocks[k].scale = scale[k];
        }
        auto y = taco::decompress(ct, cfg);
        std::memcpy(out, y.data(), n * sizeof(float));
    });
}

// compress -> decompress of one tensor (the round trip bench.py times)
int ref_roundtrip(const float* x, uint64_t n, uint32_t b, int fmt, float* out) {
    return guarded([&] {
        auto cfg = make_cfg(b, 1.0f, 1e-12f, fmt, 0);
        auto y = taco::decompress(taco::compress(std::span<const float>(x, n), cfg), cfg);
        std::memcpy(out, y.data(), n * sizeof(float));
    });
}

// taco::allreduce (collective.hpp:28); inputs rank-major [p][n]
int ref_allreduce(const float* inputs, uint32_t p, uint64_t n, uint32_t b, int fmt, int kind,
                  int algorithm, uint64_t chunk, float* result, float* exact, uint64_t* steps,
                  uint64_t* bytes) {
    return guarded([&] {
        taco::RankSet rs;
        for (uint32_t r = 0; r < p; ++r) rs.inputs.emplace_back(inputs + r * n, inputs + (r + 1) * n);
        rs.algorithm = static_cast<taco::Algorithm>(algorithm);
        rs.codec = make_cfg(b, 1.0f, 1e-12f, fmt, kind);
        rs.chunk_elements = chunk;
        auto out = taco::allreduce(rs);
        std::memcpy(result, out.result.data(), n * sizeof(float));
        std::memcpy(exact, out.exact.data(), n * sizeof(float));
        *steps = out.compress_invocations;
        *bytes = out.bytes_on_wire;
    });
}

// taco::generate (analysis.hpp:37): kind 0 gaussian, 1 near-zero mixture
int ref_generate(int kind, uint64_t n, uint64_t seed, double dense_sigma, double tail_sigma,
                 double tail_fraction, float* out) {
    return guarded([&] {
        taco::SyntheticSpec spec;
        spec.kind = static_cast<taco::SyntheticKind>(kind);
        spec.n = n;
        spec.seed = seed;
        spec.dense_sigma = dense_sigma;
        spec.tail_sigma = tail_sigma;
        spec.tail_fraction = tail_fraction;
        auto x = taco::generate(spec);
        std::memcpy(out, x.data(), n * sizeof(float));
    });
}

// taco::archive_bytes (serialize.hpp:15) of compress(x): writes up to cap bytes
int ref_archive(const float* x, uint64_t n, uint32_t b, int fmt, uint8_t* out, uint64_t cap,
                uint64_t* size) {
    return guarded([&] {
        auto cfg = make_cfg(b, 1.0f, 1e-12f, fmt, 0);
        auto bytes = taco::archive_bytes(taco::compress(std::span<const float>(x, n), cfg));
        *size = bytes.size();
        std::memcpy(out, bytes.data(), std::min<uint64_t>(cap, bytes.size()));
    });
}

uint64_t ref_archive_size(uint32_t b, int kind, uint64_t n) {
    return taco::archive_size_bytes(make_cfg(b, 1.0f, 1e-12f, 0, kind), n);
}

double ref_compressed_ratio(uint32_t b, int kind, uint64_t n) {
    return taco::compressed_ratio(make_cfg(b, 1.0f, 1e-12f, 0, kind), n);
}

// compress with every CodecConfig field (DirectFp8 scope included)
int ref_compress2(const float* x, uint64_t n, uint32_t b, float tau, float eps, int fmt, int kind, int scope,
                  uint8_t* codes, float* alpha, float* scale) {
    return guarded([&] {
        auto cfg = make_cfg(b, tau, eps, fmt, kind);
        cfg.direct_scale = static_cast<taco::DirectScaleScope>(scope);
        auto ct = taco::compress(std::span<const float>(x, n), cfg);
        const size_t pay = ct.blocks.empty() ? 0 : ct.blocks[0].payload.size();
        for (size_t k = 0; k < ct.blocks.size(); ++k) {
            std::memcpy(codes + k * pay, ct.blocks[k].payload.data(), pay);
            alpha[k] = ct.blocks[k].alpha;
            scale[k] = ct.blocks[k].scale;
        }
    });
}

// archive_bytes(compress(x)) for any kind / scope
int ref_archive2(const float* x, uint64_t n, uint32_t b, int fmt, int kind, int scope, uint8_t* out, uint64_t cap,
                 uint64_t* size) {
    return guarded([&] {
        auto cfg = make_cfg(b, 1.0f, 1e-12f, fmt, kind);
        cfg.direct_scale = static_cast<taco::DirectScaleScope>(scope);
        auto bytes = taco::archive_bytes(taco::compress(std::span<const float>(x, n), cfg));
        *size = bytes.size();
        std::memcpy(out, bytes.data(), std::min<uint64_t>(cap, bytes.size()));
    });
}

// archive_parse -> decompress (the import path) of a byte stream
int ref_archive_decode(const uint8_t* bytes, uint64_t size, float* out, uint64_t cap, uint64_t* n) {
    return guarded([&] {
        auto ct = taco::archive_parse(std::span<const uint8_t>(bytes, size));
        auto y = taco::decompress(ct);
        *n = y.size();
        std::memcpy(out, y.data(), std::min<uint64_t>(cap, y.size()) * sizeof(float));
    });
}

// taco::scaled_spectrum (codec.hpp:70)
int ref_scaled_spectrum(const float* x, uint64_t n, uint32_t b, int fmt, int kind, float* out) {
    return guarded([&] {
        auto y = taco::scaled_spectrum(std::span<const float>(x, n), make_cfg(b, 1.0f, 1e-12f, fmt, kind));
        std::memcpy(out, y.data(), y.size() * sizeof(float));
    });
}

// taco::error_report (analysis.hpp:42): out8 = mse, rel_l2, max_abs, zero_collapse, kurtosis,
// defined, first edge, last edge; counts[bins]
int ref_error_report(const float* x, const float* y, uint64_t n, uint32_t bins, double* out8, uint64_t* counts) {
    return guarded([&] {
        auto r = taco::error_report(std::span<const float>(x, n), std::span<const float>(y, n), bins);
        out8[0] = r.mse;
        out8[1] = r.relative_l2;
        out8[2] = r.max_abs_error;
        out8[3] = r.zero_collapse_fraction;
        out8[4] = r.kurtosis;
        out8[5] = r.kurtosis_defined ? 1.0 : 0.0;
        out8[6] = r.histogram.bin_edges.front();
        out8[7] = r.histogram.bin_edges.back();
        for (uint32_t i = 0; i < bins; ++i) counts[i] = r.histogram.counts[i];
    });
}

uint8_t ref_fp8_encode(float x, int fmt) {
    return taco::fp8_encode(x, fmt ? taco::Fp8Format::e5m2() : taco::Fp8Format::e4m3());
}

}  // extern "C"
