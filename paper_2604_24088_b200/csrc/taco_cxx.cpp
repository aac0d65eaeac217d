// taco_cxx.cpp -- the reference's C++ API (include/taco/*.hpp, same declarations as
// proj/include/taco/{error,fp8,transform,codec,collective}.hpp) implemented on top of
// the B200 C ABI.  Relinking a reference caller against libtaco_b200.so moves
// compress / decompress / allreduce(TwoShot) onto the GPU unchanged.
//
// compress, decompress and allreduce never compute on the host: they marshal the
// reference's AoS CompressedTensor <-> the device SoA message and call K1/K2/K3.
// The scalar helpers (fp8_encode, block_rms, the double FWHT utilities, partition)
// stay host code because their signatures are host-scalar / host-span utilities.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <mutex>
#include <stdexcept>

#include "taco/codec.hpp"
#include "taco/collective.hpp"
#include "taco/error.hpp"
#include "taco/fp8.hpp"
#include "taco/transform.hpp"
#include "taco_b200.h"

namespace taco {

namespace {

[[noreturn]] void raise_status(int rc) {
    const char* msg = taco_last_error();
    switch (rc) {
        case TACO_ERR_USAGE: fail(ErrorCode::Usage, msg);
        case TACO_ERR_CONFIG: fail(ErrorCode::Config, msg);
        case TACO_ERR_INPUT: fail(ErrorCode::Input, msg);
        case TACO_ERR_IO: fail(ErrorCode::Io, msg);
        case TACO_ERR_CORRUPT: fail(ErrorCode::Corrupt, msg);
        default: throw std::runtime_error(std::string("taco_b200: ") + msg);
    }
}

void check(int rc) {
    if (rc != TACO_OK) raise_status(rc);
}

// One context per process, created on first use on the current device.
taco_ctx* context() {
    static std::once_flag once;
    static taco_ctx* ctx = nullptr;
    static int rc = TACO_OK;
    std::call_once(once, [] { rc = taco_ctx_create(0, &ctx); });
    check(rc);
    return ctx;
}

taco_config to_c(const CodecConfig& cfg) {
    taco_config c;
    c.block_size = static_cast<uint32_t>(std::min<size_t>(cfg.block_size, 0xffffffffu));
    c.target_energy = cfg.target_energy;
    c.stability_epsilon = cfg.stability_epsilon;
    c.format = cfg.format == Fp8Variant::E5M2 ? 1u : 0u;
    c.kind = static_cast<uint32_t>(cfg.kind);
    c.direct_scale = static_cast<uint32_t>(cfg.direct_scale);
    return c;
}

size_t payload_bytes(CodecKind k, size_t b) { return k == CodecKind::Identity ? 4 * b : b; }

constexpr Fp8Format kE4M3{Fp8Variant::E4M3, 4, 3, 7, 448.0f, false};
constexpr Fp8Format kE5M2{Fp8Variant::E5M2, 5, 2, 15, 57344.0f, true};

std::array<float, 256> make_table(const Fp8Format& f) {
    std::array<float, 256> t{};
    const int emax = (1 << f.exponent_bits) - 1, fmask = (1 << f.mantissa_bits) - 1;
    for (int c = 0; c < 256; ++c) {
        const int e = (c >> f.mantissa_bits) & emax, fr = c & fmask;
        float v;
        if (e == 0)
            v = std::ldexp(static_cast<float>(fr), 1 - f.bias - f.mantissa_bits);
        else if (e == emax && f.has_infinity)
            v = fr == 0 ? std::numeric_limits<float>::infinity() : std::numeric_limits<float>::quiet_NaN();
        else if (e == emax && fr == fmask)
            v = std::numeric_limits<float>::quiet_NaN();
        else
            v = std::ldexp(1.0f + static_cast<float>(fr) / static_cast<float>(1 << f.mantissa_bits), e - f.bias);
        t[c] = (c & 0x80) ? -v : v;
    }
    return t;
}

}  // namespace

// ------------------------------------------------------------------------- fp8 ---
const Fp8Format& Fp8Format::e4m3() { return kE4M3; }
const Fp8Format& Fp8Format::e5m2() { return kE5M2; }
const Fp8Format& Fp8Format::from_variant(Fp8Variant v) { return v == Fp8Variant::E5M2 ? kE5M2 : kE4M3; }

const std::array<float, 256>& fp8_decode_table(const Fp8Format& fmt) {
    static const std::array<float, 256> t4 = make_table(kE4M3), t5 = make_table(kE5M2);
    return fmt.variant == Fp8Variant::E5M2 ? t5 : t4;
}

float fp8_decode(Fp8Code code, const Fp8Format& fmt) { return fp8_decode_table(fmt)[code]; }

// nearest-even on the fp8 grid, saturating (the device uses cvt.rn.satfinite)
Fp8Code fp8_encode(float x, const Fp8Format& fmt) {
    if (std::isnan(x)) return 0x7F;
    uint32_t u;
    std::memcpy(&u, &x, 4);
    const Fp8Code sign = static_cast<Fp8Code>((u >> 24) & 0x80u);
    const float ax = std::fabs(x);
    if (ax > fmt.q_max) return sign | (fmt.has_infinity ? 0x7B : 0x7E);
    if (ax < std::ldexp(1.0f, 1 - fmt.bias)) {
        const double q = std::nearbyint(static_cast<double>(ax) * std::ldexp(1.0, fmt.bias + fmt.mantissa_bits - 1));
        return sign | static_cast<Fp8Code>(q);
    }
    uint32_t a;
    std::memcpy(&a, &ax, 4);
    a -= static_cast<uint32_t>(127 - fmt.bias) << 23;
    const int drop = 23 - fmt.mantissa_bits;
    a += (1u << (drop - 1)) - 1u + ((a >> drop) & 1u);
    return sign | static_cast<Fp8Code>(a >> drop);
}

float fp8_ulp(float x, const Fp8Format& fmt) {
    const float ax = std::fabs(x), mn = std::ldexp(1.0f, 1 - fmt.bias);
    if (!(ax >= mn)) return std::ldexp(1.0f, 1 - fmt.bias - fmt.mantissa_bits);
    return std::ldexp(1.0f, std::ilogb(ax) - fmt.mantissa_bits);
}

// ------------------------------------------------------------------- transform ---
bool is_valid_block_size(size_t b) { return b >= kMinBlockSize && b <= kMaxBlockSize && (b & (b - 1)) == 0; }

void validate_block_size(size_t b) {
    if (b == 0 || (b & (b - 1)) != 0) fail(ErrorCode::Config, "block size must be a power of two");
    if (b < kMinBlockSize || b > kMaxBlockSize) fail(ErrorCode::Config, "block size must be between 2 and 32768");
}

std::vector<Block> partition(std::span<const float> x, size_t block_size) {
    validate_block_size(block_size);
    if (x.empty()) fail(ErrorCode::Input, "input tensor is empty");
    std::vector<Block> out((x.size() + block_size - 1) / block_size);
    for (size_t k = 0; k < out.size(); ++k) {
        const size_t at = k * block_size, valid = std::min(block_size, x.size() - at);
        out[k].values.assign(block_size, 0.0f);
        std::copy_n(x.begin() + static_cast<ptrdiff_t>(at), valid, out[k].values.begin());
        out[k].block_index = k;
        out[k].valid_length = valid;
    }
    return out;
}

void fwht_orthonormal_inplace(std::span<double> v) {
    const size_t n = v.size();
    if (n == 0 || (n & (n - 1)) != 0) fail(ErrorCode::Config, "transform length must be a power of two");
    for (size_t h = 1; h < n; h *= 2)
        for (size_t i = 0; i < n; i += 2 * h)
            for (size_t j = i; j < i + h; ++j) {
                const double a = v[j], b = v[j + h];
                v[j] = a + b;
                v[j + h] = a - b;
            }
    const double norm = 1.0 / std::sqrt(static_cast<double>(n));
    for (double& e : v) e *= norm;
}

std::vector<float> fwht_orthonormal(std::span<const float> v) {
    std::vector<double> w(v.begin(), v.end());
    fwht_orthonormal_inplace(w);
    return std::vector<float>(w.begin(), w.end());
}

std::vector<float> fwht_inverse(std::span<const float> v) { return fwht_orthonormal(v); }

// ----------------------------------------------------------------------- codec ---
void validate_config(const CodecConfig& cfg) {
    validate_block_size(cfg.block_size);
    if (!(cfg.target_energy > 0.0f) || !std::isfinite(cfg.target_energy))
        fail(ErrorCode::Config, "target energy must be positive and finite");
    if (!(cfg.stability_epsilon > 0.0f) || !std::isfinite(cfg.stability_epsilon))
        fail(ErrorCode::Config, "stability epsilon must be positive and finite");
}

float block_rms(std::span<const float> g, float eps) {
    double acc = 0.0;
    for (float v : g) acc += static_cast<double>(v) * v;
    return static_cast<float>(std::sqrt(acc / static_cast<double>(g.size()) + static_cast<double>(eps)));
}

float adaptive_scale(float sigma, float tau) { return tau / sigma; }

CompressedTensor compress(std::span<const float> x, const CodecConfig& cfg) {
    validate_config(cfg);
    if (x.empty()) fail(ErrorCode::Input, "input tensor is empty");
    const taco_config c = to_c(cfg);
    const uint64_t b = cfg.block_size, m = (x.size() + b - 1) / b, pb = payload_bytes(cfg.kind, b);
    taco_layout lay;
    check(taco_msg_layout(&c, m, &lay));
    std::vector<uint8_t> msg(lay.msg_bytes);
    check(taco_compress_host(context(), &c, x.data(), TACO_DT_F32, x.size(), msg.data()));
    CompressedTensor ct;
    ct.kind = cfg.kind;
    ct.format = cfg.format;
    ct.block_size = static_cast<uint32_t>(b);
    ct.original_length = x.size();
    ct.blocks.resize(m);
    const float* scal = reinterpret_cast<const float*>(msg.data() + lay.scal_offset);
    for (uint64_t k = 0; k < m; ++k) {
        ct.blocks[k].payload.assign(msg.data() + k * pb, msg.data() + (k + 1) * pb);
        ct.blocks[k].alpha = scal[2 * k];
        ct.blocks[k].scale = scal[2 * k + 1];
    }
    return ct;
}

TensorBuffer decompress(const CompressedTensor& ct) {
    CodecConfig cfg;
    cfg.kind = ct.kind;
    cfg.format = ct.format;
    cfg.block_size = ct.block_size;
    return decompress(ct, cfg);
}

TensorBuffer decompress(const CompressedTensor& ct, const CodecConfig& cfg) {
    if (cfg.kind != ct.kind || cfg.format != ct.format || cfg.block_size != ct.block_size)
        fail(ErrorCode::Corrupt, "codec config does not match the compressed tensor");
    const size_t b = ct.block_size;
    validate_block_size(b);
    const uint64_t n = ct.original_length;
    if (n == 0) fail(ErrorCode::Corrupt, "compressed tensor declares zero elements");
    const uint64_t m = (n + b - 1) / b;
    if (ct.blocks.size() != m) fail(ErrorCode::Corrupt, "block count does not match the declared length");
    const size_t payload = ct.kind == CodecKind::Identity ? 4 * b : b;
    for (const auto& blk : ct.blocks) {
        if (blk.payload.size() != payload) fail(ErrorCode::Corrupt, "block payload has the wrong size");
        if (!std::isfinite(blk.alpha) || !std::isfinite(blk.scale) || blk.scale == 0.0f || blk.alpha == 0.0f)
            fail(ErrorCode::Corrupt, "block scalars must be finite and nonzero");
    }
    taco_config c = to_c(cfg);
    taco_layout lay;
    check(taco_msg_layout(&c, m, &lay));
    std::vector<uint8_t> msg(lay.msg_bytes);
    float* scal = reinterpret_cast<float*>(msg.data() + lay.scal_offset);
    for (uint64_t k = 0; k < m; ++k) {
        std::memcpy(msg.data() + k * payload, ct.blocks[k].payload.data(), payload);
        scal[2 * k] = ct.blocks[k].alpha;
        scal[2 * k + 1] = ct.blocks[k].scale;
    }
    TensorBuffer out(n);
    check(taco_decompress_host(context(), &c, msg.data(), n, out.data(), TACO_DT_F32));
    return out;
}

double compressed_ratio(const CodecConfig& cfg, uint64_t n) {
    if (n == 0) fail(ErrorCode::Input, "element count must be positive");
    if (cfg.kind == CodecKind::Identity) return 1.0;
    const taco_config c = to_c(cfg);
    return taco_compressed_ratio(&c, n);
}

TensorBuffer scaled_spectrum(std::span<const float> x, const CodecConfig& cfg) {
    validate_config(cfg);
    if (x.empty()) fail(ErrorCode::Input, "input tensor is empty");
    const taco_config c = to_c(cfg);
    const uint64_t b = cfg.block_size, m = (x.size() + b - 1) / b;
    TensorBuffer out(m * b);
    check(taco_scaled_spectrum_host(context(), &c, x.data(), x.size(), out.data()));
    return out;
}

const char* codec_kind_name(CodecKind k) {
    switch (k) {
        case CodecKind::Taco: return "taco";
        case CodecKind::DirectFp8: return "direct_fp8";
        case CodecKind::Int8Uniform: return "int8";
        case CodecKind::Identity: return "identity";
        case CodecKind::AshInt8: return "ash_int8";
    }
    return "unknown";
}

// ------------------------------------------------------------------ collective ---
const char* algorithm_name(Algorithm a) {
    switch (a) {
        case Algorithm::TwoShot: return "twoshot";
        case Algorithm::Ring: return "ring";
        case Algorithm::Tree: return "tree";
    }
    return "?";
}

namespace {
// collective.cpp:50-58: wire bytes of one transfer, chunk framing rounds to blocks
uint64_t message_bytes(const CodecConfig& cfg, uint64_t n, size_t chunk_elements) {
    const taco_config c = to_c(cfg);
    if (chunk_elements == 0) return taco_archive_size(&c, n);
    const uint64_t b = cfg.block_size, chunk = ((chunk_elements + b - 1) / b) * b;
    uint64_t total = 0;
    for (uint64_t at = 0; at < n; at += chunk) total += taco_archive_size(&c, std::min(chunk, n - at));
    return total;
}
}  // namespace

namespace {

// Schedule shape (collective.cpp:75-254) in closed form: compressed transfer steps and wire
// bytes.  Two-shot: two batched steps of P(P-1) shard messages.  Ring: P-1 codec hops of the
// whole tensor plus P-1 forwards of the final archive.  Tree over q = 2^floor(log2 P) ranks:
// an optional fold step (P-q whole padded tensors), log2 q halving rounds in which each of the
// P origins is carried as 2^k pieces of padded/2^(k+1) elements, log2 q doubling rounds in
// which every rank forwards the 2^k slice archives it holds, and an optional unfold step.
void schedule_shape(const RankSet& rs, uint64_t& steps, uint64_t& bytes) {
    const uint64_t p = rs.inputs.size(), n = rs.inputs[0].size();
    auto mb = [&](uint64_t len) { return message_bytes(rs.codec, len, rs.chunk_elements); };
    steps = bytes = 0;
    if (rs.algorithm == Algorithm::TwoShot) {
        steps = 2;
        bytes = 2 * p * (p - 1) * mb((n + p - 1) / p);
        return;
    }
    if (rs.algorithm == Algorithm::Ring) {
        steps = 2 * (p - 1);
        bytes = 2 * (p - 1) * mb(n);
        return;
    }
    uint64_t q = 1, levels = 0;
    while (2 * q <= p) q *= 2, ++levels;
    const uint64_t padded = (n + q - 1) / q * q, slice = padded / q, extra = p - q;
    steps = 2 * levels + (extra ? 2 : 0);
    bytes = extra * mb(padded) + extra * q * mb(slice);
    for (uint64_t k = 0, pieces = p, len = padded / 2; k < levels; ++k, pieces *= 2, len /= 2)
        bytes += pieces * mb(len);
    for (uint64_t k = 0, held = 1; k < levels; ++k, held *= 2) bytes += q * held * mb(slice);
}

AllReduceOutcome run_schedule(const RankSet& rs, double* rel_l2) {
    if (rs.inputs.size() < 2) fail(ErrorCode::Usage, "allreduce needs at least 2 ranks");
    const size_t n = rs.inputs[0].size();
    if (n == 0) fail(ErrorCode::Input, "input tensor is empty");
    for (const auto& in : rs.inputs)
        if (in.size() != n) fail(ErrorCode::Input, "all rank inputs must have the same length");
    validate_config(rs.codec);
    const size_t p = rs.inputs.size();
    std::vector<float> flat(p * n);
    for (size_t r = 0; r < p; ++r) std::copy(rs.inputs[r].begin(), rs.inputs[r].end(), flat.begin() + r * n);
    AllReduceOutcome out;
    out.result.resize(n);
    out.exact.resize(n);
    const taco_config c = to_c(rs.codec);
    check(taco_allreduce_schedule_host(context(), &c, static_cast<int>(rs.algorithm), flat.data(),
                                       static_cast<uint32_t>(p), n, out.result.data(), out.exact.data(), rel_l2));
    schedule_shape(rs, out.compress_invocations, out.bytes_on_wire);
    return out;
}

}  // namespace

AllReduceOutcome allreduce(const RankSet& rs) { return run_schedule(rs, nullptr); }

// collective.cpp:270-294: the three schedules on the same inputs; the relative L2 of each
// comes from the device error report of its result against the exact sum.
std::vector<AlgorithmRow> error_vs_frequency(const RankSet& rs) {
    std::vector<AlgorithmRow> rows;
    for (Algorithm a : {Algorithm::TwoShot, Algorithm::Ring, Algorithm::Tree}) {
        RankSet run = rs;
        run.algorithm = a;
        AlgorithmRow row{a, 0.0, 0, 0};
        const AllReduceOutcome o = run_schedule(run, &row.relative_l2);
        row.compress_invocations = o.compress_invocations;
        row.bytes_on_wire = o.bytes_on_wire;
        rows.push_back(row);
    }
    const uint64_t fewest = std::min(rows[1].compress_invocations, rows[2].compress_invocations);
    if (rows[0].compress_invocations > fewest) throw std::logic_error("twoshot must use the fewest compressed steps");
    return rows;
}

}  // namespace taco
