// taco_synth.cpp -- synthetic TP tensors with the reference's exact values, on the host.
//
// The benchmark and the collectives' per-rank inputs must be the values the reference's
// own generator produces ("Generate on the host with the reference's own
// taco::generate, so CPU and GPU see identical values").  The reference draws them from
// one sequential xoshiro256++ stream (proj/src/rng.cpp:21-67) inside taco::generate
// (proj/src/analysis.cpp:70-95); a sequential stream with rejection sampling has no
// parallel decomposition, so this stays a host routine that fills a caller buffer, which
// the caller then uploads once (the data is an input, not part of the timed path).
//
// Bit-exactness against the reference generator is pinned by
// tests/test_abi.py::test_generate_matches_reference.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <utility>

#include "taco_b200.h"

// taco_abi.cu: records the message taco_last_error() returns
extern "C" int taco_set_error(int code, const char* msg);

namespace {

// xoshiro256++ (rng.cpp:27-37) whose four state words come from a splitmix64 walk of the
// seed (rng.cpp:9-25).
class Xoshiro {
  public:
    explicit Xoshiro(uint64_t seed) {
        uint64_t walk = seed;
        for (uint64_t& w : s_) {
            walk += 0x9e3779b97f4a7c15ull;
            uint64_t z = walk;
            z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
            z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
            w = z ^ (z >> 31);
        }
    }
    uint64_t u64() {
        const uint64_t out = rotl(s_[0] + s_[3], 23) + s_[0];
        const uint64_t t = s_[1] << 17;
        s_[2] ^= s_[0];
        s_[3] ^= s_[1];
        s_[1] ^= s_[2];
        s_[0] ^= s_[3];
        s_[2] ^= t;
        s_[3] = rotl(s_[3], 45);
        return out;
    }
    // uniform in [0, n) by rejection of the low remainder band (rng.cpp:39-46)
    uint64_t below(uint64_t n) {
        const uint64_t reject = (0 - n) % n;
        uint64_t r;
        do r = u64();
        while (r < reject);
        return r % n;
    }
    // 53-bit uniform in [0, 1) (rng.cpp:48-50)
    double unit() { return static_cast<double>(u64() >> 11) * 0x1.0p-53; }
    // Marsaglia polar method, the second variate of each accepted pair cached
    // (rng.cpp:52-67)
    double normal() {
        if (spare_ok_) {
            spare_ok_ = false;
            return spare_;
        }
        for (;;) {
            const double u = 2.0 * unit() - 1.0, v = 2.0 * unit() - 1.0;
            const double r2 = u * u + v * v;
            if (!(r2 > 0.0 && r2 < 1.0)) continue;
            const double f = std::sqrt(-2.0 * std::log(r2) / r2);
            spare_ = v * f;
            spare_ok_ = true;
            return u * f;
        }
    }

  private:
    static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
    uint64_t s_[4];
    bool spare_ok_ = false;
    double spare_ = 0.0;
};

}  // namespace

extern "C" int taco_generate_host(int kind, uint64_t n, uint64_t seed, double dense_sigma, double tail_sigma,
                                  double tail_fraction, float* out) {
    // error texts: analysis.cpp:76,83,85
    if (n == 0) return taco_set_error(TACO_ERR_CONFIG, "synthetic tensor length must be positive");
    if (out == nullptr || (kind != 0 && kind != 1)) return taco_set_error(TACO_ERR_USAGE, "bad generate arguments");
    Xoshiro rng(seed);
    if (kind == 0) {  // Gaussian: one N(0,1) draw per element
        for (uint64_t i = 0; i < n; ++i) out[i] = static_cast<float>(rng.normal());
        return TACO_OK;
    }
    if (!(tail_fraction >= 0.0 && tail_fraction <= 1.0))
        return taco_set_error(TACO_ERR_CONFIG, "tail fraction must be in [0, 1]");
    if (!(dense_sigma > 0.0) || !(tail_sigma > 0.0))
        return taco_set_error(TACO_ERR_CONFIG, "mixture sigmas must be positive");
    // near-zero mixture: the dense body first, then the tail, then one Fisher-Yates pass
    const uint64_t tail = static_cast<uint64_t>(std::llround(tail_fraction * static_cast<double>(n)));
    const uint64_t body = n - tail;
    for (uint64_t i = 0; i < n; ++i)
        out[i] = static_cast<float>((i < body ? dense_sigma : tail_sigma) * rng.normal());
    for (uint64_t i = n; i > 1; --i) std::swap(out[i - 1], out[rng.below(i)]);
    return TACO_OK;
}
