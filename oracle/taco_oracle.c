/*
 * taco_oracle.c -- plain-C, double-precision restatement of the TACO codec path.
 *
 * TEST INFRASTRUCTURE ONLY: used by tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py as the checker.  The product
 * (paper_2604_24088_b200/) never links or calls it.
 *
 * Every function cites the reference lines it restates (paths relative to
 * /root/reference/proj).  Parity of this file is pinned by tests/test_oracle.py
 * against the reference's known-answer tests and against fixtures produced by
 * the reference itself (oracle/_ref, oracle/make_golden.py).
 */
#include "taco_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local const char* g_err = "";

const char* tor_last_error(void) { return g_err; }

static int fail_with(int code, const char* msg) {
    g_err = msg;
    return code;
}

/* ---------------------------------------------------------------- fp8 --- */

/* format constants: src/fp8.cpp:11-12 (E4M3: 4/3/bias 7/448/no-inf,
 * E5M2: 5/2/bias 15/57344/inf) */
typedef struct {
    int ebits, mbits, bias;
    float qmax;
    int has_inf;
} fmt_t;

static const fmt_t kFmt[2] = {{4, 3, 7, 448.0f, 0}, {5, 2, 15, 57344.0f, 1}};

static float fmt_qmax(int format) { return kFmt[format ? 1 : 0].qmax; }

/* decode table: src/fp8.cpp:16-40 (sign / exponent / fraction split, subnormal
 * f*2^(1-bias-m), E5M2 inf/NaN at emax, E4M3 NaN only at S.1111.111) */
void tor_fp8_decode_table(int format, float out[256]) {
    const fmt_t* f = &kFmt[format ? 1 : 0];
    const int emax = (1 << f->ebits) - 1;
    const int fmask = (1 << f->mbits) - 1;
    for (int code = 0; code < 256; ++code) {
        const int neg = code >> 7;
        const int e = (code >> f->mbits) & emax;
        const int frac = code & fmask;
        float v;
        if (e == 0) {
            v = ldexpf((float)frac, 1 - f->bias - f->mbits);
        } else if (e == emax && f->has_inf) {
            v = frac == 0 ? INFINITY : NAN;
        } else if (e == emax && !f->has_inf && frac == fmask) {
            v = NAN;
        } else {
            v = ldexpf(1.0f + (float)frac / (float)(1 << f->mbits), e - f->bias);
        }
        out[code] = neg ? -v : v;
    }
}

/* encode: src/fp8.cpp:66-91.  NaN -> 0x7F; |x| > q_max saturates to the top
 * finite code (0x7E / 0x7B, :43-45); subnormal range rounds |x|/step with
 * nearbyint (ties-to-even) in double; normal range re-biases the fp32 exponent
 * and rounds the mantissa to m bits, ties to even, carry into the exponent. */
uint8_t tor_fp8_encode(float x, int format) {
    const fmt_t* f = &kFmt[format ? 1 : 0];
    if (isnan(x)) return 0x7F;
    uint32_t bits;
    memcpy(&bits, &x, 4);
    const uint8_t sign = (uint8_t)((bits >> 24) & 0x80u);
    const float ax = fabsf(x);
    if (ax > f->qmax) return (uint8_t)(sign | (f->has_inf ? 0x7B : 0x7E));
    const float min_normal = ldexpf(1.0f, 1 - f->bias);
    if (ax < min_normal) {
        const double step = ldexp(1.0, 1 - f->bias - f->mbits);
        const int q = (int)nearbyint((double)ax / step);
        return (uint8_t)(sign | q);
    }
    uint32_t a;
    memcpy(&a, &ax, 4);
    a -= (uint32_t)(127 - f->bias) << 23;
    const int shift = 23 - f->mbits;
    a += ((1u << (shift - 1)) - 1u) + ((a >> shift) & 1u);
    return (uint8_t)(sign | (uint8_t)(a >> shift));
}

/* ---------------------------------------------------------- transform --- */

static int is_pow2(size_t b) { return b != 0 && (b & (b - 1)) == 0; }

/* src/transform.cpp:41-58: unnormalised butterflies with stride h = 1, 2, ...,
 * n/2 (natural / Sylvester order), then one 1/sqrt(n) pass, all in double. */
int tor_fwht_inplace(double* v, size_t n) {
    if (!is_pow2(n)) return fail_with(TOR_CONFIG, "transform length must be a power of two");
    for (size_t h = 1; h < n; h <<= 1) {
        for (size_t base = 0; base < n; base += 2 * h) {
            for (size_t j = base; j < base + h; ++j) {
                const double lo = v[j], hi = v[j + h];
                v[j] = lo + hi;
                v[j + h] = lo - hi;
            }
        }
    }
    const double norm = 1.0 / sqrt((double)n);
    for (size_t i = 0; i < n; ++i) v[i] *= norm;
    return TOR_OK;
}

/* -------------------------------------------------------------- codec --- */

/* src/transform.cpp:13-20 and src/codec.cpp:189-197 (same messages, same order) */
int tor_validate_config(const tor_cfg* cfg) {
    const size_t b = cfg->block_size;
    if (!is_pow2(b)) return fail_with(TOR_CONFIG, "block size must be a power of two");
    if (b < 2 || b > 32768) return fail_with(TOR_CONFIG, "block size must be between 2 and 32768");
    if (!(cfg->target_energy > 0.0f) || !isfinite(cfg->target_energy))
        return fail_with(TOR_CONFIG, "target energy must be positive and finite");
    if (!(cfg->stability_epsilon > 0.0f) || !isfinite(cfg->stability_epsilon))
        return fail_with(TOR_CONFIG, "stability epsilon must be positive and finite");
    return TOR_OK;
}

/* src/codec.cpp:208-254 (driver) + :45-62 (rotate_block) + :64-76
 * (compress_block_taco).  Per block k: zero-padded load (:23-28); sequential
 * double sum of squares over all B slots; sigma = sqrt(acc/B + (double)eps)
 * rounded to float; alpha = tau/sigma in float (:206); v *= alpha in double;
 * FWHT; s = zmax==0 ? 1 : float(zmax/q_max); code = enc(float(z/double(s))). */
int tor_compress(const float* x, size_t n, const tor_cfg* cfg, uint8_t* codes, float* alpha,
                 float* scale) {
    int rc = tor_validate_config(cfg);
    if (rc) return rc;
    if (n == 0) return fail_with(TOR_INPUT, "input tensor is empty");
    for (size_t i = 0; i < n; ++i)
        if (!isfinite(x[i])) return fail_with(TOR_INPUT, "input tensor contains NaN or Inf");

    const size_t b = cfg->block_size;
    const size_t blocks = (n + b - 1) / b;
    const double qmax = (double)fmt_qmax(cfg->format);
    double* v = (double*)malloc(b * sizeof(double));
    for (size_t k = 0; k < blocks; ++k) {
        const size_t begin = k * b;
        const size_t valid = n - begin < b ? n - begin : b;
        for (size_t i = 0; i < b; ++i) v[i] = i < valid ? (double)x[begin + i] : 0.0;
        double acc = 0.0;
        for (size_t i = 0; i < b; ++i) acc += v[i] * v[i];
        const float sigma = (float)sqrt(acc / (double)b + (double)cfg->stability_epsilon);
        const float a = cfg->target_energy / sigma;
        for (size_t i = 0; i < b; ++i) v[i] *= (double)a;
        tor_fwht_inplace(v, b);
        double zmax = 0.0;
        for (size_t i = 0; i < b; ++i) zmax = fabs(v[i]) > zmax ? fabs(v[i]) : zmax;
        const float s = zmax == 0.0 ? 1.0f : (float)(zmax / qmax);
        for (size_t i = 0; i < b; ++i)
            codes[begin + i] = tor_fp8_encode((float)(v[i] / (double)s), cfg->format);
        alpha[k] = a;
        scale[k] = s;
    }
    free(v);
    return TOR_OK;
}

/* src/codec.cpp:264-296 (checks) + :144-155 (Taco block): z = double(table[c]) *
 * double(s); FWHT in double; out = float(z/double(alpha)) for the valid prefix. */
int tor_decompress(const uint8_t* codes, const float* alpha, const float* scale, size_t n,
                   const tor_cfg* cfg, float* out) {
    const size_t b = cfg->block_size;
    if (!is_pow2(b)) return fail_with(TOR_CONFIG, "block size must be a power of two");
    if (b < 2 || b > 32768) return fail_with(TOR_CONFIG, "block size must be between 2 and 32768");
    if (n == 0) return fail_with(TOR_CORRUPT, "compressed tensor declares zero elements");
    const size_t blocks = (n + b - 1) / b;
    for (size_t k = 0; k < blocks; ++k) {
        if (!isfinite(alpha[k]) || !isfinite(scale[k]) || scale[k] == 0.0f || alpha[k] == 0.0f)
            return fail_with(TOR_CORRUPT, "block scalars must be finite and nonzero");
    }
    float table[256];
    tor_fp8_decode_table(cfg->format, table);
    double* v = (double*)malloc(b * sizeof(double));
    for (size_t k = 0; k < blocks; ++k) {
        const size_t begin = k * b;
        const size_t valid = n - begin < b ? n - begin : b;
        for (size_t i = 0; i < b; ++i) v[i] = (double)table[codes[begin + i]] * (double)scale[k];
        tor_fwht_inplace(v, b);
        for (size_t i = 0; i < valid; ++i) out[begin + i] = (float)(v[i] / (double)alpha[k]);
    }
    free(v);
    return TOR_OK;
}

/* ---------------------------------------------------------- collective --- */

/* one rank-to-rank message in bytes: src/serialize.cpp:172-177 */
static uint64_t archive_size(const tor_cfg* cfg, uint64_t n) {
    const uint64_t b = cfg->block_size;
    return 22 + ((n + b - 1) / b) * (b + 8);
}

/* src/collective.cpp:24-33 (validation), :36-41 (exact sum), :75-111 (two-shot):
 * shard = ceil(n/p), inputs zero-padded to shard*p; every rank compresses every
 * shard slice; owner s sums decompress(shard s of rank r) in fp32 for r = 0..p-1
 * ascending (own shard through the codec too); compress(acc) then decompress
 * once; result truncated to n.  bytes = 2 * p(p-1) * archive(shard). */
int tor_allreduce_twoshot(const float* inputs, size_t p, size_t n, const tor_cfg* cfg,
                          float* result, float* exact, float* stage1, uint64_t* bytes_on_wire) {
    if (p < 2) return fail_with(TOR_USAGE, "allreduce needs at least 2 ranks");
    if (n == 0) return fail_with(TOR_INPUT, "input tensor is empty");
    int rc = tor_validate_config(cfg);
    if (rc) return rc;

    const size_t b = cfg->block_size;
    const size_t shard = (n + p - 1) / p;
    const size_t m = (shard + b - 1) / b; /* blocks per shard message */
    uint8_t* codes = (uint8_t*)malloc(p * p * m * b);
    float* al = (float*)malloc(p * p * m * sizeof(float));
    float* sc = (float*)malloc(p * p * m * sizeof(float));
    float* slice = (float*)malloc(shard * sizeof(float));
    float* acc = (float*)malloc(shard * sizeof(float));
    float* part = (float*)malloc(shard * sizeof(float));
    uint8_t* c2 = (uint8_t*)malloc(m * b);
    float* al2 = (float*)malloc(m * sizeof(float));
    float* sc2 = (float*)malloc(m * sizeof(float));

    /* phase 1: rank r compresses shard s into message (r, s) */
    for (size_t r = 0; r < p && rc == TOR_OK; ++r) {
        for (size_t s = 0; s < p && rc == TOR_OK; ++s) {
            for (size_t i = 0; i < shard; ++i) {
                const size_t g = s * shard + i;
                slice[i] = g < n ? inputs[r * n + g] : 0.0f;
            }
            const size_t msg = r * p + s;
            rc = tor_compress(slice, shard, cfg, codes + msg * m * b, al + msg * m, sc + msg * m);
        }
    }
    /* owner reduce (ascending rank, fp32), re-encode, every rank decodes it */
    for (size_t s = 0; s < p && rc == TOR_OK; ++s) {
        for (size_t r = 0; r < p && rc == TOR_OK; ++r) {
            const size_t msg = r * p + s;
            float* dst = r == 0 ? acc : part;
            rc = tor_decompress(codes + msg * m * b, al + msg * m, sc + msg * m, shard, cfg, dst);
            if (r > 0)
                for (size_t i = 0; i < shard; ++i) acc[i] += part[i];
        }
        if (rc) break;
        if (stage1) memcpy(stage1 + s * shard, acc, shard * sizeof(float));
        rc = tor_compress(acc, shard, cfg, c2, al2, sc2);
        if (rc) break;
        rc = tor_decompress(c2, al2, sc2, shard, cfg, part);
        for (size_t i = 0; i < shard; ++i) {
            const size_t g = s * shard + i;
            if (g < n) result[g] = part[i];
        }
    }
    if (rc == TOR_OK && exact) {
        for (size_t i = 0; i < n; ++i) exact[i] = inputs[i];
        for (size_t r = 1; r < p; ++r)
            for (size_t i = 0; i < n; ++i) exact[i] += inputs[r * n + i];
    }
    if (bytes_on_wire) *bytes_on_wire = 2ull * p * (p - 1) * archive_size(cfg, shard);
    free(codes); free(al); free(sc); free(slice); free(acc); free(part);
    free(c2); free(al2); free(sc2);
    return rc;
}

/* ----------------------------------------------------------------- rng --- */

/* src/rng.cpp:9-67: splitmix64 seeding, xoshiro256++, 53-bit doubles,
 * Marsaglia polar normals with one cached value, rejection-sampled next_below,
 * Fisher-Yates shuffle (rng.hpp:19-25). */
typedef struct {
    uint64_t s[4];
    int has_cached;
    double cached;
} rng_t;

static uint64_t splitmix(uint64_t* x) {
    uint64_t z = (*x += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

static uint64_t rotl64(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }

static void rng_init(rng_t* r, uint64_t seed) {
    uint64_t sm = seed;
    for (int i = 0; i < 4; ++i) r->s[i] = splitmix(&sm);
    r->has_cached = 0;
    r->cached = 0.0;
}

static uint64_t rng_u64(rng_t* r) {
    uint64_t* s = r->s;
    const uint64_t out = rotl64(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return out;
}

static uint64_t rng_below(rng_t* r, uint64_t n) {
    const uint64_t threshold = (0 - n) % n;
    for (;;) {
        const uint64_t v = rng_u64(r);
        if (v >= threshold) return v % n;
    }
}

static double rng_unit(rng_t* r) { return (double)(rng_u64(r) >> 11) * 0x1.0p-53; }

static double rng_normal(rng_t* r) {
    if (r->has_cached) {
        r->has_cached = 0;
        return r->cached;
    }
    for (;;) {
        const double u = 2.0 * rng_unit(r) - 1.0;
        const double w = 2.0 * rng_unit(r) - 1.0;
        const double q = u * u + w * w;
        if (q > 0.0 && q < 1.0) {
            const double k = sqrt(-2.0 * log(q) / q);
            r->cached = w * k;
            r->has_cached = 1;
            return u * k;
        }
    }
}

/* the reference tests' gaussian(n, seed, sigma) helper
 * (tests/test_codec.cpp:19-24; generate() Gaussian kind is sigma = 1,
 * src/analysis.cpp:76-80) */
void tor_gaussian(size_t n, uint64_t seed, double sigma, float* out) {
    rng_t r;
    rng_init(&r, seed);
    for (size_t i = 0; i < n; ++i) out[i] = (float)(sigma * rng_normal(&r));
}

/* src/analysis.cpp:81-94: dense block then tail block, then shuffle */
int tor_mixture(size_t n, uint64_t seed, double dense_sigma, double tail_sigma,
                double tail_fraction, float* out) {
    if (n == 0) return fail_with(TOR_CONFIG, "synthetic tensor length must be positive");
    if (!(tail_fraction >= 0.0 && tail_fraction <= 1.0))
        return fail_with(TOR_CONFIG, "tail fraction must be in [0, 1]");
    if (!(dense_sigma > 0.0) || !(tail_sigma > 0.0))
        return fail_with(TOR_CONFIG, "mixture sigmas must be positive");
    rng_t r;
    rng_init(&r, seed);
    const size_t n_tail = (size_t)llround(tail_fraction * (double)n);
    const size_t n_dense = n - n_tail;
    for (size_t i = 0; i < n_dense; ++i) out[i] = (float)(dense_sigma * rng_normal(&r));
    for (size_t i = n_dense; i < n; ++i) out[i] = (float)(tail_sigma * rng_normal(&r));
    for (size_t i = n; i > 1; --i) {
        const size_t j = (size_t)rng_below(&r, i);
        const float t = out[i - 1];
        out[i - 1] = out[j];
        out[j] = t;
    }
    return TOR_OK;
}
