/*
 * taco_oracle.h -- CPU restatement of the TACO codec path, TEST INFRASTRUCTURE ONLY.
 *
 * This header and taco_oracle.c restate, in plain C and double precision, the
 * reference algorithm of arxiv/paper_2604_24088 (proj/src/{fp8,transform,codec,
 * collective,rng,analysis}.cpp) so that tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg can check the B200 path against it.  Nothing in
 * paper_2604_24088_b200/ may link, import or call this code.
 *
 * Parity of this restatement is pinned (tests/test_oracle.py) against
 *   (1) the golden vectors / known-answer tests of the reference's own tests,
 *   (2) the reference itself compiled from /root/reference into oracle/_ref/
 *       (fixtures under tests/golden/ are generated from it by
 *       oracle/make_golden.py).
 */
#ifndef TACO_ORACLE_H
#define TACO_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes mirror taco::ErrorCode (proj/include/taco/error.hpp:10-16), +1 */
enum { TOR_OK = 0, TOR_USAGE = 1, TOR_CONFIG = 2, TOR_INPUT = 3, TOR_IO = 4, TOR_CORRUPT = 5 };

typedef struct {
    uint32_t block_size;      /* B, power of two in [2, 32768] */
    float target_energy;      /* tau */
    float stability_epsilon;  /* eps */
    int format;               /* 0 = E4M3, 1 = E5M2 */
} tor_cfg;

const char* tor_last_error(void);

/* fp8 (proj/src/fp8.cpp) */
uint8_t tor_fp8_encode(float x, int format);
void tor_fp8_decode_table(int format, float out[256]);

/* transform (proj/src/transform.cpp) */
int tor_fwht_inplace(double* v, size_t n);

/* codec, Taco kind (proj/src/codec.cpp) */
int tor_validate_config(const tor_cfg* cfg);
int tor_compress(const float* x, size_t n, const tor_cfg* cfg, uint8_t* codes, float* alpha,
                 float* scale);
int tor_decompress(const uint8_t* codes, const float* alpha, const float* scale, size_t n,
                   const tor_cfg* cfg, float* out);

/* collective, two-shot schedule (proj/src/collective.cpp:75-111).
 * inputs: P*n floats, rank-major.  result/exact: n floats.  stage1 (optional,
 * may be NULL): P*shard floats = the fp32 ascending-rank sums before re-encode. */
int tor_allreduce_twoshot(const float* inputs, size_t p, size_t n, const tor_cfg* cfg,
                          float* result, float* exact, float* stage1, uint64_t* bytes_on_wire);

/* synthetic inputs (proj/src/rng.cpp, proj/src/analysis.cpp:70-95) */
void tor_gaussian(size_t n, uint64_t seed, double sigma, float* out);
int tor_mixture(size_t n, uint64_t seed, double dense_sigma, double tail_sigma,
                double tail_fraction, float* out);

#ifdef __cplusplus
}
#endif
#endif
