// taco_r2.cuh -- K1 "r2": the register geometry of taco_kernels.cuh (E = 64 values per
// lane, L = B/64 lanes per block, two shuffle stages at B = 256) with the per-tile
// overheads that the r1a/t1 profiles exposed taken out:
//
//   * staging through the TMA engine: one cp.async.bulk per 2048-element warp tile into a
//     D-deep per-warp ring, completion on an mbarrier (no per-lane LDGSTS / address math);
//   * bf16 unpack fused into the first butterfly: add/sub.rn.f32.bf16 (FHADD.BF16) take
//     the low half straight from the packed word, one rounding, exact operands;
//   * sum of squares without the XU pipe when TACO_SUMSQ == 1: fma.rn.f32.bf16 (FHFMA)
//     in 8 fp32 chains, alpha within 5e-7 relative (north-star bound 1e-6).  TACO_SUMSQ
//     == 0 keeps the exact fp64 sum (cvt.f64.bf16 + DFMA), alpha bit-exact;
//   * branch-free per-block scalars when TACO_FAST_SCALARS == 1: alpha = tau / sigma as a
//     double Newton quotient (correctly rounded to float: the exact quotient of two
//     24-bit floats is >= 2^-48 relative away from a float midpoint), s = zmax * (1/qmax),
//     k = g / s by a Newton reciprocal (k only feeds the cvt);
//   * overflow handled by a rare redo: the fast path never pre-scales; a tile whose
//     butterfly overflowed fp32 (only possible when the block sum of squares >= 2^160) is
//     recomputed with the exact power-of-two pre-scale of the register kernels.
#pragma once

#include "taco_kernels.cuh"
#include "taco_tile.cuh"

#ifndef TACO_SUMSQ
#define TACO_SUMSQ 0
#endif
#ifndef TACO_FAST_SCALARS
#define TACO_FAST_SCALARS 1
#endif
#ifndef TACO_FHADD
#define TACO_FHADD 0
#endif
#ifndef TACO_R2_STAGES
#define TACO_R2_STAGES 3
#endif

namespace taco_dev {
namespace r2 {

using tile::add_bf16;
using tile::bf16_to_f64;
using tile::bulk_g2s;
using tile::fence_mbar_init;
using tile::fence_proxy_async;
using tile::mbar_arrive;
using tile::mbar_arrive_tx;
using tile::mbar_init;
using tile::mbar_wait;
using tile::sub_bf16;

constexpr int kWarps = 4;

__device__ __forceinline__ float fma_bf16(uint32_t h16, float c) {  // h*h + c, h = bf16
    float d;
    asm("fma.rn.f32.bf16 %0, %1, %1, %2;" : "=f"(d) : "h"((unsigned short)h16), "f"(c));
    return d;
}

// double reciprocal, Newton from MUFU.RCP64H; ITER = 1 -> ~2^-40, 2 -> full precision
template <int ITER>
__device__ __forceinline__ double rcp_nr(double d) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
#pragma unroll
    for (int i = 0; i < ITER; ++i) {
        const double e = fma(-d, r, 1.0);
        r = fma(r, e, r);
    }
    return r;
}

// sigma = float(sqrt(acc/B + eps)), alpha = tau / sigma (codec.cpp:50-54)
__device__ __forceinline__ float alpha_of(double ss, const CodecConsts& c) {
#if TACO_FAST_SCALARS
    const float sigma = __double2float_rn(__dsqrt_rn(fma(ss, c.inv_b, (double)c.eps)));
    return __double2float_rn((double)c.tau * rcp_nr<2>((double)sigma));
#else
    return block_alpha(ss, c);
#endif
}

// s = float(zmax / qmax) and the multiplier k with Z/s = y * k (see block_scale)
__device__ __forceinline__ void scale_of(double ymax, float alpha, float p2, const CodecConsts& c, float& s,
                                         double& k) {
#if TACO_FAST_SCALARS
    const double g = (double)alpha / (double)p2 * c.norm;  // p2 is a power of two: exact
    const double zmax = ymax * g;
    s = zmax == 0.0 ? 1.0f : __double2float_rn(zmax * c.inv_qmax);
    k = g * rcp_nr<1>((double)s);
#else
    block_scale(ymax, alpha, p2, c, s, k);
#endif
}

template <int E2>
__device__ __forceinline__ void mul_k(float2 (&w)[E2], double k) {
    const bool in_range = fabs(k) < 0x1p126 && (k == 0.0 || fabs(k) >= 0x1p-126);
    if (__all_sync(kFull, in_range)) scale2<E2>(w, (float)k);
    else mul_wide<E2>(w, k);
}

template <int B, typename TIn>
struct Cfg {
    using Gm = Geo<B, 64, 8>;
    static constexpr int E = Gm::E, E2 = Gm::E2, L = Gm::L, G = Gm::G, NV = Gm::NV;
    static constexpr int TILE = G * B;  // elements per warp tile
    static constexpr int D = TACO_R2_STAGES;
    static constexpr int STAGE = TILE * (int)sizeof(TIn);
    static constexpr int WORDS = E * (int)sizeof(TIn) / 4;  // raw 32-bit words per lane
    static constexpr size_t SMEM = (size_t)kWarps * D * (STAGE + 8 + 4);
};

// raw words of lane (g, q): vector j (8 elements) at block position (j*L + q)*8
template <int B, typename TIn>
__device__ __forceinline__ void load_raw(const unsigned char* st, int g, int q, uint32_t (&raw)[Cfg<B, TIn>::WORDS]) {
    using C = Cfg<B, TIn>;
    constexpr int WPV = 8 * (int)sizeof(TIn) / 4;  // words per 8-element vector
    const TIn* blk = reinterpret_cast<const TIn*>(st) + g * B;
#pragma unroll
    for (int j = 0; j < C::NV; ++j) {
        const uint4* p = reinterpret_cast<const uint4*>(blk + (j * C::L + q) * 8);
#pragma unroll
        for (int h = 0; h < WPV / 4; ++h) {
            const uint4 u = p[h];
            raw[j * WPV + 4 * h + 0] = u.x;
            raw[j * WPV + 4 * h + 1] = u.y;
            raw[j * WPV + 4 * h + 2] = u.z;
            raw[j * WPV + 4 * h + 3] = u.w;
        }
    }
}

// lane-partial sum of squares of the raw words: exact fp64 (x^2 exact in double) ...
template <int B, typename TIn>
__device__ __forceinline__ double lane_sumsq_f64(const uint32_t (&raw)[Cfg<B, TIn>::WORDS]) {
    using C = Cfg<B, TIn>;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < C::WORDS; ++i) {
        if constexpr (sizeof(TIn) == 2) {
            const double d0 = bf16_to_f64(raw[i] & 0xffffu), d1 = bf16_to_f64(raw[i] >> 16);
            acc[(2 * i) & 3] = fma(d0, d0, acc[(2 * i) & 3]);
            acc[(2 * i + 1) & 3] = fma(d1, d1, acc[(2 * i + 1) & 3]);
        } else {
            const double d = (double)__uint_as_float(raw[i]);
            acc[i & 3] = fma(d, d, acc[i & 3]);
        }
    }
    return (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

// ... or fp32 (FHFMA.BF16 / FFMA, 8 chains): relative error <= ~12 u
template <int B, typename TIn>
__device__ __forceinline__ float lane_sumsq_f32(const uint32_t (&raw)[Cfg<B, TIn>::WORDS]) {
    using C = Cfg<B, TIn>;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if constexpr (sizeof(TIn) == 2) {
#pragma unroll
        for (int i = 0; i < C::WORDS; ++i) {
            acc[(2 * i) & 7] = fma_bf16(raw[i] & 0xffffu, acc[(2 * i) & 7]);
            acc[(2 * i + 1) & 7] = fma_bf16(raw[i] >> 16, acc[(2 * i + 1) & 7]);
        }
    } else {
#pragma unroll
        for (int i = 0; i < C::WORDS; ++i) {
            const float x = __uint_as_float(raw[i]);
            acc[i & 7] = fmaf(x, x, acc[i & 7]);
        }
    }
    return ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
}

template <int B, typename TIn>
__device__ __forceinline__ double lane_sumsq(const uint32_t (&raw)[Cfg<B, TIn>::WORDS]) {
#if TACO_SUMSQ == 1
    // fp32 squares are exact for bf16 inputs; fall back to fp64 where fp32 could overflow
    // (|x| >= 2^50) or lose the squares to its subnormal range (|x| < 2^-50)
    const float sl = lane_sumsq_f32<B, TIn>(raw);
    if (__any_sync(kFull, !(sl < 0x1p100f) || (sl > 0.0f && sl < 0x1p-100f))) return lane_sumsq_f64<B, TIn>(raw);
    return (double)sl;
#else
    return lane_sumsq_f64<B, TIn>(raw);
#endif
}

// first butterfly (position bit 0) straight from the raw words, optional exact pre-scale
template <int B, typename TIn>
__device__ __forceinline__ void pair_from_raw(const uint32_t (&raw)[Cfg<B, TIn>::WORDS], float2 (&w)[Cfg<B, TIn>::E2],
                                              float p2, bool scaled) {
    using C = Cfg<B, TIn>;
#pragma unroll
    for (int i = 0; i < C::E2; ++i) {
        if constexpr (sizeof(TIn) == 2) {
            if (!scaled && TACO_FHADD) {
                const float x1 = __uint_as_float(raw[i] & 0xffff0000u);
                w[i] = make_float2(add_bf16(raw[i] & 0xffffu, x1), sub_bf16(raw[i] & 0xffffu, x1));
            } else if (!scaled) {
                const float x0 = __uint_as_float(raw[i] << 16), x1 = __uint_as_float(raw[i] & 0xffff0000u);
                w[i] = make_float2(x0 + x1, x0 - x1);
            } else {
                const float x0 = __uint_as_float(raw[i] << 16) * p2, x1 = __uint_as_float(raw[i] & 0xffff0000u) * p2;
                w[i] = make_float2(x0 + x1, x0 - x1);
            }
        } else {
            float x0 = __uint_as_float(raw[2 * i]), x1 = __uint_as_float(raw[2 * i + 1]);
            if (scaled) {
                x0 *= p2;
                x1 *= p2;
            }
            w[i] = make_float2(x0 + x1, x0 - x1);
        }
    }
}

// butterflies over every position bit except bit 0 (register bits, then lane bits) --
// the stage order of fwht() in taco_device.cuh
template <int L, int E2>
__device__ __forceinline__ void fwht_rest(float2 (&w)[E2], int q) {
    const float2 neg1 = make_float2(-1.0f, -1.0f);
#pragma unroll
    for (int h = 1; h < E2; h <<= 1) {
#pragma unroll
        for (int i = 0; i < E2; ++i) {
            if ((i & h) == 0) {
                const float2 a = w[i], cc = w[i + h];
                w[i] = __fadd2_rn(a, cc);
                w[i + h] = __ffma2_rn(cc, neg1, a);
            }
        }
    }
#pragma unroll
    for (int m = 1; m < L; m <<= 1) {
        const float s = (q & m) ? -1.0f : 1.0f;
        const float2 sgn = make_float2(s, s);
#pragma unroll
        for (int i = 0; i < E2; ++i) {
            const float2 o = make_float2(__shfl_xor_sync(kFull, w[i].x, m), __shfl_xor_sync(kFull, w[i].y, m));
            w[i] = __ffma2_rn(w[i], sgn, o);
        }
    }
}

template <int L, int E2>
__device__ __forceinline__ float group_absmax(const float2 (&w)[E2]) {
    float m[E2];
#pragma unroll
    for (int i = 0; i < E2; ++i) m[i] = fmaxf(fabsf(w[i].x), fabsf(w[i].y));
#pragma unroll
    for (int h = 1; h < E2; h <<= 1)
#pragma unroll
        for (int i = 0; i + h < E2; i += 2 * h) m[i] = fmaxf(m[i], m[i + h]);
    float v = m[0];
#pragma unroll
    for (int o = 1; o < L; o <<= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, o));
    return v;
}

template <int B, typename TIn>
__device__ __forceinline__ void fill_slow(unsigned char* st, const TIn* __restrict__ x, const ShardArgs& a,
                                          uint64_t p, uint64_t kk0, int lane) {
    using C = Cfg<B, TIn>;
    TIn* d = reinterpret_cast<TIn*>(st);
    for (int i = lane; i < C::TILE; i += 32) {
        const uint64_t kk = kk0 + (uint64_t)(i / B);
        const int pos = i % B;
        float v = 0.0f;
        if (kk < a.nblk) {
            const uint64_t k = a.blk0 + kk;
            const int valid =
                clamp_valid((int64_t)a.S - (int64_t)(k * B), (int64_t)a.n - (int64_t)(p * a.S + k * B), B);
            if (pos < valid) v = to_f32(x[p * a.S + k * B + pos]);
        }
        store_one(d + i, v);
    }
}

// Cold path: the block again, straight from global memory, with the exact pre-scale
// p2 = 2^floor(log2 alpha) where its sum of squares reached 2^160 (no fp32 overflow is
// then possible), quantised and stored.  Out of line so the hot loop's registers are
// untouched.
template <int B, typename TIn>
__device__ __noinline__ void redo_tile(const TIn* __restrict__ x, ShardArgs a, uint64_t p, uint64_t kk0, int g,
                                       int q, double ss, float alpha, CodecConsts c, uint8_t* m, uint64_t kk) {
    using C = Cfg<B, TIn>;
    using Gm = typename C::Gm;
    constexpr int L = C::L;
    const bool huge = !(ss < 0x1p160);
    const float p2 = huge ? pow2_near(alpha) : 1.0f;
    float2 w[C::E2];
    int valid = 0;
    if (kk < a.nblk) {
        const uint64_t k = a.blk0 + kk;
        valid = clamp_valid((int64_t)a.S - (int64_t)(k * B), (int64_t)a.n - (int64_t)(p * a.S + k * B), B);
    }
    const TIn* src = x + (p * a.S + (a.blk0 + kk) * B);
#pragma unroll
    for (int j = 0; j < C::NV; ++j)
#pragma unroll
        for (int r = 0; r < 8; r += 2) {
            const int pos = Gm::pos(j, q) + r;
            const float x0 = pos < valid ? to_f32(src[pos]) * p2 : 0.0f;
            const float x1 = pos + 1 < valid ? to_f32(src[pos + 1]) * p2 : 0.0f;
            w[j * 4 + r / 2] = make_float2(x0 + x1, x0 - x1);
        }
    fwht_rest<L, C::E2>(w, q);
    const float ymax = group_absmax<L, C::E2>(w);
    float s;
    double k;
    scale_of((double)ymax, alpha, p2, c, s, k);
    mul_wide<C::E2>(w, k);
    if (m) {
#pragma unroll
        for (int j = 0; j < C::NV; ++j) store_codes<0, 8>(m + kk * B + Gm::pos(j, q), &w[j * 4]);
        if (q == 0) {
            *reinterpret_cast<float2*>(m + a.scal_off + kk * 8) = make_float2(alpha, s);
            if (!isfinite(ss) || !isfinite(ymax)) raise_flag(a.flags, 1);
        }
    }
}

// Work distribution: tiles are claimed dynamically from a per-launch counter (one
// atomicAdd per tile per warp), so every warp stays busy until the tensor is exhausted
// and the kernel's tail is one tile, not the static round-robin's 4-vs-5-tile imbalance
// (r2 ab1 profile: 20 % of SM cycles idle).  Claims are issued D-1 tiles ahead together
// with the TMA fetch; the claimed index travels to the consumer through shared memory.
// Every warp makes exactly D failed claims, so the claim that returns
// ntiles + D * nwarps - 1 is the last one and resets the counter for the next launch.
template <int B, typename TIn>
__global__ void __launch_bounds__(kWarps * 32, 4)
    k_compress_r2(const TIn* __restrict__ x, uint8_t* __restrict__ msgs, ShardArgs a, CodecConsts c, FastDiv tps,
                  uint32_t* __restrict__ counter) {
    using C = Cfg<B, TIn>;
    using Gm = typename C::Gm;
    constexpr int D = C::D, L = C::L, G = C::G;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, q = lane & (L - 1), g = lane / L;
    unsigned char* stage = smem + (size_t)warp * D * C::STAGE;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)kWarps * D * C::STAGE) + warp * D;
    uint32_t* slot_tile = reinterpret_cast<uint32_t*>(smem + (size_t)kWarps * D * (C::STAGE + 8)) + warp * D;
    const uint32_t ntiles = a.P * tps.d;
    const uint32_t last_claim = ntiles + (uint32_t)D * gridDim.x * kWarps - 1;

    // lane 0: claim the next tile for `slot` and start its fetch
    auto refill = [&](int slot) {
        const uint32_t t = atomicAdd(counter, 1u);
        if (t == last_claim) atomicExch(counter, 0u);
        slot_tile[slot] = t;
        if (t < ntiles) {
            const uint32_t p = tps.div(t);
            const uint64_t kk0 = (uint64_t)(t - p * tps.d) * G;
            if (tile_full<B, G>(a, p, kk0)) {
                fence_proxy_async();
                mbar_arrive_tx(&bars[slot], C::STAGE);
                bulk_g2s(stage + slot * C::STAGE, x + (p * a.S + (a.blk0 + kk0) * B), C::STAGE, &bars[slot]);
                return;
            }
        }
        mbar_arrive(&bars[slot]);  // ragged tile (filled by the consumer) or no tile
    };
    if (lane == 0) {
#pragma unroll
        for (int d = 0; d < D; ++d) mbar_init(&bars[d], 1);
        fence_mbar_init();
#pragma unroll
        for (int d = 0; d < D; ++d) refill(d);
    }
    __syncwarp();
    int slot = 0;
    uint32_t par = 0;
    for (;;) {
        mbar_wait(&bars[slot], (par >> slot) & 1);
        par ^= 1u << slot;
        const uint32_t t = slot_tile[slot];
        if (t >= ntiles) break;
        const uint32_t p = tps.div(t);
        const uint64_t kk0 = (uint64_t)(t - p * tps.d) * G;
        unsigned char* st = stage + slot * C::STAGE;
        if (!tile_full<B, G>(a, p, kk0)) {
            fill_slow<B, TIn>(st, x, a, p, kk0, lane);
            __syncwarp();
        }
        uint32_t raw[C::WORDS];
        load_raw<B, TIn>(st, g, q, raw);
        double ss = lane_sumsq<B, TIn>(raw);
#pragma unroll
        for (int o = 1; o < L; o <<= 1) ss += __shfl_xor_sync(kFull, ss, o);
        const float alpha = alpha_of(ss, c);
        float2 w[C::E2];
        pair_from_raw<B, TIn>(raw, w, 1.0f, false);
        __syncwarp();  // every lane has read the slot: refill it
        if (lane == 0) refill(slot);
        fwht_rest<L, C::E2>(w, q);
        const float ymax = group_absmax<L, C::E2>(w);
        const uint64_t kk = kk0 + g;
        uint8_t* m = msgs + p * a.msg_stride;
        // fp32 overflow inside the butterfly (block sum of squares >= 2^160): redo the
        // tile with the exact power-of-two pre-scale, out of line (warp-uniform, rare).
        // The slot was refilled already, so the redo reads the tile from global memory.
        const bool redo = !isfinite(ymax) && isfinite(ss) && !(ss < 0x1p160);
        if (__any_sync(kFull, redo)) {
            redo_tile<B, TIn>(x, a, p, kk0, g, q, ss, alpha, c, kk < a.nblk ? m : nullptr, kk);
        } else {
            float s;
            double k;
            scale_of((double)ymax, alpha, 1.0f, c, s, k);
            mul_k<C::E2>(w, k);
            if (kk < a.nblk) {
#pragma unroll
                for (int j = 0; j < C::NV; ++j) store_codes<0, 8>(m + kk * B + Gm::pos(j, q), &w[j * 4]);
                if (q == 0) {
                    *reinterpret_cast<float2*>(m + a.scal_off + kk * 8) = make_float2(alpha, s);
                    if (!isfinite(ss) || !isfinite(ymax)) raise_flag(a.flags, 1);
                }
            }
        }
        slot = slot + 1 == D ? 0 : slot + 1;
    }
}

}  // namespace r2
}  // namespace taco_dev
