// taco_xk.cuh -- "exchange butterfly" TACO kernels for E4M3 at 64 <= B <= 512 (sm_100a).
//
//   K1 k1x   x (bf16|f32)          -> message(s): FP8 codes + (alpha, s)
//   K2 k2x   message(s)            -> y (bf16|f32)
//   K3 k3x   P messages of a shard -> fp32 ascending-rank sum [-> acc_out] -> message
//
// Same operator contract as the register / tile kernels (taco_kernels.cuh, taco_tile.cuh):
// codec.cpp:45-76 (rotate_block + compress_block_taco), :144-155 (decompress_block),
// collective.cpp:95-104 (the owner's reduce + re-encode).  What changes is how a block's
// Walsh-Hadamard butterfly is spread over a warp, to cut instructions per element:
//
// * Geometry.  A block of B = 64 L elements is held by L lanes, 64 fp32 values per lane in
//   32 float2 pairs (pair index i, bits i0..i4 = "slot" bits 1..5; slot bit 0 is the pair
//   half).  A warp carries G = 32 / L blocks.
// * Pair-bit stage fused into the unpack.  The butterfly over the bit that lives inside a
//   pair cannot use the packed FP32 pipe.  It is done while unpacking: (a + b, a - b) of
//   the two bf16 halves of one input word by two sm_100 mixed-precision FMAs
//   (fma.rn.f32.bf16 -> FHFMA.BF16, hi * +-1 + lo, one rounding of the exact sum, i.e. the
//   same value as an fp32 FADD), and for E4M3 codes cvt.rn.f16x2.e4m3x2 plus
//   fma.rn.f32.f16.  Every other stage is a packed FADD2 / FFMA2 over two pairs.
// * Exchange stages.  A butterfly over a lane bit normally costs one SHFL per value plus an
//   FFMA2 per pair.  Here a lane keeps half its values and trades the other half with its
//   partner (one SHFL per two values): the stage before the exchange places its outputs
//   lane-dependently (fma(b, +-1, a)), so that lane q_e = 0 holds the "sum" half and lane
//   q_e = 1 the "difference" half in the same registers; after the swap each lane owns one
//   output index of that bit and runs an ordinary packed stage over the lane bit.  A lane
//   bit and a register bit trade places (a transpose for free); lanes with q_e = 1 compute
//   own - partner, i.e. the negated difference, for their upper outputs.  That sign is a
//   fixed function of (lane, pair) and is folded into the final per-pair multiplier.
// * Canonical zeros.  The final multiply is fma(v, +-k, +0), so an exact zero comes out +0
//   whatever the sign bookkeeping (x - x = +0 in the reference's double arithmetic too).
//
// Butterfly order (pinned; K3's re-encode runs exactly K1's operations on the fp32 sum):
//   K1 (lane bits q_e = position b(3+e), pair bits i0 = b1, i1 = b2, i2..i4 = j0..j2 =
//       b(3+logL) .. b(5+logL)):  b0 [unpack], then for e = 0..logL-1: placed stage over
//       j(2-e), exchange with lane bit e; then b1, b2, then the remaining j bits ascending.
//   K2 / K3 decode (lane q owns 64 contiguous codes: lane bits = b6.., pair bits = b1..b5):
//       b0 [decode], for e: placed stage over b(3+e), exchange with lane bit e; then b1, b2,
//       then b(3+logL) .. b5.  It ends in K1's input layout (lane bits b3..), so K3 re-encodes
//       its sum without a transpose; only the pair-bit <-> position map differs (EncPlan J).
#pragma once

#include "taco_kernels.cuh"

namespace taco_dev {
namespace xk {

constexpr int kWarps = 4;    // warps per CTA (persistent grid)
#ifndef TACO_XK_MINCTAS
#define TACO_XK_MINCTAS 4
#endif
constexpr int kMinCtas = TACO_XK_MINCTAS;  // 4: 16 warps per SM (registers capped at 128)

#ifndef TACO_XK_K1_F32_DIRECT
// fp32-input K1 without shared-memory staging: 119.9 -> 72.2 us (0.54 -> 0.89 of HBM) on
// configs[3]; the staged form saturated the MIO pipe (16 LDGSTS + 16 LDS.128 + 70 SHFL per
// lane-tile, mio_throttle 2.4 and short_scoreboard 2.8 stalls per issue, issue active 0.28).
// bf16 keeps the staging (direct loads: 55.7 vs 50.7 us).
#define TACO_XK_K1_F32_DIRECT 1
#endif
#ifndef TACO_XK_K2_DIRECT_L
#define TACO_XK_K2_DIRECT_L 0x1  // K2 codes straight into registers at B = 64 (33.5 -> 32.1 us at the configs[2] shape); staged elsewhere (B = 256: 36.4 vs 33.1 us direct)
#endif
#ifndef TACO_XK_K1_BF16_DIRECT_L
// bf16 K1 loads straight into registers for these lanes-per-block (bit log2 L): B = 64
// (LDG.256, 50.3 -> 36.3 us at the configs[2] shape) and B = 128 (42.4 -> 39.4 us); B = 256
// keeps the cp.async staging (direct: 55.7 vs 50.7 us on configs[3])
#define TACO_XK_K1_BF16_DIRECT_L 0x3
#endif
#ifndef TACO_XK_SUMSQ_BF16
#define TACO_XK_SUMSQ_BF16 1  // K1 bf16: sum of squares by fma.rn.f32.bf16 on the inputs (51.35 -> 50.75 us, configs[3])
#endif
#ifndef TACO_XK_WARP_MAJOR
#define TACO_XK_WARP_MAJOR 0
#endif
// first tile of a persistent warp (then every gridDim.x * kWarps-th): CTA-major gives the
// trailing partial round to the first CTAs, warp-major spreads it over every CTA (and SM)
// (measured, configs[1] / configs[3] tensors: warp-major K2 13.9 / 47.3 us vs 14.3 / 47.6;
// K1 15.7 / 51.4 vs 15.6 / 51.2 -- K1 stays CTA-major)
#ifndef TACO_XK_K2_WARP_MAJOR
#define TACO_XK_K2_WARP_MAJOR 1
#endif
template <bool WARP_MAJOR = (TACO_XK_WARP_MAJOR != 0)>
__device__ __forceinline__ uint32_t first_tile(int warp) {
    return WARP_MAJOR ? (uint32_t)warp * gridDim.x + blockIdx.x : blockIdx.x * kWarps + (uint32_t)warp;
}

__host__ __device__ constexpr int ilog2c(int v) { return v <= 1 ? 0 : 1 + ilog2c(v >> 1); }
__host__ __device__ constexpr int bit(int v, int b) { return (v >> b) & 1; }

// ------------------------------------------------------------------ primitives ---

// (lo + hi, lo - hi) of the two bf16 halves of u (element 2k in the low half)
__device__ __forceinline__ float2 bf16_b0(uint32_t u) {
    float s, d;
    asm("{\n\t.reg .b16 l, h, one, mone;\n\t.reg .b32 t;\n\t"
        "mov.b32 {l, h}, %2;\n\tshl.b32 t, %2, 16;\n\t"
        "mov.b16 one, 0x3F80;\n\tmov.b16 mone, 0xBF80;\n\t"
        "fma.rn.f32.bf16 %0, h, one, t;\n\tfma.rn.f32.bf16 %1, h, mone, t;\n\t}"
        : "=f"(s), "=f"(d)
        : "r"(u));
    return make_float2(s, d);
}

// four E4M3 codes (byte k = position 4w + k) -> (c0 + c1, c0 - c1), (c2 + c3, c2 - c3); every
// E4M3 value is an f16 value, so the cvt is exact and the FMAs round once like an fp32 add
__device__ __forceinline__ void e4m3_b0(uint32_t u, float2& p, float2& q) {
    asm("{\n\t.reg .b16 c01, c23, l, h, l2, h2, one, mone;\n\t.reg .b32 h01, h23;\n\t.reg .f32 a, b;\n\t"
        "mov.b32 {c01, c23}, %4;\n\t"
        "cvt.rn.f16x2.e4m3x2 h01, c01;\n\tcvt.rn.f16x2.e4m3x2 h23, c23;\n\t"
        "mov.b32 {l, h}, h01;\n\tmov.b32 {l2, h2}, h23;\n\t"
        "cvt.f32.f16 a, l;\n\tcvt.f32.f16 b, l2;\n\t"
        "mov.b16 one, 0x3C00;\n\tmov.b16 mone, 0xBC00;\n\t"
        "fma.rn.f32.f16 %0, h, one, a;\n\tfma.rn.f32.f16 %1, h, mone, a;\n\t"
        "fma.rn.f32.f16 %2, h2, one, b;\n\tfma.rn.f32.f16 %3, h2, mone, b;\n\t}"
        : "=f"(p.x), "=f"(p.y), "=f"(q.x), "=f"(q.y)
        : "r"(u));
}

__device__ __forceinline__ float2 b0_f32(float2 v) { return make_float2(v.x + v.y, v.x - v.y); }

// packed butterfly over pair bit T
template <int T>
__device__ __forceinline__ void st(float2 (&w)[32]) {
    const float2 m1 = make_float2(-1.0f, -1.0f);
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        if (!(i & (1 << T))) {
            const float2 a = w[i], b = w[i | (1 << T)];
            w[i] = __fadd2_rn(a, b);
            w[i | (1 << T)] = __ffma2_rn(b, m1, a);  // a - b, one rounding
        }
    }
}

// butterfly over pair bit T with lane-dependent output placement: m = +1 puts a + b at the
// lower pair, m = -1 puts a - b there (and a + b at the upper one)
template <int T>
__device__ __forceinline__ void st_placed(float2 (&w)[32], float m) {
    const float2 mp = make_float2(m, m), mn = make_float2(-m, -m);
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        if (!(i & (1 << T))) {
            const float2 a = w[i], b = w[i | (1 << T)];
            w[i] = __ffma2_rn(b, mp, a);
            w[i | (1 << T)] = __ffma2_rn(b, mn, a);
        }
    }
}

// exchange over lane bit LB: trade the upper half (pair bit T set) with the partner lane,
// then butterfly own (lower) against partner's (upper)
template <int T, int LB>
__device__ __forceinline__ void xch(float2 (&w)[32]) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        if (i & (1 << T)) {
            w[i].x = __shfl_xor_sync(kFull, w[i].x, 1 << LB);
            w[i].y = __shfl_xor_sync(kFull, w[i].y, 1 << LB);
        }
    }
    st<T>(w);
}

__device__ __forceinline__ float lane_sign(int q, int e) { return (q >> e) & 1 ? -1.0f : 1.0f; }

// ------------------------------------------------------------------ plans ---------

// Encode plan (K1 order).  J0..J2: the pair bits that hold the logical bits j0..j2 =
// b(3+logL) .. b(5+logL) when the encode starts (K1: 2, 3, 4; K3 after its decode: see Dec).
template <int L, int J0, int J1, int J2>
struct EncPlan {
    static constexpr int LOGL = ilog2c(L);
    __host__ __device__ static constexpr int J(int k) { return k == 0 ? J0 : k == 1 ? J1 : J2; }
    // position bit (within the lane's 64 contiguous outputs) of pair bit t after the encode
    __host__ __device__ static constexpr int posbit(int t) {
        return t == 0 ? 1 : t == 1 ? 2
             : (t == J(2) ? (LOGL > 0 ? 3 : 3 + LOGL + 2)
                          : t == J(1) ? (LOGL > 1 ? 4 : 3 + LOGL + 1) : (LOGL > 2 ? 5 : 3 + LOGL));
    }
    __host__ __device__ static constexpr int pos_of_pair(int i) {
        return (bit(i, 0) << posbit(0)) | (bit(i, 1) << posbit(1)) | (bit(i, 2) << posbit(2)) |
               (bit(i, 3) << posbit(3)) | (bit(i, 4) << posbit(4));
    }
    __host__ __device__ static constexpr int pair_at(int pos) {  // pos even, < 64
        return (bit(pos, posbit(0)) << 0) | (bit(pos, posbit(1)) << 1) | (bit(pos, posbit(2)) << 2) |
               (bit(pos, posbit(3)) << 3) | (bit(pos, posbit(4)) << 4);
    }
    // sign index of pair i: bit e = pair bit J(2-e) (the exchange-e output index)
    __host__ __device__ static constexpr int sidx(int i) {
        return (LOGL > 0 ? bit(i, J(2)) : 0) | (LOGL > 1 ? bit(i, J(1)) << 1 : 0) | (LOGL > 2 ? bit(i, J(0)) << 2 : 0);
    }
    // pair index (in this plan) of K1's pair i: the sum-of-squares walk order
    __host__ __device__ static constexpr int k1_pair(int i) {
        return bit(i, 0) | (bit(i, 1) << 1) | (bit(i, 2) << J(0)) | (bit(i, 3) << J(1)) | (bit(i, 4) << J(2));
    }
    // block offset of lane q's 64 outputs: lane bit e holds logical j(2-e) = b(5+logL-e)
    __device__ static __forceinline__ int lane_off(int q) {
        int o = 0;
#pragma unroll
        for (int e = 0; e < LOGL; ++e) o |= ((q >> e) & 1) << (5 + LOGL - e);
        return o;
    }
    // the stages after b0
    __device__ static __forceinline__ void stages(float2 (&w)[32], int q) {
        if constexpr (LOGL >= 1) { st_placed<J2>(w, lane_sign(q, 0)); xch<J2, 0>(w); }
        if constexpr (LOGL >= 2) { st_placed<J1>(w, lane_sign(q, 1)); xch<J1, 1>(w); }
        if constexpr (LOGL >= 3) { st_placed<J0>(w, lane_sign(q, 2)); xch<J0, 2>(w); }
        st<0>(w);
        st<1>(w);
        if constexpr (LOGL <= 2) st<J0>(w);
        if constexpr (LOGL <= 1) st<J1>(w);
        if constexpr (LOGL == 0) st<J2>(w);
    }
};

// Decode plan (K2, K3): lane q owns codes [64 q, 64 q + 64) of its block.
template <int L>
struct DecPlan {
    static constexpr int LOGL = ilog2c(L);
    __device__ static __forceinline__ void stages(float2 (&w)[32], int q) {
        if constexpr (LOGL >= 1) { st_placed<2>(w, lane_sign(q, 0)); xch<2, 0>(w); }
        if constexpr (LOGL >= 2) { st_placed<3>(w, lane_sign(q, 1)); xch<3, 1>(w); }
        if constexpr (LOGL >= 3) { st_placed<4>(w, lane_sign(q, 2)); xch<4, 2>(w); }
        st<0>(w);
        st<1>(w);
        if constexpr (LOGL <= 0) st<2>(w);
        if constexpr (LOGL <= 1) st<3>(w);
        if constexpr (LOGL <= 2) st<4>(w);
    }
    // after the decode: position bit (in the block) of pair bit t = 2..4, lane bit e = b(3+e)
    __host__ __device__ static constexpr int posbit(int t) { return t - 2 < LOGL ? 6 + (t - 2) : t + 1; }
    // block position of the 8-element vector of pairs 4v .. 4v+3
    __host__ __device__ static constexpr int vec_pos(int v) {
        return (bit(v, 0) << posbit(2)) | (bit(v, 1) << posbit(3)) | (bit(v, 2) << posbit(4));
    }
    __device__ static __forceinline__ int lane_off(int q) { return q << 3; }
    // sign index of pair i: bit e = pair bit 2+e
    __host__ __device__ static constexpr int sidx(int i) { return (i >> 2) & ((1 << LOGL) - 1); }
    // the pair bit holding logical j_k = b(3+logL+k) after the decode (K3's EncPlan)
    __host__ __device__ static constexpr int jbit(int k) {
        return 3 + LOGL + k >= 6 ? 2 + (LOGL + k - 3) : 3 + LOGL + k - 1;
    }
    using Enc = EncPlan<L, jbit(0), jbit(1), jbit(2)>;
};

// multipliers k * (+-1) per sign index: bit e of the index negates for lanes with q_e = 1
template <int LOGL>
__device__ __forceinline__ void signed_mults(float k, int q, float (&mk)[1 << LOGL]) {
#pragma unroll
    for (int s = 0; s < (1 << LOGL); ++s) mk[s] = (__popc(s & q) & 1) ? -k : k;
}

// v = v * m (+0): sign bookkeeping and zero canonicalisation in one FFMA2 per pair
template <int LOGL, typename SIdx>
__device__ __forceinline__ void apply_mults(float2 (&w)[32], const float (&mk)[1 << LOGL], SIdx sidx) {
    const float2 z = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int i = 0; i < 32; ++i) w[i] = __ffma2_rn(w[i], make_float2(mk[sidx(i)], mk[sidx(i)]), z);
}

// scale by a double factor that may lie outside the fp32 range: exact powers of two first
// (mul_wide's split), returns the remaining float factor
__device__ __forceinline__ float wide_prescale(float2 (&w)[32], double k) {
#pragma unroll 1
    for (int i = 0; i < 4 && isfinite(k) && (fabs(k) >= 0x1p126 || (k != 0.0 && fabs(k) < 0x1p-126)); ++i) {
        const double step = fabs(k) >= 0x1p126 ? 0x1p63 : 0x1p-63;
        scale2<32>(w, (float)step);
        k /= step;
    }
    return (float)k;
}

template <int L>
__device__ __forceinline__ float absmax32(const float2 (&w)[32]) {
    float m[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) m[r] = fmaxf(fabsf(w[r].x), fabsf(w[r].y));
#pragma unroll
    for (int i = 8; i < 32; ++i) m[i & 7] = fmaxf(m[i & 7], fmaxf(fabsf(w[i].x), fabsf(w[i].y)));
    float a = fmaxf(fmaxf(m[0], m[1]), fmaxf(m[2], m[3]));
    float b = fmaxf(fmaxf(m[4], m[5]), fmaxf(m[6], m[7]));
    a = fmaxf(a, b);
#pragma unroll
    for (int o = 1; o < L; o <<= 1) a = fmaxf(a, __shfl_xor_sync(kFull, a, o));
    return a;
}

// fp32 sum of squares of the b0-stage outputs in K1's pair order (4 FFMA2 chains), halved:
// (a + b)^2 + (a - b)^2 = 2 (a^2 + b^2)
template <typename Plan>
__device__ __forceinline__ float sumsq_b0(const float2 (&w)[32]) {
    float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i & 3] = __ffma2_rn(w[Plan::k1_pair(i)], w[Plan::k1_pair(i)], acc[i & 3]);
    const float2 t = __fadd2_rn(__fadd2_rn(acc[0], acc[1]), __fadd2_rn(acc[2], acc[3]));
    return (t.x + t.y) * 0.5f;
}

// fp64 sum of squares of plain (pre-b0) values in K1's pair order (the out-of-range path)
template <typename Plan>
__device__ __forceinline__ double sumsq_plain_f64(const float2 (&w)[32]) {
    double d[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        const float2 v = w[Plan::k1_pair(i)];
        d[(2 * i) & 3] = fma((double)v.x, (double)v.x, d[(2 * i) & 3]);
        d[(2 * i + 1) & 3] = fma((double)v.y, (double)v.y, d[(2 * i + 1) & 3]);
    }
    return (d[0] + d[1]) + (d[2] + d[3]);
}

// whether the lane's fp32 sum of squares is inside the range where it is trusted
__device__ __forceinline__ bool sf_ok(float sf) { return sf < 0x1p100f && !(sf > 0.0f && sf < 0x1p-100f); }

// Per-block scalars + rotation + quantisation of a lane's b0-stage values (the part of
// rotate_block / compress_block_taco, codec.cpp:45-76, after the pair-bit butterfly).
// `reload(w)` refills w with the plain block values (the out-of-range path: fp64 sum of
// squares and the exact power-of-two pre-scale, taken per lane / per block as the register
// K1 does).  On return w holds the FP8-ready Z/s with canonical signs and zeros.
template <int L, typename Plan, typename Reload>
__device__ __forceinline__ void encode(float2 (&w)[32], int q, const CodecConsts& c, float& alpha, float& s,
                                       double& ss, Reload reload, float sf_pre = -1.0f) {
    // sf_pre >= 0: the lane's fp32 sum of squares was taken from the bf16 inputs (mixed-precision
    // FMAs off the packed-FP32 pipe); otherwise from the b0-stage outputs
    const float sf = sf_pre >= 0.0f ? sf_pre : sumsq_b0<Plan>(w);
    const bool lane_slow = !sf_ok(sf);
    float p2 = 1.0f;
    double sl = (double)sf;
    if (__any_sync(kFull, lane_slow)) {  // rare: re-derive from the plain values
        reload(w);
        if (lane_slow) sl = sumsq_plain_f64<Plan>(w);
        const double ss0 = group_sum<L>(sl);
        const bool huge = !(ss0 < 0x1p160);
        p2 = huge ? pow2_near(block_alpha_fast(ss0, c)) : 1.0f;
#pragma unroll
        for (int i = 0; i < 32; ++i) w[i] = b0_f32(make_float2(w[i].x * p2, w[i].y * p2));
    }
    // the scalar chain sits in the same basic block as the butterfly, which does not depend
    // on it (alpha enters only through k), so the scheduler overlaps its latency
    ss = group_sum<L>(sl);
    alpha = block_alpha_xk(ss, c);
    Plan::stages(w, q);
    const float ymax = absmax32<L>(w);
    double k;
    block_scale_fast((double)ymax, alpha, p2, c, s, k);
    const float kf = wide_prescale(w, k);
    float mk[1 << Plan::LOGL];
    signed_mults<Plan::LOGL>(kf, q, mk);
    apply_mults<Plan::LOGL>(w, mk, [](int i) { return Plan::sidx(i); });
}

// the lane's 64 codes (positions lane_off .. +64 of the block) as 4 x 16 bytes
template <typename Plan>
__device__ __forceinline__ void pack_codes(const float2 (&w)[32], uint4 (&out)[4]) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        uint32_t wd[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int pos = 16 * u + 4 * k;
            wd[k] = enc2<0>(w[Plan::pair_at(pos)]) | (enc2<0>(w[Plan::pair_at(pos + 2)]) << 16);
        }
        out[u] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
    }
}

// 16-byte global store that does not allocate in L1 (streamed output: measured 43.5 vs
// 46.3 us for K2's access pattern alone, tools/mempat2.cu)
__device__ __forceinline__ void st16_na(void* p, uint4 v) {
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}

// 256-bit global accesses (sm_100: LDG.256 / STG.256), 32-byte aligned addresses only
__device__ __forceinline__ void ldg32_f32(const float* p, float2 (&o)[4]) {
    asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=f"(o[0].x), "=f"(o[0].y), "=f"(o[1].x), "=f"(o[1].y), "=f"(o[2].x), "=f"(o[2].y), "=f"(o[3].x),
                   "=f"(o[3].y)
                 : "l"(p));
}
__device__ __forceinline__ void ldg32_u4x2(const void* p, uint4& a, uint4& b) {
    asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
                 : "l"(p));
}
__device__ __forceinline__ void stg32_u4x2(void* p, const uint4& a, const uint4& b) {
    asm volatile("st.global.L1::no_allocate.v8.u32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(a.x),
                 "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
                 : "memory");
}
__device__ __forceinline__ void stg32_f32(float* p, const float2* v) {
    asm volatile("st.global.L1::no_allocate.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "f"(v[0].x),
                 "f"(v[0].y), "f"(v[1].x), "f"(v[1].y), "f"(v[2].x), "f"(v[2].y), "f"(v[3].x), "f"(v[3].y)
                 : "memory");
}

// 8 contiguous outputs (4 pairs) of type T; wide: 32-byte aligned (one 256-bit store for fp32)
template <typename T>
__device__ __forceinline__ void store8(T* p, const float2* v, bool wide = false) {
    if constexpr (sizeof(T) == 2) {
        st16_na(p, make_uint4(pack_bf16x2(v[0]), pack_bf16x2(v[1]), pack_bf16x2(v[2]), pack_bf16x2(v[3])));
    } else if (wide) {
        stg32_f32(p, v);
    } else {
        st16_na(p, make_uint4(__float_as_uint(v[0].x), __float_as_uint(v[0].y), __float_as_uint(v[1].x),
                              __float_as_uint(v[1].y)));
        st16_na(p + 4, make_uint4(__float_as_uint(v[2].x), __float_as_uint(v[2].y), __float_as_uint(v[3].x),
                                  __float_as_uint(v[3].y)));
    }
}
template <typename T>
__device__ __forceinline__ void store8_guarded(T* p, int pos, int valid, const float2* v) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        if (pos + 2 * r < valid) store_one(p + 2 * r, v[r].x);
        if (pos + 2 * r + 1 < valid) store_one(p + 2 * r + 1, v[r].y);
    }
}

// K2/K3 decode output layout: lane q holds, for vector v (pairs 4v..4v+3), the 8 outputs at
// block position lane_off(q) + vec_pos(v)
template <int L, typename T>
__device__ __forceinline__ void store_decoded(T* blk, int q, int valid, int vec_ok, const float2 (&w)[32]) {
    using D = DecPlan<L>;
    const int lo = D::lane_off(q);
    if (vec_ok && valid == 64 * L) {
        if constexpr (L == 1 && sizeof(T) == 2) {  // one lane per block: 64 contiguous outputs
            if (vec_ok >= 2) {  // (32-byte aligned block starts, see wide_ok)
#pragma unroll
                for (int v = 0; v < 8; v += 2) {
                    static_assert(D::vec_pos(1) == 8, "B = 64 lanes own contiguous 8-element vectors");
                    const float2* a = &w[4 * v];
                    const float2* b = &w[4 * v + 4];
                    stg32_u4x2(blk + D::vec_pos(v),
                               make_uint4(pack_bf16x2(a[0]), pack_bf16x2(a[1]), pack_bf16x2(a[2]), pack_bf16x2(a[3])),
                               make_uint4(pack_bf16x2(b[0]), pack_bf16x2(b[1]), pack_bf16x2(b[2]), pack_bf16x2(b[3])));
                }
                return;
            }
        }
#pragma unroll
        for (int v = 0; v < 8; ++v) store8<T>(blk + lo + D::vec_pos(v), &w[4 * v], vec_ok >= 2);
    } else {
#pragma unroll
        for (int v = 0; v < 8; ++v) {
            const int pos = lo + D::vec_pos(v);
            if (vec_ok && pos + 8 <= valid) store8<T>(blk + pos, &w[4 * v]);
            else store8_guarded<T>(blk + pos, pos, valid, &w[4 * v]);
        }
    }
}

// ------------------------------------------------------------- async copies -------
// Codes of a warp tile (G blocks x B codes = 2 KB = 128 16-byte units) are copied coalesced
// (instruction c, lane l -> unit 32 c + l) into a shared-memory tile whose 16-byte units are
// XOR-swizzled (unit u at u ^ ((u >> 3) & 3)), so that the decode's per-lane reads (lane (g, q)
// takes units 16 g + 4 q + c, its 64 contiguous codes) are bank-conflict free.  The half-sector
// per-lane copies this replaces bound K2 at 53.4 us on configs[3] (tools/mempat.cu).
__device__ __forceinline__ int swz_unit(int u) { return u ^ ((u >> 3) & 3); }
__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// --------------------------------------------------------------------- K1 --------
template <int L, typename TIn>
struct K1X {
    static constexpr int B = 64 * L, G = 32 / L;
    static constexpr int EPC = 16 / (int)sizeof(TIn);  // elements per 16-byte chunk
    static constexpr int NCH = 64 / EPC;              // chunks per lane per tile
    // fp32 input (TACO_XK_K1_F32_DIRECT): no shared-memory staging -- the lane's chunks are
    // loaded straight into registers (the ragged path's vector loads), which leaves the MIO
    // pipe to the exchanges; 16 warps per SM hide the load latency
    // B = 64 bf16 (one lane per block: its 64 inputs are one contiguous 128-byte run) likewise:
    // the staged form is MIO-bound there (profiles/r3s_block_sweep_configs2.txt)
    static constexpr bool DIRECT = (sizeof(TIn) == 4 && TACO_XK_K1_F32_DIRECT) ||
                                   (sizeof(TIn) == 2 && ((TACO_XK_K1_BF16_DIRECT_L >> ilog2c(L)) & 1));
    static constexpr int STAGES = DIRECT ? 0 : 2;
    static constexpr int STAGE_U4 = NCH * 32;
#ifndef TACO_XK_CSTORE
#define TACO_XK_CSTORE 1  // codes staged through shared memory: 54.0 -> 51.4 us (configs[3], bf16)
#endif
#if TACO_XK_CSTORE
    static constexpr int CODE_U4 = 128;  // the tile's codes, staged for coalesced stores
#else
    static constexpr int CODE_U4 = 0;
#endif
    static constexpr int WARP_U4 = STAGES * STAGE_U4 + CODE_U4;
    static constexpr size_t SMEM = (size_t)kWarps * WARP_U4 * 16;
    // element offset (in the block) of chunk ch of lane q: vector j = ch / (8 / EPC)
    __device__ static __forceinline__ int chunk_off(int ch, int q) {
        constexpr int CPV = 8 / EPC;
        return ((ch / CPV) * L + q) * 8 + (ch % CPV) * EPC;
    }
};

// plain values of vector j (natural K1 layout) from 16-byte chunks
template <typename TIn>
__device__ __forceinline__ void plain_from_chunk(uint4 u, float2* dst) {
    if constexpr (sizeof(TIn) == 2) {
        dst[0] = bf16x2_to_f2(u.x); dst[1] = bf16x2_to_f2(u.y);
        dst[2] = bf16x2_to_f2(u.z); dst[3] = bf16x2_to_f2(u.w);
    } else {
        dst[0] = make_float2(__uint_as_float(u.x), __uint_as_float(u.y));
        dst[1] = make_float2(__uint_as_float(u.z), __uint_as_float(u.w));
    }
}

template <int L, typename TIn, bool PUSH>
__global__ void __launch_bounds__(kWarps * 32, kMinCtas)
    k1x(const TIn* __restrict__ x, uint8_t* __restrict__ msgs, ShardArgs a, CodecConsts c, FastDiv tps) {
    using K = K1X<L, TIn>;
    using Plan = EncPlan<L, 2, 3, 4>;
    constexpr int B = K::B, G = K::G, NCH = K::NCH, EPC = K::EPC;
    extern __shared__ uint4 smem_dyn[];
    const int lane = threadIdx.x & 31, q = lane & (L - 1), g = lane / L, warp = threadIdx.x >> 5;
    uint4* stage_base = smem_dyn + (size_t)warp * K::WARP_U4 + lane;
    uint4* code_buf = smem_dyn + (size_t)warp * K::WARP_U4 + K::STAGES * K::STAGE_U4;
    const uint32_t ntiles = a.P * tps.d;
    const uint32_t stride = gridDim.x * kWarps;
    const int qoff = q * 8;  // lane's element offset inside a vector row (chunk_off(0, q))
    uint32_t t = first_tile(warp);

    // tile tt -> shard p, first block kk0 of the chunk, whether every block is whole
    struct Tile {
        uint32_t p;
        uint32_t kk0;
        bool full;
    };
    // whole-block limits as 32-bit (run_xk requires nblk < 2^31)
    const uint32_t fmid = (uint32_t)a.full_mid, flast = (uint32_t)a.full_last, plast = a.P - 1;
    auto info = [&](uint32_t tt) -> Tile {
        const uint32_t p = tps.div(tt);
        const uint32_t kk0 = (tt - p * tps.d) * G;
        return Tile{p, kk0, a.vec_ok && kk0 + G <= (p == plast ? flast : fmid)};
    };
    auto issue = [&](const Tile& tl, int stage) {
        if (tl.full && !K::DIRECT) {
            const TIn* src = x + (tl.p * a.S + (a.blk0 + tl.kk0 + g) * B) + qoff;
            uint4* sb = stage_base + stage * K::STAGE_U4;
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) cp16(sb + ch * 32, src + K::chunk_off(ch, 0));
        }
        cp_async_commit();
    };

    grid_dep_wait();
    if constexpr (PUSH) peer_pre(a);  // fused peer mode: the peers have finished reading the slots this K1 writes
    Tile cur{0, 0, false};
    if (t < ntiles) {
        cur = info(t);
        issue(cur, 0);
    }
    for (int it = 0; t < ntiles; t += stride, ++it) {
        Tile nxt{0, 0, false};
        if (t + stride < ntiles) {
            nxt = info(t + stride);
            issue(nxt, (it + 1) & 1);
        } else {
            cp_async_commit();
        }
        const uint64_t kk = cur.kk0 + g;
        const uint32_t p = cur.p;
        const uint4* sb = stage_base + (it & 1) * K::STAGE_U4;
        const bool full = cur.full;
        // plain (pre-b0) values of the lane in the natural layout: pair 4j + r/2
        auto load_plain = [&](float2 (&w)[32]) {
            if (full && !K::DIRECT) {
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) plain_from_chunk<TIn>(sb[ch * 32], &w[ch * (EPC / 2)]);
            } else {
                const uint64_t k = a.blk0 + kk;
                const int valid = kk < a.nblk ? clamp_valid((int64_t)a.S - (int64_t)(k * B),
                                                            (int64_t)a.n - (int64_t)(p * a.S + k * B), B)
                                              : 0;
                const TIn* src = x + (p * a.S + k * B);
                // lane index re-read through a volatile move: the ragged path's offsets are
                // not hoisted into (and kept live through) the whole-tile loop
                int qq;
                asm volatile("mov.b32 %0, %1;" : "=r"(qq) : "r"(q));
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int pos = (j * L + qq) * 8;
                    float2 tmp[4];
                    if (sizeof(TIn) == 4 && a.vec_ok >= 2 && pos + 8 <= valid)
                        ldg32_f32(reinterpret_cast<const float*>(src + pos), tmp);
                    else if (a.vec_ok && pos + 8 <= valid) load_vec<TIn, 8>(src + pos, tmp);
                    else load_vec_guarded<TIn, 8>(src + pos, pos, valid, tmp);
#pragma unroll
                    for (int r = 0; r < 4; ++r) w[4 * j + r] = tmp[r];
                }
            }
        };
        float2 w[32];
        if (full && !K::DIRECT) cp_wait<1>();  // this lane's chunks of tile t have landed
        float sf_pre = -1.0f;
        if (sizeof(TIn) == 2 && full) {
#if TACO_XK_SUMSQ_BF16
            float sq[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#endif
            uint4 cw[NCH];
            if constexpr (K::DIRECT) {  // B = 64: the lane's block, straight from global memory
                const TIn* src = x + (p * a.S + (a.blk0 + kk) * B) + qoff;
                if (L == 1 && a.vec_ok >= 2 && (a.P == 1 || (a.S & 15) == 0)) {  // 32-byte aligned block starts
#pragma unroll
                    for (int m2 = 0; m2 < NCH / 2; ++m2) ldg32_u4x2(src + 16 * m2, cw[2 * m2], cw[2 * m2 + 1]);
                } else {
#pragma unroll
                    for (int ch = 0; ch < NCH; ++ch) cw[ch] = __ldg(reinterpret_cast<const uint4*>(src + K::chunk_off(ch, 0)));
                }
            } else {
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) cw[ch] = sb[ch * 32];
            }
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) {
                const uint4 u = cw[ch];
                w[4 * ch + 0] = bf16_b0(u.x);
                w[4 * ch + 1] = bf16_b0(u.y);
                w[4 * ch + 2] = bf16_b0(u.z);
                w[4 * ch + 3] = bf16_b0(u.w);
#if TACO_XK_SUMSQ_BF16
                const uint32_t uu[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    sq[k] = fma_bf16_sq(uu[k] & 0xffffu, sq[k]);
                    sq[k] = fma_bf16_sq(uu[k] >> 16, sq[k]);
                }
#endif
            }
#if TACO_XK_SUMSQ_BF16
            sf_pre = (sq[0] + sq[1]) + (sq[2] + sq[3]);
#endif
        } else {
            load_plain(w);
#if TACO_XK_SUMSQ_BF16
            if (sizeof(TIn) == 2) {  // the full path's sum, same operations in the same order
                float sq[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    sq[i & 3] = __fmaf_rn(w[i].x, w[i].x, sq[i & 3]);
                    sq[i & 3] = __fmaf_rn(w[i].y, w[i].y, sq[i & 3]);
                }
                sf_pre = (sq[0] + sq[1]) + (sq[2] + sq[3]);
            }
#endif
#pragma unroll
            for (int i = 0; i < 32; ++i) w[i] = b0_f32(w[i]);
        }
        float alpha, s;
        double ss;
        encode<L, Plan>(w, q, c, alpha, s, ss, load_plain, sf_pre);
#if TACO_XK_CSTORE
        {
            uint4 cv[4];
            pack_codes<Plan>(w, cv);
            const int u0 = (g * B + Plan::lane_off(q)) / 16;
            __syncwarp();  // the previous tile's codes were read out
#pragma unroll
            for (int u = 0; u < 4; ++u) code_buf[swz_unit(u0 + u)] = cv[u];
            __syncwarp();
            uint4 ov[4];
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) ov[c4] = code_buf[swz_unit(32 * c4 + lane)];
            const uint64_t kk0 = cur.kk0;
            auto put = [&](uint8_t* m) {
                uint8_t* base = m + kk0 * B + 16 * lane;  // unit u = 32 c4 + lane at base + 512 c4
                if (full) {
#pragma unroll
                    for (int c4 = 0; c4 < 4; ++c4) st16_na(base + 512 * c4, ov[c4]);
                } else {
#pragma unroll
                    for (int c4 = 0; c4 < 4; ++c4)
                        if (kk0 + (uint64_t)((16 * (32 * c4 + lane)) / B) < a.nblk) st16_na(base + 512 * c4, ov[c4]);
                }
                if (q == 0 && (full || kk < a.nblk))
                    *reinterpret_cast<float2*>(m + a.scal_off + kk * 8) = make_float2(alpha, s);
            };
            if constexpr (PUSH) {
                if (a.bcast)
                    for (uint32_t d = 0; d < a.ndst; ++d) put(a.dst[d]);
                else
                    put(a.dst[p]);
            } else {
                put(msgs + p * a.msg_stride);
            }
            if (q == 0 && (full || kk < a.nblk) && !isfinite(ss)) raise_flag(a.flags, 1);
        }
#else
        if (full || kk < a.nblk) {
            uint4 cv[4];
            pack_codes<Plan>(w, cv);
            const int lo = Plan::lane_off(q);
            auto put = [&](uint8_t* m) {
                uint4* dst = reinterpret_cast<uint4*>(m + kk * B + lo);
#pragma unroll
                for (int u = 0; u < 4; ++u) dst[u] = cv[u];
                if (q == 0) *reinterpret_cast<float2*>(m + a.scal_off + kk * 8) = make_float2(alpha, s);
            };
            if constexpr (PUSH) {
                if (a.bcast)
                    for (uint32_t d = 0; d < a.ndst; ++d) put(a.dst[d]);
                else
                    put(a.dst[p]);
            } else {
                put(msgs + p * a.msg_stride);
            }
            if (q == 0 && !isfinite(ss)) raise_flag(a.flags, 1);  // any NaN/Inf element poisons the block sum
        }
#endif
        cur = nxt;
    }
    if constexpr (PUSH) peer_post(a);  // ... and every rank's pushes of this phase have landed
}

// --------------------------------------------------------------------- K2 --------
template <int L>
struct K2X {
    static constexpr int B = 64 * L, G = 32 / L;
    static constexpr int STAGES = 4;
    // per stage: the tile's 128 code units (swizzled), then the G blocks' (alpha, s) pairs
    static constexpr int STAGE_U4 = 128 + G / 2;
    static constexpr size_t SMEM = (size_t)kWarps * STAGES * STAGE_U4 * 16;
};

__device__ __forceinline__ void cp8(void* smem, const void* gmem) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}

// coalesced copy of a tile's codes (blocks kk0 .. kk0+G-1 of message m, live blocks only) and
// scalars into one stage
template <int L>
__device__ __forceinline__ void stage_tile(uint4* sb, const uint8_t* m, uint64_t kk0, uint64_t nblk,
                                           uint64_t scal_off, int lane) {
    constexpr int B = 64 * L, G = 32 / L;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int u = 32 * c + lane;
        if (kk0 + (uint64_t)((16 * u) / B) < nblk) cp16(sb + swz_unit(u), m + kk0 * B + 16 * (uint64_t)u);
    }
    if (lane < G && kk0 + lane < nblk) cp8(reinterpret_cast<float2*>(sb + 128) + lane, m + scal_off + (kk0 + lane) * 8);
}

// this lane's 64 codes (units 16 g + 4 q + c for L = 4; generally (g B + 64 q) / 16 + c)
template <int L>
__device__ __forceinline__ void read_lane_codes(const uint4* sb, int g, int q, uint4 (&u)[4]) {
    const int u0 = (g * 64 * L + 64 * q) / 16;
#pragma unroll
    for (int c = 0; c < 4; ++c) u[c] = sb[swz_unit(u0 + c)];
}

// decode 64 codes (4 x 16 bytes, positions 16 ch + ..) into b0-stage pairs
__device__ __forceinline__ void decode64(const uint4 (&u)[4], float2 (&w)[32]) {
#pragma unroll
    for (int ch = 0; ch < 4; ++ch) {
        e4m3_b0(u[ch].x, w[8 * ch + 0], w[8 * ch + 1]);
        e4m3_b0(u[ch].y, w[8 * ch + 2], w[8 * ch + 3]);
        e4m3_b0(u[ch].z, w[8 * ch + 4], w[8 * ch + 5]);
        e4m3_b0(u[ch].w, w[8 * ch + 6], w[8 * ch + 7]);
    }
}

// the decode of one lane's 64 codes of a block with scalars sc = (alpha, s): K2's exact
// arithmetic (decompress_block, codec.cpp:146-153: out = float(H(table[c] * s) * norm / alpha))
template <int L>
__device__ __forceinline__ void decode_block(const uint4 (&u)[4], float2 sc, bool live, int q, const CodecConsts& c,
                                             float2 (&w)[32]) {
    using D = DecPlan<L>;
    decode64(u, w);
    D::stages(w, q);
    const float mf = wide_prescale(w, block_dequant(live ? sc.x : 1.0f, live ? sc.y : 1.0f, c));
    float mk[1 << D::LOGL];
    signed_mults<D::LOGL>(mf, q, mk);
    apply_mults<D::LOGL>(w, mk, [](int i) { return D::sidx(i); });
}

template <int L, typename TOut>
__global__ void __launch_bounds__(kWarps * 32, kMinCtas)
    k2x(const uint8_t* __restrict__ msgs, TOut* __restrict__ out, ShardArgs a, CodecConsts c, FastDiv tps) {
    using K = K2X<L>;
    constexpr int B = K::B, G = K::G, NS = K::STAGES;
    extern __shared__ uint4 smem_dyn[];
    const int lane = threadIdx.x & 31, q = lane & (L - 1), g = lane / L, warp = threadIdx.x >> 5;
    uint4* stage_base = smem_dyn + (size_t)warp * NS * K::STAGE_U4;
    const uint32_t ntiles = a.P * tps.d;
    const uint32_t stride = gridDim.x * kWarps;

    constexpr bool DIRECT = (TACO_XK_K2_DIRECT_L >> ilog2c(L)) & 1;  // codes straight into registers
    auto issue = [&](uint32_t tt, int stage) {
        if (DIRECT) return;
        if (tt < ntiles) {
            const uint32_t p = tps.div(tt);
            const uint64_t kk0 = (uint64_t)(tt - p * tps.d) * G;
            stage_tile<L>(stage_base + stage * K::STAGE_U4, msgs + p * a.msg_stride, kk0, a.nblk, a.scal_off, lane);
        }
        cp_async_commit();
    };

    grid_dep_wait();
    peer_pre(a);  // fused peer mode: every rank's K3 has finished (its messages are in the gather slots)
    uint32_t t = first_tile<TACO_XK_WARP_MAJOR || TACO_XK_K2_WARP_MAJOR>(warp);
    if constexpr (DIRECT) {
        for (; t < ntiles; t += stride) {
            const uint32_t p = tps.div(t);
            const uint64_t kk = (uint64_t)(t - p * tps.d) * G + g;
            const bool live = kk < a.nblk;
            uint4 u[4];
            float2 sc = make_float2(1.0f, 1.0f);
            if (live) {  // the lane's 64 codes are one contiguous 64-byte run of the message
                const uint8_t* m = msgs + p * a.msg_stride;
                const uint4* src = reinterpret_cast<const uint4*>(m + kk * B + 64 * q);
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) u[ch] = __ldg(src + ch);
                sc = __ldg(reinterpret_cast<const float2*>(m + a.scal_off + kk * 8));
            } else {
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) u[ch] = make_uint4(0, 0, 0, 0);
            }
            float2 w[32];
            decode_block<L>(u, sc, live, q, c, w);
            if (!live) continue;
            if (q == 0 && !scalars_ok(sc.x, sc.y)) raise_flag(a.flags, 2);
            const uint64_t k = a.blk0 + kk;
            const int valid = clamp_valid((int64_t)a.S - (int64_t)(k * B), (int64_t)a.n - (int64_t)(p * a.S + k * B), B);
            const int vok = (sizeof(TOut) == 2 && a.P > 1 && (a.S & 15)) ? (a.vec_ok ? 1 : 0) : a.vec_ok;
            store_decoded<L, TOut>(out + (p * a.S + k * B), q, valid, vok, w);
        }
    } else {
#pragma unroll
        for (int i = 0; i < NS - 1; ++i) issue(t + i * stride, i);
        int cur = 0;
        for (; t < ntiles; t += stride) {
            __syncwarp();  // every lane is done with the stage about to be refilled
            issue(t + (NS - 1) * stride, cur == 0 ? NS - 1 : cur - 1);
            const uint32_t p = tps.div(t);
            const uint64_t kk = (uint64_t)(t - p * tps.d) * G + g;
            const bool live = kk < a.nblk;
            cp_wait<NS - 1>();
            __syncwarp();  // the other lanes' copies of this tile are visible
            const uint4* sb = stage_base + cur * K::STAGE_U4;
            cur = cur == NS - 1 ? 0 : cur + 1;
            uint4 u[4];
            float2 sc = make_float2(1.0f, 1.0f);
            if (live) {
                read_lane_codes<L>(sb, g, q, u);
                sc = reinterpret_cast<const float2*>(sb + 128)[g];
            } else {
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) u[ch] = make_uint4(0, 0, 0, 0);
            }
            float2 w[32];
            decode_block<L>(u, sc, live, q, c, w);
            if (!live) continue;
            if (q == 0 && !scalars_ok(sc.x, sc.y)) raise_flag(a.flags, 2);
            const uint64_t k = a.blk0 + kk;
            const int valid = clamp_valid((int64_t)a.S - (int64_t)(k * B), (int64_t)a.n - (int64_t)(p * a.S + k * B), B);
            // 256-bit bf16 stores need 32-byte aligned shard starts (S % 16), fp32 ones S % 8 (vec_ok)
            const int vok = (sizeof(TOut) == 2 && a.P > 1 && (a.S & 15)) ? (a.vec_ok ? 1 : 0) : a.vec_ok;
            store_decoded<L, TOut>(out + (p * a.S + k * B), q, valid, vok, w);
        }
    }
}

// --------------------------------------------------------------------- K3 --------
// One warp per tile of G blocks (non-persistent), ranks walked in ascending order with the
// next rank's codes copied while the current one is decoded.
template <int L>
struct K3X {
    static constexpr int B = 64 * L, G = 32 / L;
    static constexpr int STAGES = 3;
    static constexpr int STAGE_U4 = K2X<L>::STAGE_U4;
    static constexpr int WARP_U4 = STAGES * STAGE_U4 + 128;  // + the re-encoded codes, staged
    static constexpr size_t SMEM = (size_t)kWarps * WARP_U4 * 16;
};

// K3 holds the running sum and one decoded rank at once (2 x 64 values): 3 CTAs per SM
constexpr int kMinCtasK3 = 3;

template <int L, typename TAcc, bool P2>
__device__ __forceinline__ void k3x_warp(const uint8_t* __restrict__ msgs, uint8_t* __restrict__ out_msg,
                                         TAcc* __restrict__ acc_out, const ShardArgs& a, const CodecConsts& c,
                                         uint64_t cta) {
    using K = K3X<L>;
    using D = DecPlan<L>;
    using Plan = typename D::Enc;
    constexpr int B = K::B, G = K::G, NS = K::STAGES;
    extern __shared__ uint4 smem_dyn[];
    const int lane = threadIdx.x & 31, q = lane & (L - 1), g = lane / L, warp = threadIdx.x >> 5;
    uint4* stage_base = smem_dyn + (size_t)warp * K::WARP_U4;
    uint4* code_buf = stage_base + NS * K::STAGE_U4;
    const uint64_t kk0 = (cta * kWarps + warp) * G;
    if (kk0 >= a.nblk) return;  // warp-uniform
    const uint64_t kk = kk0 + g;
    const bool live = kk < a.nblk;
    const int valid = live ? clamp_valid((int64_t)a.S - (int64_t)((a.blk0 + kk) * B), (int64_t)B, B) : 0;
    auto msg_of = [&](uint32_t r) -> const uint8_t* { return a.nsrc ? a.src[r] : msgs + r * a.msg_stride; };
    auto issue = [&](uint32_t r, int stage) {
        if (r < a.P) stage_tile<L>(stage_base + stage * K::STAGE_U4, msg_of(r), kk0, a.nblk, a.scal_off, lane);
        cp_async_commit();
    };
#pragma unroll
    for (int i = 0; i < NS - 1; ++i) issue(i, i);
    float2 acc[32];
    bool ok = true;
    int cur = 0;
    if constexpr (P2) {
        // two ranks (TP = 2): both tiles are staged by the prologue; the two decodes are one
        // straight-line block the scheduler interleaves (no wait / barrier between them)
        cp_wait<0>();
        __syncwarp();
        uint4 u0[4], u1[4];
        float2 sc0 = make_float2(1.0f, 1.0f), sc1 = make_float2(1.0f, 1.0f);
        if (live) {
            read_lane_codes<L>(stage_base, g, q, u0);
            sc0 = reinterpret_cast<const float2*>(stage_base + 128)[g];
            read_lane_codes<L>(stage_base + K::STAGE_U4, g, q, u1);
            sc1 = reinterpret_cast<const float2*>(stage_base + K::STAGE_U4 + 128)[g];
        } else {
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) u0[ch] = u1[ch] = make_uint4(0, 0, 0, 0);
        }
        ok = scalars_ok(sc0.x, sc0.y) && scalars_ok(sc1.x, sc1.y);
        float2 y[32];
        decode_block<L>(u0, sc0, live, q, c, acc);  // acc = decompress(rank 0) (collective.cpp:96)
        decode_block<L>(u1, sc1, live, q, c, y);
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[i] = __fadd2_rn(acc[i], y[i]);  // acc[i] += part[i] (:99)
    }
    for (uint32_t r = 0; !P2 && r < a.P; ++r) {
        __syncwarp();  // every lane is done with the stage about to be refilled
        issue(r + NS - 1, cur == 0 ? NS - 1 : cur - 1);
        cp_wait<NS - 1>();
        __syncwarp();  // the other lanes' copies of this rank's tile are visible
        const uint4* sb = stage_base + cur * K::STAGE_U4;
        cur = cur == NS - 1 ? 0 : cur + 1;
        uint4 u[4];
        float2 sc = make_float2(1.0f, 1.0f);
        if (live) {
            read_lane_codes<L>(sb, g, q, u);
            sc = reinterpret_cast<const float2*>(sb + 128)[g];
        } else {
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) u[ch] = make_uint4(0, 0, 0, 0);
        }
        ok &= scalars_ok(sc.x, sc.y);
        float2 y[32];
        decode_block<L>(u, sc, live, q, c, y);
        if (r == 0) {
#pragma unroll
            for (int i = 0; i < 32; ++i) acc[i] = y[i];  // acc = decompress(rank 0) (collective.cpp:96)
        } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) acc[i] = __fadd2_rn(acc[i], y[i]);  // acc[i] += part[i] (:99)
        }
    }
    // positions past the shard end are zero padding of the re-encoded slice (collective.cpp:101)
    const int lo = D::lane_off(q);
    auto zero_tail = [&](float2 (&v)[32]) {
        if (__any_sync(kFull, valid < B)) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const int pos = lo + D::vec_pos(i >> 2) + 2 * (i & 3);
                if (pos >= valid) v[i].x = 0.0f;
                if (pos + 1 >= valid) v[i].y = 0.0f;
            }
        }
    };
    zero_tail(acc);
    if (acc_out && live) store_decoded<L, TAcc>(acc_out + (a.blk0 + kk) * B, q, valid, a.vec_ok, acc);
    if (out_msg == nullptr) {  // reduce-scatter: the fp32 sum is the product
        if (live && q == 0 && !ok) raise_flag(a.flags, 2);
        return;
    }
    // ---- re-encode: K1's operations on the fp32 sum (Plan = K1's order on this layout)
    // out-of-range path: recompute the plain sum from the messages (direct loads)
    auto reload = [&](float2 (&v)[32]) {
        for (uint32_t r = 0; r < a.P; ++r) {
            const uint8_t* m = msg_of(r);
            float2 sc = make_float2(1.0f, 1.0f);
            uint4 u[4];
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) u[ch] = make_uint4(0, 0, 0, 0);
            if (live) {
                sc = __ldg(reinterpret_cast<const float2*>(m + a.scal_off + kk * 8));
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) u[ch] = __ldg(reinterpret_cast<const uint4*>(m + kk * B + 64 * q + 16 * ch));
            }
            float2 y[32];
            decode_block<L>(u, sc, live, q, c, y);
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = r == 0 ? y[i] : __fadd2_rn(v[i], y[i]);
        }
        zero_tail(v);
    };
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = b0_f32(acc[i]);
    float alpha, s;
    double ss;
    encode<L, Plan>(acc, q, c, alpha, s, ss, reload);
    uint4 cv[4];
    pack_codes<Plan>(acc, cv);
    // codes staged through shared memory and stored coalesced (as K1)
    const int u0 = (g * B + Plan::lane_off(q)) / 16;
#pragma unroll
    for (int u = 0; u < 4; ++u) code_buf[swz_unit(u0 + u)] = cv[u];
    __syncwarp();
    uint4 ov[4];
#pragma unroll
    for (int c4 = 0; c4 < 4; ++c4) ov[c4] = code_buf[swz_unit(32 * c4 + lane)];
    const uint32_t nd = a.ndst ? a.ndst : 1;
    for (uint32_t d = 0; d < nd; ++d) {  // peer mode: the same message into every rank's buffer
        uint8_t* o = a.ndst ? a.dst[d] : out_msg;
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {
            const int u = 32 * c4 + lane;
            if (kk0 + (uint64_t)((16 * u) / B) < a.nblk) st16_na(o + kk0 * B + 16 * (uint64_t)u, ov[c4]);
        }
        if (live && q == 0) *reinterpret_cast<float2*>(o + a.scal_off + kk * 8) = make_float2(alpha, s);
    }
    if (live && q == 0 && !ok) raise_flag(a.flags, 2);
}

template <int L, typename TAcc, bool P2>
__global__ void __launch_bounds__(kWarps * 32, kMinCtasK3)
    k3x(const uint8_t* __restrict__ msgs, uint8_t* __restrict__ out_msg, TAcc* __restrict__ acc_out, ShardArgs a,
        CodecConsts c) {
    grid_dep_wait();
    k3x_warp<L, TAcc, P2>(msgs, out_msg, acc_out, a, c, blockIdx.x);
}

}  // namespace xk
}  // namespace taco_dev
