// taco_tile.cuh -- "tile" variants of K1 / K2 / K3 for E4M3 and 64 <= B <= 512 (the
// block sizes of the north-star sweep; B = 256 is the default).
//
// Why a second geometry.  The r1a profile (profiles/README.md) showed the register-only
// kernels issue/latency bound: 4 warps per scheduler (128 registers) and 2 SHFL per
// element for the lane butterflies.  Here a block of B = 2^NB values is owned by 8 lanes
// with E = B/8 values each (32 at B = 256, ~70 registers, 5 CTAs x 4 warps per SM), and
// the butterflies over the three "lane" bits run in registers after a transpose through
// shared memory (one STS.128 + one LDS.128 per 4 values instead of 3 SHFL per value).
//
//   staging   tiles of 4 blocks are fetched with the TMA engine (cp.async.bulk 1D, one
//             instruction per tile, completion on an mbarrier), D tiles in flight per warp
//   phase 1   lane q of block g holds positions  r[0..2] | q<<3 | r[3..]<<6   (r = register)
//             -> butterflies over position bits 0,1,2,6,7,.. (pair bit fused with the
//                bf16 unpack: add/sub.rn.f32.bf16 = FHADD.BF16, one rounding, exact
//                operands); fp64 sum of squares from cvt.f64.bf16
//   transpose fp32 tile through a per-warp buffer, 16-byte chunks XOR-swizzled so both the
//             phase-1 writes and the phase-2 reads are bank-conflict free
//   phase 2   lane q holds positions r[0..LO-1] | q[..]<<LO | r[LO..LO+2]<<3 | q[..]<<6
//             -> butterflies over bits 3,4,5, block max over the 8 lanes, quantise
//   output    codes staged through the same buffer and written with coalesced 128-bit
//             stores; (alpha, s) by one lane per block.
//
// Butterfly order: bits 0,1,2,6,7,..,3,4,5.  For B = 256 this is exactly the order of
// the register kernels' Geo<256, 32, 8> (taco_device.cuh), so K2 here and the K3 decode
// agree bit for bit.  Every stage is the reference's (a+b, a-b) (transform.cpp:46-55).
#pragma once

#include "taco_kernels.cuh"

namespace taco_dev {
namespace tile {

// --------------------------------------------------------------- PTX helpers ---
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
#ifndef TACO_TMA_ISSUE_FENCE
#define TACO_TMA_ISSUE_FENCE 0  // proxy fence before every TMA refill: only needed after generic
                                // writes to the slot (ragged tiles fence there); -3.5 % K2 fp32
#endif
#ifndef TACO_K2_MIN_CTAS
#define TACO_K2_MIN_CTAS 5
#endif
#ifndef TACO_K2_SUB
#define TACO_K2_SUB 1  // 4-block sub-tiles per K2 TMA stage
#endif

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "TACO_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra TACO_DONE;\n\t"
        "bra TACO_WAIT;\n"
        "TACO_DONE:\n\t}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 1D bulk copy global -> shared through the TMA engine (UBLKCP); 16-byte aligned, size % 16 == 0
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// mixed-precision adds (sm_100): fp32 result of a bf16 / f16 operand and an fp32 operand,
// one rounding -- identical to the fp32 add of the widened (exact) operand
__device__ __forceinline__ float add_bf16(uint32_t h16, float c) {
    float d;
    asm("add.rn.f32.bf16 %0, %1, %2;" : "=f"(d) : "h"((unsigned short)h16), "f"(c));
    return d;
}
__device__ __forceinline__ float sub_bf16(uint32_t h16, float c) {
    float d;
    asm("sub.rn.f32.bf16 %0, %1, %2;" : "=f"(d) : "h"((unsigned short)h16), "f"(c));
    return d;
}
__device__ __forceinline__ double bf16_to_f64(uint32_t h16) {
    double d;
    asm("cvt.f64.bf16 %0, %1;" : "=d"(d) : "h"((unsigned short)h16));
    return d;
}
__device__ __forceinline__ float add_f16(uint32_t h16, float c) {
    float d;
    asm("add.rn.f32.f16 %0, %1, %2;" : "=f"(d) : "h"((unsigned short)h16), "f"(c));
    return d;
}
__device__ __forceinline__ float sub_f16(uint32_t h16, float c) {
    float d;
    asm("sub.rn.f32.f16 %0, %1, %2;" : "=f"(d) : "h"((unsigned short)h16), "f"(c));
    return d;
}
__device__ __forceinline__ float f16_to_f32(uint32_t h16) {
    float d;
    asm("cvt.f32.f16 %0, %1;" : "=f"(d) : "h"((unsigned short)h16));
    return d;
}
// two E4M3 codes (low 16 bits) -> f16x2 (exact)
__device__ __forceinline__ uint32_t e4m3x2_to_f16x2(uint32_t two) {
    const __half2_raw h = __nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)(two & 0xffffu), __NV_E4M3);
    return (uint32_t)h.x | ((uint32_t)h.y << 16);
}

// ----------------------------------------------------------------- geometry ---
constexpr int kLanes = 8;       // lanes per block
constexpr int kBlocks = 4;      // blocks per warp tile
constexpr int kTileWarps = 4;   // warps per CTA

template <int NB>
struct TG {
    static_assert(NB >= 6 && NB <= 9, "tile kernels cover 64 <= B <= 512");
    static constexpr int B = 1 << NB;
    static constexpr int NE = NB - 3;  // log2 values per lane
    static constexpr int E = 1 << NE;
    static constexpr int E2 = E / 2;
    static constexpr int TILE = kBlocks * B;
    static constexpr int LO = NE - 3;  // phase-2 contiguous low bits
    static constexpr int VW = 1 << LO;  // phase-2 run length (elements)
    // phase 1: register r of lane q -> block position
    __host__ __device__ static constexpr int pos1(int r, int q) { return (r & 7) | (q << 3) | ((r >> 3) << 6); }
    // phase 2: register r of lane q -> block position
    __host__ __device__ static constexpr int pos2(int r, int q) {
        return (r & (VW - 1)) | ((q & ((1 << (3 - LO)) - 1)) << LO) | ((r >> LO) << 3) | ((q >> (3 - LO)) << 6);
    }
};

// XOR swizzle of 16-byte chunk indices: the chunk's bank group (low 3 bits) absorbs the
// XOR-fold of every higher 3-bit group.  Linear over GF(2), so lane and register parts of
// an index (disjoint bits) can be swizzled separately and XOR-ed.
__host__ __device__ constexpr uint32_t swz(uint32_t k) {
    return k ^ (((k >> 3) ^ (k >> 6) ^ (k >> 9) ^ (k >> 12)) & 7u);
}

// ------------------------------------------------------------- butterflies ----
// packed register stages over float2-index bits [lo, hi)
template <int E2, int LO_BIT, int HI_BIT>
__device__ __forceinline__ void stages(float2 (&w)[E2]) {
    const float2 neg1 = make_float2(-1.0f, -1.0f);
#pragma unroll
    for (int b = LO_BIT; b < HI_BIT; ++b) {
        const int h = 1 << b;
#pragma unroll
        for (int i = 0; i < E2; ++i) {
            if ((i & h) == 0) {
                const float2 a = w[i], c = w[i + h];
                w[i] = __fadd2_rn(a, c);
                w[i + h] = __ffma2_rn(c, neg1, a);  // a - c, one rounding
            }
        }
    }
}

// same, over float2-index bits HI_BIT-1 down to LO_BIT (the last butterfly then writes
// the adjacent pairs w[2c], w[2c+1] that one 128-bit store takes)
template <int E2, int LO_BIT, int HI_BIT>
__device__ __forceinline__ void stages_rev(float2 (&w)[E2]) {
    const float2 neg1 = make_float2(-1.0f, -1.0f);
#pragma unroll
    for (int b = HI_BIT - 1; b >= LO_BIT; --b) {
        const int h = 1 << b;
#pragma unroll
        for (int i = 0; i < E2; ++i) {
            if ((i & h) == 0) {
                const float2 a = w[i], c = w[i + h];
                w[i] = __fadd2_rn(a, c);
                w[i + h] = __ffma2_rn(c, neg1, a);
            }
        }
    }
}

// the pair bit (position bit 3 in the phase-2 layout of B = 64)
template <int E2>
__device__ __forceinline__ void pair_stage(float2 (&w)[E2]) {
#pragma unroll
    for (int i = 0; i < E2; ++i) w[i] = make_float2(w[i].x + w[i].y, w[i].x - w[i].y);
}

template <typename T>
struct InTraits;
template <>
struct InTraits<__nv_bfloat16> {
    static constexpr int WORDS8 = 4;  // u32 words per 8 elements
};
template <>
struct InTraits<float> {
    static constexpr int WORDS8 = 8;
};

// ------------------------------------------------------------ tile transpose ---
// Phase-1 registers -> fp32 tile buffer (natural position g*B + pos, swizzled chunks).
template <int NB>
__device__ __forceinline__ void xpose_write(float* xb, const float2 (&w)[TG<NB>::E2], int g, int q) {
    using Gm = TG<NB>;
    const uint32_t kl = swz((uint32_t)(g * Gm::B + Gm::pos1(0, q)) >> 2);
#pragma unroll
    for (int c = 0; c < Gm::E / 4; ++c) {
        const uint32_t kr = swz((uint32_t)Gm::pos1(4 * c, 0) >> 2);
        *reinterpret_cast<float4*>(xb + 4 * (kl ^ kr)) = make_float4(w[2 * c].x, w[2 * c].y, w[2 * c + 1].x,
                                                                     w[2 * c + 1].y);
    }
}

// fp32 tile buffer -> phase-2 registers
template <int NB>
__device__ __forceinline__ void xpose_read(const float* xb, float2 (&w)[TG<NB>::E2], int g, int q) {
    using Gm = TG<NB>;
    const uint32_t p0 = (uint32_t)(g * Gm::B + Gm::pos2(0, q));
    const uint32_t kl = swz(p0 >> 2);
    if constexpr (Gm::VW >= 4) {
#pragma unroll
        for (int c = 0; c < Gm::E / 4; ++c) {
            const uint32_t kr = swz((uint32_t)Gm::pos2(4 * c, 0) >> 2);
            const float4 v = *reinterpret_cast<const float4*>(xb + 4 * (kl ^ kr));
            w[2 * c] = make_float2(v.x, v.y);
            w[2 * c + 1] = make_float2(v.z, v.w);
        }
    } else if constexpr (Gm::VW == 2) {
#pragma unroll
        for (int c = 0; c < Gm::E2; ++c) {
            const uint32_t pr = (uint32_t)Gm::pos2(2 * c, 0);
            const uint32_t kr = swz(pr >> 2);
            // word offset inside the chunk: bits 0,1 of (p0 | pr) -- p0 and pr are disjoint
            w[c] = *reinterpret_cast<const float2*>(xb + 4 * (kl ^ kr) + ((p0 | pr) & 3));
        }
    } else {
#pragma unroll
        for (int c = 0; c < Gm::E2; ++c) {
            float v2[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t pr = (uint32_t)Gm::pos2(2 * c + h, 0);
                v2[h] = xb[4 * (kl ^ swz(pr >> 2)) + ((p0 | pr) & 3)];
            }
            w[c] = make_float2(v2[0], v2[1]);
        }
    }
}

// ------------------------------------------------------------------- K1 ------
template <int NB, typename TIn>
struct K1T {
    using Gm = TG<NB>;
    static constexpr int D = NB >= 9 ? 2 : 3;                      // tiles in flight per warp
    static constexpr int STAGE = Gm::TILE * (int)sizeof(TIn);       // bytes per staged tile
    static constexpr int XB = Gm::TILE * 4;                         // fp32 transpose buffer
    static constexpr int WARP_BYTES = D * STAGE + XB;
    static constexpr size_t SMEM = (size_t)kTileWarps * WARP_BYTES + (size_t)kTileWarps * D * 8;
};

// Quantise the phase-2 registers of one block (8-lane group) and return the scalars.
// ss: block sum of squares (all lanes), p2: the exact pre-scale used (1 unless huge).
template <int NB>
__device__ __forceinline__ void tile_quantise(float2 (&w)[TG<NB>::E2], double ss, float p2, const CodecConsts& c,
                                              float& alpha, float& s) {
    using Gm = TG<NB>;
#if TACO_FAST_SCALARS_REG
    alpha = block_alpha_fast(ss, c);
#else
    alpha = block_alpha(ss, c);
#endif
    float m[Gm::E2];
#pragma unroll
    for (int i = 0; i < Gm::E2; ++i) m[i] = fmaxf(fabsf(w[i].x), fabsf(w[i].y));
#pragma unroll
    for (int h = 1; h < Gm::E2; h <<= 1)
#pragma unroll
        for (int i = 0; i + h < Gm::E2; i += 2 * h) m[i] = fmaxf(m[i], m[i + h]);
    float ymax = m[0];
#pragma unroll
    for (int o = 1; o < kLanes; o <<= 1) ymax = fmaxf(ymax, __shfl_xor_sync(kFull, ymax, o));
    double k;
#if TACO_FAST_SCALARS_REG
    block_scale_fast((double)ymax, alpha, p2, c, s, k);
#else
    block_scale((double)ymax, alpha, p2, c, s, k);
#endif
    mul_wide<Gm::E2>(w, k);
}

// Phase-2 codes -> code staging (bytes, natural order, 16-byte chunks swizzled) in xb.
template <int NB>
__device__ __forceinline__ void stage_codes(uint8_t* cb, const float2 (&w)[TG<NB>::E2], int g, int q) {
    using Gm = TG<NB>;
    const uint32_t p0 = (uint32_t)(g * Gm::B + Gm::pos2(0, q));
#pragma unroll
    for (int mid = 0; mid < 8; ++mid) {
        const uint32_t pr = (uint32_t)Gm::pos2(mid * Gm::VW, 0);
        const uint32_t p = p0 | pr;
        uint8_t* dst = cb + 16 * swz(p >> 4) + (p & 15);
        const float2* v = &w[mid * Gm::VW / 2];
        if constexpr (Gm::VW == 8) {
            *reinterpret_cast<uint2*>(dst) = make_uint2(enc2<0>(v[0]) | (enc2<0>(v[1]) << 16),
                                                        enc2<0>(v[2]) | (enc2<0>(v[3]) << 16));
        } else if constexpr (Gm::VW == 4) {
            *reinterpret_cast<uint32_t*>(dst) = enc2<0>(v[0]) | (enc2<0>(v[1]) << 16);
        } else if constexpr (Gm::VW == 2) {
            *reinterpret_cast<uint16_t*>(dst) = (uint16_t)enc2<0>(v[0]);
        } else {
            // VW == 1: registers 2i, 2i+1 are positions 8*mid apart -- one code each
            const uint32_t two = enc2<0>(w[mid / 2]);
            *dst = (uint8_t)((mid & 1) ? (two >> 8) : two);
        }
    }
}

// Load + rotate one staged tile (natural order, TIn) into phase-2 registers.
// Returns the block's sum of squares (reduced over the 8 lanes) and the pre-scale p2.
template <int NB, typename TIn>
__device__ __forceinline__ void tile_rotate(const unsigned char* st, float* xb, float2 (&w)[TG<NB>::E2], int g,
                                            int q, const CodecConsts& c, double& ss, float& p2) {
    using Gm = TG<NB>;
    constexpr int NTOP = Gm::E / 8;  // 8-element runs per lane
    const TIn* src = reinterpret_cast<const TIn*>(st) + g * Gm::B + Gm::pos1(0, q);
    // raw words of the lane's runs (run j = positions j*64 + q*8 + 0..7)
    uint32_t raw[NTOP * InTraits<TIn>::WORDS8];
#pragma unroll
    for (int j = 0; j < NTOP; ++j) {
        const uint4* p = reinterpret_cast<const uint4*>(src + j * 64);
#pragma unroll
        for (int h = 0; h < InTraits<TIn>::WORDS8 / 4; ++h) {
            const uint4 u = p[h];
            raw[j * InTraits<TIn>::WORDS8 + 4 * h + 0] = u.x;
            raw[j * InTraits<TIn>::WORDS8 + 4 * h + 1] = u.y;
            raw[j * InTraits<TIn>::WORDS8 + 4 * h + 2] = u.z;
            raw[j * InTraits<TIn>::WORDS8 + 4 * h + 3] = u.w;
        }
    }
    // fp64 sum of squares (x^2 exact in double), four chains
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < Gm::E2; ++i) {
        double d0, d1;
        if constexpr (sizeof(TIn) == 2) {
            d0 = bf16_to_f64(raw[i] & 0xffffu);
            d1 = bf16_to_f64(raw[i] >> 16);
        } else {
            d0 = (double)__uint_as_float(raw[2 * i]);
            d1 = (double)__uint_as_float(raw[2 * i + 1]);
        }
        acc[(2 * i) & 3] = fma(d0, d0, acc[(2 * i) & 3]);
        acc[(2 * i + 1) & 3] = fma(d1, d1, acc[(2 * i + 1) & 3]);
    }
    double sl = (acc[0] + acc[1]) + (acc[2] + acc[3]);
    // Exact power-of-two pre-scale only where the butterfly could overflow fp32
    // (lane-local test, warp-uniform branch; NaN/Inf also take it).
    const bool huge = !(sl < 0x1p150);
    p2 = 1.0f;
    ss = sl;
#pragma unroll
    for (int o = 1; o < kLanes; o <<= 1) ss += __shfl_xor_sync(kFull, ss, o);
    if (__any_sync(kFull, huge)) {
        p2 = pow2_near(block_alpha(ss, c));
#pragma unroll
        for (int i = 0; i < Gm::E2; ++i) {
            float x0, x1;
            if constexpr (sizeof(TIn) == 2) {
                x0 = __uint_as_float(raw[i] << 16);
                x1 = __uint_as_float(raw[i] & 0xffff0000u);
            } else {
                x0 = __uint_as_float(raw[2 * i]);
                x1 = __uint_as_float(raw[2 * i + 1]);
            }
            x0 *= p2;
            x1 *= p2;
            w[i] = make_float2(x0 + x1, x0 - x1);
        }
    } else {
#pragma unroll
        for (int i = 0; i < Gm::E2; ++i) {
            if constexpr (sizeof(TIn) == 2) {
                const float x1 = __uint_as_float(raw[i] & 0xffff0000u);
                w[i] = make_float2(add_bf16(raw[i] & 0xffffu, x1), sub_bf16(raw[i] & 0xffffu, x1));
            } else {
                const float x0 = __uint_as_float(raw[2 * i]), x1 = __uint_as_float(raw[2 * i + 1]);
                w[i] = make_float2(x0 + x1, x0 - x1);
            }
        }
    }
    // phase 1: position bits 1, 2, 6, 7, .. (float2 index bits 0 .. NE-2)
    stages_rev<Gm::E2, 0, Gm::NE - 1>(w);
    __syncwarp();  // the transpose buffer is free (previous tile fully read out)
    xpose_write<NB>(xb, w, g, q);
    __syncwarp();
    xpose_read<NB>(xb, w, g, q);
    // phase 2: position bits 3, 4, 5
    if constexpr (Gm::LO == 0) {
        pair_stage<Gm::E2>(w);
        stages<Gm::E2, 0, 2>(w);
    } else {
        stages<Gm::E2, Gm::LO - 1, Gm::LO + 2>(w);
    }
}

// Zero-padded natural-order copy of a ragged / unaligned tile into the staging slot.
template <int NB, typename TIn>
__device__ __forceinline__ void fill_slow(unsigned char* st, const TIn* __restrict__ x, const ShardArgs& a,
                                          uint64_t p, uint64_t kk0, int lane) {
    using Gm = TG<NB>;
    TIn* d = reinterpret_cast<TIn*>(st);
    for (int i = lane; i < Gm::TILE; i += 32) {
        const uint64_t kk = kk0 + (uint64_t)(i >> NB);
        const int pos = i & (Gm::B - 1);
        float v = 0.0f;
        if (kk < a.nblk) {
            const uint64_t k = a.blk0 + kk;
            const int valid = clamp_valid((int64_t)a.S - (int64_t)(k * Gm::B),
                                          (int64_t)a.n - (int64_t)(p * a.S + k * Gm::B), Gm::B);
            if (pos < valid) v = to_f32(x[p * a.S + k * Gm::B + pos]);
        }
        store_one(d + i, v);
    }
}

template <int NB, typename TIn>
__global__ void __launch_bounds__(kTileWarps * 32, 5)
    k_compress_tile(const TIn* __restrict__ x, uint8_t* __restrict__ msgs, ShardArgs a, CodecConsts c, FastDiv tps) {
    using Gm = TG<NB>;
    using Cf = K1T<NB, TIn>;
    constexpr int D = Cf::D, B = Gm::B;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 3, q = lane & 7;
    unsigned char* stage = smem + warp * Cf::WARP_BYTES;
    float* xb = reinterpret_cast<float*>(stage + D * Cf::STAGE);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kTileWarps * Cf::WARP_BYTES) + warp * D;
    if (lane == 0) {
#pragma unroll
        for (int d = 0; d < D; ++d) mbar_init(&bars[d], 1);
        fence_mbar_init();
    }
    __syncwarp();
    const uint32_t ntiles = a.P * tps.d;
    const uint32_t stride = gridDim.x * kTileWarps;
    const uint32_t t0 = blockIdx.x * kTileWarps + warp;

    auto issue = [&](uint32_t t, int slot) {  // lane 0
        const uint32_t p = tps.div(t);
        const uint64_t kk0 = (uint64_t)(t - p * tps.d) * kBlocks;
        if (tile_full<B, kBlocks>(a, p, kk0)) {
#if TACO_TMA_ISSUE_FENCE
            fence_proxy_async();
#endif
            mbar_arrive_tx(&bars[slot], Cf::STAGE);
            bulk_g2s(stage + slot * Cf::STAGE, x + (p * a.S + (a.blk0 + kk0) * B), Cf::STAGE, &bars[slot]);
        } else {
            mbar_arrive(&bars[slot]);  // keeps the slot's phase sequence; filled by fill_slow
        }
    };
    grid_dep_wait();
    if (lane == 0) {
#pragma unroll
        for (int d = 0; d < D - 1; ++d)
            if (t0 + d * stride < ntiles) issue(t0 + d * stride, d);
    }
    int slot = 0;
    uint32_t par = 0;  // bit d = parity to wait for on slot d
    for (uint32_t t = t0; t < ntiles; t += stride) {
        const uint32_t tn = t + (D - 1) * stride;
        if (lane == 0 && tn < ntiles) issue(tn, slot == 0 ? D - 1 : slot - 1);
        mbar_wait(&bars[slot], (par >> slot) & 1);
        par ^= 1u << slot;
        const uint32_t p = tps.div(t);
        const uint64_t kk0 = (uint64_t)(t - p * tps.d) * kBlocks;
        unsigned char* st = stage + slot * Cf::STAGE;
        const bool full = tile_full<B, kBlocks>(a, p, kk0);
        if (!full) {
            fill_slow<NB, TIn>(st, x, a, p, kk0, lane);
            __syncwarp();
            fence_proxy_async();  // these generic writes before any later TMA write of the slot
        }
        float2 w[Gm::E2];
        double ss;
        float p2;
        tile_rotate<NB, TIn>(st, xb, w, g, q, c, ss, p2);
        float alpha, s;
        tile_quantise<NB>(w, ss, p2, c, alpha, s);
        __syncwarp();  // every lane has read its phase-2 values out of xb
        uint8_t* cb = reinterpret_cast<uint8_t*>(xb);
        stage_codes<NB>(cb, w, g, q);
        __syncwarp();
        const uint64_t kk = kk0 + g;
        // coalesced copy-out: chunk j (16 codes) of the tile belongs to block j*16/B
        // (peer all-gather: the same message to every rank)
        const uint32_t nd = a.bcast ? a.ndst : 1;
        for (uint32_t d = 0; d < nd; ++d) {
            uint8_t* m = a.bcast ? a.dst[d] : shard_msg(msgs, a, p);
#pragma unroll
            for (int j = lane; j < Gm::TILE / 16; j += 32) {
                const uint4 v = *reinterpret_cast<const uint4*>(cb + 16 * swz((uint32_t)j));
                if (full || kk0 + (uint64_t)((j * 16) >> NB) < a.nblk)
                    *reinterpret_cast<uint4*>(m + kk0 * B + 16 * (uint64_t)j) = v;
            }
            if (q == 0 && kk < a.nblk) *reinterpret_cast<float2*>(m + a.scal_off + kk * 8) = make_float2(alpha, s);
        }
        if (q == 0 && kk < a.nblk && !isfinite(ss)) raise_flag(a.flags, 1);
        slot = slot + 1 == D ? 0 : slot + 1;
    }
}

// ------------------------------------------------------------------- K2 ------
template <int NB, typename TOut>
struct K2T {
    using Gm = TG<NB>;
    static constexpr int D = 3;
    static constexpr int SUB = TACO_K2_SUB;                     // 4-block sub-tiles per TMA stage
    static constexpr int KB = SUB * kBlocks;                    // blocks per stage
    static constexpr int STAGE = SUB * (Gm::TILE + kBlocks * 8);  // [codes of KB blocks][their (alpha, s)]
    static constexpr int XB = Gm::TILE * 4;
    static constexpr int WARP_BYTES = D * STAGE + XB;
    static constexpr size_t SMEM = (size_t)kTileWarps * WARP_BYTES + (size_t)kTileWarps * D * 8;
};

// Decode one staged tile (codes in natural order) into phase-2 registers and apply the
// per-block dequantisation multiplier: out = H(table[c]) * float(s*norm/alpha).
// Shared by K2 and K3 so both produce bit-identical fp32 slices.
template <int NB>
__device__ __forceinline__ bool tile_decode(const uint8_t* codes, float2 sc, float* xb, float2 (&w)[TG<NB>::E2],
                                            int g, int q, const CodecConsts& c) {
    using Gm = TG<NB>;
    constexpr int NTOP = Gm::E / 8;
    const uint8_t* src = codes + g * Gm::B + Gm::pos1(0, q);
#pragma unroll
    for (int j = 0; j < NTOP; ++j) {
        const uint2 u = *reinterpret_cast<const uint2*>(src + j * 64);
        const uint32_t wd[2] = {u.x, u.y};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t lo = e4m3x2_to_f16x2(wd[h]), hi = e4m3x2_to_f16x2(wd[h] >> 16);
            const float l1 = f16_to_f32(lo >> 16), h1 = f16_to_f32(hi >> 16);
            w[j * 4 + 2 * h] = make_float2(add_f16(lo & 0xffffu, l1), sub_f16(lo & 0xffffu, l1));
            w[j * 4 + 2 * h + 1] = make_float2(add_f16(hi & 0xffffu, h1), sub_f16(hi & 0xffffu, h1));
        }
    }
    stages_rev<Gm::E2, 0, Gm::NE - 1>(w);
    __syncwarp();
    xpose_write<NB>(xb, w, g, q);
    __syncwarp();
    xpose_read<NB>(xb, w, g, q);
    if constexpr (Gm::LO == 0) {
        pair_stage<Gm::E2>(w);
        stages<Gm::E2, 0, 2>(w);
    } else {
        stages<Gm::E2, Gm::LO - 1, Gm::LO + 2>(w);
    }
#if TACO_FAST_SCALARS_REG
    // s * norm / alpha with a Newton reciprocal (2 steps: the float rounding of the
    // multiplier matches the correctly rounded quotient except in double-rounding cases)
    mul_wide<Gm::E2>(w, (double)sc.y * c.norm * rcp_newton((double)sc.x, 2));
#else
    mul_wide<Gm::E2>(w, block_dequant(sc.x, sc.y, c));
#endif
    return scalars_ok(sc.x, sc.y);
}

// Phase-2 fp32 values -> output staging (natural order, 16-byte chunks swizzled) in xb.
template <int NB, typename TOut>
__device__ __forceinline__ void stage_out(unsigned char* ob, const float2 (&w)[TG<NB>::E2], int g, int q) {
    using Gm = TG<NB>;
    constexpr int EPC = 16 / (int)sizeof(TOut);  // elements per 16-byte chunk
    const uint32_t p0 = (uint32_t)(g * Gm::B + Gm::pos2(0, q));
    if constexpr (Gm::VW >= 2) {
#pragma unroll
        for (int mid = 0; mid < 8; ++mid) {
            const uint32_t pr = (uint32_t)Gm::pos2(mid * Gm::VW, 0);
            // a run may span several 16-byte chunks (fp32, VW = 8): one store per chunk
            constexpr int PIECE = Gm::VW < EPC ? Gm::VW : EPC;
#pragma unroll
            for (int e = 0; e < Gm::VW; e += PIECE) {
                const uint32_t p = (p0 | pr) + (uint32_t)e;
                unsigned char* dst = ob + 16 * swz(p / EPC) + (p % EPC) * sizeof(TOut);
                store_vec<TOut, PIECE>(reinterpret_cast<TOut*>(dst), &w[(mid * Gm::VW + e) / 2]);
            }
        }
    } else {
#pragma unroll
        for (int r = 0; r < Gm::E; ++r) {
            const uint32_t p = p0 | (uint32_t)Gm::pos2(r, 0);
            const float v = (r & 1) ? w[r / 2].y : w[r / 2].x;
            store_one(reinterpret_cast<TOut*>(ob + 16 * swz(p / EPC) + (p % EPC) * sizeof(TOut)), v);
        }
    }
}

template <int NB, typename TOut>
__global__ void __launch_bounds__(kTileWarps * 32, TACO_K2_MIN_CTAS)
    k_decompress_tile(const uint8_t* __restrict__ msgs, TOut* __restrict__ out, ShardArgs a, CodecConsts c,
                      FastDiv tps) {
    using Gm = TG<NB>;
    using Cf = K2T<NB, TOut>;
    constexpr int D = Cf::D, B = Gm::B;
    constexpr int EPC = 16 / (int)sizeof(TOut);
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 3, q = lane & 7;
    unsigned char* stage = smem + warp * Cf::WARP_BYTES;
    float* xb = reinterpret_cast<float*>(stage + D * Cf::STAGE);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kTileWarps * Cf::WARP_BYTES) + warp * D;
    if (lane == 0) {
#pragma unroll
        for (int d = 0; d < D; ++d) mbar_init(&bars[d], 1);
        fence_mbar_init();
    }
    __syncwarp();
    const uint32_t ntiles = a.P * tps.d;
    const uint32_t stride = gridDim.x * kTileWarps;
    const uint32_t t0 = blockIdx.x * kTileWarps + warp;

    constexpr int SUB = Cf::SUB, KB = Cf::KB, CODES = SUB * Gm::TILE;
    auto issue = [&](uint32_t t, int slot) {  // lane 0
        const uint32_t p = tps.div(t);
        const uint64_t kk0 = (uint64_t)(t - p * tps.d) * KB;
        const uint8_t* m = msgs + p * a.msg_stride;
        if (kk0 + KB <= a.nblk) {
#if TACO_TMA_ISSUE_FENCE
            fence_proxy_async();
#endif
            mbar_arrive_tx(&bars[slot], Cf::STAGE);
            unsigned char* st = stage + slot * Cf::STAGE;
            bulk_g2s(st, m + kk0 * B, CODES, &bars[slot]);
            bulk_g2s(st + CODES, m + a.scal_off + kk0 * 8, KB * 8, &bars[slot]);
        } else {
            mbar_arrive(&bars[slot]);
        }
    };
    grid_dep_wait();
    if (lane == 0) {
#pragma unroll
        for (int d = 0; d < D - 1; ++d)
            if (t0 + d * stride < ntiles) issue(t0 + d * stride, d);
    }
    int slot = 0;
    uint32_t par = 0;
    for (uint32_t t = t0; t < ntiles; t += stride) {
        const uint32_t tn = t + (D - 1) * stride;
        if (lane == 0 && tn < ntiles) issue(tn, slot == 0 ? D - 1 : slot - 1);
        mbar_wait(&bars[slot], (par >> slot) & 1);
        par ^= 1u << slot;
        const uint32_t p = tps.div(t);
        const uint64_t kk0 = (uint64_t)(t - p * tps.d) * KB;
        unsigned char* st = stage + slot * Cf::STAGE;
        const uint8_t* m = msgs + p * a.msg_stride;
        if (kk0 + KB > a.nblk) {  // ragged stage: live blocks' codes, unit scalars elsewhere
            for (int i = lane; i < CODES / 4; i += 32) {
                const uint64_t kk = kk0 + (uint64_t)((4 * i) >> NB);
                reinterpret_cast<uint32_t*>(st)[i] =
                    kk < a.nblk ? *reinterpret_cast<const uint32_t*>(m + kk0 * B + 4 * (uint64_t)i) : 0u;
            }
            if (lane < KB)
                reinterpret_cast<float2*>(st + CODES)[lane] =
                    kk0 + lane < a.nblk ? *reinterpret_cast<const float2*>(m + a.scal_off + (kk0 + lane) * 8)
                                        : make_float2(1.0f, 1.0f);
            __syncwarp();
            fence_proxy_async();  // these generic writes before any later TMA write of the slot
        }
#pragma unroll 1
        for (int h = 0; h < SUB; ++h) {
            const uint64_t kh = kk0 + (uint64_t)h * kBlocks;  // first block of the sub-tile
            if (kh >= a.nblk) break;                          // warp-uniform
            const float2 sc = reinterpret_cast<const float2*>(st + CODES)[h * kBlocks + g];
            float2 w[Gm::E2];
            const bool ok = tile_decode<NB>(st + h * Gm::TILE, sc, xb, w, g, q, c);
            const uint64_t kk = kh + g;
            if (q == 0 && kk < a.nblk && !ok) raise_flag(a.flags, 2);
            // whole sub-tile valid and vector-aligned -> staged, coalesced 128-bit stores
            const bool full = tile_full<B, kBlocks>(a, p, kh);
            TOut* dst = out + (p * a.S + (a.blk0 + kh) * B);
            if (__all_sync(kFull, full)) {
                // (direct 8-byte stores from the phase-2 registers measured 22.7 vs 18.5 us)
                __syncwarp();
                unsigned char* ob = reinterpret_cast<unsigned char*>(xb);
                stage_out<NB, TOut>(ob, w, g, q);
                __syncwarp();
#pragma unroll
                for (int j = lane; j < Gm::TILE / EPC; j += 32) {
                    *reinterpret_cast<uint4*>(dst + (uint64_t)j * EPC) =
                        *reinterpret_cast<const uint4*>(ob + 16 * swz((uint32_t)j));
                }
            } else if (kk < a.nblk) {
                const uint64_t k = a.blk0 + kk;
                const int valid =
                    clamp_valid((int64_t)a.S - (int64_t)(k * B), (int64_t)a.n - (int64_t)(p * a.S + k * B), B);
                TOut* bd = out + (p * a.S + k * B);
#pragma unroll
                for (int r = 0; r < Gm::E; ++r) {
                    const int pos = Gm::pos2(r, q);
                    if (pos < valid) store_one(bd + pos, (r & 1) ? w[r / 2].y : w[r / 2].x);
                }
            }
        }
        slot = slot + 1 == D ? 0 : slot + 1;
    }
}

// ------------------------------------------------------------------- K3 ------
// Owner step of the two-shot (collective.cpp:95-101): decode the P ranks' copies of a
// tile with tile_decode (so every rank's slice is bit-identical to what K2 produces),
// sum in fp32 in ascending rank order, zero the positions past the shard end, then
// re-encode with exactly K1's fp32 operations (so the result equals compress(sum), the
// property test_collective.cpp:123-156 pins).  The sum goes from the decode's phase-2
// registers to K1's phase-1 registers through one swizzled transpose (no natural-order
// round trip).  One warp per tile; the next rank's codes and scalars are prefetched into
// registers while the current rank is decoded.
template <int NB>
struct K3T {
    using Gm = TG<NB>;
    static constexpr int SLOT = Gm::TILE + kBlocks * 8;  // codes + scalars of one rank's tile
    static constexpr int XB = Gm::TILE * 4;
    static constexpr int WARP_BYTES = SLOT + XB;
    static constexpr size_t SMEM = (size_t)kTileWarps * WARP_BYTES;
    static constexpr int CHUNKS = Gm::TILE / 16;         // 16-byte code chunks per tile
    static constexpr int PER_LANE = (CHUNKS + 31) / 32;
};

// phase-2 registers -> fp32 tile buffer (the inverse of xpose_read), and the phase-1 read
// back (the inverse of xpose_write): same swizzle, so both directions stay conflict-free
template <int NB>
__device__ __forceinline__ void xpose_write2(float* xb, const float2 (&w)[TG<NB>::E2], int g, int q) {
    using Gm = TG<NB>;
    const uint32_t p0 = (uint32_t)(g * Gm::B + Gm::pos2(0, q));
    const uint32_t kl = swz(p0 >> 2);
    if constexpr (Gm::VW >= 4) {
#pragma unroll
        for (int c = 0; c < Gm::E / 4; ++c) {
            const uint32_t kr = swz((uint32_t)Gm::pos2(4 * c, 0) >> 2);
            *reinterpret_cast<float4*>(xb + 4 * (kl ^ kr)) =
                make_float4(w[2 * c].x, w[2 * c].y, w[2 * c + 1].x, w[2 * c + 1].y);
        }
    } else {
#pragma unroll
        for (int r = 0; r < Gm::E; ++r) {
            const uint32_t pr = (uint32_t)Gm::pos2(r, 0);
            xb[4 * (kl ^ swz(pr >> 2)) + ((p0 | pr) & 3)] = (r & 1) ? w[r / 2].y : w[r / 2].x;
        }
    }
}

template <int NB>
__device__ __forceinline__ void xpose_read1(const float* xb, float2 (&w)[TG<NB>::E2], int g, int q) {
    using Gm = TG<NB>;
    const uint32_t kl = swz((uint32_t)(g * Gm::B + Gm::pos1(0, q)) >> 2);
#pragma unroll
    for (int c = 0; c < Gm::E / 4; ++c) {
        const uint32_t kr = swz((uint32_t)Gm::pos1(4 * c, 0) >> 2);
        const float4 v = *reinterpret_cast<const float4*>(xb + 4 * (kl ^ kr));
        w[2 * c] = make_float2(v.x, v.y);
        w[2 * c + 1] = make_float2(v.z, v.w);
    }
}

template <int NB, typename TAcc>
__global__ void __launch_bounds__(kTileWarps * 32, NB <= 8 ? 4 : 2)
    k_reduce_encode_tile(const uint8_t* __restrict__ msgs, uint8_t* __restrict__ out_msg, TAcc* __restrict__ acc_out,
                         ShardArgs a, CodecConsts c) {
    using Gm = TG<NB>;
    using Cf = K3T<NB>;
    constexpr int B = Gm::B;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 3, q = lane & 7;
    unsigned char* slot = smem + warp * Cf::WARP_BYTES;
    float* xb = reinterpret_cast<float*>(slot + Cf::SLOT);
    const uint64_t tile = (uint64_t)blockIdx.x * kTileWarps + warp;
    const uint64_t kk0 = tile * kBlocks;
    grid_dep_wait();
    if (kk0 >= a.nblk) return;  // warp-uniform
    const uint64_t kk = kk0 + g;
    const bool live = kk < a.nblk;
    const int valid = live ? clamp_valid((int64_t)a.S - (int64_t)((a.blk0 + kk) * B), (int64_t)B, B) : 0;

    // rank r's codes + scalars of this tile, in registers (prefetched one rank ahead)
    uint4 pre[Cf::PER_LANE];
    float2 pre_sc = make_float2(1.0f, 1.0f);
    auto fetch = [&](uint32_t r) {
        const uint8_t* m = a.nsrc ? a.src[r] : msgs + r * a.msg_stride;
#pragma unroll
        for (int h = 0; h < Cf::PER_LANE; ++h) {
            const int i = lane + 32 * h;
            const bool bl = i < Cf::CHUNKS && kk0 + (uint64_t)((16 * i) >> NB) < a.nblk;
            pre[h] = bl ? __ldg(reinterpret_cast<const uint4*>(m + kk0 * B + 16 * (uint64_t)i)) : make_uint4(0, 0, 0, 0);
        }
        if (lane < kBlocks)
            pre_sc = kk0 + lane < a.nblk ? __ldg(reinterpret_cast<const float2*>(m + a.scal_off + (kk0 + lane) * 8))
                                         : make_float2(1.0f, 1.0f);
    };
    fetch(0);
    float2 acc[Gm::E2];
    bool ok = true;
    for (uint32_t r = 0; r < a.P; ++r) {
        __syncwarp();  // previous rank's slot contents fully consumed
#pragma unroll
        for (int h = 0; h < Cf::PER_LANE; ++h) {
            const int i = lane + 32 * h;
            if (i < Cf::CHUNKS) reinterpret_cast<uint4*>(slot)[i] = pre[h];
        }
        if (lane < kBlocks) reinterpret_cast<float2*>(slot + Gm::TILE)[lane] = pre_sc;
        __syncwarp();
        if (r + 1 < a.P) fetch(r + 1);
        const float2 sc = reinterpret_cast<const float2*>(slot + Gm::TILE)[g];
        float2 w[Gm::E2];
        ok &= tile_decode<NB>(slot, sc, xb, w, g, q, c);
        if (r == 0) {
#pragma unroll
            for (int i = 0; i < Gm::E2; ++i) acc[i] = w[i];  // keeps -0.0 like the reference
        } else {
#pragma unroll
            for (int i = 0; i < Gm::E2; ++i) acc[i] = __fadd2_rn(acc[i], w[i]);
        }
    }
    // positions past the shard end are padding of the re-encoded slice (collective.cpp:101)
#pragma unroll
    for (int rr = 0; rr < Gm::E; ++rr) {
        if (Gm::pos2(rr, q) >= valid) {
            if (rr & 1) acc[rr / 2].y = 0.0f;
            else acc[rr / 2].x = 0.0f;
        }
    }
    if (acc_out) {  // the stage-1 sum (the SP reduce-scatter output)
        if (__all_sync(kFull, tile_full<B, kBlocks>(a, 0, kk0))) {
            // whole tile: staged through xb, coalesced 128-bit stores (as K2's output)
            constexpr int EPC = 16 / (int)sizeof(TAcc);
            __syncwarp();
            unsigned char* ob = reinterpret_cast<unsigned char*>(xb);
            stage_out<NB, TAcc>(ob, acc, g, q);
            __syncwarp();
            TAcc* dst = acc_out + (a.blk0 + kk0) * B;
#pragma unroll
            for (int j = lane; j < Gm::TILE / EPC; j += 32)
                *reinterpret_cast<uint4*>(dst + (uint64_t)j * EPC) =
                    *reinterpret_cast<const uint4*>(ob + 16 * swz((uint32_t)j));
        } else if (live) {
            TAcc* dst = acc_out + (a.blk0 + kk) * B;
#pragma unroll
            for (int rr = 0; rr < Gm::E; ++rr) {
                const int pos = Gm::pos2(rr, q);
                if (pos < valid) store_one(dst + pos, (rr & 1) ? acc[rr / 2].y : acc[rr / 2].x);
            }
        }
    }
    if (out_msg == nullptr) {  // reduce-scatter: the fp32 sum is the product
        if (live && q == 0 && !ok) raise_flag(a.flags, 2);
        return;
    }
    // ---- re-encode: exactly K1's operations on an fp32 tile (tile_rotate<NB, float>), with
    // the tile taken from registers instead of a natural-order load
    __syncwarp();  // xb free (the last tile_decode read it)
    xpose_write2<NB>(xb, acc, g, q);
    __syncwarp();
    xpose_read1<NB>(xb, acc, g, q);  // phase-1 registers: tile_rotate's raw words
    double ss;
    float p2 = 1.0f;
    {
        double d4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int i = 0; i < Gm::E2; ++i) {
            const double d0 = (double)acc[i].x, d1 = (double)acc[i].y;
            d4[(2 * i) & 3] = fma(d0, d0, d4[(2 * i) & 3]);
            d4[(2 * i + 1) & 3] = fma(d1, d1, d4[(2 * i + 1) & 3]);
        }
        const double sl = (d4[0] + d4[1]) + (d4[2] + d4[3]);
        ss = sl;
#pragma unroll
        for (int o = 1; o < kLanes; o <<= 1) ss += __shfl_xor_sync(kFull, ss, o);
        if (__any_sync(kFull, !(sl < 0x1p150))) {
            p2 = pow2_near(block_alpha(ss, c));
#pragma unroll
            for (int i = 0; i < Gm::E2; ++i) {
                const float x0 = acc[i].x * p2, x1 = acc[i].y * p2;
                acc[i] = make_float2(x0 + x1, x0 - x1);
            }
        } else {
#pragma unroll
            for (int i = 0; i < Gm::E2; ++i) acc[i] = make_float2(acc[i].x + acc[i].y, acc[i].x - acc[i].y);
        }
    }
    stages_rev<Gm::E2, 0, Gm::NE - 1>(acc);
    __syncwarp();
    xpose_write<NB>(xb, acc, g, q);
    __syncwarp();
    xpose_read<NB>(xb, acc, g, q);
    if constexpr (Gm::LO == 0) {
        pair_stage<Gm::E2>(acc);
        stages<Gm::E2, 0, 2>(acc);
    } else {
        stages<Gm::E2, Gm::LO - 1, Gm::LO + 2>(acc);
    }
    float alpha, s;
    tile_quantise<NB>(acc, ss, p2, c, alpha, s);
    __syncwarp();
    uint8_t* cb = reinterpret_cast<uint8_t*>(xb);
    stage_codes<NB>(cb, acc, g, q);
    __syncwarp();
    uint4 cv[Cf::PER_LANE];
#pragma unroll
    for (int h = 0; h < Cf::PER_LANE; ++h) {
        const int j = lane + 32 * h;
        if (j < Cf::CHUNKS) cv[h] = *reinterpret_cast<const uint4*>(cb + 16 * swz((uint32_t)j));
    }
    const uint32_t nd = a.ndst ? a.ndst : 1;
    for (uint32_t d = 0; d < nd; ++d) {  // peer mode: the same message into every rank's buffer
        uint8_t* o = a.ndst ? a.dst[d] : out_msg;
#pragma unroll
        for (int h = 0; h < Cf::PER_LANE; ++h) {
            const int j = lane + 32 * h;
            if (j < Cf::CHUNKS && kk0 + (uint64_t)((j * 16) >> NB) < a.nblk)
                *reinterpret_cast<uint4*>(o + kk0 * B + 16 * (uint64_t)j) = cv[h];
        }
        if (live && q == 0) *reinterpret_cast<float2*>(o + a.scal_off + kk * 8) = make_float2(alpha, s);
    }
    if (live && q == 0 && !ok) raise_flag(a.flags, 2);
}

}  // namespace tile
}  // namespace taco_dev
