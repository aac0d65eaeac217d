// taco_kernels.cuh -- the three fused TACO kernels, templated on block size and types.
//
//   K1 k_compress        x (bf16|f32)          -> message(s): FP8 codes + (alpha, s)
//   K2 k_decompress      message(s)            -> y (bf16|f32), valid prefix only
//   K3 k_reduce_encode   P messages of a shard -> fp32 ascending-rank sum -> message
//
// Warp kernels (B <= 1024) keep a whole block in registers of an L-lane group
// (taco_device.cuh); big-block kernels (B >= 2048) stage one block per CTA in shared
// memory.  All of them read their input once and write their output once.
#pragma once

#include "taco_device.cuh"

namespace taco_dev {

struct ShardArgs {
    uint64_t n;           // logical elements of the tensor (K1/K2)
    uint64_t S;           // shard length
    uint32_t P;           // shards (K1/K2) or ranks (K3)
    uint64_t blk0;        // first block of the chunk, per shard
    uint64_t nblk;        // blocks per shard in the chunk
    uint64_t msg_stride;  // bytes between consecutive messages
    uint64_t scal_off;    // byte offset of the (alpha, s) array in a message
    int vec_ok;           // element pointers allow V-wide vector access
    int* flags;           // device error flags (may be null)
};

constexpr int kWarpThreads = 256;  // 8 warps per CTA
constexpr int kBigThreads = 512;   // one block per CTA for B >= 2048

__device__ __forceinline__ void raise_flag(int* flags, int bit) {
    if (flags) atomicOr(flags, bit);
}

__device__ __forceinline__ int clamp_valid(int64_t a, int64_t b, int B) {
    int64_t v = a < b ? a : b;
    v = v < (int64_t)B ? v : (int64_t)B;
    return v < 0 ? 0 : (int)v;
}

// Rotate + quantise a register-resident block (rotate_block codec.cpp:45-62 and
// compress_block_taco :64-76).  On return v holds Z/s, ready for the FP8 cvt.
template <int V, int L, int E>
__device__ __forceinline__ void quantise_regs(float (&v)[E], int q, const CodecConsts& c, float& alpha,
                                              float& s, double& sumsq) {
    double ss = 0.0;
#pragma unroll
    for (int i = 0; i < E; ++i) ss = fma((double)v[i], (double)v[i], ss);  // x^2 exact in double
    ss = group_sum<L>(ss);
    sumsq = ss;
    alpha = block_alpha(ss, c);
    const float p2 = pow2_near(alpha);
#pragma unroll
    for (int i = 0; i < E; ++i) v[i] *= p2;
    fwht<V, L, E>(v, q);
    float ym = 0.0f;
#pragma unroll
    for (int i = 0; i < E; ++i) ym = fmaxf(ym, fabsf(v[i]));
    ym = group_max<L>(ym);
    float k;
    block_scale(ym, alpha, p2, c, s, k);
#pragma unroll
    for (int i = 0; i < E; ++i) v[i] *= k;
}

// Decode one block of a message into registers: yhat*m (decompress_block :144-155).
// Every lane of the warp executes the butterfly (dead groups on zeros) so the
// shuffles stay converged.
template <int FMT, int V, int L, int E>
__device__ __forceinline__ void dequantise_regs(float (&v)[E], bool live, const uint8_t* __restrict__ codes,
                                                float2 sc, int q, const CodecConsts& c) {
    if (live) {
#pragma unroll
        for (int j = 0; j < E / V; ++j) load_codes<FMT, V>(codes + (j * L + q) * V, &v[j * V]);
    } else {
#pragma unroll
        for (int i = 0; i < E; ++i) v[i] = 0.0f;
    }
    fwht<V, L, E>(v, q);
    const float m = live ? block_dequant(sc.x, sc.y, c) : 0.0f;
#pragma unroll
    for (int i = 0; i < E; ++i) v[i] *= m;
}

// --------------------------------------------------------------------------- K1 ---
template <int B, typename TIn, int FMT, int EMAX, int VMAX>
__global__ void __launch_bounds__(kWarpThreads) k_compress(const TIn* __restrict__ x, uint8_t* __restrict__ msgs,
                                                           ShardArgs a, CodecConsts c) {
    using Gm = Geo<B, EMAX, VMAX>;
    constexpr int E = Gm::E, V = Gm::V, L = Gm::L, G = Gm::G, NV = Gm::NV;
    const int lane = threadIdx.x & 31, q = lane & (L - 1), g = lane / L;
    const uint64_t warp = (uint64_t)blockIdx.x * (kWarpThreads / 32) + (threadIdx.x >> 5);
    const uint64_t job = warp * G + g;
    const bool live = job < (uint64_t)a.P * a.nblk;
    const uint64_t p = live ? job / a.nblk : 0;
    const uint64_t kk = live ? job - p * a.nblk : 0;
    const uint64_t k = a.blk0 + kk;
    const int valid = live ? clamp_valid((int64_t)a.S - (int64_t)(k * B),
                                         (int64_t)a.n - (int64_t)(p * a.S + k * B), B)
                           : 0;
    const TIn* src = x + (p * a.S + k * B);

    float v[E];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const int pos = Gm::pos(j, q);
        if (a.vec_ok && pos + V <= valid) {
            load_vec<TIn, V>(src + pos, &v[j * V]);
        } else {
#pragma unroll
            for (int r = 0; r < V; ++r) v[j * V + r] = pos + r < valid ? to_f32(src[pos + r]) : 0.0f;
        }
    }
    float alpha, s;
    double ss;
    quantise_regs<V, L, E>(v, q, c, alpha, s, ss);
    if (!live) return;
    if (q == 0 && !isfinite(ss)) raise_flag(a.flags, 1);
    uint8_t* m = msgs + p * a.msg_stride;
#pragma unroll
    for (int j = 0; j < NV; ++j) store_codes<FMT, V>(m + kk * B + Gm::pos(j, q), &v[j * V]);
    if (q == 0) *reinterpret_cast<float2*>(m + a.scal_off + kk * 8) = make_float2(alpha, s);
}

// --------------------------------------------------------------------------- K2 ---
template <int B, typename TOut, int FMT, int EMAX, int VMAX>
__global__ void __launch_bounds__(kWarpThreads) k_decompress(const uint8_t* __restrict__ msgs, TOut* __restrict__ out,
                                                             ShardArgs a, CodecConsts c) {
    using Gm = Geo<B, EMAX, VMAX>;
    constexpr int E = Gm::E, V = Gm::V, L = Gm::L, G = Gm::G, NV = Gm::NV;
    const int lane = threadIdx.x & 31, q = lane & (L - 1), g = lane / L;
    const uint64_t warp = (uint64_t)blockIdx.x * (kWarpThreads / 32) + (threadIdx.x >> 5);
    const uint64_t job = warp * G + g;
    const bool live = job < (uint64_t)a.P * a.nblk;
    const uint64_t p = live ? job / a.nblk : 0;
    const uint64_t kk = live ? job - p * a.nblk : 0;
    const uint64_t k = a.blk0 + kk;
    const int valid = live ? clamp_valid((int64_t)a.S - (int64_t)(k * B),
                                         (int64_t)a.n - (int64_t)(p * a.S + k * B), B)
                           : 0;
    const uint8_t* m = msgs + p * a.msg_stride;
    float v[E];
    const float2 sc = live ? __ldg(reinterpret_cast<const float2*>(m + a.scal_off + kk * 8)) : make_float2(1.0f, 1.0f);
    dequantise_regs<FMT, V, L, E>(v, live, m + kk * B, sc, q, c);
    if (!live) return;
    if (q == 0 && !scalars_ok(sc.x, sc.y)) raise_flag(a.flags, 2);
    TOut* dst = out + (p * a.S + k * B);
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const int pos = Gm::pos(j, q);
        if (a.vec_ok && pos + V <= valid) {
            store_vec<TOut, V>(dst + pos, &v[j * V]);
        } else {
#pragma unroll
            for (int r = 0; r < V; ++r)
                if (pos + r < valid) store_one(dst + pos + r, v[j * V + r]);
        }
    }
}

// --------------------------------------------------------------------------- K3 ---
// msgs: nranks messages (rank r at msgs + r*msg_stride) of one shard chunk.
template <int B, typename TAcc, int FMT, int EMAX, int VMAX>
__global__ void __launch_bounds__(kWarpThreads) k_reduce_encode(const uint8_t* __restrict__ msgs,
                                                                uint8_t* __restrict__ out_msg,
                                                                TAcc* __restrict__ acc_out, ShardArgs a,
                                                                CodecConsts c) {
    using Gm = Geo<B, EMAX, VMAX>;
    constexpr int E = Gm::E, V = Gm::V, L = Gm::L, G = Gm::G, NV = Gm::NV;
    const int lane = threadIdx.x & 31, q = lane & (L - 1), g = lane / L;
    const uint64_t warp = (uint64_t)blockIdx.x * (kWarpThreads / 32) + (threadIdx.x >> 5);
    const uint64_t kk = warp * G + g;
    const bool live = kk < a.nblk;
    const uint64_t k = a.blk0 + kk;
    const int valid = live ? clamp_valid((int64_t)a.S - (int64_t)(k * B), (int64_t)B, B) : 0;

    float acc[E];
#pragma unroll
    for (int i = 0; i < E; ++i) acc[i] = 0.0f;
    bool bad = false;
    for (uint32_t r = 0; r < a.P; ++r) {
        const uint8_t* m = msgs + r * a.msg_stride;
        float d[E];
        const float2 sc = live ? __ldg(reinterpret_cast<const float2*>(m + a.scal_off + kk * 8)) : make_float2(1.0f, 1.0f);
        bad |= !scalars_ok(sc.x, sc.y);
        dequantise_regs<FMT, V, L, E>(d, live, m + kk * B, sc, q, c);
        if (r == 0) {
#pragma unroll
            for (int i = 0; i < E; ++i) acc[i] = d[i];  // acc = dec(rank 0), keeps -0.0
        } else {
#pragma unroll
            for (int i = 0; i < E; ++i) acc[i] += d[i];
        }
    }
    // positions past the shard end are padding of the re-encoded slice (collective.cpp:101)
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const int pos = Gm::pos(j, q);
#pragma unroll
        for (int r = 0; r < V; ++r)
            if (pos + r >= valid) acc[j * V + r] = 0.0f;
    }
    if (live && acc_out) {
        TAcc* dst = acc_out + k * B;
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            const int pos = Gm::pos(j, q);
            if (a.vec_ok && pos + V <= valid) {
                store_vec<TAcc, V>(dst + pos, &acc[j * V]);
            } else {
#pragma unroll
                for (int r = 0; r < V; ++r)
                    if (pos + r < valid) store_one(dst + pos + r, acc[j * V + r]);
            }
        }
    }
    float alpha, s;
    double ss;
    quantise_regs<V, L, E>(acc, q, c, alpha, s, ss);
    if (!live) return;
    if (q == 0 && bad) raise_flag(a.flags, 2);
#pragma unroll
    for (int j = 0; j < NV; ++j) store_codes<FMT, V>(out_msg + kk * B + Gm::pos(j, q), &acc[j * V]);
    if (q == 0) *reinterpret_cast<float2*>(out_msg + a.scal_off + kk * 8) = make_float2(alpha, s);
}

// ===================================================== big blocks (B >= 2048) ===
// One CTA of kBigThreads per block.  Thread t owns positions t + i*T (i < PER) in
// registers; butterflies run through shared memory.

template <int B>
__device__ __forceinline__ void smem_fwht(float* sm) {
    constexpr int T = kBigThreads;
#pragma unroll 1
    for (int h = 1; h < B; h <<= 1) {
        __syncthreads();
        for (int t = threadIdx.x; t < B / 2; t += T) {
            const int i = (t / h) * 2 * h + (t % h);
            const float a = sm[i], b = sm[i + h];
            sm[i] = a + b;
            sm[i + h] = a - b;
        }
    }
    __syncthreads();
}

__device__ __forceinline__ double cta_sum(double v, double* red) {
#pragma unroll
    for (int m = 1; m < 32; m <<= 1) v += __shfl_xor_sync(kFull, v, m);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < kBigThreads / 32; ++w) t += red[w];  // same order in every thread
    return t;
}

__device__ __forceinline__ float cta_max(float v, float* red) {
#pragma unroll
    for (int m = 1; m < 32; m <<= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, m));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    float t = 0.0f;
    for (int w = 0; w < kBigThreads / 32; ++w) t = fmaxf(t, red[w]);
    return t;
}

// Quantise the register block r[PER] (positions t + i*T); writes codes + scalars.
template <int B, int FMT>
__device__ __forceinline__ void big_quantise_store(float (&r)[B / kBigThreads], float* sm, double* red,
                                                   const CodecConsts& c, uint8_t* codes, float2* scal,
                                                   int* flags) {
    constexpr int T = kBigThreads, PER = B / T;
    double ss = 0.0;
#pragma unroll
    for (int i = 0; i < PER; ++i) ss = fma((double)r[i], (double)r[i], ss);
    ss = cta_sum(ss, red);
    const float alpha = block_alpha(ss, c);
    const float p2 = pow2_near(alpha);
#pragma unroll
    for (int i = 0; i < PER; ++i) sm[threadIdx.x + i * T] = r[i] * p2;
    smem_fwht<B>(sm);
    float ym = 0.0f;
#pragma unroll
    for (int i = 0; i < PER; ++i) ym = fmaxf(ym, fabsf(sm[threadIdx.x + i * T]));
    ym = cta_max(ym, reinterpret_cast<float*>(red));
    float s, k;
    block_scale(ym, alpha, p2, c, s, k);
    for (int t = threadIdx.x; t < B / 2; t += T)
        reinterpret_cast<uint16_t*>(codes)[t] = (uint16_t)enc2<FMT>(sm[2 * t] * k, sm[2 * t + 1] * k);
    if (threadIdx.x == 0) {
        *scal = make_float2(alpha, s);
        if (!isfinite(ss)) raise_flag(flags, 1);
    }
}

// decode one block into sm (H(table[c]) * m), returns validity of its scalars
template <int B, int FMT>
__device__ __forceinline__ bool big_dequantise(const uint8_t* codes, float2 sc, float* sm, const CodecConsts& c) {
    __syncthreads();
    for (int t = threadIdx.x; t < B / 2; t += kBigThreads) {
        const uint32_t two = reinterpret_cast<const uint16_t*>(codes)[t];
        dec2<FMT>(two, sm[2 * t], sm[2 * t + 1]);
    }
    smem_fwht<B>(sm);
    const float m = block_dequant(sc.x, sc.y, c);
    for (int t = threadIdx.x; t < B; t += kBigThreads) sm[t] *= m;
    __syncthreads();
    return scalars_ok(sc.x, sc.y);
}

template <int B, typename TIn, int FMT>
__global__ void __launch_bounds__(kBigThreads) k_compress_big(const TIn* __restrict__ x, uint8_t* __restrict__ msgs,
                                                              ShardArgs a, CodecConsts c) {
    extern __shared__ float sm[];
    __shared__ double red[kBigThreads / 32];
    constexpr int T = kBigThreads, PER = B / T;
    const uint64_t job = blockIdx.x;
    const uint64_t p = job / a.nblk, kk = job - p * a.nblk, k = a.blk0 + kk;
    const int valid = clamp_valid((int64_t)a.S - (int64_t)(k * B), (int64_t)a.n - (int64_t)(p * a.S + k * B), B);
    const TIn* src = x + (p * a.S + k * B);
    float r[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int pos = threadIdx.x + i * T;
        r[i] = pos < valid ? to_f32(src[pos]) : 0.0f;
    }
    uint8_t* m = msgs + p * a.msg_stride;
    big_quantise_store<B, FMT>(r, sm, red, c, m + kk * B, reinterpret_cast<float2*>(m + a.scal_off + kk * 8),
                               a.flags);
}

template <int B, typename TOut, int FMT>
__global__ void __launch_bounds__(kBigThreads) k_decompress_big(const uint8_t* __restrict__ msgs, TOut* __restrict__ out,
                                                                ShardArgs a, CodecConsts c) {
    extern __shared__ float sm[];
    const uint64_t job = blockIdx.x;
    const uint64_t p = job / a.nblk, kk = job - p * a.nblk, k = a.blk0 + kk;
    const int valid = clamp_valid((int64_t)a.S - (int64_t)(k * B), (int64_t)a.n - (int64_t)(p * a.S + k * B), B);
    const uint8_t* m = msgs + p * a.msg_stride;
    const float2 sc = *reinterpret_cast<const float2*>(m + a.scal_off + kk * 8);
    const bool ok = big_dequantise<B, FMT>(m + kk * B, sc, sm, c);
    if (threadIdx.x == 0 && !ok) raise_flag(a.flags, 2);
    TOut* dst = out + (p * a.S + k * B);
    for (int t = threadIdx.x; t < valid; t += kBigThreads) store_one(dst + t, sm[t]);
}

template <int B, typename TAcc, int FMT>
__global__ void __launch_bounds__(kBigThreads) k_reduce_encode_big(const uint8_t* __restrict__ msgs,
                                                                   uint8_t* __restrict__ out_msg,
                                                                   TAcc* __restrict__ acc_out, ShardArgs a,
                                                                   CodecConsts c) {
    extern __shared__ float sm[];
    __shared__ double red[kBigThreads / 32];
    constexpr int T = kBigThreads, PER = B / T;
    const uint64_t kk = blockIdx.x, k = a.blk0 + kk;
    const int valid = clamp_valid((int64_t)a.S - (int64_t)(k * B), (int64_t)B, B);
    float acc[PER];
    bool ok = true;
    for (uint32_t r = 0; r < a.P; ++r) {
        const uint8_t* m = msgs + r * a.msg_stride;
        const float2 sc = *reinterpret_cast<const float2*>(m + a.scal_off + kk * 8);
        ok &= big_dequantise<B, FMT>(m + kk * B, sc, sm, c);
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const float d = sm[threadIdx.x + i * T];
            acc[i] = r == 0 ? d : acc[i] + d;
        }
    }
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int pos = threadIdx.x + i * T;
        if (pos >= valid) acc[i] = 0.0f;
        else if (acc_out) store_one(acc_out + k * B + pos, acc[i]);
    }
    __syncthreads();
    big_quantise_store<B, FMT>(acc, sm, red, c, out_msg + kk * B,
                               reinterpret_cast<float2*>(out_msg + a.scal_off + kk * 8), nullptr);
    if (threadIdx.x == 0 && !ok) raise_flag(a.flags, 2);
}

}  // namespace taco_dev
