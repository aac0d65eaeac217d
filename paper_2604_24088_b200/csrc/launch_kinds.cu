// launch_kinds.cu -- the reference's other codec kinds on the device:
//
//   DirectFp8    (codec.cpp:92-115)   fp8_encode(x / s), s = GlobalMax | Unit | PerBlockMax
//   Int8Uniform  (codec.cpp:117-130)  nearbyint(double(x) / delta), delta = max|x| / 127
//   Identity     (codec.cpp:132-138)  the raw fp32 bits, 4 B per element
//   AshInt8      (codec.cpp:78-90)    the Taco rotation with an int8 payload (q_top 127)
//   scaled_spectrum (codec.cpp:306-326)  Z / s of the Taco / AshInt8 rotation
//
// These are comparison baselines and analysis paths, not the north-star hot path, so the
// kernels favour bit-exactness over speed:
//   * the elementwise kinds use one warp per block; every operation is the reference's
//     float (or double) operation, so codes, scales and decoded values are bit-identical;
//   * "GlobalMax" / Int8Uniform scales are per shard (the reference calls compress on each
//     shard slice, collective.cpp:82-88): a pre-pass reduces max|x| per shard;
//   * AshInt8 and scaled_spectrum replay rotate_block (codec.cpp:45-62) in fp64 with one
//     CTA per block, in the reference's own operation order (sequential sum of squares,
//     butterflies h = 1 .. B/2, one 1/sqrt(B) pass), so they are bit-identical too.
#include <cmath>

#include "taco_b200.h"
#include "taco_kernels.cuh"
#include "taco_launch.h"

namespace taco_impl {
using namespace taco_dev;

namespace {

__device__ __forceinline__ float elem(const void* x, int dtype, uint64_t i) {
    return dtype == TACO_DT_BF16 ? __bfloat162float(static_cast<const __nv_bfloat16*>(x)[i])
                                 : static_cast<const float*>(x)[i];
}

__device__ __forceinline__ void put(void* out, int dtype, uint64_t i, float v) {
    if (dtype == TACO_DT_BF16) static_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(v);
    else static_cast<float*>(out)[i] = v;
}

// number of valid elements of block k of shard p (codec.cpp:20-28, collective.cpp:76-87)
__device__ __forceinline__ int valid_of(const ShardArgs& a, uint64_t p, uint64_t k, int B) {
    return clamp_valid((int64_t)a.S - (int64_t)(k * B), (int64_t)a.n - (int64_t)(p * a.S + k * B), B);
}

__device__ __forceinline__ uint8_t enc1(float v, int fmt) {
    return (uint8_t)(fmt ? enc2<1>(make_float2(v, 0.0f)) : enc2<0>(make_float2(v, 0.0f)));
}
__device__ __forceinline__ float dec1(uint8_t c, int fmt) { return fmt ? dec2<1>(c).x : dec2<0>(c).x; }

// quantize_int8 (codec.cpp:36-41): nearbyint (round half to even), clamp to +-127
__device__ __forceinline__ uint8_t q_int8(double v) {
    double r = rint(v);
    r = r > 127.0 ? 127.0 : (r < -127.0 ? -127.0 : r);
    return (uint8_t)(int8_t)r;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// ------------------------------------------------------------------- pre-pass ---
// max|x| of every shard's valid elements, as float bits (non-negative floats order like
// their bit patterns) OR-ed into a zeroed slot; NaN/Inf raise the input flag.
__global__ void k_shard_absmax(const void* __restrict__ x, int dtype, ShardArgs a, uint32_t* __restrict__ smax) {
    const uint64_t p = blockIdx.y;
    const uint64_t len = p * a.S >= a.n ? 0 : (a.n - p * a.S < a.S ? a.n - p * a.S : a.S);
    // the scale covers the whole shard, whatever block range [blk0, blk0+nblk) is encoded,
    // so every chunk of a chunked compress agrees with the unchunked one
    float m = 0.0f;
    bool bad = false;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (uint64_t)gridDim.x * blockDim.x) {
        const float v = elem(x, dtype, p * a.S + i);
        bad |= !isfinite(v);
        m = fmaxf(m, fabsf(v));
    }
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0 && m > 0.0f) atomicMax(smax + p, __float_as_uint(m));
    if (bad) raise_flag(a.flags, 1);
}

// ---------------------------------------------------------- elementwise kinds ---
// one warp per block; kind 1 DirectFp8, 2 Int8Uniform, 3 Identity
__global__ void k_compress_elem(const void* __restrict__ x, int dtype, uint8_t* __restrict__ msgs, ShardArgs a,
                                int B, int kind, int scope, int fmt, float qmax, const uint32_t* __restrict__ smax) {
    const uint64_t p = blockIdx.y;
    const uint64_t kk = (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (kk >= a.nblk) return;
    const uint64_t k = a.blk0 + kk;
    const int valid = valid_of(a, p, k, B);
    const uint64_t base = p * a.S + k * (uint64_t)B;
    uint8_t* m = msgs + p * a.msg_stride;
    float2* scal = reinterpret_cast<float2*>(m + a.scal_off) + kk;
    bool bad = false;
    if (kind == 3) {  // Identity: raw fp32 bits, zero padding
        float* pay = reinterpret_cast<float*>(m) + kk * (uint64_t)B;
        for (int i = lane; i < B; i += 32) {
            const float v = i < valid ? elem(x, dtype, base + i) : 0.0f;
            bad |= !isfinite(v);
            pay[i] = v;
        }
        if (lane == 0) *scal = make_float2(1.0f, 1.0f);
    } else if (kind == 1) {  // DirectFp8
        float s;
        if (scope == 2) {  // PerBlockMax (codec.cpp:101-105)
            float mx = 0.0f;
            for (int i = lane; i < valid; i += 32) mx = fmaxf(mx, fabsf(elem(x, dtype, base + i)));
            mx = warp_max(mx);
            s = mx == 0.0f ? 1.0f : __fdiv_rn(mx, qmax);
        } else if (scope == 1) {  // Unit
            s = 1.0f;
        } else {  // GlobalMax (codec.cpp:223-226)
            const float mx = __uint_as_float(smax[p]);
            s = mx == 0.0f ? 1.0f : __fdiv_rn(mx, qmax);
        }
        uint8_t* pay = m + kk * (uint64_t)B;
        for (int i = lane; i < B; i += 32) {
            uint8_t code = 0;
            if (i < valid) {
                const float v = elem(x, dtype, base + i);
                bad |= !isfinite(v);
                code = enc1(__fdiv_rn(v, s), fmt);
            }
            pay[i] = code;
        }
        if (lane == 0) *scal = make_float2(1.0f, s);
    } else {  // Int8Uniform (codec.cpp:117-130, delta = max / 127.0f at :227-228)
        const float delta = __fdiv_rn(__uint_as_float(smax[p]), 127.0f);
        uint8_t* pay = m + kk * (uint64_t)B;
        for (int i = lane; i < B; i += 32) {
            uint8_t code = 0;
            if (i < valid) {
                const float v = elem(x, dtype, base + i);
                bad |= !isfinite(v);
                if (delta > 0.0f) code = q_int8(__ddiv_rn((double)v, (double)delta));
            }
            pay[i] = code;
        }
        if (lane == 0) *scal = make_float2(1.0f, delta > 0.0f ? delta : 1.0f);
    }
    if (bad) raise_flag(a.flags, 1);
}

__global__ void k_decompress_elem(const uint8_t* __restrict__ msgs, void* __restrict__ out, int dtype, ShardArgs a,
                                  int B, int kind, int fmt) {
    const uint64_t p = blockIdx.y;
    const uint64_t kk = (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (kk >= a.nblk) return;
    const uint64_t k = a.blk0 + kk;
    const int valid = valid_of(a, p, k, B);
    const uint64_t base = p * a.S + k * (uint64_t)B;
    const uint8_t* m = msgs + p * a.msg_stride;
    const float2 sc = reinterpret_cast<const float2*>(m + a.scal_off)[kk];
    if (lane == 0 && !scalars_ok(sc.x, sc.y)) raise_flag(a.flags, 2);
    if (kind == 3) {
        const float* pay = reinterpret_cast<const float*>(m) + kk * (uint64_t)B;
        for (int i = lane; i < valid; i += 32) put(out, dtype, base + i, pay[i]);
    } else if (kind == 1) {  // table[c] * s (codec.cpp:167-172)
        const uint8_t* pay = m + kk * (uint64_t)B;
        for (int i = lane; i < valid; i += 32) put(out, dtype, base + i, __fmul_rn(dec1(pay[i], fmt), sc.y));
    } else {  // float(int8) * s (codec.cpp:173-178)
        const uint8_t* pay = m + kk * (uint64_t)B;
        for (int i = lane; i < valid; i += 32) put(out, dtype, base + i, __fmul_rn((float)(int8_t)pay[i], sc.y));
    }
}

// ----------------------------------------------------------------- AshInt8 -----
// rotate_block (codec.cpp:45-62) in fp64 with the reference's operation order; one CTA of
// 256 threads per block, the block in shared memory.
constexpr int kAshThreads = 256;

__device__ void ash_fwht(double* v, int B) {  // transform.cpp:41-58
    for (int h = 1; h < B; h <<= 1) {
        __syncthreads();
        for (int t = threadIdx.x; t < B / 2; t += kAshThreads) {
            const int i = (t / h) * 2 * h + (t % h);
            const double x0 = v[i], x1 = v[i + h];
            v[i] = x0 + x1;
            v[i + h] = x0 - x1;
        }
    }
    __syncthreads();
}

// mode 0: AshInt8 compress (q_top 127, int8 payload); mode 1: scaled_spectrum (float out,
// q_top = qtop: 127 for AshInt8, q_max of the fp8 format for Taco)
__global__ void k_ash_rotate(const void* __restrict__ x, int dtype, uint8_t* __restrict__ msgs, float* __restrict__ spec,
                             ShardArgs a, int B, CodecConsts c, double qtop, int mode) {
    extern __shared__ double sv[];
    __shared__ float s_alpha, s_s;
    const uint64_t p = blockIdx.y, kk = blockIdx.x, k = a.blk0 + kk;
    const int valid = valid_of(a, p, k, B);
    const uint64_t base = p * a.S + k * (uint64_t)B;
    bool bad = false;
    for (int i = threadIdx.x; i < B; i += kAshThreads) {
        const float v = i < valid ? elem(x, dtype, base + i) : 0.0f;
        bad |= !isfinite(v);
        sv[i] = (double)v;
    }
    if (bad) raise_flag(a.flags, 1);
    __syncthreads();
    if (threadIdx.x == 0) {  // sequential double sum of squares, like the reference
        double acc = 0.0;
        for (int i = 0; i < B; ++i) acc += sv[i] * sv[i];
        const double sigma = sqrt(acc / (double)B + (double)c.eps);
        s_alpha = __fdiv_rn(c.tau, (float)sigma);  // adaptive_scale(float(sigma), tau)
    }
    __syncthreads();
    const double al = (double)s_alpha;
    for (int i = threadIdx.x; i < B; i += kAshThreads) sv[i] *= al;
    ash_fwht(sv, B);
    for (int i = threadIdx.x; i < B; i += kAshThreads) sv[i] *= c.norm;  // transform.cpp:56-57
    __syncthreads();
    if (threadIdx.x == 0) {
        double zmax = 0.0;
        for (int i = 0; i < B; ++i) zmax = fmax(zmax, fabs(sv[i]));
        s_s = zmax == 0.0 ? 1.0f : (float)(zmax / qtop);
    }
    __syncthreads();
    const double s = (double)s_s;
    if (mode == 1) {  // scaled_spectrum: float(Z / s) for all B slots (codec.cpp:318-321)
        float* o = spec + (p * (uint64_t)a.nblk + kk) * (uint64_t)B;
        for (int i = threadIdx.x; i < B; i += kAshThreads) o[i] = (float)(sv[i] / s);
        return;
    }
    uint8_t* m = msgs + p * a.msg_stride;
    for (int i = threadIdx.x; i < B; i += kAshThreads) m[kk * (uint64_t)B + i] = q_int8(sv[i] / s);
    if (threadIdx.x == 0) reinterpret_cast<float2*>(m + a.scal_off)[kk] = make_float2(s_alpha, s_s);
}

// decompress_block AshInt8 (codec.cpp:156-166): int8 * s in double, FWHT, / alpha
__global__ void k_ash_decode(const uint8_t* __restrict__ msgs, void* __restrict__ out, int dtype, ShardArgs a, int B,
                             CodecConsts c) {
    extern __shared__ double sv[];
    const uint64_t p = blockIdx.y, kk = blockIdx.x, k = a.blk0 + kk;
    const int valid = valid_of(a, p, k, B);
    const uint64_t base = p * a.S + k * (uint64_t)B;
    const uint8_t* m = msgs + p * a.msg_stride;
    const float2 sc = reinterpret_cast<const float2*>(m + a.scal_off)[kk];
    if (threadIdx.x == 0 && !scalars_ok(sc.x, sc.y)) raise_flag(a.flags, 2);
    for (int i = threadIdx.x; i < B; i += kAshThreads) sv[i] = (double)(int8_t)m[kk * (uint64_t)B + i] * (double)sc.y;
    ash_fwht(sv, B);
    for (int i = threadIdx.x; i < valid; i += kAshThreads) put(out, dtype, base + i, (float)(sv[i] * c.norm / (double)sc.x));
}

}  // namespace

// taco_config.kind != Taco: compress (and the per-shard max pre-pass where needed)
cudaError_t launch_compress_kind(const Launch& l, const ShardArgs& a, const CodecConsts& c, int kind, int scope,
                                 uint32_t* smax) {
    if (a.nblk == 0 || a.P == 0) return cudaSuccess;
    const int B = (int)l.block_size;
    if (kind == 4) {
        const size_t smem = (size_t)B * sizeof(double);
        if (smem > 48 * 1024) cudaFuncSetAttribute(k_ash_rotate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_ash_rotate<<<dim3((unsigned)a.nblk, a.P), kAshThreads, smem, l.stream>>>(
            l.in, l.dtype, static_cast<uint8_t*>(l.out), nullptr, a, B, c, 127.0, 0);
        return cudaGetLastError();
    }
    const bool need_max = kind == 2 || (kind == 1 && scope == 0);
    if (need_max) {
        if (cudaError_t e = cudaMemsetAsync(smax, 0, a.P * sizeof(uint32_t), l.stream)) return e;
        const uint64_t S = a.S;
        unsigned gx = (unsigned)((S + 255) / 256);
        gx = gx > 1184 ? 1184 : (gx == 0 ? 1 : gx);
        k_shard_absmax<<<dim3(gx, a.P), 256, 0, l.stream>>>(l.in, l.dtype, a, smax);
    }
    const unsigned wpb = 8;
    k_compress_elem<<<dim3((unsigned)((a.nblk + wpb - 1) / wpb), a.P), wpb * 32, 0, l.stream>>>(
        l.in, l.dtype, static_cast<uint8_t*>(l.out), a, B, kind, scope, l.format, (float)c.qmax, smax);
    return cudaGetLastError();
}

cudaError_t launch_decompress_kind(const Launch& l, const ShardArgs& a, const CodecConsts& c, int kind) {
    if (a.nblk == 0 || a.P == 0) return cudaSuccess;
    const int B = (int)l.block_size;
    if (kind == 4) {
        const size_t smem = (size_t)B * sizeof(double);
        if (smem > 48 * 1024) cudaFuncSetAttribute(k_ash_decode, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_ash_decode<<<dim3((unsigned)a.nblk, a.P), kAshThreads, smem, l.stream>>>(static_cast<const uint8_t*>(l.in),
                                                                                    l.out, l.dtype, a, B, c);
        return cudaGetLastError();
    }
    const unsigned wpb = 8;
    k_decompress_elem<<<dim3((unsigned)((a.nblk + wpb - 1) / wpb), a.P), wpb * 32, 0, l.stream>>>(
        static_cast<const uint8_t*>(l.in), l.out, l.dtype, a, B, kind, l.format);
    return cudaGetLastError();
}

cudaError_t launch_scaled_spectrum(const Launch& l, const ShardArgs& a, const CodecConsts& c, double qtop) {
    if (a.nblk == 0 || a.P == 0) return cudaSuccess;
    const int B = (int)l.block_size;
    const size_t smem = (size_t)B * sizeof(double);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_ash_rotate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_ash_rotate<<<dim3((unsigned)a.nblk, a.P), kAshThreads, smem, l.stream>>>(l.in, l.dtype, nullptr,
                                                                              static_cast<float*>(l.out), a, B, c,
                                                                              qtop, 1);
    return cudaGetLastError();
}

}  // namespace taco_impl
