// ubench.cu -- issue-rate microbenchmarks of the instructions the codec kernels are built
// from (sm_100a): warp instructions per SMSP per cycle with 4 / 8 warps per scheduler and
// 8 independent chains per thread.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o
// tools/ubench tools/ubench.cu ; ./tools/ubench
#include <cuda_bf16.h>
#include <cuda_fp8.h>
#include <cstdio>
#include <cstdint>

constexpr int ITERS = 2048;
constexpr int CH = 8;

#define KERNEL(NAME, T, INIT, BODY)                                                              \
    __global__ void NAME(T* out, long long* cyc, float seed) {                                    \
        T v[CH];                                                                                  \
        _Pragma("unroll") for (int c = 0; c < CH; ++c) { INIT; }                                  \
        __syncthreads();                                                                          \
        long long t0 = clock64();                                                                 \
        for (int it = 0; it < ITERS; ++it) {                                                      \
            _Pragma("unroll") for (int c = 0; c < CH; ++c) { BODY; }                              \
        }                                                                                         \
        long long t1 = clock64();                                                                 \
        T acc = v[0];                                                                             \
        _Pragma("unroll") for (int c = 1; c < CH; ++c) acc = acc_op(acc, v[c]);                   \
        out[blockIdx.x * blockDim.x + threadIdx.x] = acc;                                         \
        if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32] = t1 - t0; \
    }

__device__ __forceinline__ float acc_op(float a, float b) { return a + b; }
__device__ __forceinline__ float2 acc_op(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ uint32_t acc_op(uint32_t a, uint32_t b) { return a ^ b; }
__device__ __forceinline__ double acc_op(double a, double b) { return a + b; }

__device__ __forceinline__ float add_bf16(uint32_t h16, float c) {
    float d;
    asm volatile("add.rn.f32.bf16 %0, %1, %2;" : "=f"(d) : "h"((unsigned short)h16), "f"(c));
    return d;
}
__device__ __forceinline__ float fma_bf16(uint32_t h16, float c) {
    float d;
    asm volatile("fma.rn.f32.bf16 %0, %1, %1, %2;" : "=f"(d) : "h"((unsigned short)h16), "f"(c));
    return d;
}
__device__ __forceinline__ float max3(float a, float b, float c) {
    float d;
    asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ float max3abs(float a, float b, float c) {
    float d;
    asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(fabsf(b)), "f"(fabsf(c)));
    return d;
}

KERNEL(k_fadd, float, v[c] = seed * (c + 1), v[c] = v[c] + 1.0001f)
KERNEL(k_ffma, float, v[c] = seed * (c + 1), v[c] = fmaf(v[c], 0.9999f, seed))
KERNEL(k_fadd2, float2, v[c] = make_float2(seed * c, seed), v[c] = __fadd2_rn(v[c], make_float2(seed, 1.0f)))
KERNEL(k_ffma2, float2, v[c] = make_float2(seed * c, seed),
       v[c] = __ffma2_rn(v[c], make_float2(-1.0f, -1.0f), make_float2(seed, 1.0f)))
KERNEL(k_fmul2, float2, v[c] = make_float2(seed * c, seed), v[c] = __fmul2_rn(v[c], make_float2(seed, 1.0f)))
KERNEL(k_shfl, float, v[c] = seed * (c + 1), v[c] = __shfl_xor_sync(0xffffffffu, v[c], 1))
KERNEL(k_f2fp, uint32_t, v[c] = __float_as_uint(seed) + c,
       v[c] = (uint32_t)__nv_cvt_float2_to_fp8x2(make_float2(__uint_as_float(v[c]), seed), __NV_SATFINITE, __NV_E4M3))
KERNEL(k_f2bf, uint32_t, v[c] = __float_as_uint(seed) + c, {
    __nv_bfloat162 h = __float22bfloat162_rn(make_float2(__uint_as_float(v[c]), seed));
    v[c] = *reinterpret_cast<uint32_t*>(&h);
})
KERNEL(k_fp8dec, uint32_t, v[c] = __float_as_uint(seed) + c, {
    __half2_raw h = __nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)(v[c] & 0xffffu), __NV_E4M3);
    v[c] = (uint32_t)h.x | ((uint32_t)h.y << 16);
})
KERNEL(k_h2f, float, v[c] = seed * (c + 1), {
    __half h = __float2half_rn(v[c]);
    v[c] = __half2float(h) + 0.0f;
})
KERNEL(k_addbf16, float, v[c] = seed * (c + 1), v[c] = add_bf16(__float_as_uint(v[c]) >> 16, v[c]))
KERNEL(k_fmabf16, float, v[c] = seed * (c + 1), v[c] = fma_bf16(__float_as_uint(v[c]) >> 16, v[c]))
KERNEL(k_fmnmx, float, v[c] = seed * (c + 1), v[c] = fmaxf(fabsf(v[c]), seed))
KERNEL(k_max3, float, v[c] = seed * (c + 1), v[c] = max3abs(v[c], seed, -seed))
KERNEL(k_lop3, uint32_t, v[c] = __float_as_uint(seed) + c, v[c] = (v[c] ^ 0x5555u) & (v[c] | 0x10u))
KERNEL(k_prmt, uint32_t, v[c] = __float_as_uint(seed) + c, v[c] = __byte_perm(v[c], 0x12345678u, 0x5140))
KERNEL(k_shl, uint32_t, v[c] = __float_as_uint(seed) + c, v[c] = v[c] << 3)
KERNEL(k_imad, uint32_t, v[c] = __float_as_uint(seed) + c, v[c] = v[c] * 3u + 7u)
KERNEL(k_dfma, double, v[c] = seed * (c + 1), v[c] = fma(v[c], 0.9999, 1e-3))

template <typename T>
void bench(const char* name, void (*kern)(T*, long long*, float), int threads, double instr_per_body) {
    const int blocks = 148;
    T* out;
    long long* cyc;
    cudaMalloc(&out, (size_t)blocks * threads * sizeof(T));
    cudaMalloc(&cyc, (size_t)blocks * (threads / 32) * 8);
    kern<<<blocks, threads>>>(out, cyc, 1.0001f);
    kern<<<blocks, threads>>>(out, cyc, 1.0001f);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("%s: %s\n", name, cudaGetErrorString(e));
        return;
    }
    const int nw = blocks * threads / 32;
    long long* h = new long long[nw];
    cudaMemcpy(h, cyc, nw * 8, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < nw; ++i) mx = h[i] > mx ? h[i] : mx;
    const double warps_per_smsp = threads / 32 / 4.0;
    const double instr = (double)ITERS * CH * instr_per_body * warps_per_smsp;
    printf("%-10s warps/SMSP=%4.1f  %.3f warp-instr/clk/SMSP  (%.2f clk per instr)\n", name, warps_per_smsp,
           instr / mx, mx / instr);
    delete[] h;
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    for (int threads : {512, 1024}) {
        bench("FADD", k_fadd, threads, 1);
        bench("FFMA", k_ffma, threads, 1);
        bench("FADD2", k_fadd2, threads, 1);
        bench("FFMA2", k_ffma2, threads, 1);
        bench("FMUL2", k_fmul2, threads, 1);
        bench("SHFL", k_shfl, threads, 1);
        bench("F2FP.e4m3", k_f2fp, threads, 1);
        bench("F2F.bf16x2", k_f2bf, threads, 1);
        bench("e4m3->f16x2", k_fp8dec, threads, 1);
        bench("h->f->h", k_h2f, threads, 2);
        bench("add.f32.bf16", k_addbf16, threads, 2);
        bench("fma.f32.bf16", k_fmabf16, threads, 2);
        bench("FMNMX", k_fmnmx, threads, 1);
        bench("max3abs", k_max3, threads, 1);
        bench("LOP3", k_lop3, threads, 2);
        bench("PRMT", k_prmt, threads, 1);
        bench("SHL", k_shl, threads, 1);
        bench("IMAD", k_imad, threads, 1);
        bench("DFMA", k_dfma, threads, 1);
    }
    return 0;
}
