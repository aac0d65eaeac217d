// ubench2.cu -- fma-pipe issue rates of the packed-FP32 forms the exchange-butterfly kernels
// use (sm_100a): FADD2, FADD2 with a negated operand, FFMA2 with an immediate -1, FFMA2 with a
// register multiplier, and mixes.  warp-instructions per SMSP per cycle, 4 warps per SMSP.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench2 tools/ubench2.cu
#include <cstdio>
#include <cstdint>

constexpr int ITERS = 4096;
constexpr int CH = 8;

__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {
    unsigned long long ra = *reinterpret_cast<unsigned long long*>(&a), rb = *reinterpret_cast<unsigned long long*>(&b), rd;
    asm volatile("sub.rn.f32x2 %0, %1, %2;" : "=l"(rd) : "l"(ra), "l"(rb));
    return *reinterpret_cast<float2*>(&rd);
}

#define KERNEL(NAME, BODY, NI)                                                                  \
    __global__ void NAME(float2* out, long long* cyc, float seed, float m) {                     \
        float2 v[CH];                                                                            \
        const float2 mm = make_float2(m, m), w = make_float2(seed, 1.0f);                        \
        _Pragma("unroll") for (int c = 0; c < CH; ++c) v[c] = make_float2(seed * c, seed);       \
        __syncthreads();                                                                         \
        long long t0 = clock64();                                                                \
        for (int it = 0; it < ITERS; ++it) {                                                     \
            _Pragma("unroll") for (int c = 0; c < CH; ++c) { BODY; }                             \
        }                                                                                        \
        long long t1 = clock64();                                                                \
        float2 acc = v[0];                                                                       \
        _Pragma("unroll") for (int c = 1; c < CH; ++c) acc = make_float2(acc.x + v[c].x, acc.y + v[c].y); \
        out[blockIdx.x * blockDim.x + threadIdx.x] = acc;                                        \
        if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32] = t1 - t0; \
    }                                                                                            \
    constexpr double NAME##_ni = NI;

KERNEL(k_fadd2, v[c] = __fadd2_rn(v[c], w), 1)
KERNEL(k_fsub2, v[c] = fsub2(v[c], w), 1)
KERNEL(k_ffma2_imm, v[c] = __ffma2_rn(w, make_float2(-1.0f, -1.0f), v[c]), 1)
KERNEL(k_ffma2_reg, v[c] = __ffma2_rn(w, mm, v[c]), 1)
KERNEL(k_mix_add_immfma, { v[c] = __fadd2_rn(v[c], w); v[c] = __ffma2_rn(w, make_float2(-1.0f, -1.0f), v[c]); }, 2)
KERNEL(k_mix_add_sub, { v[c] = __fadd2_rn(v[c], w); v[c] = fsub2(v[c], w); }, 2)
KERNEL(k_fadd, { v[c].x = v[c].x + w.x; }, 1)
KERNEL(k_ffma_imm, { v[c].x = fmaf(v[c].x, -1.0f, w.x); }, 1)

void bench(const char* name, void (*kern)(float2*, long long*, float, float), double ni, int threads) {
    const int blocks = 148;
    float2* out;
    long long* cyc;
    cudaMalloc(&out, (size_t)blocks * threads * sizeof(float2));
    cudaMalloc(&cyc, (size_t)blocks * (threads / 32) * 8);
    kern<<<blocks, threads>>>(out, cyc, 1.0001f, -1.0f);
    kern<<<blocks, threads>>>(out, cyc, 1.0001f, -1.0f);
    cudaDeviceSynchronize();
    const int nw = blocks * threads / 32;
    long long* h = new long long[nw];
    cudaMemcpy(h, cyc, nw * 8, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < nw; ++i) mx = h[i] > mx ? h[i] : mx;
    const double wps = threads / 32 / 4.0;
    const double instr = (double)ITERS * CH * ni * wps;
    printf("%-16s warps/SMSP=%4.1f  %.3f warp-instr/clk/SMSP\n", name, wps, instr / mx);
    delete[] h;
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    for (int threads : {512, 1024}) {
#define B(K) bench(#K, K, K##_ni, threads);
        B(k_fadd2) B(k_fsub2) B(k_ffma2_imm) B(k_ffma2_reg) B(k_mix_add_immfma) B(k_mix_add_sub) B(k_fadd) B(k_ffma_imm)
    }
    return 0;
}
