// mempat.cu -- HBM ceiling of the codec kernels' access patterns, no arithmetic: the same
// persistent warps, per-lane cp.async rings and store shapes as K1x / K2x (taco_xk.cuh, B = 256,
// bf16), with the math replaced by a byte pick.  nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -o tools/mempat tools/mempat.cu ; ./tools/mempat
#include <cstdio>
#include <cstdint>

constexpr int W = 4;  // warps per CTA
__device__ __forceinline__ void cp16(void* s, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((uint32_t)__cvta_generic_to_shared(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N> __device__ __forceinline__ void wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// K1 shape: tile = 8 blocks x 256 bf16 (4 KB), lane (g, q) copies 8 chunks at g*512 + j*64 + q*16;
// writes 64 codes per lane: CONTIG=1 as 4 x 16 B at lane_off (lane stride 64 B, K1x), CONTIG=0
// as 4 x 16 B with 16 B lane stride (coalesced per instruction)
template <int CONTIG>
__global__ void __launch_bounds__(128, 4) k1pat(const uint16_t* x, uint8_t* out, uint32_t ntiles) {
    extern __shared__ uint4 sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, q = lane & 3;
    uint4* sb = sm + warp * 2 * 256 + lane;
    const uint32_t stride = gridDim.x * W;
    uint32_t t = blockIdx.x * W + warp;
    auto issue = [&](uint32_t tt, int st) {
        const uint16_t* src = x + (uint64_t)tt * 2048 + g * 256 + q * 8;
        for (int j = 0; j < 8; ++j) cp16(sb + st * 256 + j * 32, src + j * 32);
        commit();
    };
    if (t < ntiles) issue(t, 0);
    for (int it = 0; t < ntiles; t += stride, ++it) {
        if (t + stride < ntiles) issue(t + stride, (it + 1) & 1); else commit();
        wait<1>();
        uint32_t acc[16];
        for (int j = 0; j < 8; ++j) {
            const uint4 u = sb[(it & 1) * 256 + j * 32];
            acc[2 * j] = u.x ^ u.y;
            acc[2 * j + 1] = u.z ^ u.w;
        }
        uint8_t* o = out + (uint64_t)t * 2048;
        for (int u = 0; u < 4; ++u) {
            const uint4 v = make_uint4(acc[4 * u], acc[4 * u + 1], acc[4 * u + 2], acc[4 * u + 3]);
            if (CONTIG) *reinterpret_cast<uint4*>(o + g * 256 + q * 64 + u * 16) = v;
            else *reinterpret_cast<uint4*>(o + u * 512 + lane * 16) = v;
        }
    }
}

// K2 shape: lane copies its 64 codes (4 x 16 B at g*256 + q*64, CONTIG=1) or coalesced 16 B at
// lane stride (CONTIG=0); writes 8 x 16 B of bf16 at g*512 + v*64 + q*16 (coalesced)
template <int CONTIG>
__global__ void __launch_bounds__(128, 4) k2pat(const uint8_t* m, uint16_t* y, uint32_t ntiles) {
    extern __shared__ uint4 sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, q = lane & 3;
    uint4* sb = sm + warp * 3 * 128 + lane;
    const uint32_t stride = gridDim.x * W;
    uint32_t t = blockIdx.x * W + warp;
    auto issue = [&](uint32_t tt, int st) {
        if (tt < ntiles) {
            const uint8_t* src = m + (uint64_t)tt * 2048;
            for (int c = 0; c < 4; ++c)
                cp16(sb + st * 128 + c * 32, CONTIG ? src + g * 256 + q * 64 + c * 16 : src + c * 512 + lane * 16);
        }
        commit();
    };
    issue(t, 0);
    issue(t + stride, 1);
    for (int it = 0; t < ntiles; t += stride, ++it) {
        issue(t + 2 * stride, (it + 2) % 3);
        wait<2>();
        uint4 u[4];
        for (int c = 0; c < 4; ++c) u[c] = sb[(it % 3) * 128 + c * 32];
        uint16_t* o = y + (uint64_t)t * 2048 + g * 256 + q * 8;
        for (int v = 0; v < 8; ++v) {
            const uint4 a = u[v & 3];
            *reinterpret_cast<uint4*>(o + v * 32) = make_uint4(a.x + v, a.y, a.z, a.w);
        }
    }
}

template <typename K, typename A, typename B>
float timeit(K k, int grid, size_t smem, A a, B b, uint32_t nt) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int i = 0; i < 3; ++i) k<<<grid, 128, smem>>>(a, b, nt);
    cudaEventRecord(e0);
    for (int i = 0; i < 50; ++i) k<<<grid, 128, smem>>>(a, b, nt);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return ms / 50;
}

int main() {
    const uint64_t n = 16384ull * 5120;  // configs[3]
    const uint32_t nt = n / 2048;
    uint16_t *x, *y; uint8_t* m;
    cudaMalloc(&x, n * 2); cudaMalloc(&y, n * 2); cudaMalloc(&m, n);
    cudaMemset(x, 1, n * 2); cudaMemset(m, 1, n);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * 4;
    const double bytes = n * 3.0;
    cudaFuncSetAttribute(k1pat<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    cudaFuncSetAttribute(k1pat<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    float a = timeit(k1pat<1>, grid, 32768, x, m, nt), b = timeit(k1pat<0>, grid, 32768, x, m, nt);
    printf("K1 pattern: codes 64B/lane %.2f us %.0f GB/s | codes coalesced %.2f us %.0f GB/s\n", a * 1e3, bytes / a / 1e6, b * 1e3, bytes / b / 1e6);
    a = timeit(k2pat<1>, grid, 24576, m, y, nt); b = timeit(k2pat<0>, grid, 24576, m, y, nt);
    printf("K2 pattern: codes 64B/lane %.2f us %.0f GB/s | codes coalesced %.2f us %.0f GB/s\n", a * 1e3, bytes / a / 1e6, b * 1e3, bytes / b / 1e6);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
