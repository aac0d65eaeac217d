// mempat2.cu -- store / load variants for the codec patterns (B = 256, bf16, configs[3] size).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mempat2 tools/mempat2.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>

constexpr int W = 4;
__device__ __forceinline__ void cp16(void* s, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((uint32_t)__cvta_generic_to_shared(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N> __device__ __forceinline__ void wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }
__device__ __forceinline__ void st_cs(void* p, uint4 v) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void st_na(void* p, uint4 v) {
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
template <int MODE> __device__ __forceinline__ void st(void* p, uint4 v) {
    if (MODE == 0) *reinterpret_cast<uint4*>(p) = v;
    else if (MODE == 1) st_cs(p, v);
    else st_na(p, v);
}
// mbarrier + bulk helpers
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* m, int n) { asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(sa(m)), "r"(n)); }
__device__ __forceinline__ void mb_expect(uint64_t* m, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(sa(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* s, const void* g, uint32_t bytes, uint64_t* m) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(s)), "l"(g), "r"(bytes), "r"(sa(m)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* m, uint32_t ph) {
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(sa(m)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* g, const void* s, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(sa(s)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N> __device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void fence_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// K2 shape.  NS stages of codes (coalesced per-lane cp16); output: STG MODE 0/1/2 or TMA bulk (3)
template <int NS, int MODE>
__global__ void __launch_bounds__(128, 4) k2v(const uint8_t* m, uint16_t* y, uint32_t ntiles) {
    extern __shared__ uint4 sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, q = lane & 3;
    uint4* sb = sm + warp * (NS * 128 + (MODE == 3 ? 2 * 256 : 0));
    uint4* ob = sb + NS * 128;
    const uint32_t stride = gridDim.x * W;
    uint32_t t = blockIdx.x * W + warp;
    auto issue = [&](uint32_t tt, int st) {
        if (tt < ntiles) {
            const uint8_t* src = m + (uint64_t)tt * 2048;
            for (int c = 0; c < 4; ++c) cp16(sb + st * 128 + c * 32 + lane, src + c * 512 + lane * 16);
        }
        commit();
    };
    for (int i = 0; i < NS - 1; ++i) issue(t + i * stride, i);
    for (int it = 0; t < ntiles; t += stride, ++it) {
        issue(t + (NS - 1) * stride, (it + NS - 1) % NS);
        wait<NS - 1>();
        uint4 u[4];
        for (int c = 0; c < 4; ++c) u[c] = sb[(it % NS) * 128 + c * 32 + lane];
        uint16_t* o = y + (uint64_t)t * 2048;
        if (MODE < 3) {
            for (int v = 0; v < 8; ++v) {
                const uint4 a = u[v & 3];
                st<MODE>(o + g * 256 + q * 8 + v * 32, make_uint4(a.x + v, a.y, a.z, a.w));
            }
        } else {
            uint4* obuf = ob + (it & 1) * 256;
            if (lane == 0) bulk_wait_read<1>();
            __syncwarp();
            for (int v = 0; v < 8; ++v) {
                const uint4 a = u[v & 3];
                obuf[v * 32 + lane] = make_uint4(a.x + v, a.y, a.z, a.w);
            }
            fence_async();
            __syncwarp();
            if (lane == 0) bulk_s2g(o, obuf, 4096);
        }
    }
    if (MODE == 3 && lane == 0) bulk_wait_read<0>();
}

// K1 shape.  IN: 0 = per-lane cp16 (8 per lane), 1 = one TMA bulk per warp tile (4 KB) with an
// mbarrier ring of NS stages.  Codes out coalesced, STG MODE 0/1/2.
template <int IN, int NS, int MODE>
__global__ void __launch_bounds__(128, 4) k1v(const uint16_t* x, uint8_t* out, uint32_t ntiles) {
    extern __shared__ uint4 sm[];
    __shared__ uint64_t mbar[W][8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, q = lane & 3;
    uint4* sb = sm + warp * NS * 256;
    const uint32_t stride = gridDim.x * W;
    uint32_t t = blockIdx.x * W + warp;
    if (IN == 1) {
        if (lane == 0) for (int s = 0; s < NS; ++s) mb_init(&mbar[warp][s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        __syncwarp();
    }
    auto issue = [&](uint32_t tt, int st) {
        if (IN == 0) {
            if (tt < ntiles) {
                const uint16_t* src = x + (uint64_t)tt * 2048 + g * 256 + q * 8;
                for (int j = 0; j < 8; ++j) cp16(sb + st * 256 + j * 32 + lane, src + j * 32);
            }
            commit();
        } else if (tt < ntiles && lane == 0) {
            mb_expect(&mbar[warp][st], 4096);
            bulk_g2s(sb + st * 256, x + (uint64_t)tt * 2048, 4096, &mbar[warp][st]);
        }
    };
    for (int i = 0; i < NS - 1; ++i) issue(t + i * stride, i);
    for (int it = 0; t < ntiles; t += stride, ++it) {
        if (IN == 1) __syncwarp();  // stage (it-1)%NS fully read before its refill
        issue(t + (NS - 1) * stride, (it + NS - 1) % NS);
        const int cur = it % NS;
        if (IN == 0) wait<NS - 1>();
        else mb_wait(&mbar[warp][cur], (it / NS) & 1);
        uint32_t acc[16];
        for (int j = 0; j < 8; ++j) {
            const uint4 u = IN == 0 ? sb[cur * 256 + j * 32 + lane] : sb[cur * 256 + g * 32 + j * 4 + q];
            acc[2 * j] = u.x ^ u.y;
            acc[2 * j + 1] = u.z ^ u.w;
        }
        uint8_t* o = out + (uint64_t)t * 2048;
        for (int u = 0; u < 4; ++u)
            st<MODE>(o + u * 512 + lane * 16, make_uint4(acc[4 * u], acc[4 * u + 1], acc[4 * u + 2], acc[4 * u + 3]));
    }
}

__global__ void k_read(const uint4* p, uint64_t n, uint4* sink) {
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint4 v = __ldcs(p + i);
        acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
    if (acc.x == 0x12345678) sink[0] = acc;
}
__global__ void k_write(uint4* p, uint64_t n) {
    for (uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = make_uint4(i, 1, 2, 3);
}

static int g_iters = 40;
template <typename K, typename... A>
float timeit(K k, dim3 grid, int threads, size_t smem, A... a) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int i = 0; i < 3; ++i) k<<<grid, threads, smem>>>(a...);
    cudaEventRecord(e0);
    for (int i = 0; i < g_iters; ++i) k<<<grid, threads, smem>>>(a...);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return ms / g_iters;
}

int main(int argc, char** argv) {
    setvbuf(stdout, nullptr, _IONBF, 0);
    if (argc > 1) g_iters = atoi(argv[1]);
    const uint64_t n = 16384ull * 5120;
    const uint32_t nt = n / 2048;
    uint16_t *x, *y; uint8_t* m; uint4* sink;
    cudaMalloc(&x, n * 2); cudaMalloc(&y, n * 2); cudaMalloc(&m, n); cudaMalloc(&sink, 64);
    cudaMemset(x, 1, n * 2); cudaMemset(m, 1, n);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * 4;
    const double bytes = n * 3.0;
#define R(name, expr) { float t_ = expr; printf("%-34s %7.2f us %6.0f GB/s\n", name, t_ * 1e3, bytes / t_ / 1e6); }
    R("K2 coalesced codes NS3 STG", timeit(k2v<3, 0>, grid, 128, W * 3 * 128 * 16, m, y, nt));
    R("K2 coalesced codes NS3 st.cs", timeit(k2v<3, 1>, grid, 128, W * 3 * 128 * 16, m, y, nt));
    R("K2 coalesced codes NS3 st.na", timeit(k2v<3, 2>, grid, 128, W * 3 * 128 * 16, m, y, nt));
    R("K2 coalesced codes NS6 STG", timeit(k2v<6, 0>, grid, 128, W * 6 * 128 * 16, m, y, nt));
    R("K2 coalesced codes NS3 TMA store", timeit(k2v<3, 3>, grid, 128, W * (3 * 128 + 512) * 16, m, y, nt));
    R("K2 coalesced codes NS6 TMA store", timeit(k2v<6, 3>, grid, 128, W * (6 * 128 + 512) * 16, m, y, nt));
    R("K1 cp16 NS2 STG", timeit(k1v<0, 2, 0>, grid, 128, W * 2 * 256 * 16, x, m, nt));
    R("K1 cp16 NS2 st.cs", timeit(k1v<0, 2, 1>, grid, 128, W * 2 * 256 * 16, x, m, nt));
    R("K1 cp16 NS3 STG", timeit(k1v<0, 3, 0>, grid, 128, W * 3 * 256 * 16, x, m, nt));
    R("K1 TMA NS2 STG", timeit(k1v<1, 2, 0>, grid, 128, W * 2 * 256 * 16, x, m, nt));
    R("K1 TMA NS3 STG", timeit(k1v<1, 3, 0>, grid, 128, W * 3 * 256 * 16, x, m, nt));
    R("K1 TMA NS3 st.cs", timeit(k1v<1, 3, 1>, grid, 128, W * 3 * 256 * 16, x, m, nt));
    {
        float tr = timeit(k_read, dim3(sms * 8), 512, 0, (const uint4*)x, n * 2 / 16, sink);
        float tw = timeit(k_write, dim3(sms * 8), 512, 0, (uint4*)y, n * 2 / 16);
        printf("read-only  %.2f us %.0f GB/s | write-only %.2f us %.0f GB/s\n", tr * 1e3, n * 2 / tr / 1e6, tw * 1e3, n * 2 / tw / 1e6);
    }
    return 0;
}
