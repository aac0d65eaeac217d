// launch_misc.cu -- small device helpers of the C ABI: the fp32 ascending-rank sum of the
// generic two-shot (collective.cpp:99) and the TACOCMP1 archive <-> message conversion
// (serialize.cpp:109-160).
#include <algorithm>
#include <cmath>
#include <vector>

#include "taco_kernels.cuh"
#include "taco_launch.h"

namespace taco_impl {
namespace {

__global__ void k_add_f32(float* __restrict__ acc, const float* __restrict__ x, uint64_t n) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        acc[i] = __fadd_rn(acc[i], x[i]);
}

struct Hdr {
    uint8_t b[22];
};

// one warp per block.  mode 0: message (SoA) -> archive: header + [payload][alpha][scale]
// per block at 22 + k*(payload+8), byte-wise (the records are not word aligned).
// mode 1: archive body -> message; non-finite scalars raise TACO_FLAG_BAD_SCALARS
// ("block scalars must be finite", serialize.cpp:150-153, checked by the caller).
__global__ void k_archive(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, uint64_t nblocks,
                          uint64_t payload, uint64_t scal_off, Hdr hdr, int mode, int* flags) {
    const uint64_t k = (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (mode == 0 && k == 0 && lane < 22) dst[lane] = hdr.b[lane];
    if (k >= nblocks) return;
    const uint64_t rec = 22 + k * (payload + 8);
    if (mode == 0) {
        for (uint64_t i = lane; i < payload; i += 32) dst[rec + i] = src[k * payload + i];
        if (lane < 8) dst[rec + payload + lane] = src[scal_off + k * 8 + lane];
    } else {
        for (uint64_t i = lane; i < payload; i += 32) dst[k * payload + i] = src[rec + i];
        if (lane < 8) dst[scal_off + k * 8 + lane] = src[rec + payload + lane];
        if (lane == 0) {
            uint32_t ab, sb;
            uint8_t t[8];
            for (int j = 0; j < 8; ++j) t[j] = src[rec + payload + j];
            ab = t[0] | (t[1] << 8) | (t[2] << 16) | ((uint32_t)t[3] << 24);
            sb = t[4] | (t[5] << 8) | (t[6] << 16) | ((uint32_t)t[7] << 24);
            if (!isfinite(__uint_as_float(ab)) || !isfinite(__uint_as_float(sb))) taco_dev::raise_flag(flags, 2);
        }
    }
}

}  // namespace

cudaError_t launch_add_f32(float* acc, const float* x, uint64_t n, cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    uint64_t blocks = (n + 255) / 256;
    k_add_f32<<<(unsigned)(blocks < 4096 ? blocks : 4096), 256, 0, stream>>>(acc, x, n);
    return cudaGetLastError();
}

cudaError_t launch_archive(const uint8_t* src, uint8_t* dst, uint64_t nblocks, uint64_t payload, uint64_t scal_off,
                           const uint8_t* hdr22, int mode, int* flags, cudaStream_t stream) {
    Hdr h{};
    if (hdr22)
        for (int i = 0; i < 22; ++i) h.b[i] = hdr22[i];
    const unsigned wpb = 8;
    const uint64_t grid = (nblocks + wpb - 1) / wpb;
    k_archive<<<(unsigned)(grid ? grid : 1), wpb * 32, 0, stream>>>(src, dst, nblocks, payload, scal_off, h, mode,
                                                                     flags);
    return cudaGetLastError();
}

}  // namespace taco_impl

// ----------------------------------------------------------- error metrics (f4) ---
// analysis.cpp:97-132 (error_report) on the device: elementwise error e = double(x) -
// y, two deterministic passes (fixed grid, per-CTA partials reduced in CTA order):
//   pass 1: sum e^2, sum x^2, max |e|, nonzero / collapsed counts, sum e, min e, max e
//   pass 2: centred moments sum d^2, sum d^4 (d = e - mean) and the histogram counts
// The final divisions / sqrt are done on the host in double, as the reference does.
namespace taco_impl {
namespace {

constexpr int kErrThreads = 256;
constexpr int kErrGrid = 592;

__device__ __forceinline__ float load_elem(const void* p, int dt, uint64_t i) {
    return dt == 1 ? __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]) : static_cast<const float*>(p)[i];
}

struct P1 {
    double se, sx, emax_abs, sum_e, emin, emax;
    unsigned long long nonzero, collapsed;
};

__device__ void block_reduce_p1(P1& v, P1* sh) {
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int s = kErrThreads / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) {
            P1& a = sh[threadIdx.x];
            const P1& b = sh[threadIdx.x + s];
            a.se += b.se; a.sx += b.sx; a.sum_e += b.sum_e;
            a.emax_abs = fmax(a.emax_abs, b.emax_abs);
            a.emin = fmin(a.emin, b.emin); a.emax = fmax(a.emax, b.emax);
            a.nonzero += b.nonzero; a.collapsed += b.collapsed;
        }
        __syncthreads();
    }
    v = sh[0];
}

__global__ void k_err_pass1(const void* x, int dx, const void* y, int dy, uint64_t n, P1* part) {
    __shared__ P1 sh[kErrThreads];
    P1 v{0.0, 0.0, 0.0, 0.0, INFINITY, -INFINITY, 0ull, 0ull};
    for (uint64_t i = (uint64_t)blockIdx.x * kErrThreads + threadIdx.x; i < n; i += (uint64_t)gridDim.x * kErrThreads) {
        const float xo = load_elem(x, dx, i), yr = load_elem(y, dy, i);
        const double e = (double)xo - (double)yr;
        v.se += e * e;
        v.sx += (double)xo * xo;
        v.emax_abs = fmax(v.emax_abs, fabs(e));
        v.sum_e += e;
        v.emin = fmin(v.emin, e);
        v.emax = fmax(v.emax, e);
        if (xo != 0.0f) {
            ++v.nonzero;
            if (yr == 0.0f) ++v.collapsed;
        }
    }
    block_reduce_p1(v, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = v;
}

struct P2 {
    double m2, m4;
};

__global__ void k_err_pass2(const void* x, int dx, const void* y, int dy, uint64_t n, double mean, double lo,
                            double hi, uint32_t bins, P2* part, unsigned long long* counts) {
    __shared__ P2 sh[kErrThreads];
    P2 v{0.0, 0.0};
    for (uint64_t i = (uint64_t)blockIdx.x * kErrThreads + threadIdx.x; i < n; i += (uint64_t)gridDim.x * kErrThreads) {
        const double e = (double)load_elem(x, dx, i) - (double)load_elem(y, dy, i);
        const double d = e - mean, d2 = d * d;
        v.m2 += d2;
        v.m4 += d2 * d2;
        const double t = (e - lo) / (hi - lo) * (double)bins;  // build_histogram (analysis.cpp:24-27)
        const unsigned idx = (unsigned)fmin(fmax(t, 0.0), (double)bins - 1.0);
        atomicAdd(counts + idx, 1ull);
    }
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int s = kErrThreads / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) {
            sh[threadIdx.x].m2 += sh[threadIdx.x + s].m2;
            sh[threadIdx.x].m4 += sh[threadIdx.x + s].m4;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

}  // namespace

int error_report_dev(const void* x, int dx, const void* y, int dy, uint64_t n, uint32_t bins, double* out8,
                     unsigned long long* counts_host, cudaStream_t st) {
    // out8: mse, relative_l2, max_abs, zero_collapse, kurtosis, kurtosis_defined, lo, hi
    P1* p1 = nullptr;
    P2* p2 = nullptr;
    unsigned long long* cnt = nullptr;
    cudaError_t e = cudaMallocAsync(&p1, kErrGrid * sizeof(P1), st);
    if (!e) e = cudaMallocAsync(&p2, kErrGrid * sizeof(P2), st);
    if (!e) e = cudaMallocAsync(&cnt, bins * sizeof(unsigned long long), st);
    if (!e) e = cudaMemsetAsync(cnt, 0, bins * sizeof(unsigned long long), st);
    std::vector<P1> h1(kErrGrid);
    std::vector<P2> h2(kErrGrid);
    if (!e) {
        k_err_pass1<<<kErrGrid, kErrThreads, 0, st>>>(x, dx, y, dy, n, p1);
        e = cudaGetLastError();
    }
    if (!e) e = cudaMemcpyAsync(h1.data(), p1, kErrGrid * sizeof(P1), cudaMemcpyDeviceToHost, st);
    if (!e) e = cudaStreamSynchronize(st);
    double se = 0, sx = 0, mx = 0, sum_e = 0, lo = INFINITY, hi = -INFINITY;
    unsigned long long nz = 0, col = 0;
    for (const P1& v : h1) {  // CTA order: deterministic
        se += v.se; sx += v.sx; sum_e += v.sum_e;
        mx = std::max(mx, v.emax_abs); lo = std::min(lo, v.emin); hi = std::max(hi, v.emax);
        nz += v.nonzero; col += v.collapsed;
    }
    if (!(hi > lo)) {
        lo -= 0.5;
        hi += 0.5;
    }
    const double mean = sum_e / (double)n;
    if (!e) {
        k_err_pass2<<<kErrGrid, kErrThreads, 0, st>>>(x, dx, y, dy, n, mean, lo, hi, bins, p2, cnt);
        e = cudaGetLastError();
    }
    if (!e) e = cudaMemcpyAsync(h2.data(), p2, kErrGrid * sizeof(P2), cudaMemcpyDeviceToHost, st);
    if (!e) e = cudaMemcpyAsync(counts_host, cnt, bins * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
    if (!e) e = cudaStreamSynchronize(st);
    cudaFreeAsync(p1, st);
    cudaFreeAsync(p2, st);
    cudaFreeAsync(cnt, st);
    if (e) return (int)e;
    double m2 = 0, m4 = 0;
    for (const P2& v : h2) {
        m2 += v.m2;
        m4 += v.m4;
    }
    m2 /= (double)n;
    m4 /= (double)n;
    out8[0] = se / (double)n;
    out8[1] = sx > 0.0 ? std::sqrt(se / sx) : (se > 0.0 ? INFINITY : 0.0);
    out8[2] = mx;
    out8[3] = nz == 0 ? 0.0 : (double)col / (double)nz;
    out8[4] = m2 <= 0.0 ? NAN : m4 / (m2 * m2) - 3.0;
    out8[5] = m2 <= 0.0 ? 0.0 : 1.0;
    out8[6] = lo;
    out8[7] = hi;
    return 0;
}

}  // namespace taco_impl

// ------------------------------------------------------ peer-memory barrier ---
// One CTA; thread q < P signals rank q and then waits for rank q's signal.  The epoch lives
// in this rank's own region so a captured CUDA graph keeps counting across replays.
namespace taco_impl {
namespace {

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void k_peer_barrier(PeerSlots f, uint32_t rank, uint32_t P, uint64_t timeout_ns, int* flags) {
    __shared__ uint32_t e;
    taco_dev::grid_dep_wait();  // the pushes of the kernel before this one have completed
    if (threadIdx.x == 0) {
        e = *f.epoch + 1;
        *f.epoch = e;
    }
    __syncthreads();
    const uint32_t q = threadIdx.x;
    if (q >= P) return;
    // the peer stores of the kernels before this one on the stream (K1 / K3 pushes) are
    // complete at this kernel's start (stream order); the system-scope fence + release
    // store publish them to the peer that acquires the signal
    __threadfence_system();
    st_release_sys(f.slot[q] + rank, e);
    const uint32_t* mine = f.slot[rank] + q;
    const uint64_t t0 = globaltimer();
    while ((int32_t)(ld_acquire_sys(mine) - e) < 0) {
        if (globaltimer() - t0 > timeout_ns) {
            taco_dev::raise_flag(flags, 4);  // TACO_FLAG_PEER_TIMEOUT
            break;
        }
        __nanosleep(64);
    }
}

}  // namespace

cudaError_t launch_peer_barrier(const PeerSlots& f, uint32_t rank, uint32_t P, uint64_t timeout_ns, int* flags,
                                cudaStream_t stream) {
    return launch_k(&k_peer_barrier, dim3(1), dim3(32), 0, stream, f, rank, P, timeout_ns, flags);
}

}  // namespace taco_impl
