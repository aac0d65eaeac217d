// launch_misc.cu -- small device helpers of the C ABI: the fp32 ascending-rank sum of the
// generic two-shot (collective.cpp:99) and the TACOCMP1 archive <-> message conversion
// (serialize.cpp:109-160).
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
