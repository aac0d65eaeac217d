// K1 dispatch: block size x input dtype x FP8 format.
#include "taco_kernels.cuh"
#include "taco_launch.h"
#include "taco_tile.cuh"
#include "taco_r2.cuh"

namespace taco_impl {
using namespace taco_dev;

namespace {
template <int B, typename T, int FMT>
cudaError_t run(const Launch& l, const ShardArgs& a, const CodecConsts& c) {
    if (a.nblk == 0 || a.P == 0) return cudaSuccess;
    if constexpr (FMT == 0 && B >= 32 && B <= 1024) {
        if (kernel_family() == 3) {
            using Cf = r2::Cfg<B, T>;
            const uint64_t tps = (a.nblk + Cf::G - 1) / Cf::G;
            auto* kern = &r2::k_compress_r2<B, T>;
            const unsigned grid = persistent_grid(kern, r2::kWarps * 32, Cf::SMEM, tps * a.P, r2::kWarps);
            uint32_t* ctr = claim_counter();
            if (!ctr) return cudaErrorMemoryAllocation;
            kern<<<grid, r2::kWarps * 32, Cf::SMEM, l.stream>>>(static_cast<const T*>(l.in),
                                                               static_cast<uint8_t*>(l.out), a, c,
                                                               make_fastdiv((uint32_t)tps), ctr);
            return cudaGetLastError();
        }
    }
    if constexpr (FMT == 0 && B >= 64 && B <= 512) {
        if (kernel_family() == 1) {
            constexpr int NB = B == 64 ? 6 : B == 128 ? 7 : B == 256 ? 8 : 9;
            using Cf = tile::K1T<NB, T>;
            const uint64_t tps = (a.nblk + tile::kBlocks - 1) / tile::kBlocks;
            auto* kern = &tile::k_compress_tile<NB, T>;
            const unsigned grid = persistent_grid(kern, tile::kTileWarps * 32, Cf::SMEM, tps * a.P, tile::kTileWarps);
            kern<<<grid, tile::kTileWarps * 32, Cf::SMEM, l.stream>>>(static_cast<const T*>(l.in),
                                                                      static_cast<uint8_t*>(l.out), a, c,
                                                                      make_fastdiv((uint32_t)tps));
            return cudaGetLastError();
        }
    }
    if constexpr (B <= 1024) {
        constexpr int VMAX = 8, EMAX = FMT == 0 ? TACO_K1_EMAX : 32;  // fp32 pairs: 64/lane; fp64: 32/lane
        using Cf = K1Cfg<B, T, FMT, EMAX, VMAX>;
        const uint64_t tps = (a.nblk + Cf::Gm::G - 1) / Cf::Gm::G;
        auto* kern = &k_compress<B, T, FMT, EMAX, VMAX>;
        const unsigned grid = persistent_grid(kern, kPipeWarps * 32, Cf::SMEM, tps * a.P, kPipeWarps);
        kern<<<grid, kPipeWarps * 32, Cf::SMEM, l.stream>>>(static_cast<const T*>(l.in), static_cast<uint8_t*>(l.out), a, c, make_fastdiv((uint32_t)tps));
    } else {
        const size_t smem = (size_t)B * sizeof(BigW<FMT, B>);
        auto* kern = &k_compress_big<B, T, FMT>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<dim3((unsigned)a.nblk, a.P), kBigThreads, smem, l.stream>>>(static_cast<const T*>(l.in),
                                                              static_cast<uint8_t*>(l.out), a, c);
    }
    return cudaGetLastError();
}

template <typename T, int FMT>
cudaError_t by_size(const Launch& l, const ShardArgs& a, const CodecConsts& c) {
    switch (l.block_size) {
#define CASE(B) \
    case B: return run<B, T, FMT>(l, a, c);
        TACO_WARP_SIZES(CASE)
        TACO_BIG_SIZES(CASE)
#undef CASE
        default: return cudaErrorInvalidValue;
    }
}
}  // namespace

cudaError_t launch_compress(const Launch& l, const ShardArgs& a, const CodecConsts& c) {
    if (l.dtype == 1) return l.format ? by_size<__nv_bfloat16, 1>(l, a, c) : by_size<__nv_bfloat16, 0>(l, a, c);
    return l.format ? by_size<float, 1>(l, a, c) : by_size<float, 0>(l, a, c);
}

}  // namespace taco_impl
