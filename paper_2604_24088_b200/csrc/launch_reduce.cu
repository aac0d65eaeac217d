// K3 dispatch: block size x stage-1 output dtype x FP8 format.
#include "taco_kernels.cuh"
#include "taco_launch.h"
#include "taco_tile.cuh"
#include "taco_xk.cuh"

#ifndef TACO_XK_K3_P2
#define TACO_XK_K3_P2 1  // TP = 2 specialisation of K3 (both decodes in one straight-line block)
#endif
namespace taco_impl {
using namespace taco_dev;

namespace {
template <int L, typename T>
cudaError_t run_xk(const Launch& l, const ShardArgs& a, const CodecConsts& c) {
    using K = xk::K3X<L>;
    auto* kern = (a.P == 2 && TACO_XK_K3_P2) ? &xk::k3x<L, T, true> : &xk::k3x<L, T, false>;
    const uint64_t tiles = (a.nblk + K::G - 1) / K::G;
    const unsigned grid = (unsigned)((tiles + xk::kWarps - 1) / xk::kWarps);
    return launch_k(kern, grid, xk::kWarps * 32, K::SMEM, l.stream, static_cast<const uint8_t*>(l.in),
                    static_cast<uint8_t*>(l.out), static_cast<T*>(l.acc), a, c);
}

template <int B, typename T, int FMT>
cudaError_t run(const Launch& l, const ShardArgs& a, const CodecConsts& c) {
    if (a.nblk == 0) return cudaSuccess;
    if (a.npre | a.npost) {  // the fused peer phases live in the exchange-butterfly K1 / K2 only (K3 is plain)
        if constexpr (!(FMT == 0 && B >= 64 && B <= 512)) return cudaErrorNotSupported;
        if (!xk_family() || a.nblk >= (1ull << 31)) return cudaErrorNotSupported;
    }
    if constexpr (FMT == 0 && B >= 64 && B <= 512) {
        if (xk_family()) return run_xk<B / 64, T>(l, a, c);
    }
    if constexpr (FMT == 0 && B >= 256 && B <= 512) {
        if (legacy_family() != 2) {  // K2's decode is the tile kernel: decode with the same code
            constexpr int NB = B == 64 ? 6 : B == 128 ? 7 : B == 256 ? 8 : 9;
            using Cf = tile::K3T<NB>;
            auto* kern = &tile::k_reduce_encode_tile<NB, T>;
            static bool attr = false;
            if (!attr) {
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cf::SMEM);
                attr = true;
            }
            const uint64_t tiles = (a.nblk + tile::kBlocks - 1) / tile::kBlocks;
            const unsigned grid = (unsigned)((tiles + tile::kTileWarps - 1) / tile::kTileWarps);
            return launch_k(kern, grid, tile::kTileWarps * 32, Cf::SMEM, l.stream, static_cast<const uint8_t*>(l.in),
                            static_cast<uint8_t*>(l.out), static_cast<T*>(l.acc), a, c);
        }
    }
    if constexpr (B <= 1024 || (B == 2048 && FMT == 0)) {
        // the decode geometry of K2 (launch_decompress.cu): fp32 butterflies over the same
        // bits in the same order, so K3's per-rank decode is bit-identical to K2's
        constexpr int VMAX = 16, EMAX = FMT == 0 ? k2_emax<B>() : 32;
        using Gm = Geo<B, EMAX, VMAX>;
        return launch_k(&k_reduce_encode<B, T, FMT, EMAX, VMAX>, warp_grid(a.nblk, Gm::G, kWarpThreads), kWarpThreads,
                        0, l.stream, static_cast<const uint8_t*>(l.in), static_cast<uint8_t*>(l.out),
                        static_cast<T*>(l.acc), a, c);
    } else {
        const size_t smem = (size_t)B * sizeof(BigW<FMT, B>);
        auto* kern = &k_reduce_encode_big<B, T, FMT>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<(unsigned)a.nblk, kBigThreads, smem, l.stream>>>(static_cast<const uint8_t*>(l.in),
                                                                static_cast<uint8_t*>(l.out),
                                                                static_cast<T*>(l.acc), a, c);
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

cudaError_t launch_reduce_encode(const Launch& l, const ShardArgs& a, const CodecConsts& c) {
    if (l.acc && l.dtype == 1)
        return l.format ? by_size<__nv_bfloat16, 1>(l, a, c) : by_size<__nv_bfloat16, 0>(l, a, c);
    return l.format ? by_size<float, 1>(l, a, c) : by_size<float, 0>(l, a, c);
}

}  // namespace taco_impl
