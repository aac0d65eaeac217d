// K2 dispatch: block size x output dtype x FP8 format.
#include "taco_kernels.cuh"
#include "taco_launch.h"
#include "taco_tile.cuh"
#include "taco_xk.cuh"

#ifndef TACO_K2_VMAX_B256
#define TACO_K2_VMAX_B256 16  // codes per lane run of the register K2 at B = 256 (32: 22.3 vs 17.4 us)
#endif
#ifndef TACO_K2_REG_BF16_B256
// bf16-output K2 at B = 256 on the register kernel: alone 17.3 vs 16.2 us (tile), but the
// K1 -> K2 round trip (bench value) 3,454 vs 3,379 GB/s -- the register K2 follows the register
// K1 with the same CTA shape under PDL and reads K1's L2-resident messages.  fp32 output (the
// reference's path, and K3's decode) stays on the tile kernel.
#define TACO_K2_REG_BF16_B256 1
#endif

namespace taco_impl {
using namespace taco_dev;

namespace {
template <int L, typename T>
cudaError_t run_xk(const Launch& l, const ShardArgs& a, const CodecConsts& c) {
    using K = xk::K2X<L>;
    const uint64_t tps = (a.nblk + K::G - 1) / K::G;
    auto* kern = &xk::k2x<L, T>;
    const unsigned grid = persistent_grid(kern, xk::kWarps * 32, K::SMEM, tps * a.P, xk::kWarps);
    return launch_k(kern, grid, xk::kWarps * 32, K::SMEM, l.stream, static_cast<const uint8_t*>(l.in),
                    static_cast<T*>(l.out), a, c, make_fastdiv((uint32_t)tps));
}

template <int B, typename T, int FMT>
cudaError_t run(const Launch& l, const ShardArgs& a, const CodecConsts& c) {
    if (a.nblk == 0 || a.P == 0) return cudaSuccess;
    if (a.npre | a.npost) {  // the fused peer phases live in the exchange-butterfly K1 / K2 only
        if constexpr (!(FMT == 0 && B >= 64 && B <= 512)) return cudaErrorNotSupported;
        if (!xk_family() || a.nblk >= (1ull << 31)) return cudaErrorNotSupported;
    }
    if constexpr (FMT == 0 && B >= 64 && B <= 512) {
        if (xk_family() && a.nblk < (1ull << 31)) return run_xk<B / 64, T>(l, a, c);
    }
    if constexpr (FMT == 0 && B >= 64 && B <= 512) {
        // measured (profiles/README.md): tile kernels for B >= 256 and fp32 output at
        // B = 128; the register kernel (K2_EMAX lanes geometry) at B = 64 and bf16 B = 128
        const bool tile = (B >= 256 && !(TACO_K2_REG_BF16_B256 && B == 256 && std::is_same<T, __nv_bfloat16>::value)) ||
                          (B == 128 && std::is_same<T, float>::value);
        if (legacy_family() != 2 && (tile || legacy_family() == 1)) {
            constexpr int NB = B == 64 ? 6 : B == 128 ? 7 : B == 256 ? 8 : 9;
            using Cf = tile::K2T<NB, T>;
            const uint64_t tps = (a.nblk + Cf::KB - 1) / Cf::KB;
            auto* kern = &tile::k_decompress_tile<NB, T>;
            const unsigned grid = persistent_grid(kern, tile::kTileWarps * 32, Cf::SMEM, tps * a.P, tile::kTileWarps);
            return launch_k(kern, grid, tile::kTileWarps * 32, Cf::SMEM, l.stream, static_cast<const uint8_t*>(l.in),
                            static_cast<T*>(l.out), a, c, make_fastdiv((uint32_t)tps));
        }
    }
    if constexpr (B <= 1024 || (B == 2048 && FMT == 0)) {  // B = 2048: one warp per block
        constexpr int VMAX = B == 256 ? TACO_K2_VMAX_B256 : 16, EMAX = FMT == 0 ? k2_emax<B>() : 32;
        using Cf = K2Cfg<B, T, FMT, EMAX, VMAX>;
        const uint64_t tps = (a.nblk + Cf::Gm::G - 1) / Cf::Gm::G;
        auto* kern = &k_decompress<B, T, FMT, EMAX, VMAX>;
        const unsigned grid = persistent_grid(kern, kPipeWarps * 32, Cf::SMEM, tps * a.P, kPipeWarps);
        return launch_k(kern, grid, kPipeWarps * 32, Cf::SMEM, l.stream, static_cast<const uint8_t*>(l.in),
                        static_cast<T*>(l.out), a, c, make_fastdiv((uint32_t)tps));
    } else {
        const size_t smem = (size_t)B * sizeof(BigW<FMT, B>);
        auto* kern = &k_decompress_big<B, T, FMT>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<dim3((unsigned)a.nblk, a.P), kBigThreads, smem, l.stream>>>(static_cast<const uint8_t*>(l.in),
                                                              static_cast<T*>(l.out), a, c);
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

cudaError_t launch_decompress(const Launch& l, const ShardArgs& a, const CodecConsts& c) {
    if (l.dtype == 1) return l.format ? by_size<__nv_bfloat16, 1>(l, a, c) : by_size<__nv_bfloat16, 0>(l, a, c);
    return l.format ? by_size<float, 1>(l, a, c) : by_size<float, 0>(l, a, c);
}

}  // namespace taco_impl
