// K1 dispatch: block size x input dtype x FP8 format.
#include "taco_kernels.cuh"
#include "taco_launch.h"
#include "taco_tile.cuh"
#include "taco_xk.cuh"
#include "taco_tc.cuh"

#include <cudaTypedefs.h>

#include <mutex>

// values per lane of the register K1 (E4M3), per block size -- measured, bf16 [8192x2560]:
// B = 64: 32 -> 19.6 us (64 -> 29.4); B = 128: 32 -> 19.2 us (64 -> 22.2)
#ifndef TACO_K1_EMAX_B64
#define TACO_K1_EMAX_B64 32
#endif
#ifndef TACO_K1_EMAX_B128
#define TACO_K1_EMAX_B128 32
#endif
#ifndef TACO_K1_EMAX_B256
#define TACO_K1_EMAX_B256 TACO_K1_EMAX
#endif
#ifndef TACO_K1_EMAX_B512
#define TACO_K1_EMAX_B512 TACO_K1_EMAX
#endif
#ifndef TACO_K1_EMAX_B1024
#define TACO_K1_EMAX_B1024 TACO_K1_EMAX
#endif
template <int B>
constexpr int k1_emax() {
    return B == 64 ? TACO_K1_EMAX_B64 : B == 128 ? TACO_K1_EMAX_B128 : B == 256 ? TACO_K1_EMAX_B256
         : B == 512 ? TACO_K1_EMAX_B512 : B == 1024 ? TACO_K1_EMAX_B1024 : TACO_K1_EMAX;
}

namespace taco_impl {
using namespace taco_dev;

namespace {

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// K1 on the tensor cores (taco_tc.cuh): bf16 input, E4M3, B = 256, every shard a whole
// number of blocks and no ragged tail, 16-byte aligned input.  Returns cudaErrorNotSupported
// when the launch is not eligible (the caller then uses the CUDA-core kernel).
cudaError_t run_tc(const Launch& l, const ShardArgs& a, const CodecConsts& c) {
    using namespace taco_dev::tc;
    if (a.S % kB != 0 || a.n != (uint64_t)a.P * a.S || (reinterpret_cast<uintptr_t>(l.in) & 15) != 0)
        return cudaErrorNotSupported;
    auto encode = tensor_map_encoder();
    if (!encode) return cudaErrorNotSupported;
    const uint64_t nrows = a.n / kB;
    CUtensorMap map;
    const cuuint64_t dims[2] = {(cuuint64_t)kB, (cuuint64_t)nrows};
    const cuuint64_t strides[1] = {(cuuint64_t)kB * 2};
    const cuuint32_t box[2] = {64, (cuuint32_t)kM};
    const cuuint32_t estr[2] = {1, 1};
    if (encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(l.in), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorNotSupported;
    static std::once_flag attr;
    std::call_once(attr, [] {
        cudaFuncSetAttribute(&k_compress_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
    });
    const uint64_t tps = (a.nblk + kM - 1) / kM;
    const uint64_t ntiles = tps * a.P;
    int sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned grid = (unsigned)(ntiles < (uint64_t)sms ? ntiles : (uint64_t)sms);
    TcArgs ta{a.S / kB, a.blk0, a.nblk, a.msg_stride, a.scal_off, a.P, a.flags};
    k_compress_tc<<<grid, kThreads, kSmem, l.stream>>>(map, static_cast<const __nv_bfloat16*>(l.in),
                                                       static_cast<uint8_t*>(l.out), ta, c,
                                                       make_fastdiv((uint32_t)tps));
    return cudaGetLastError();
}

// exchange-butterfly K1 (taco_xk.cuh): E4M3, 64 <= B <= 512
template <int L, typename T>
cudaError_t run_xk(const Launch& l, const ShardArgs& a, const CodecConsts& c) {
    using K = xk::K1X<L, T>;
    const uint64_t tps = (a.nblk + K::G - 1) / K::G;
    auto* kern = a.ndst ? &xk::k1x<L, T, true> : &xk::k1x<L, T, false>;
    const unsigned grid = persistent_grid(kern, xk::kWarps * 32, K::SMEM, tps * a.P, xk::kWarps);
    return launch_k(kern, grid, xk::kWarps * 32, K::SMEM, l.stream, static_cast<const T*>(l.in),
                    static_cast<uint8_t*>(l.out), a, c, make_fastdiv((uint32_t)tps));
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
    if constexpr (FMT == 0 && B == 256 && std::is_same<T, __nv_bfloat16>::value) {
        if (legacy_family() == 5 && a.ndst == 0) {
            const cudaError_t e = run_tc(l, a, c);
            if (e != cudaErrorNotSupported) return e;
        }
    }
    if constexpr (FMT == 0 && B >= 64 && B <= 512) {
        const int fam = legacy_family();
        // fp32 input: the tile kernel for 128 <= B <= 512; at B = 64 the register kernel
        // (31.8 vs 41.3 us, profiles/README.md)
        if (fam == 1 || (fam == 0 && std::is_same<T, float>::value && B >= 128)) {
            constexpr int NB = B == 64 ? 6 : B == 128 ? 7 : B == 256 ? 8 : 9;
            using Cf = tile::K1T<NB, T>;
            const uint64_t tps = (a.nblk + tile::kBlocks - 1) / tile::kBlocks;
            auto* kern = &tile::k_compress_tile<NB, T>;
            const unsigned grid = persistent_grid(kern, tile::kTileWarps * 32, Cf::SMEM, tps * a.P, tile::kTileWarps);
            return launch_k(kern, grid, tile::kTileWarps * 32, Cf::SMEM, l.stream, static_cast<const T*>(l.in),
                            static_cast<uint8_t*>(l.out), a, c, make_fastdiv((uint32_t)tps));
        }
    }
    // E4M3 B = 2048: one warp per block (32 lanes x 64 values, 5 shuffle stages) instead of
    // the CTA-per-block shared-memory kernel
    if constexpr (B <= 1024 || (B == 2048 && FMT == 0)) {
        constexpr int VMAX = 8, EMAX = FMT == 0 ? k1_emax<B>() : 32;
        using Cf = K1Cfg<B, T, FMT, EMAX, VMAX>;
        const uint64_t tps = (a.nblk + Cf::Gm::G - 1) / Cf::Gm::G;
        auto* kern = a.ndst ? &k_compress<B, T, FMT, EMAX, VMAX, true> : &k_compress<B, T, FMT, EMAX, VMAX, false>;
        const unsigned grid = persistent_grid(kern, kPipeWarps * 32, Cf::SMEM, tps * a.P, kPipeWarps);
        uint32_t* ctr = nullptr;
        if (k1_dynamic()) {
            ctr = claim_counter();
            if (!ctr) return cudaErrorMemoryAllocation;
        }
        return launch_k(kern, grid, kPipeWarps * 32, Cf::SMEM, l.stream, static_cast<const T*>(l.in),
                        static_cast<uint8_t*>(l.out), a, c, make_fastdiv((uint32_t)tps), ctr);
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
