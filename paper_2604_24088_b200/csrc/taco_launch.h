// taco_launch.h -- host-side launch descriptors shared by the kernel dispatch units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "taco_kernels.cuh"

namespace taco_impl {

// One kernel launch: B, element dtype (0 f32, 1 bf16), FP8 format, pointers.
struct Launch {
    uint32_t block_size;
    int dtype;   // K1: input, K2: output, K3: acc_out (ignored when acc == nullptr)
    int format;  // 0 E4M3, 1 E5M2
    const void* in;
    void* out;
    void* acc;   // K3 only
    cudaStream_t stream;
};

cudaError_t launch_compress(const Launch& l, const taco_dev::ShardArgs& a, const taco_dev::CodecConsts& c);
cudaError_t launch_decompress(const Launch& l, const taco_dev::ShardArgs& a, const taco_dev::CodecConsts& c);
cudaError_t launch_reduce_encode(const Launch& l, const taco_dev::ShardArgs& a, const taco_dev::CodecConsts& c);

// persistent grid: enough CTAs to fill every SM at the kernel's occupancy, never more
// than there are tiles.  Occupancy (and the >48 KB smem opt-in) is resolved once per
// (kernel, device) -- kernels of one signature share a function type, so key by address.
int resident_ctas(const void* kernel, int threads, size_t smem);

template <typename K>
inline unsigned persistent_grid(K kernel, int threads, size_t smem, uint64_t tiles, int warps_per_cta) {
    const uint64_t ctas = (uint64_t)resident_ctas(reinterpret_cast<const void*>(kernel), threads, smem);
    const uint64_t need = (tiles + warps_per_cta - 1) / warps_per_cta;
    return (unsigned)(need < ctas ? need : ctas);
}

// Kernel family for E4M3 (TACO_B200_KERNELS, read once).  0 = default, the measured best
// per case (profiles/README.md): K1 register kernel for bf16 input, K1 tile kernel for fp32
// input (64 <= B <= 512), K2/K3 tile kernels.  5 = "tc": K1 on the tensor cores for bf16,
// B = 256 (taco_tc.cuh; parity-exact, slower today).  1 = "tile" (K1 tile for bf16 too),
// 2 = "reg" (the register kernels everywhere), 3 = "r2" (K1 r2).
// 6 = "r1": round 1's default dispatch (the register / tile kernels below instead of the
// exchange-butterfly family of taco_xk.cuh, which is the default for E4M3 at 64 <= B <= 512).
int kernel_family();
// the family the register / tile / tc dispatch sees ("r1" = its default)
inline int legacy_family() { const int f = kernel_family(); return f == 6 ? 0 : f; }
// whether E4M3 at 64 <= B <= 512 runs the exchange-butterfly kernels (taco_xk.cuh)
inline bool xk_family() { return kernel_family() == 0; }

// A zeroed device counter for one launch of a dynamically scheduled kernel (ring of
// counters per device; each kernel leaves its counter at zero when it finishes).
uint32_t* claim_counter();

// P zero-able 32-bit scratch words (per-shard scales of the non-Taco codec kinds).
uint32_t* claim_scratch(uint32_t words);

// the other codec kinds (launch_kinds.cu) and small helpers (launch_misc.cu)
cudaError_t launch_compress_kind(const Launch& l, const taco_dev::ShardArgs& a, const taco_dev::CodecConsts& c,
                                 int kind, int scope, uint32_t* smax);
cudaError_t launch_decompress_kind(const Launch& l, const taco_dev::ShardArgs& a, const taco_dev::CodecConsts& c,
                                   int kind);
cudaError_t launch_scaled_spectrum(const Launch& l, const taco_dev::ShardArgs& a, const taco_dev::CodecConsts& c,
                                   double qtop);
cudaError_t launch_add_f32(float* acc, const float* x, uint64_t n, cudaStream_t stream);
// analysis error_report on the device (synchronous; out8 = mse, relative_l2, max_abs,
// zero_collapse, kurtosis, kurtosis_defined, hist lo, hist hi); returns a cudaError_t
int error_report_dev(const void* x, int dx, const void* y, int dy, uint64_t n, uint32_t bins, double* out8,
                     unsigned long long* counts_host, cudaStream_t st);
// mode 0: SoA message -> TACOCMP1 archive (header from hdr22); mode 1: archive body -> message
cudaError_t launch_archive(const uint8_t* src, uint8_t* dst, uint64_t nblocks, uint64_t payload, uint64_t scal_off,
                           const uint8_t* hdr22, int mode, int* flags, cudaStream_t stream);

// peer-memory barrier: slot[q] = rank q's arrival array (kMaxPeers u32) as mapped here,
// epoch = this rank's barrier counter
struct PeerSlots {
    uint32_t* slot[taco_dev::kMaxPeers];
    uint32_t* epoch;
};
cudaError_t launch_peer_barrier(const PeerSlots& f, uint32_t rank, uint32_t P, uint64_t timeout_ns, int* flags,
                                cudaStream_t stream);

// values per lane of the register K2 / K3 decode (E4M3), per block size: K3 decodes with
// exactly K2's geometry so its stage-1 sums are bit-identical to K2 decodes
#ifndef TACO_K2_EMAX_B64
#define TACO_K2_EMAX_B64 TACO_K2_EMAX
#endif
#ifndef TACO_K2_EMAX_B1024
#define TACO_K2_EMAX_B1024 TACO_K2_EMAX
#endif
#ifndef TACO_K2_EMAX_B256
#define TACO_K2_EMAX_B256 TACO_K2_EMAX  // the register decode at B = 256 (family "reg" only)
#endif
template <int B>
constexpr int k2_emax() {
    return B == 2048 ? 64 : B == 64 ? TACO_K2_EMAX_B64 : B == 1024 ? TACO_K2_EMAX_B1024 : B == 256 ? TACO_K2_EMAX_B256
                                                                                         : TACO_K2_EMAX;
}

// Programmatic dependent launch (sm_90+): the kernel may be scheduled while the previous
// kernel on the stream drains; it runs its prologue (shared-memory / mbarrier setup,
// index math) and then blocks in griddepcontrol.wait until the previous grid has completed
// and its memory is visible (taco_dev::grid_dep_wait, before ANY global access).  Hides
// the launch gap and the ramp of back-to-back codec kernels.  TACO_PDL=0 disables it.
bool pdl_enabled();
// register K1 tile schedule: dynamic claims (TACO_K1_DYNAMIC=1) or static round robin
bool k1_dynamic();

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

inline taco_dev::FastDiv make_fastdiv(uint32_t d) {
    uint32_t s = 0;
    while ((1ull << s) < d) ++s;
    const uint32_t m = (uint32_t)((((1ull << s) - d) << 32) / d + 1);
    return taco_dev::FastDiv{d, m, s};
}

// grid for the warp kernels: one L-lane group per block job
inline unsigned warp_grid(uint64_t jobs, int blocks_per_warp, int threads) {
    const uint64_t warps = (jobs + blocks_per_warp - 1) / blocks_per_warp;
    const uint64_t wpc = threads / 32;
    return (unsigned)((warps + wpc - 1) / wpc);
}

}  // namespace taco_impl

// Instantiate `MACRO(B)` for every supported block size.
#define TACO_WARP_SIZES(M) M(2) M(4) M(8) M(16) M(32) M(64) M(128) M(256) M(512) M(1024)
#define TACO_BIG_SIZES(M) M(2048) M(4096) M(8192) M(16384) M(32768)
