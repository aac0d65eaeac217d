// taco_tc.cuh -- K1 on the 5th-generation tensor cores (tcgen05) for bf16 input, E4M3,
// B = 256: the Hadamard rotation as a GEMM.
//
// Why.  The CUDA-core K1 spends ~1000 warp instructions per 2048 elements, 40 % of them in
// the butterfly, and is issue bound at ~45 % of HBM (profiles/README.md).  Here the
// rotation runs on the tensor pipe and the CUDA cores only do the per-block epilogue.
//
// Math.  Sylvester order: H256 = H4 (x) H64, so for a block x = [x0|x1|x2|x3] (4 x 64)
//     P_i = x_i H64  (i = 0..3),   y[64q + j] = sum_i (-1)^popcount(q & i) P_i[j].
// The P_i are tcgen05.mma.kind::f16 products (bf16 x bf16 -> fp32 in TMEM): the products
// x * (+-1) are exact and the 64-term sums accumulate in fp32; the last two butterfly
// levels (bits 6 and 7: a = P0+P1, b = P0-P1, c = P2+P3, d = P2-P3, y = a+-c, b+-d) are
// fp32 adds in the epilogue, like every stage of the reference's (a+b, a-b) recursion
// (transform.cpp:46-55).  The block max needs no extra pass: max(|a+c|, |a-c|) =
// |a| + |c| exactly, and the fp32 rounding of that sum is the rounding of the larger.
// H64 as the B operand is 8 KB, which leaves shared memory for three 64 KB stages.
//
// Tiles.  M = 128 blocks (32768 elements) per tile, one block per TMEM lane.
//   warp 0      TMA producer: four 2D boxes of [128 rows x 64 bf16] with the 128-byte
//               swizzle = the canonical K-major SW128 UMMA layout (2 stages, 64 KB each)
//   warp 1      TMEM allocator + MMA issuer (one elected lane): 4 x 4 MMAs of
//               M=128, N=64, K=16 per tile into a 256-column TMEM buffer
//   warps 2-5   sum of squares (fp64, or fp32 with TACO_SUMSQ) and alpha, one thread per
//               block row, straight from the staged tile; the stage is released as soon as
//               they and the MMA are done, so TMA runs ahead of the epilogue
//   warps 6-21  epilogue: two groups of 8 warps (group g takes tiles i = g mod 2 from TMEM
//               buffer g, so the MMA of tile i+1 overlaps the epilogue of tile i); in a
//               group, 4 TMEM lane quarters x 2 column halves: each thread owns 128 of its
//               block's 256 outputs, written as four full 32-byte sectors (st.global.v8).
// B operand: H64 (8 KB, bf16 +-1) written once into shared memory by all threads.
#pragma once

#include <cuda.h>

#include "taco_kernels.cuh"

#ifndef TACO_TC_DEBUG
#define TACO_TC_DEBUG 0
#endif

namespace taco_dev {
namespace tc {

constexpr int kB = 256;              // block size served
constexpr int kM = 128;              // blocks per tile (UMMA M)
constexpr int kStages = 3;           // A stages
constexpr int kSlab = kM * 128;      // one 64-element K slab of the tile: 128 rows x 128 B
constexpr int kStageBytes = 4 * kSlab;  // 64 KB: the whole 128 x 256 bf16 tile
constexpr int kBBytes = 64 * 128;    // H64: 64 rows (n) x 64 k x bf16 = one K slab
constexpr int kBufs = 2;             // TMEM accumulator buffers
#ifndef TACO_TC_GROUPS
#define TACO_TC_GROUPS 2
#endif
constexpr int kEpiGroups = TACO_TC_GROUPS;  // epilogue groups: group g takes tiles i = g mod groups
constexpr int kGroupWarps = 8;              // 4 lane quarters x 2 column halves
constexpr int kEpiWarps = kEpiGroups * kGroupWarps;
constexpr int kSsWarps = 4;          // sum-of-squares warps: one thread per block row
constexpr int kEpi0 = 2 + kSsWarps;  // first epilogue warp
constexpr int kThreads = (kEpi0 + kEpiWarps) * 32;
constexpr int kTmemCols = 512;       // 2 buffers x (128 P + 128 Q) fp32 columns

struct Smem {  // byte offsets inside the 1024-aligned dynamic shared memory
    static constexpr int A = 0;
    static constexpr int B = A + kStages * kStageBytes;
    static constexpr int SS = B + kBBytes;               // [2 parity][128 rows] double: sum of squares
    static constexpr int AL = SS + 2 * kM * 8;           // [2 parity][128 rows] float: alpha
    static constexpr int RED_MX = AL + 2 * kM * 4;       // [groups][2][2 halves][128 rows] float
    static constexpr int BARS = RED_MX + kEpiGroups * 2 * 2 * kM * 4; // full, empty [kStages]; tfull, tempty, ssfull, ssempty [kBufs]
    static constexpr int TMEM = BARS + (2 * kStages + 4 * kBufs) * 8;
    static constexpr int TOTAL = TMEM + 16;
};
constexpr size_t kSmem = Smem::TOTAL + 1024;  // + alignment slack

struct TcArgs {
    uint64_t rows_per_shard;  // S / B
    uint64_t blk0;            // first block of the chunk, per shard
    uint64_t nblk;            // blocks per shard in the chunk
    uint64_t msg_stride;
    uint64_t scal_off;
    uint32_t P;
    int* flags;
};

// ------------------------------------------------------------------ PTX ----
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(dst),
        "l"(map), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void mbar_init_u(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive_u(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait_u(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "TACO_TCW:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra TACO_TCD;\n\t"
        "bra TACO_TCW;\n"
        "TACO_TCD:\n\t}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// UMMA shared-memory descriptor, K-major, 128-byte swizzle (canonical layout
// Swizzle<3,4,3> o ((8,n),2):((8,SBO),1) in 16-byte units): LBO = 1, SBO = 1024 B.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t addr) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3fff);       // start address
    d |= (uint64_t)1 << 16;                      // leading byte offset (ignored for SW128 K-major)
    d |= (uint64_t)(1024 >> 4) << 32;            // stride byte offset: 8 rows x 128 B
    d |= (uint64_t)1 << 46;                      // version (sm_100)
    d |= (uint64_t)2 << 61;                      // layout: SWIZZLE_128B
    return d;
}

// instruction descriptor: D f32, A/B bf16, both K-major, N = 64, M = 128
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(kIdesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}

// 32 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// 16 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
// 8 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// --------------------------------------------------------------- epilogue ----
// Sum of squares of one 64-element K slab of the thread's block from the staged
// (swizzled) tile: row r is 128 B at slab + r*128, chunk c at position c ^ (r & 7).
__device__ __forceinline__ double slab_sumsq(const unsigned char* slab, int r) {
    const unsigned char* row = slab + r * 128;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
#if TACO_SUMSQ == 1
    float facc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#endif
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const uint4 u = *reinterpret_cast<const uint4*>(row + ((c ^ (r & 7)) << 4));
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
#if TACO_SUMSQ == 1
            facc[(2 * i) & 7] = fma_bf16_sq(w[i] & 0xffffu, facc[(2 * i) & 7]);
            facc[(2 * i + 1) & 7] = fma_bf16_sq(w[i] >> 16, facc[(2 * i + 1) & 7]);
#else
            const double d0 = tile::bf16_to_f64(w[i] & 0xffffu), d1 = tile::bf16_to_f64(w[i] >> 16);
            acc[(2 * i) & 3] = fma(d0, d0, acc[(2 * i) & 3]);
            acc[(2 * i + 1) & 3] = fma(d1, d1, acc[(2 * i + 1) & 3]);
#endif
        }
    }
#if TACO_SUMSQ == 1
    const float sf = ((facc[0] + facc[1]) + (facc[2] + facc[3])) + ((facc[4] + facc[5]) + (facc[6] + facc[7]));
    if (sf < 0x1p100f && !(sf > 0.0f && sf < 0x1p-100f)) return (double)sf;
    // out of the fp32 squares' exact range: the fp64 sum (thread-local, rare)
#pragma unroll 1
    for (int c = 0; c < 8; ++c) {
        const uint4 u = *reinterpret_cast<const uint4*>(row + ((c ^ (r & 7)) << 4));
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
        for (int i = 0; i < 4; ++i) {
            const double d0 = tile::bf16_to_f64(w[i] & 0xffffu), d1 = tile::bf16_to_f64(w[i] >> 16);
            acc[0] = fma(d0, d0, acc[0]);
            acc[1] = fma(d1, d1, acc[1]);
        }
    }
#endif
    return (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

__device__ __forceinline__ void named_bar(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// Rare fallback for one block whose fp32 accumulators overflowed (|x| >~ 1e36): the
// butterfly in fp32 with the exact power-of-two pre-scale, from global memory, in one
// thread (local-memory array), then quantise + store.
__device__ __noinline__ void block_slow(const __nv_bfloat16* __restrict__ xb, double ss, float alpha, CodecConsts c,
                                        uint8_t* codes, float* s_out) {
    float v[kB];
    const float p2 = pow2_near(alpha);
    for (int i = 0; i < kB; ++i) v[i] = __bfloat162float(xb[i]) * p2;
    for (int h = 1; h < kB; h <<= 1)
        for (int i = 0; i < kB; ++i)
            if ((i & h) == 0) {
                const float a = v[i], b = v[i + h];
                v[i] = a + b;
                v[i + h] = a - b;
            }
    float ymax = 0.0f;
    for (int i = 0; i < kB; ++i) ymax = fmaxf(ymax, fabsf(v[i]));
    float s;
    double k;
    block_scale((double)ymax, alpha, p2, c, s, k);
    for (int i = 0; i < kB; i += 2) {
        float2 w[1] = {make_float2(v[i], v[i + 1])};
        mul_wide<1>(w, k);
        *reinterpret_cast<uint16_t*>(codes + i) = (uint16_t)enc2<0>(w[0]);
    }
    *s_out = s;
}

// -------------------------------------------------------------------- K1 -----
__global__ void __launch_bounds__(kThreads, 1)
    k_compress_tc(const __grid_constant__ CUtensorMap xmap, const __nv_bfloat16* __restrict__ x,
                  uint8_t* __restrict__ msgs, TcArgs a, CodecConsts c, FastDiv tps) {
    extern __shared__ unsigned char smem_raw[];
    // 1024-byte alignment by offsetting the shared array itself (keeps LDS/STS addressing)
    unsigned char* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
    const uint32_t sbase = su32(smem);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t bar_full = sbase + Smem::BARS, bar_empty = bar_full + 8 * kStages,
                   bar_tfull = bar_empty + 8 * kStages, bar_tempty = bar_tfull + 8 * kBufs,
                   bar_ssfull = bar_tempty + 8 * kBufs, bar_ssempty = bar_ssfull + 8 * kBufs;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + Smem::TMEM);

    // H64 (B operand, N x K K-major SW128): element (n, k) = (-1)^popcount(n & k)
    for (int id = threadIdx.x; id < kBBytes / 16; id += blockDim.x) {
        const int n = id >> 3, ch = id & 7;
        uint32_t wv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int k0 = ch * 8 + 2 * e;
            const uint32_t lo = (__popc(n & k0) & 1) ? 0xBF80u : 0x3F80u;
            const uint32_t hi = (__popc(n & (k0 + 1)) & 1) ? 0xBF80u : 0x3F80u;
            wv[e] = lo | (hi << 16);
        }
        *reinterpret_cast<uint4*>(smem + Smem::B + n * 128 + ((ch ^ (n & 7)) << 4)) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init_u(bar_full + 8 * i, 1);
            mbar_init_u(bar_empty + 8 * i, 1 + kSsWarps);  // MMA commit + the sum-of-squares warps
        }
        for (int i = 0; i < kBufs; ++i) {
            mbar_init_u(bar_tfull + 8 * i, 1);
            mbar_init_u(bar_tempty + 8 * i, kGroupWarps);
            mbar_init_u(bar_ssfull + 8 * i, kSsWarps);
            mbar_init_u(bar_ssempty + 8 * i, kGroupWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                     "n"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic H128 writes -> tensor core reads
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t ntiles = a.P * tps.d;

    if (warp == 0) {
        // ============================ TMA producer ============================
        if (lane == 0) {
            uint32_t i = 0;
            for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
                const int s = i % kStages;
                mbar_wait_u(bar_empty + 8 * s, ((i / kStages) & 1) ^ 1);
                const uint32_t p = tps.div(t);
                const int row0 = (int)(p * a.rows_per_shard + a.blk0 + (uint64_t)(t - p * tps.d) * kM);
                mbar_expect_tx(bar_full + 8 * s, kStageBytes);
#pragma unroll
                for (int slab = 0; slab < 4; ++slab)
                    tma_load_2d(sbase + Smem::A + s * kStageBytes + slab * kSlab, &xmap, slab * 64, row0,
                                bar_full + 8 * s);
            }
        }
    } else if (warp == 1) {
        // ============================ MMA issuer ==============================
        if (lane == 0) {
            uint32_t i = 0;
            for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
                const int s = i % kStages, buf = i % kBufs;
                mbar_wait_u(bar_tempty + 8 * buf, ((i / kBufs) & 1) ^ 1);
                mbar_wait_u(bar_full + 8 * s, (i / kStages) & 1);
                tc_fence_after();
                const uint32_t a0 = sbase + Smem::A + s * kStageBytes, b0 = sbase + Smem::B;
#pragma unroll
                for (int qi = 0; qi < 4; ++qi) {  // P_qi = x_qi H64 -> columns 64 qi .. 64 qi + 63
                    const uint32_t d = tmem + buf * 256 + qi * 64;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        umma_bf16(d, sw128_desc(a0 + qi * kSlab + kk * 32), sw128_desc(b0 + kk * 32), kk != 0);
                }
                umma_commit(bar_empty + 8 * s);
                umma_commit(bar_tfull + 8 * buf);
            }
        }
    } else if (warp < kEpi0) {
        // ========================== sum of squares ============================
        // one thread per block row: the whole staged row (4 slabs), alpha; the stage is
        // released as soon as these warps and the MMA are done with it
        const int r = (warp - 2) * 32 + lane;
        double* ss_buf = reinterpret_cast<double*>(smem + Smem::SS);
        float* al_buf = reinterpret_cast<float*>(smem + Smem::AL);
        uint32_t i = 0;
        for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
            const int s = i % kStages, par = i & 1;
            mbar_wait_u(bar_full + 8 * s, (i / kStages) & 1);
            const unsigned char* st = smem + Smem::A + s * kStageBytes;
#if TACO_TC_DEBUG & 1
            const double ss = 1.0 + (double)st[r];  // A/B experiment: no sum of squares
#else
            const double ss = (slab_sumsq(st, r) + slab_sumsq(st + kSlab, r)) +
                              (slab_sumsq(st + 2 * kSlab, r) + slab_sumsq(st + 3 * kSlab, r));
#endif
            __syncwarp();
            if (lane == 0) mbar_arrive_u(bar_empty + 8 * s);
            const float alpha = block_alpha_fast(ss, c);
            mbar_wait_u(bar_ssempty + 8 * par, ((i >> 1) & 1) ^ 1);
            ss_buf[par * kM + r] = ss;
            al_buf[par * kM + r] = alpha;
            __syncwarp();
            if (lane == 0) mbar_arrive_u(bar_ssfull + 8 * par);  // release: makes the writes visible
        }
    } else {
        // ============================== epilogue ==============================
        // group g = tiles i with i % 2 == g, TMEM buffer g.  Warp (quarter, h): TMEM lanes
        // 32*quarter.. = blocks; columns j in [32h, 32h+32) of P0..P3, i.e. outputs
        // 64q + 32h + j' (q = 0..3) of each of its 32 blocks -> four 32-byte code runs per
        // thread (full-sector 256-bit stores).  Pass 1 finds the block max (combined with
        // the other half through shared memory), pass 2 re-reads TMEM and quantises.
        const int e = warp - kEpi0, grp = e / kGroupWarps, quarter = warp & 3, h = (e % kGroupWarps) >> 2;
        const int r = quarter * 32 + lane;  // TMEM lane = block row of the tile
        const double* ss_buf = reinterpret_cast<const double*>(smem + Smem::SS);
        const float* al_buf = reinterpret_cast<const float*>(smem + Smem::AL);
        float* red_mx = reinterpret_cast<float*>(smem + Smem::RED_MX);  // [grp][pp][h][row]
        const float2 neg1 = make_float2(-1.0f, -1.0f);
        uint32_t i = grp;
        uint32_t t = blockIdx.x + grp * gridDim.x;
        for (; t < ntiles; t += kEpiGroups * gridDim.x, i += kEpiGroups) {
            const int pp = (i / kEpiGroups) & 1, buf = i % kBufs, par = i & 1;
            const uint32_t p = tps.div(t);
            const uint64_t kk = (uint64_t)(t - p * tps.d) * kM + r;  // block within the chunk
            const bool live = kk < a.nblk;
            mbar_wait_u(bar_tfull + 8 * buf, (i / kBufs) & 1);
            tc_fence_after();
            const uint32_t tl = tmem + ((uint32_t)(quarter * 32) << 16) + buf * 256 + h * 32;
            float mx = 0.0f;
#pragma unroll
            for (int sub = 0; sub < 4; ++sub) {  // 8 columns at a time: P0..P3 in 32 registers
                float P0[8], P1[8], P2[8], P3[8];
                tmem_ld8(tl + sub * 8, P0);
                tmem_ld8(tl + 64 + sub * 8, P1);
                tmem_ld8(tl + 128 + sub * 8, P2);
                tmem_ld8(tl + 192 + sub * 8, P3);
                tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float2 p0 = make_float2(P0[2 * j], P0[2 * j + 1]), p1 = make_float2(P1[2 * j], P1[2 * j + 1]);
                    const float2 p2 = make_float2(P2[2 * j], P2[2 * j + 1]), p3 = make_float2(P3[2 * j], P3[2 * j + 1]);
                    const float2 A = __fadd2_rn(p0, p1), Bv = __ffma2_rn(p1, neg1, p0);
                    const float2 Cv = __fadd2_rn(p2, p3), Dv = __ffma2_rn(p3, neg1, p2);
                    // bit 7: max(|a+c|, |a-c|) = |a| + |c|
                    mx = fmaxf(mx, fmaxf(fabsf(A.x) + fabsf(Cv.x), fabsf(A.y) + fabsf(Cv.y)));
                    mx = fmaxf(mx, fmaxf(fabsf(Bv.x) + fabsf(Dv.x), fabsf(Bv.y) + fabsf(Dv.y)));
                }
            }
            float* red = red_mx + ((grp * 2 + pp) * 2) * kM;
            red[h * kM + r] = mx;
            named_bar(1 + grp * 4 + quarter, 64);
            const float ymax = fmaxf(red[r], red[kM + r]);
            mbar_wait_u(bar_ssfull + 8 * par, (i >> 1) & 1);
            const double ss = ss_buf[par * kM + r];
            const float alpha = al_buf[par * kM + r];
            __syncwarp();
            if (lane == 0) mbar_arrive_u(bar_ssempty + 8 * par);
            uint8_t* m = msgs + p * a.msg_stride;
            const bool overflow = !isfinite(ymax) && isfinite(ss);
            float s_blk;
            double k;
            block_scale_fast((double)ymax, alpha, 1.0f, c, s_blk, k);
            const bool kfast = fabs(k) < 0x1p126 && (k == 0.0 || fabs(k) >= 0x1p-126);
            const float2 kk2 = make_float2((float)k, (float)k);
            uint32_t code[4][8];  // [q][word]: codes of outputs 64q + 32h .. +31
#pragma unroll
            for (int sub = 0; sub < 4; ++sub) {
                float P0[8], P1[8], P2[8], P3[8];
                tmem_ld8(tl + sub * 8, P0);
                tmem_ld8(tl + 64 + sub * 8, P1);
                tmem_ld8(tl + 128 + sub * 8, P2);
                tmem_ld8(tl + 192 + sub * 8, P3);
                tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 4; j += 2) {
                    float2 Y[4][2];
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int jj = j + u;
                        const float2 p0 = make_float2(P0[2 * jj], P0[2 * jj + 1]);
                        const float2 p1 = make_float2(P1[2 * jj], P1[2 * jj + 1]);
                        const float2 p2 = make_float2(P2[2 * jj], P2[2 * jj + 1]);
                        const float2 p3 = make_float2(P3[2 * jj], P3[2 * jj + 1]);
                        const float2 A = __fadd2_rn(p0, p1), Bv = __ffma2_rn(p1, neg1, p0);
                        const float2 Cv = __fadd2_rn(p2, p3), Dv = __ffma2_rn(p3, neg1, p2);
                        // y[64q + ...]: q = 0 a+c, 1 b+d, 2 a-c, 3 b-d
                        Y[0][u] = __fadd2_rn(A, Cv);
                        Y[1][u] = __fadd2_rn(Bv, Dv);
                        Y[2][u] = __ffma2_rn(Cv, neg1, A);
                        Y[3][u] = __ffma2_rn(Dv, neg1, Bv);
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        if (kfast) {
                            Y[q][0] = __fmul2_rn(Y[q][0], kk2);
                            Y[q][1] = __fmul2_rn(Y[q][1], kk2);
                        } else {
                            mul_wide<2>(Y[q], k);
                        }
                        code[q][sub * 2 + j / 2] = enc2<0>(Y[q][0]) | (enc2<0>(Y[q][1]) << 16);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_u(bar_tempty + 8 * buf);
            if (live && !overflow && !(TACO_TC_DEBUG & 2)) {
                uint8_t* cp = m + kk * kB + h * 32;
                if ((reinterpret_cast<uintptr_t>(m) & 31) == 0) {  // messages past the first may be 16-aligned only
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(cp + 64 * q),
                                     "r"(code[q][0]), "r"(code[q][1]), "r"(code[q][2]), "r"(code[q][3]),
                                     "r"(code[q][4]), "r"(code[q][5]), "r"(code[q][6]), "r"(code[q][7])
                                     : "memory");
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        *reinterpret_cast<uint4*>(cp + 64 * q) = make_uint4(code[q][0], code[q][1], code[q][2], code[q][3]);
                        *reinterpret_cast<uint4*>(cp + 64 * q + 16) =
                            make_uint4(code[q][4], code[q][5], code[q][6], code[q][7]);
                    }
                }
            }
            if (live && h == 0) {
                if (overflow) {
                    const __nv_bfloat16* xb = x + (p * a.rows_per_shard + a.blk0 + kk) * kB;
                    block_slow(xb, ss, alpha, c, m + kk * kB, &s_blk);
                }
                *reinterpret_cast<float2*>(m + a.scal_off + kk * 8) = make_float2(alpha, s_blk);
                if (!isfinite(ss)) raise_flag(a.flags, 1);  // any NaN/Inf element poisons the sum
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols) : "memory");
    }
}

}  // namespace tc
}  // namespace taco_dev
