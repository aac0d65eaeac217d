// taco_kernels.cuh -- the three fused TACO kernels, templated on block size and types.
//
//   K1 k_compress        x (bf16|f32)          -> message(s): FP8 codes + (alpha, s)
//   K2 k_decompress      message(s)            -> y (bf16|f32), valid prefix only
//   K3 k_reduce_encode   P messages of a shard -> fp32 ascending-rank sum -> message
//
// Warp kernels (B <= 32*EMAX) keep whole blocks in registers of L-lane groups
// (taco_device.cuh); big-block kernels (B >= 2048) stage one block per CTA in shared
// memory.  All of them read their input once and write their output once.
// Grid: blockIdx.y = shard (K1/K2), blockIdx.x * warps * G + g = block of the chunk.
#pragma once

#include "taco_device.cuh"

#ifndef TACO_K1_WARP_MAJOR
#define TACO_K1_WARP_MAJOR 0
#endif
#ifndef TACO_FAST_SCALARS_REG
#define TACO_FAST_SCALARS_REG 1  // branch-free scalar chain (+2.5 % K1, profiles/README.md)
#endif

namespace taco_dev {

constexpr int kMaxPeers = 8;  // peer-memory collectives: ranks of one NVLink domain (TP <= 8)

struct ShardArgs {
    uint64_t n;           // logical elements of the tensor (K1/K2)
    uint64_t S;           // shard length
    uint32_t P;           // shards (K1/K2) or ranks (K3)
    uint64_t blk0;        // first block of the chunk, per shard
    uint64_t nblk;        // blocks per shard in the chunk
    uint64_t msg_stride;  // bytes between consecutive messages
    uint64_t scal_off;    // byte offset of the (alpha, s) array in a message
    int vec_ok;           // element pointers allow V-wide vector access
    int* flags;           // device error flags (may be null)
    // leading blocks of the chunk that are whole (no shard / tensor tail) in a shard other
    // than the last and in the last one (host-computed by with_full_blocks)
    uint64_t full_mid = 0, full_last = 0;
    // peer-memory collectives (ndst > 0): K1 writes shard p's message to dst[p] and K3
    // writes its re-encoded shard to every dst[0..ndst) -- stores straight into the
    // peers' receive buffers over NVLink.  Their visibility to the peers is established
    // by the next kernel on the stream, the peer barrier (fence.sc.sys, then a
    // st.release.sys signal), not by per-thread fences (one per warp of a 5,120-CTA K3
    // cost 2.3x its run time)
    uint8_t* dst[kMaxPeers] = {};
    uint32_t ndst = 0;
    uint32_t bcast = 0;  // K1 with ndst > 0: shard 0's message to every dst (all-gather)
    // K3 with nsrc > 0: rank r's message is read from src[r] (any address, e.g. a peer's
    // buffer over NVLink) instead of msgs + r * msg_stride
    const uint8_t* src[kMaxPeers] = {};
    uint32_t nsrc = 0;
    // fused peer signalling (taco_peer_*_dev; the exchange-butterfly K1 / K2 only, K3 stays
    // plain).  "pre" (kernel start, after grid_dep_wait): CTA 0 publishes this rank's epoch
    // into pre_sig[0..npre) -- one word per peer, "the kernels before this one are done with
    // the slots" -- then every CTA waits until this rank's words pre_wait[0..npre) reach it.
    // "post" (kernel end): the last CTA to finish opens the next epoch, publishes it into
    // post_sig[0..npost) and waits until post_wait[0..npost) reach it, so the next kernel on
    // the stream only reads slots every peer has finished writing (peer_pre / peer_post).
    uint32_t* pre_sig[kMaxPeers] = {};
    const uint32_t* pre_wait = nullptr;
    uint32_t npre = 0;
    uint32_t* post_sig[kMaxPeers] = {};
    const uint32_t* post_wait = nullptr;
    uint32_t npost = 0;
    uint32_t* epoch = nullptr;   // this rank's epoch word (own region)
    uint32_t* ticket = nullptr;  // CTA completion count of this launch (own region, left at 0)
    uint64_t timeout_ns = 0;
};

// programmatic dependent launch (taco_launch.h launch_k): let the next kernel on the stream
// be scheduled, then wait until the previous one has completed and its writes are visible.
// Called before a kernel's first global memory access; a no-op without the launch attribute.
__device__ __forceinline__ void grid_dep_wait() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

__device__ __forceinline__ void st_release_sys_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void raise_flag(int* flags, int bit);

// Thread-local poll of n words of this rank's region until each reaches e (system-scope
// acquire).  A peer that never signals sets TACO_FLAG_PEER_TIMEOUT (4) after timeout_ns
// instead of hanging the stream.
__device__ __forceinline__ void wait_words(const uint32_t* w, uint32_t n, uint32_t e, uint64_t timeout_ns,
                                           int* flags) {
    const uint64_t t0 = global_ns();
    for (uint32_t q = 0; q < n; ++q)
        while ((int32_t)(ld_acquire_sys_u32(w + q) - e) < 0) {
            if (global_ns() - t0 > timeout_ns) {
                raise_flag(flags, 4);
                return;
            }
            __nanosleep(64);
        }
}

// Phase at kernel start (after grid_dep_wait: the kernels before this one on the stream
// have completed and their stores are visible on this GPU).  CTA 0 makes them visible
// system-wide (fence.sc.sys, cumulative over what this thread observed) and releases the
// epoch into every peer's word; every CTA then acquires all of this rank's words.
__device__ __forceinline__ void peer_pre(const ShardArgs& a) {
    if (a.npre == 0) return;
    if (threadIdx.x == 0) {
        const uint32_t e = *reinterpret_cast<volatile const uint32_t*>(a.epoch);
        if (blockIdx.x == 0) {
            __threadfence_system();
#pragma unroll
            for (uint32_t q = 0; q < kMaxPeers; ++q)  // static indices: the parameter array stays in the constant bank
                if (q < a.npre) st_release_sys_u32(a.pre_sig[q], e);
        }
        wait_words(a.pre_wait, a.npre, e, a.timeout_ns, a.flags);
    }
    __syncthreads();
}

// Phase at kernel end (every thread of every CTA, after its last store).  The barrier
// orders the CTA's stores (peer memory over NVLink included) before thread 0's release at
// GPU scope (atom.release.gpu on the ticket); the CTA that completes the count has acquired
// every CTA's release, so its fence.sc.sys is cumulative over the whole grid's stores and
// its st.release.sys of the new epoch publishes them (PTX causality order is transitive
// across the GPU- and system-scope links).  That CTA then waits for every peer's word of
// the phase: the kernel completes only when every rank's stores of this phase have landed.
// One system fence and one waiting CTA per launch.
__device__ __forceinline__ void peer_post(const ShardArgs& a) {
    if (a.npost == 0) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t;
        asm volatile("atom.release.gpu.global.add.u32 %0, [%1], 1;" : "=r"(t) : "l"(a.ticket) : "memory");
        if (t == gridDim.x * gridDim.y - 1) {
            *reinterpret_cast<volatile uint32_t*>(a.ticket) = 0;  // the next launch counts from zero
            __threadfence_system();
            const uint32_t e = *reinterpret_cast<volatile uint32_t*>(a.epoch) + 1;
            *reinterpret_cast<volatile uint32_t*>(a.epoch) = e;
#pragma unroll
            for (uint32_t q = 0; q < kMaxPeers; ++q)
                if (q < a.npost) st_release_sys_u32(a.post_sig[q], e);
            wait_words(a.post_wait, a.npost, e, a.timeout_ns, a.flags);
        }
    }
}

__device__ __forceinline__ uint8_t* shard_msg(uint8_t* msgs, const ShardArgs& a, uint64_t p) {
    return a.ndst ? a.dst[p] : msgs + p * a.msg_stride;
}

// number of whole blocks of a chunk; every kernel's "is this tile full" is one compare
__host__ __device__ inline void with_full_blocks(ShardArgs& a, uint64_t B) {
    auto whole = [&](uint64_t valid) -> uint64_t {
        const uint64_t wb = valid / B;
        return wb <= a.blk0 ? 0 : (wb - a.blk0 < a.nblk ? wb - a.blk0 : a.nblk);
    };
    const uint64_t last_valid = a.P == 0 ? 0 : (a.n > (uint64_t)(a.P - 1) * a.S ? a.n - (uint64_t)(a.P - 1) * a.S : 0);
    a.full_mid = whole(a.S);
    a.full_last = whole(last_valid < a.S ? last_valid : a.S);
}

constexpr int kWarpThreads = 256;  // 8 warps per CTA
constexpr int kBigThreads = 512;   // one block per CTA for B >= 2048

// E4M3 rotates in packed fp32, E5M2 in fp64 (see RegsD)
template <int FMT, int E>
using RegsFor = typename std::conditional<FMT == 0, RegsF<E>, RegsD<E>>::type;

__device__ __forceinline__ void raise_flag(int* flags, int bit) {
    if (flags) atomicOr(flags, bit);
}

__device__ __forceinline__ int clamp_valid(int64_t a, int64_t b, int B) {
    int64_t v = a < b ? a : b;
    v = v < (int64_t)B ? v : (int64_t)B;
    return v < 0 ? 0 : (int)v;
}

// Rotate + quantise a register-resident block (rotate_block codec.cpp:45-62 and
// compress_block_taco :64-76).  On return the values hold Z/s, ready for the cvt.
template <int L, typename R>
__device__ __forceinline__ void quantise(R& v, int q, const CodecConsts& c, float& alpha, float& s, double& ss) {
    ss = group_sum<L>(v.sumsq());
#if TACO_FAST_SCALARS_REG
    alpha = block_alpha_fast(ss, c);
#else
    alpha = block_alpha(ss, c);
#endif
    // Exact power-of-two pre-scale, only where the butterfly could overflow fp32
    // (|y| <= B*max|x| <= B*sqrt(ss)); elsewhere p2 = 1 and the multiply is skipped.
    const bool huge = !(ss < 0x1p160);
    float p2 = 1.0f;
    if (__any_sync(kFull, huge)) {
        p2 = huge ? pow2_near(alpha) : 1.0f;
        v.mul(p2);
    }
    v.template hadamard<L>(q);
    auto ymax = v.absmax();
#pragma unroll
    for (int m = 1; m < L; m <<= 1) ymax = fmax(ymax, __shfl_xor_sync(kFull, ymax, m));
    double k;
#if TACO_FAST_SCALARS_REG
    block_scale_fast((double)ymax, alpha, p2, c, s, k);
#else
    block_scale((double)ymax, alpha, p2, c, s, k);
#endif
    v.mul(k);
}

// ------------------------------------------------------------ async-copy pipeline ---
// Persistent warps walk tiles of G consecutive blocks (one L-lane group per block).
// For full tiles every lane cp.async-es its own 16-byte chunks of tile t+1 into a
// private double-buffered smem slot (chunk c of lane l at (c*32 + l)*16: conflict-free
// LDS.128, and each lane only ever reads what it copied, so no barrier is needed)
// while it computes tile t.  Ragged tiles (shard tails, unaligned shards) take the
// guarded direct-load path.

// n / d for n < 2^31 with a host-computed magic number (Granlund-Montgomery)
struct FastDiv {
    uint32_t d, m, s;
    __device__ __forceinline__ uint32_t div(uint32_t n) const { return (__umulhi(n, m) + n) >> s; }
};

constexpr int kPipeWarps = 4;    // warps per CTA of the persistent kernels
#ifndef TACO_PIPE_MIN_CTAS
#define TACO_PIPE_MIN_CTAS 4
#endif
constexpr int kPipeMinCtas = TACO_PIPE_MIN_CTAS;  // 4: >= 16 resident warps per SM (caps registers at 128)

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// raw 16 bytes of T -> pairs
template <typename T>
__device__ __forceinline__ void unpack16(const uint4 u, float2* out) {
    if constexpr (sizeof(T) == 2) {
        out[0] = bf16x2_to_f2(u.x); out[1] = bf16x2_to_f2(u.y);
        out[2] = bf16x2_to_f2(u.z); out[3] = bf16x2_to_f2(u.w);
    } else {
        out[0] = f2(__uint_as_float(u.x), __uint_as_float(u.y));
        out[1] = f2(__uint_as_float(u.z), __uint_as_float(u.w));
    }
}

// whether the G blocks of a tile starting at block kk0 of shard p are all whole and the
// element pointers allow vector access
template <int B, int G>
__device__ __forceinline__ bool tile_full(const ShardArgs& a, uint64_t p, uint64_t kk0) {
    return a.vec_ok && kk0 + G <= (p + 1 == a.P ? a.full_last : a.full_mid);
}

template <int B, typename TIn, int FMT, int EMAX, int VMAX>
struct K1Cfg {
    using Gm = Geo<B, EMAX, VMAX>;
    static constexpr int VB = Gm::V * (int)sizeof(TIn);  // bytes per lane-vector
    static constexpr bool PIPE = VB % 16 == 0;
    static constexpr int CPV = PIPE ? VB / 16 : 1;         // 16-byte chunks per vector
    static constexpr int NCH = Gm::NV * CPV;               // chunks per lane per tile
    static constexpr int STAGE_U4 = NCH * 32;              // uint4 per warp stage
    static constexpr size_t SMEM = PIPE ? (size_t)kPipeWarps * 2 * STAGE_U4 * 16 : 0;
};

// --------------------------------------------------------------------------- K1 ---
// PUSH: peer-memory mode (ShardArgs::dst), a separate instantiation so the default
// kernel keeps its register allocation
// ctr (optional): dynamic schedule -- each warp's first tile is static (t < nwarps), later
// tiles are claimed from a per-launch counter one tile ahead of the prefetch, so warps
// that finish early take more work instead of idling through the static 4-vs-5-tile tail.
// Every warp makes exactly two failed claims; the claim that returns the last raw value
// resets the counter for the next launch that draws the same ring slot.
template <int B, typename TIn, int FMT, int EMAX, int VMAX, bool PUSH = false>
__global__ void __launch_bounds__(kPipeWarps * 32, kPipeMinCtas) k_compress(const TIn* __restrict__ x, uint8_t* __restrict__ msgs,
                                                              ShardArgs a, CodecConsts c, FastDiv tps,
                                                              uint32_t* __restrict__ ctr) {
    using Cf = K1Cfg<B, TIn, FMT, EMAX, VMAX>;
    using Gm = typename Cf::Gm;
    constexpr int E = Gm::E, V = Gm::V, L = Gm::L, G = Gm::G, NV = Gm::NV, CPV = Cf::CPV;
    constexpr int EPC = 16 / (int)sizeof(TIn);  // elements per chunk
    extern __shared__ uint4 smem_dyn[];
    const int lane = threadIdx.x & 31, q = lane & (L - 1), g = lane / L, warp = threadIdx.x >> 5;
    uint4* stage_base = smem_dyn + (size_t)warp * 2 * Cf::STAGE_U4;
    const uint32_t ntiles = a.P * tps.d;
    const uint32_t stride = gridDim.x * kPipeWarps;
#if TACO_K1_WARP_MAJOR
    // warp-major numbering: the warps that get one tile more than the others (tiles do not
    // divide evenly) are spread over all SMs instead of piling onto the first CTAs' SMs
    uint32_t t = warp * gridDim.x + blockIdx.x;
#else
    uint32_t t = blockIdx.x * kPipeWarps + warp;
#endif

    auto issue = [&](uint32_t tt, int stage) {
        if constexpr (Cf::PIPE) {
            const uint32_t p = tps.div(tt);
        const uint64_t kk0 = (uint64_t)(tt - p * tps.d) * G;
            if (tile_full<B, G>(a, p, kk0)) {
                const TIn* src = x + (p * a.S + (a.blk0 + kk0 + g) * B);
                uint4* st = stage_base + stage * Cf::STAGE_U4;
#pragma unroll
                for (int j = 0; j < NV; ++j)
#pragma unroll
                    for (int h = 0; h < CPV; ++h)
                        cp_async16(st + (j * CPV + h) * 32 + lane, src + Gm::pos(j, q) + h * EPC);
            }
        }
        cp_async_commit();  // possibly empty: keeps the group count uniform
    };

    grid_dep_wait();
    const uint32_t last_raw = (ntiles > stride ? ntiles - stride : 0u) + 2u * stride - 1u;
    auto claim = [&]() -> uint32_t {  // lane 0's raw claim (other lanes: 0)
        uint32_t r = 0;
        if (lane == 0) {
            r = atomicAdd(ctr, 1u);
            if (r == last_raw) atomicExch(ctr, 0u);
        }
        return r;
    };
    uint32_t tn = ctr ? stride + __shfl_sync(kFull, claim(), 0) : t + stride;  // the tile after t
    if (t < ntiles) issue(t, 0);
    else if (ctr) claim();  // an idle warp still makes its two failed claims
    for (int it = 0; t < ntiles; ++it) {
        const uint32_t pend = ctr ? claim() : 0u;  // the tile after tn (used next iteration)
        if (tn < ntiles) issue(tn, (it + 1) & 1);
        else cp_async_commit();
        const uint32_t p = tps.div(t);
        const uint64_t kk0 = (uint64_t)(t - p * tps.d) * G;
        const uint64_t kk = kk0 + g;
        const bool live = kk < a.nblk;
        const uint64_t k = a.blk0 + kk;
        RegsFor<FMT, E> v;
        if (Cf::PIPE && tile_full<B, G>(a, p, kk0)) {
            cp_async_wait_1();  // this lane's chunks of tile t have landed
            const uint4* st = stage_base + (it & 1) * Cf::STAGE_U4;
#pragma unroll
            for (int j = 0; j < NV; ++j) {
                float2 tmp[V / 2];
#pragma unroll
                for (int h = 0; h < CPV; ++h) unpack16<TIn>(st[(j * CPV + h) * 32 + lane], &tmp[h * EPC / 2]);
                v.template load_pairs<V>(j, tmp);
            }
        } else {
            const int valid = live ? clamp_valid((int64_t)a.S - (int64_t)(k * B),
                                                 (int64_t)a.n - (int64_t)(p * a.S + k * B), B)
                                   : 0;
            const TIn* src = x + (p * a.S + k * B);
#pragma unroll
            for (int j = 0; j < NV; ++j) {
                const int pos = Gm::pos(j, q);
                if (a.vec_ok && pos + V <= valid) v.template load<TIn, V>(j, src + pos);
                else v.template load_guarded<TIn, V>(j, src + pos, pos, valid);
            }
        }
        float alpha, s;
        double ss;
        quantise<L>(v, q, c, alpha, s, ss);
        if (live) {
            auto put = [&](uint8_t* m) {
#pragma unroll
                for (int j = 0; j < NV; ++j) v.template store_codes_at<FMT, V>(j, m + kk * B + Gm::pos(j, q));
                if (q == 0) *reinterpret_cast<float2*>(m + a.scal_off + kk * 8) = make_float2(alpha, s);
            };
            if constexpr (PUSH) {
                if (a.bcast)
                    for (uint32_t d = 0; d < a.ndst; ++d) put(a.dst[d]);
                else
                    put(a.dst[p]);
            } else {
                put(msgs + p * a.msg_stride);
            }
            if (q == 0 && !isfinite(ss)) raise_flag(a.flags, 1);  // any NaN/Inf element poisons the block sum
        }
        t = tn;
        tn = ctr ? stride + __shfl_sync(kFull, pend, 0) : tn + stride;
    }
}

template <int B, typename TOut, int FMT, int EMAX, int VMAX>
struct K2Cfg {
    using Gm = Geo<B, EMAX, VMAX>;
    static constexpr bool PIPE = Gm::V % 16 == 0;       // 16 codes per chunk
    static constexpr int NCH = PIPE ? Gm::NV * (Gm::V / 16) : 1;
    static constexpr int STAGE_U4 = NCH * 32;
    static constexpr size_t SMEM = PIPE ? (size_t)kPipeWarps * 2 * STAGE_U4 * 16 : 0;
};

// --------------------------------------------------------------------------- K2 ---
template <int B, typename TOut, int FMT, int EMAX, int VMAX>
__global__ void __launch_bounds__(kPipeWarps * 32, kPipeMinCtas) k_decompress(const uint8_t* __restrict__ msgs,
                                                                TOut* __restrict__ out, ShardArgs a, CodecConsts c,
                                                                FastDiv tps) {
    using Cf = K2Cfg<B, TOut, FMT, EMAX, VMAX>;
    using Gm = typename Cf::Gm;
    constexpr int E = Gm::E, V = Gm::V, L = Gm::L, G = Gm::G, NV = Gm::NV;
    constexpr int CPV = Cf::PIPE ? V / 16 : 1;
    extern __shared__ uint4 smem_dyn[];
    const int lane = threadIdx.x & 31, q = lane & (L - 1), g = lane / L, warp = threadIdx.x >> 5;
    uint4* stage_base = smem_dyn + (size_t)warp * 2 * Cf::STAGE_U4;
    const uint32_t ntiles = a.P * tps.d;
    const uint32_t stride = gridDim.x * kPipeWarps;
    uint32_t t = blockIdx.x * kPipeWarps + warp;
    float2 sc_next = make_float2(1.0f, 1.0f);

    auto issue = [&](uint32_t tt, int stage) {
        const uint32_t p = tps.div(tt);
        const uint64_t kk0 = (uint64_t)(tt - p * tps.d) * G;
        const uint8_t* m = msgs + p * a.msg_stride;
        if (kk0 + g < a.nblk) sc_next = __ldg(reinterpret_cast<const float2*>(m + a.scal_off + (kk0 + g) * 8));
        if constexpr (Cf::PIPE) {
            if (kk0 + G <= a.nblk) {  // codes of a message are always aligned
                const uint8_t* src = m + (kk0 + g) * B;
                uint4* st = stage_base + stage * Cf::STAGE_U4;
#pragma unroll
                for (int j = 0; j < NV; ++j)
#pragma unroll
                    for (int h = 0; h < CPV; ++h) cp_async16(st + (j * CPV + h) * 32 + lane, src + Gm::pos(j, q) + h * 16);
            }
        }
        cp_async_commit();
    };

    grid_dep_wait();
    if (t < ntiles) issue(t, 0);
    for (int it = 0; t < ntiles; t += stride, ++it) {
        const float2 sc = sc_next;
        if (t + stride < ntiles) issue(t + stride, (it + 1) & 1);
        else cp_async_commit();
        const uint32_t p = tps.div(t);
        const uint64_t kk0 = (uint64_t)(t - p * tps.d) * G;
        const uint64_t kk = kk0 + g;
        const bool live = kk < a.nblk;
        const uint64_t k = a.blk0 + kk;
        const uint8_t* m = msgs + p * a.msg_stride;
        RegsFor<FMT, E> v;
        if (Cf::PIPE && kk0 + G <= a.nblk) {
            cp_async_wait_1();
            const uint4* st = stage_base + (it & 1) * Cf::STAGE_U4;
#pragma unroll
            for (int j = 0; j < NV; ++j) {
                float2 tmp[V / 2];
#pragma unroll
                for (int h = 0; h < CPV; ++h) {
                    const uint4 u = st[(j * CPV + h) * 32 + lane];
                    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        tmp[h * 8 + 2 * i] = dec2<FMT>(w[i]);
                        tmp[h * 8 + 2 * i + 1] = dec2<FMT>(w[i] >> 16);
                    }
                }
                v.template load_pairs<V>(j, tmp);
            }
        } else if (live) {
#pragma unroll
            for (int j = 0; j < NV; ++j) v.template load_codes_at<FMT, V>(j, m + kk * B + Gm::pos(j, q));
        } else {
            v.zero();
        }
        v.template hadamard<L>(q);  // every lane takes part: the shuffles stay converged
        v.mul(block_dequant(live ? sc.x : 1.0f, live ? sc.y : 1.0f, c));
        if (!live) continue;
        if (q == 0 && !scalars_ok(sc.x, sc.y)) raise_flag(a.flags, 2);
        const int valid = clamp_valid((int64_t)a.S - (int64_t)(k * B), (int64_t)a.n - (int64_t)(p * a.S + k * B), B);
        TOut* dst = out + (p * a.S + k * B);
        if (a.vec_ok && valid == B) {
#pragma unroll
            for (int j = 0; j < NV; ++j) v.template store<TOut, V>(j, dst + Gm::pos(j, q));
        } else {
#pragma unroll
            for (int j = 0; j < NV; ++j) {
                const int pos = Gm::pos(j, q);
                if (a.vec_ok && pos + V <= valid) v.template store<TOut, V>(j, dst + pos);
                else v.template store_guarded<TOut, V>(j, dst + pos, pos, valid);
            }
        }
    }
}

// --------------------------------------------------------------------------- K3 ---
// msgs: nranks messages (rank r at msgs + r*msg_stride) of one shard chunk.
template <int B, typename TAcc, int FMT, int EMAX, int VMAX>
__global__ void __launch_bounds__(kWarpThreads) k_reduce_encode(const uint8_t* __restrict__ msgs,
                                                                uint8_t* __restrict__ out_msg,
                                                                TAcc* __restrict__ acc_out, ShardArgs a,
                                                                CodecConsts c) {
    using Gm = Geo<B, EMAX, VMAX>;
    constexpr int E = Gm::E, V = Gm::V, L = Gm::L, G = Gm::G, NV = Gm::NV;
    const int lane = threadIdx.x & 31, q = lane & (L - 1), g = lane / L;
    const uint64_t kk = ((uint64_t)blockIdx.x * (kWarpThreads / 32) + (threadIdx.x >> 5)) * G + g;
    const bool live = kk < a.nblk;
    const uint64_t k = a.blk0 + kk;
    const int valid = live ? clamp_valid((int64_t)a.S - (int64_t)(k * B), (int64_t)B, B) : 0;
    grid_dep_wait();

    RegsFor<FMT, E> acc;
    bool bad = false;
    for (uint32_t r = 0; r < a.P; ++r) {
        const uint8_t* m = a.nsrc ? a.src[r] : msgs + r * a.msg_stride;
        RegsFor<FMT, E> d;
        float2 sc = make_float2(1.0f, 1.0f);
        if (live) {
            sc = __ldg(reinterpret_cast<const float2*>(m + a.scal_off + kk * 8));
#pragma unroll
            for (int j = 0; j < NV; ++j) d.template load_codes_at<FMT, V>(j, m + kk * B + Gm::pos(j, q));
        } else {
            d.zero();
        }
        bad |= !scalars_ok(sc.x, sc.y);
        d.template hadamard<L>(q);
        d.mul(block_dequant(sc.x, sc.y, c));
        d.round_to_f32();  // the decoded slice is an fp32 tensor in the reference
        if (r == 0) acc = d;  // acc = dec(rank 0): keeps -0.0 like the reference
        else acc.add(d);      // fp32, ascending rank (collective.cpp:95-100)
    }
    // positions past the shard end are padding of the re-encoded slice (collective.cpp:101)
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const int pos = Gm::pos(j, q);
        if (pos + V > valid) acc.zero_from(j, V, pos, valid);
    }
    if (live && acc_out) {
        TAcc* dst = acc_out + k * B;
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            const int pos = Gm::pos(j, q);
            if (a.vec_ok && pos + V <= valid) acc.template store<TAcc, V>(j, dst + pos);
            else acc.template store_guarded<TAcc, V>(j, dst + pos, pos, valid);
        }
    }
    if (out_msg == nullptr) {  // reduce-scatter: the fp32 sum is the product, no re-encode
        if (live && q == 0 && bad) raise_flag(a.flags, 2);
        return;
    }
    float alpha, s;
    double ss;
    quantise<L>(acc, q, c, alpha, s, ss);
    if (!live) return;
    const uint32_t nd = a.ndst ? a.ndst : 1;
    for (uint32_t d = 0; d < nd; ++d) {  // peer mode: the same message into every rank's buffer
        uint8_t* o = a.ndst ? a.dst[d] : out_msg;
#pragma unroll
        for (int j = 0; j < NV; ++j) acc.template store_codes_at<FMT, V>(j, o + kk * B + Gm::pos(j, q));
        if (q == 0) *reinterpret_cast<float2*>(o + a.scal_off + kk * 8) = make_float2(alpha, s);
    }
    if (q == 0 && bad) raise_flag(a.flags, 2);
}

// ===================================================== big blocks (B >= 2048) ===
// One CTA of kBigThreads per block.  Thread t owns positions t + i*T (i < PER) in
// registers; the butterflies run through shared memory of type W (fp32 for E4M3,
// fp64 for E5M2 up to B = 16384 -- 128 KB).

template <int FMT, int B>
using BigW = typename std::conditional<FMT == 1 && B <= 16384, double, float>::type;

template <int B, typename W>
__device__ __forceinline__ void smem_fwht(W* sm) {
    constexpr int T = kBigThreads;
#pragma unroll 1
    for (int h = 1; h < B; h <<= 1) {
        __syncthreads();
        for (int t = threadIdx.x; t < B / 2; t += T) {
            const int i = (t / h) * 2 * h + (t % h);
            const W a = sm[i], b = sm[i + h];
            sm[i] = a + b;
            sm[i + h] = a - b;
        }
    }
    __syncthreads();
}

__device__ __forceinline__ double cta_sum(double v, double* red) {
#pragma unroll
    for (int m = 1; m < 32; m <<= 1) v += __shfl_xor_sync(kFull, v, m);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < kBigThreads / 32; ++w) t += red[w];  // same order in every thread
    return t;
}

__device__ __forceinline__ double cta_max(double v, double* red) {
#pragma unroll
    for (int m = 1; m < 32; m <<= 1) v = fmax(v, __shfl_xor_sync(kFull, v, m));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < kBigThreads / 32; ++w) t = fmax(t, red[w]);
    return t;
}

// Quantise the register block r[PER] (positions t + i*T); writes codes + scalars.
template <int B, int FMT, typename W>
__device__ __forceinline__ void big_quantise_store(float (&r)[B / kBigThreads], W* sm, double* red,
                                                   const CodecConsts& c, uint8_t* codes, float2* scal,
                                                   int* flags) {
    constexpr int T = kBigThreads, PER = B / T;
    double ss = 0.0;
#pragma unroll
    for (int i = 0; i < PER; ++i) ss = fma((double)r[i], (double)r[i], ss);
    ss = cta_sum(ss, red);
    const float alpha = block_alpha(ss, c);
    const float p2 = pow2_near(alpha);
#pragma unroll
    for (int i = 0; i < PER; ++i) sm[threadIdx.x + i * T] = (W)(r[i] * p2);
    smem_fwht<B, W>(sm);
    double ym = 0.0;
#pragma unroll
    for (int i = 0; i < PER; ++i) ym = fmax(ym, fabs((double)sm[threadIdx.x + i * T]));
    ym = cta_max(ym, red);
    float s;
    double k;
    block_scale(ym, alpha, p2, c, s, k);
    // k in double: s may be subnormal, which puts k outside the fp32 range
    for (int t = threadIdx.x; t < B / 2; t += T)
        reinterpret_cast<uint16_t*>(codes)[t] =
            (uint16_t)enc2<FMT>(make_float2((float)((double)sm[2 * t] * k), (float)((double)sm[2 * t + 1] * k)));
    if (threadIdx.x == 0) {
        *scal = make_float2(alpha, s);
        if (!isfinite(ss)) raise_flag(flags, 1);
    }
}

// decode one block into sm (H(table[c]) * m); returns validity of its scalars
template <int B, int FMT, typename W>
__device__ __forceinline__ bool big_dequantise(const uint8_t* codes, float2 sc, W* sm, const CodecConsts& c) {
    __syncthreads();
    for (int t = threadIdx.x; t < B / 2; t += kBigThreads) {
        const float2 d = dec2<FMT>(reinterpret_cast<const uint16_t*>(codes)[t]);
        sm[2 * t] = d.x;
        sm[2 * t + 1] = d.y;
    }
    smem_fwht<B, W>(sm);
    const double m = block_dequant(sc.x, sc.y, c);
    for (int t = threadIdx.x; t < B; t += kBigThreads) sm[t] = (W)(float)((double)sm[t] * m);
    __syncthreads();
    return scalars_ok(sc.x, sc.y);
}

template <int B, typename TIn, int FMT>
__global__ void __launch_bounds__(kBigThreads) k_compress_big(const TIn* __restrict__ x, uint8_t* __restrict__ msgs,
                                                              ShardArgs a, CodecConsts c) {
    using W = BigW<FMT, B>;
    extern __shared__ __align__(16) unsigned char smraw[];
    W* sm = reinterpret_cast<W*>(smraw);
    __shared__ double red[kBigThreads / 32];
    constexpr int T = kBigThreads, PER = B / T;
    const uint64_t p = blockIdx.y, kk = blockIdx.x, k = a.blk0 + kk;
    const int valid = clamp_valid((int64_t)a.S - (int64_t)(k * B), (int64_t)a.n - (int64_t)(p * a.S + k * B), B);
    const TIn* src = x + (p * a.S + k * B);
    float r[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int pos = threadIdx.x + i * T;
        r[i] = pos < valid ? to_f32(src[pos]) : 0.0f;
    }
    uint8_t* m = msgs + p * a.msg_stride;
    big_quantise_store<B, FMT, W>(r, sm, red, c, m + kk * B, reinterpret_cast<float2*>(m + a.scal_off + kk * 8),
                                  a.flags);
}

template <int B, typename TOut, int FMT>
__global__ void __launch_bounds__(kBigThreads) k_decompress_big(const uint8_t* __restrict__ msgs,
                                                                TOut* __restrict__ out, ShardArgs a, CodecConsts c) {
    using W = BigW<FMT, B>;
    extern __shared__ __align__(16) unsigned char smraw[];
    W* sm = reinterpret_cast<W*>(smraw);
    const uint64_t p = blockIdx.y, kk = blockIdx.x, k = a.blk0 + kk;
    const int valid = clamp_valid((int64_t)a.S - (int64_t)(k * B), (int64_t)a.n - (int64_t)(p * a.S + k * B), B);
    const uint8_t* m = msgs + p * a.msg_stride;
    const float2 sc = *reinterpret_cast<const float2*>(m + a.scal_off + kk * 8);
    const bool ok = big_dequantise<B, FMT, W>(m + kk * B, sc, sm, c);
    if (threadIdx.x == 0 && !ok) raise_flag(a.flags, 2);
    TOut* dst = out + (p * a.S + k * B);
    for (int t = threadIdx.x; t < valid; t += kBigThreads) store_one(dst + t, (float)sm[t]);
}

template <int B, typename TAcc, int FMT>
__global__ void __launch_bounds__(kBigThreads) k_reduce_encode_big(const uint8_t* __restrict__ msgs,
                                                                   uint8_t* __restrict__ out_msg,
                                                                   TAcc* __restrict__ acc_out, ShardArgs a,
                                                                   CodecConsts c) {
    using W = BigW<FMT, B>;
    extern __shared__ __align__(16) unsigned char smraw[];
    W* sm = reinterpret_cast<W*>(smraw);
    __shared__ double red[kBigThreads / 32];
    constexpr int T = kBigThreads, PER = B / T;
    const uint64_t kk = blockIdx.x, k = a.blk0 + kk;
    const int valid = clamp_valid((int64_t)a.S - (int64_t)(k * B), (int64_t)B, B);
    float acc[PER];
    bool ok = true;
    for (uint32_t r = 0; r < a.P; ++r) {
        const uint8_t* m = msgs + r * a.msg_stride;
        const float2 sc = *reinterpret_cast<const float2*>(m + a.scal_off + kk * 8);
        ok &= big_dequantise<B, FMT, W>(m + kk * B, sc, sm, c);
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const float d = (float)sm[threadIdx.x + i * T];
            acc[i] = r == 0 ? d : acc[i] + d;
        }
    }
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int pos = threadIdx.x + i * T;
        if (pos >= valid) acc[i] = 0.0f;
        else if (acc_out) store_one(acc_out + k * B + pos, acc[i]);
    }
    if (out_msg == nullptr) {
        if (threadIdx.x == 0 && !ok) raise_flag(a.flags, 2);
        return;
    }
    __syncthreads();
    big_quantise_store<B, FMT, W>(acc, sm, red, c, out_msg + kk * B,
                                  reinterpret_cast<float2*>(out_msg + a.scal_off + kk * 8), nullptr);
    if (threadIdx.x == 0 && !ok) raise_flag(a.flags, 2);
}

}  // namespace taco_dev
