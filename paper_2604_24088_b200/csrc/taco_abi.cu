// taco_abi.cu -- the extern "C" boundary (include/taco_b200.h): validation with the
// reference's exact messages, shard/message geometry, kernel launches, the one-device
// RankSet simulation and the pipelined host API.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "taco_b200.h"
#include "taco_kernels.cuh"
#include "taco_launch.h"

using taco_dev::CodecConsts;
using taco_dev::ShardArgs;
using taco_impl::Launch;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail(TACO_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define TACO_CUDA(call)                                        \
    do {                                                       \
        cudaError_t e_ = (call);                               \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call);    \
    } while (0)

// Switches the calling thread to `device` for the scope and restores the caller's device
// on exit: host entry points must not leave the caller's current device changed.
struct DeviceGuard {
    int prev = -1;
    cudaError_t err = cudaSuccess;
    explicit DeviceGuard(int device) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != device) err = cudaSetDevice(device);
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

bool pow2(uint64_t b) { return b != 0 && (b & (b - 1)) == 0; }

uint64_t align16(uint64_t v) { return (v + 15) & ~uint64_t(15); }

uint64_t div_up(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

size_t dtype_size(int dt) { return dt == TACO_DT_BF16 ? 2 : 4; }

// transform.cpp:13-20, codec.cpp:189-197 -- same order, same messages
int check_config(const taco_config* cfg) {
    if (!cfg) return fail(TACO_ERR_USAGE, "null codec config");
    const uint64_t b = cfg->block_size;
    if (!pow2(b)) return fail(TACO_ERR_CONFIG, "block size must be a power of two");
    if (b < 2 || b > 32768) return fail(TACO_ERR_CONFIG, "block size must be between 2 and 32768");
    if (!(cfg->target_energy > 0.0f) || !std::isfinite(cfg->target_energy))
        return fail(TACO_ERR_CONFIG, "target energy must be positive and finite");
    if (!(cfg->stability_epsilon > 0.0f) || !std::isfinite(cfg->stability_epsilon))
        return fail(TACO_ERR_CONFIG, "stability epsilon must be positive and finite");
    if (cfg->format > 1) return fail(TACO_ERR_CONFIG, "unknown fp8 format");
    if (cfg->kind > 4) return fail(TACO_ERR_CONFIG, "unknown codec kind");
    if (cfg->direct_scale > 2) return fail(TACO_ERR_CONFIG, "unknown direct-scale scope");
    return TACO_OK;
}

// payload bytes per block: B codes, or 4B raw bytes for Identity (codec.hpp:39)
uint64_t payload_of(const taco_config* cfg) {
    return cfg->kind == 3 ? 4ull * cfg->block_size : (uint64_t)cfg->block_size;
}

int check_dtype(int dt) {
    if (dt != TACO_DT_F32 && dt != TACO_DT_BF16) return fail(TACO_ERR_USAGE, "unknown element dtype");
    return TACO_OK;
}

CodecConsts consts_of(const taco_config* cfg) {
    CodecConsts c;
    c.tau = cfg->target_energy;
    c.eps = cfg->stability_epsilon;
    c.inv_b = 1.0 / (double)cfg->block_size;
    c.norm = 1.0 / std::sqrt((double)cfg->block_size);  // transform.cpp:56
    c.qmax = cfg->format ? 57344.0 : 448.0;             // fp8.cpp:11-12
    c.inv_qmax = 1.0 / c.qmax;
    return c;
}

taco_layout layout_of(uint64_t pb, uint64_t nblocks) {  // pb = payload bytes per block
    taco_layout l;
    l.nblocks = nblocks;
    l.codes_bytes = nblocks * pb;
    l.scal_offset = align16(l.codes_bytes);
    l.msg_bytes = l.scal_offset + 8 * nblocks;
    l.msg_stride = align16(l.msg_bytes);
    return l;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
// ShardArgs::vec_ok: 2 = 32-byte aligned (256-bit vector access), 1 = 16-byte aligned, 0 = scalar
int vec_align(const void* p) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    return (a & 31u) == 0 ? 2 : (a & 15u) == 0 ? 1 : 0;
}

// Messages are read and written with 16-byte vector / TMA accesses: every message base must
// be 16-byte aligned, i.e. the buffer and (with more than one message) the stride.
int check_msg_buffer(const void* p, uint64_t stride, uint64_t count, const char* what) {
    if (!aligned16(p) || (count > 1 && stride % 16 != 0))
        return fail(TACO_ERR_USAGE, std::string(what) + " must be 16-byte aligned (buffer and stride)");
    return TACO_OK;
}

int check_range(uint64_t m, uint64_t blk_begin, uint64_t blk_end) {
    if (blk_begin > blk_end || blk_end > m)
        return fail(TACO_ERR_USAGE, "block range exceeds the shard's block count");
    return TACO_OK;
}

}  // namespace

namespace taco_impl {
int set_error(int code, const char* msg) { return fail(code, msg); }
}  // namespace taco_impl

namespace taco_impl {
bool k1_dynamic() {
    static const bool on = [] {
        const char* v = std::getenv("TACO_K1_DYNAMIC");
        return v && std::strcmp(v, "1") == 0;
    }();
    return on;
}
bool pdl_enabled() {
    static const bool on = [] {
        const char* v = std::getenv("TACO_PDL");
        return !(v && std::strcmp(v, "0") == 0);
    }();
    return on;
}
}  // namespace taco_impl

namespace taco_impl {
int kernel_family() {
    static const int fam = [] {
        const char* v = std::getenv("TACO_B200_KERNELS");
        if (v && std::strcmp(v, "reg") == 0) return 2;
        if (v && std::strcmp(v, "tile") == 0) return 1;
        if (v && std::strcmp(v, "tc") == 0) return 5;
        if (v && std::strcmp(v, "r1") == 0) return 6;
        return 0;
    }();
    return fam;
}

uint32_t* claim_counter() {
    constexpr int kRing = 1024;
    static std::mutex mu;
    static std::map<int, uint32_t*> rings;
    static std::map<int, uint32_t> next;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    uint32_t*& ring = rings[dev];
    if (!ring) {
        if (cudaMalloc(&ring, kRing * sizeof(uint32_t)) != cudaSuccess) return ring = nullptr;
        if (cudaMemset(ring, 0, kRing * sizeof(uint32_t)) != cudaSuccess) return nullptr;
    }
    return ring + (next[dev]++ % kRing);
}

uint32_t* claim_scratch(uint32_t words) {
    constexpr uint32_t kWords = 1u << 16;
    static std::mutex mu;
    static std::map<int, uint32_t*> rings;
    static std::map<int, uint32_t> next;
    if (words == 0 || words > kWords) return nullptr;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    uint32_t*& ring = rings[dev];
    if (!ring && cudaMalloc(&ring, kWords * sizeof(uint32_t)) != cudaSuccess) return ring = nullptr;
    uint32_t& at = next[dev];
    if (at + words > kWords) at = 0;
    uint32_t* p = ring + at;
    at += words;
    return p;
}

int resident_ctas(const void* kernel, int threads, size_t smem) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find({kernel, dev});
    if (it != cache.end()) return it->second;
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (smem > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
    const int ctas = sms * (per_sm > 0 ? per_sm : 1);
    cache[{kernel, dev}] = ctas;
    return ctas;
}
}  // namespace taco_impl

// =================================================================== metadata ====
extern "C" {

int taco_abi_version(void) { return TACO_B200_ABI_VERSION; }

int taco_set_error(int code, const char* msg) { return fail(code, msg); }

const char* taco_last_error(void) { return g_err.c_str(); }

taco_config taco_default_config(void) {
    taco_config c;
    c.block_size = 256;
    c.target_energy = 1.0f;
    c.stability_epsilon = 1e-12f;
    c.format = 0;
    c.kind = 0;
    c.direct_scale = 0;
    return c;
}

int taco_validate_config(const taco_config* cfg) { return check_config(cfg); }

int taco_msg_layout(const taco_config* cfg, uint64_t nblocks, taco_layout* out) {
    if (int rc = check_config(cfg)) return rc;
    *out = layout_of(payload_of(cfg), nblocks);
    return TACO_OK;
}

double taco_compressed_ratio(const taco_config* cfg, uint64_t n) {
    if (n == 0 || !cfg) return 0.0;
    if (cfg->kind == 3) return 1.0;  // Identity (codec.cpp:300)
    const double blocks = (double)div_up(n, cfg->block_size);
    return 4.0 * (double)n / (blocks * ((double)cfg->block_size + 8.0));  // codec.cpp:298-304
}

uint64_t taco_archive_size(const taco_config* cfg, uint64_t n) {
    return 22 + div_up(n, cfg->block_size) * (payload_of(cfg) + 8);  // serialize.cpp:172-177
}

int taco_flags_status(int flags) {
    // a timed-out peer phase comes first: the kernels after it ran on slots that never landed
    if (flags & TACO_FLAG_PEER_TIMEOUT) return fail(TACO_ERR_CUDA, "peer barrier timed out");
    if (flags & TACO_FLAG_NONFINITE_INPUT) return fail(TACO_ERR_INPUT, "input tensor contains NaN or Inf");
    if (flags & TACO_FLAG_BAD_SCALARS) return fail(TACO_ERR_CORRUPT, "block scalars must be finite and nonzero");
    return TACO_OK;
}

// ================================================================= device API ====

int taco_compress_dev(const taco_config* cfg, const void* x, int dtype, uint64_t n, uint32_t shards,
                      uint64_t blk_begin, uint64_t blk_end, void* msgs, uint64_t msg_stride, int* d_flags,
                      void* stream) {
    if (int rc = check_config(cfg)) return rc;
    if (int rc = check_dtype(dtype)) return rc;
    if (n == 0) return fail(TACO_ERR_INPUT, "input tensor is empty");
    if (shards == 0) return fail(TACO_ERR_USAGE, "shard count must be positive");
    const uint64_t b = cfg->block_size, S = div_up(n, shards), m = div_up(S, b);
    if (int rc = check_range(m, blk_begin, blk_end)) return rc;
    const taco_layout lay = layout_of(payload_of(cfg), blk_end - blk_begin);
    if (shards > 1 && msg_stride < lay.msg_bytes) return fail(TACO_ERR_USAGE, "message stride too small");
    if (int rc = check_msg_buffer(msgs, msg_stride, shards, "messages")) return rc;
    ShardArgs a{n, S, shards, blk_begin, blk_end - blk_begin, msg_stride, lay.scal_offset,
                ((shards == 1 || S % 8 == 0) ? vec_align(x) : 0), d_flags};
    taco_dev::with_full_blocks(a, b);
    Launch l{cfg->block_size, dtype, (int)cfg->format, x, msgs, nullptr, (cudaStream_t)stream};
    if (cfg->kind != 0) {
        uint32_t* smax = taco_impl::claim_scratch(shards);
        if (!smax) return fail(TACO_ERR_CUDA, "scratch allocation failed");
        if (cudaError_t e = taco_impl::launch_compress_kind(l, a, consts_of(cfg), (int)cfg->kind,
                                                            (int)cfg->direct_scale, smax))
            return cuda_fail(e, "compress launch");
        return TACO_OK;
    }
    if (cudaError_t e = taco_impl::launch_compress(l, a, consts_of(cfg))) return cuda_fail(e, "K1 compress launch");
    return TACO_OK;
}

int taco_decompress_dev(const taco_config* cfg, const void* msgs, uint64_t msg_stride, uint32_t shards, uint64_t n,
                        uint64_t blk_begin, uint64_t blk_end, void* out, int out_dtype, int* d_flags, void* stream) {
    if (int rc = check_config(cfg)) return rc;
    if (int rc = check_dtype(out_dtype)) return rc;
    if (n == 0) return fail(TACO_ERR_CORRUPT, "compressed tensor declares zero elements");
    if (shards == 0) return fail(TACO_ERR_USAGE, "shard count must be positive");
    const uint64_t b = cfg->block_size, S = div_up(n, shards), m = div_up(S, b);
    if (int rc = check_range(m, blk_begin, blk_end)) return rc;
    const taco_layout lay = layout_of(payload_of(cfg), blk_end - blk_begin);
    if (shards > 1 && msg_stride < lay.msg_bytes) return fail(TACO_ERR_USAGE, "message stride too small");
    if (int rc = check_msg_buffer(msgs, msg_stride, shards, "messages")) return rc;
    ShardArgs a{n, S, shards, blk_begin, blk_end - blk_begin, msg_stride, lay.scal_offset,
                ((shards == 1 || S % 8 == 0) ? vec_align(out) : 0), d_flags};
    taco_dev::with_full_blocks(a, b);
    Launch l{cfg->block_size, out_dtype, (int)cfg->format, msgs, out, nullptr, (cudaStream_t)stream};
    if (cfg->kind != 0) {
        if (cudaError_t e = taco_impl::launch_decompress_kind(l, a, consts_of(cfg), (int)cfg->kind))
            return cuda_fail(e, "decompress launch");
        return TACO_OK;
    }
    if (cudaError_t e = taco_impl::launch_decompress(l, a, consts_of(cfg)))
        return cuda_fail(e, "K2 decompress launch");
    return TACO_OK;
}

int taco_reduce_encode_dev(const taco_config* cfg, const void* msgs, uint64_t rank_stride, uint32_t nranks,
                           uint64_t shard_len, uint64_t blk_begin, uint64_t blk_end, void* out_msg, void* acc_out,
                           int acc_dtype, int* d_flags, void* stream) {
    if (int rc = check_config(cfg)) return rc;
    if (acc_out)
        if (int rc = check_dtype(acc_dtype)) return rc;
    if (nranks == 0) return fail(TACO_ERR_USAGE, "reduction needs at least one rank");
    if (!out_msg && !acc_out) return fail(TACO_ERR_USAGE, "reduce-encode needs out_msg or acc_out");
    if (shard_len == 0) return fail(TACO_ERR_INPUT, "input tensor is empty");
    if (cfg->kind != 0)
        return fail(TACO_ERR_USAGE, "the fused reduce-encode serves CodecKind::Taco (use decompress + compress)");
    const uint64_t b = cfg->block_size, m = div_up(shard_len, b);
    if (int rc = check_range(m, blk_begin, blk_end)) return rc;
    const taco_layout lay = layout_of(b, blk_end - blk_begin);
    if (nranks > 1 && rank_stride < lay.msg_bytes) return fail(TACO_ERR_USAGE, "message stride too small");
    if (int rc = check_msg_buffer(msgs, rank_stride, nranks, "messages")) return rc;
    if (out_msg)
        if (int rc = check_msg_buffer(out_msg, 0, 1, "out_msg")) return rc;
    ShardArgs a{shard_len, shard_len, nranks, blk_begin, blk_end - blk_begin, rank_stride, lay.scal_offset,
                acc_out ? vec_align(acc_out) : 0, d_flags};
    taco_dev::with_full_blocks(a, b);
    a.full_last = a.full_mid;  // every rank's message covers the same (single) shard
    Launch l{cfg->block_size, acc_dtype, (int)cfg->format, msgs, out_msg, acc_out, (cudaStream_t)stream};
    if (cudaError_t e = taco_impl::launch_reduce_encode(l, a, consts_of(cfg)))
        return cuda_fail(e, "K3 reduce-encode launch");
    return TACO_OK;
}

// ------------------------------------------------------------ peer-memory two-shot ---

int taco_peer_alloc(int device, uint64_t bytes, void** ptr, taco_ipc_handle* handle) {
    static_assert(sizeof(cudaIpcMemHandle_t) == sizeof(taco_ipc_handle), "IPC handle size");
    if (!ptr || !handle || bytes == 0) return fail(TACO_ERR_USAGE, "peer allocation needs a size and outputs");
    DeviceGuard dg(device);
    TACO_CUDA(dg.err);
    void* p = nullptr;
    TACO_CUDA(cudaMalloc(&p, bytes));
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaMemset(p, 0, bytes);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p);
    if (e != cudaSuccess) {
        cudaFree(p);
        return cuda_fail(e, "peer allocation");
    }
    std::memcpy(handle->bytes, &h, sizeof(h));
    *ptr = p;
    return TACO_OK;
}

int taco_peer_open(int device, const taco_ipc_handle* handle, void** ptr) {
    if (!ptr || !handle) return fail(TACO_ERR_USAGE, "peer open needs a handle");
    DeviceGuard dg(device);
    TACO_CUDA(dg.err);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle->bytes, sizeof(h));
    TACO_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return TACO_OK;
}

int taco_peer_check_access(int device, int peer_device) {
    if (device == peer_device) return TACO_OK;  // processes sharing one GPU: IPC within the device
    int can = 0;
    TACO_CUDA(cudaDeviceCanAccessPeer(&can, device, peer_device));
    if (!can)
        return fail(TACO_ERR_USAGE, "no peer-to-peer path from GPU " + std::to_string(device) + " to GPU " +
                                        std::to_string(peer_device) + " (NVLink / PCIe P2P unavailable)");
    return TACO_OK;
}

int taco_peer_close(void* ptr) {
    TACO_CUDA(cudaIpcCloseMemHandle(ptr));
    return TACO_OK;
}

int taco_peer_free(void* ptr) {
    TACO_CUDA(cudaFree(ptr));
    return TACO_OK;
}

// barrier mode: words [0, 8) arrival slots, word 8 the epoch; fused mode (taco_peer_*_dev
// below): the same epoch, phase-A slots words [16, 24), phase-B slots [24, 32), per-kernel
// CTA tickets words 32..34
uint64_t taco_peer_flags_bytes(void) { return 160; }

namespace {
int check_peers(const taco_peers* peers) {
    if (!peers) return fail(TACO_ERR_USAGE, "null peer set");
    if (peers->nranks == 0 || peers->nranks > TACO_MAX_PEERS)
        return fail(TACO_ERR_USAGE, "peer collectives support 1 to 8 ranks");
    if (peers->rank >= peers->nranks) return fail(TACO_ERR_USAGE, "rank outside the peer set");
    for (uint32_t q = 0; q < peers->nranks; ++q)
        if (!peers->base[q]) return fail(TACO_ERR_USAGE, "peer region not mapped");
    return TACO_OK;
}

int check_push_cfg(const taco_config* cfg) {
    if (int rc = check_config(cfg)) return rc;
    if (cfg->kind != 0) return fail(TACO_ERR_USAGE, "peer collectives serve CodecKind::Taco");
    if (cfg->block_size > 1024) return fail(TACO_ERR_USAGE, "peer collectives support block sizes up to 1024");
    return TACO_OK;
}
}  // namespace

int taco_peer_barrier_dev(const taco_peers* peers, uint64_t flags_offset, uint32_t timeout_ms, int* d_flags,
                          void* stream) {
    if (int rc = check_peers(peers)) return rc;
    if (flags_offset % 16) return fail(TACO_ERR_USAGE, "peer flag offset must be 16-byte aligned");
    taco_impl::PeerSlots f{};
    for (uint32_t q = 0; q < peers->nranks; ++q)
        f.slot[q] = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(peers->base[q]) + flags_offset);
    f.epoch = f.slot[peers->rank] + TACO_MAX_PEERS;
    if (cudaError_t e = taco_impl::launch_peer_barrier(f, peers->rank, peers->nranks,
                                                       (uint64_t)timeout_ms * 1000000ull, d_flags,
                                                       (cudaStream_t)stream))
        return cuda_fail(e, "peer barrier launch");
    return TACO_OK;
}

int taco_compress_push_dev(const taco_config* cfg, const void* x, int dtype, uint64_t n, const taco_peers* peers,
                           uint64_t blk_begin, uint64_t blk_end, uint64_t dst_offset, uint64_t slot_stride,
                           int* d_flags, void* stream) {
    if (int rc = check_push_cfg(cfg)) return rc;
    if (int rc = check_peers(peers)) return rc;
    if (int rc = check_dtype(dtype)) return rc;
    if (n == 0) return fail(TACO_ERR_INPUT, "input tensor is empty");
    const uint32_t P = peers->nranks;
    const uint64_t b = cfg->block_size, S = div_up(n, P), m = div_up(S, b);
    if (int rc = check_range(m, blk_begin, blk_end)) return rc;
    const taco_layout lay = layout_of(b, blk_end - blk_begin);
    if (P > 1 && slot_stride < lay.msg_bytes) return fail(TACO_ERR_USAGE, "message stride too small");
    if ((dst_offset | slot_stride) % 16) return fail(TACO_ERR_USAGE, "peer slots must be 16-byte aligned");
    ShardArgs a{n, S, P, blk_begin, blk_end - blk_begin, lay.msg_stride, lay.scal_offset,
                ((P == 1 || S % 8 == 0) ? vec_align(x) : 0), d_flags};
    taco_dev::with_full_blocks(a, b);
    for (uint32_t q = 0; q < P; ++q)
        a.dst[q] = static_cast<uint8_t*>(peers->base[q]) + dst_offset + (uint64_t)peers->rank * slot_stride;
    a.ndst = P;
    Launch l{cfg->block_size, dtype, (int)cfg->format, x, a.dst[0], nullptr, (cudaStream_t)stream};
    if (cudaError_t e = taco_impl::launch_compress(l, a, consts_of(cfg))) return cuda_fail(e, "K1 compress launch");
    return TACO_OK;
}

int taco_compress_bcast_dev(const taco_config* cfg, const void* x, int dtype, uint64_t n, const taco_peers* peers,
                            uint64_t blk_begin, uint64_t blk_end, uint64_t dst_offset, uint64_t slot_stride,
                            int* d_flags, void* stream) {
    if (int rc = check_push_cfg(cfg)) return rc;
    if (int rc = check_peers(peers)) return rc;
    if (int rc = check_dtype(dtype)) return rc;
    if (n == 0) return fail(TACO_ERR_INPUT, "input tensor is empty");
    const uint64_t b = cfg->block_size, m = div_up(n, b);
    if (int rc = check_range(m, blk_begin, blk_end)) return rc;
    const taco_layout lay = layout_of(b, blk_end - blk_begin);
    if (peers->nranks > 1 && slot_stride < lay.msg_bytes) return fail(TACO_ERR_USAGE, "message stride too small");
    if ((dst_offset | slot_stride) % 16) return fail(TACO_ERR_USAGE, "peer slots must be 16-byte aligned");
    ShardArgs a{n, n, 1, blk_begin, blk_end - blk_begin, lay.msg_stride, lay.scal_offset, vec_align(x), d_flags};
    taco_dev::with_full_blocks(a, b);
    for (uint32_t q = 0; q < peers->nranks; ++q)
        a.dst[q] = static_cast<uint8_t*>(peers->base[q]) + dst_offset + (uint64_t)peers->rank * slot_stride;
    a.ndst = peers->nranks;
    a.bcast = 1;
    Launch l{cfg->block_size, dtype, (int)cfg->format, x, a.dst[0], nullptr, (cudaStream_t)stream};
    if (cudaError_t e = taco_impl::launch_compress(l, a, consts_of(cfg))) return cuda_fail(e, "K1 compress launch");
    return TACO_OK;
}

int taco_reduce_encode_push_dev(const taco_config* cfg, const void* msgs, uint64_t rank_stride,
                                const taco_peers* peers, uint64_t shard_len, uint64_t blk_begin, uint64_t blk_end,
                                uint64_t dst_offset, uint64_t slot_stride, void* acc_out, int acc_dtype,
                                int* d_flags, void* stream) {
    if (int rc = check_push_cfg(cfg)) return rc;
    if (int rc = check_peers(peers)) return rc;
    if (acc_out)
        if (int rc = check_dtype(acc_dtype)) return rc;
    if (shard_len == 0) return fail(TACO_ERR_INPUT, "input tensor is empty");
    const uint32_t P = peers->nranks;
    const uint64_t b = cfg->block_size, m = div_up(shard_len, b);
    if (int rc = check_range(m, blk_begin, blk_end)) return rc;
    const taco_layout lay = layout_of(b, blk_end - blk_begin);
    if (P > 1 && rank_stride < lay.msg_bytes) return fail(TACO_ERR_USAGE, "message stride too small");
    if (P > 1 && slot_stride < lay.msg_bytes) return fail(TACO_ERR_USAGE, "message stride too small");
    if ((dst_offset | slot_stride) % 16) return fail(TACO_ERR_USAGE, "peer slots must be 16-byte aligned");
    ShardArgs a{shard_len, shard_len, P, blk_begin, blk_end - blk_begin, rank_stride, lay.scal_offset,
                acc_out ? vec_align(acc_out) : 0, d_flags};
    taco_dev::with_full_blocks(a, b);
    a.full_last = a.full_mid;
    for (uint32_t q = 0; q < P; ++q)
        a.dst[q] = static_cast<uint8_t*>(peers->base[q]) + dst_offset + (uint64_t)peers->rank * slot_stride;
    a.ndst = P;
    Launch l{cfg->block_size, acc_dtype, (int)cfg->format, msgs, a.dst[0], acc_out, (cudaStream_t)stream};
    if (cudaError_t e = taco_impl::launch_reduce_encode(l, a, consts_of(cfg)))
        return cuda_fail(e, "K3 reduce-encode launch");
    return TACO_OK;
}

// ------------------------------------------------ fused peer collectives (3 / 2 launches) ---
namespace {
constexpr uint32_t kEpochWord = TACO_MAX_PEERS, kPhaseA = 16, kPhaseB = 24, kTicket = 32;

uint32_t* flag_words(const taco_peers* peers, uint32_t q, uint64_t flags_offset) {
    return reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(peers->base[q]) + flags_offset);
}

// this rank's words of `phase` in its own region, and its word [rank] of that phase in
// every peer's region
void phase_words(const taco_peers* peers, uint64_t flags_offset, uint32_t phase, const uint32_t*& own,
                 uint32_t* (&at_peers)[taco_dev::kMaxPeers]) {
    own = flag_words(peers, peers->rank, flags_offset) + phase;
    for (uint32_t q = 0; q < peers->nranks; ++q) at_peers[q] = flag_words(peers, q, flags_offset) + phase + peers->rank;
}

void set_common(ShardArgs& a, const taco_peers* peers, uint64_t flags_offset, uint32_t timeout_ms) {
    uint32_t* own = flag_words(peers, peers->rank, flags_offset);
    a.epoch = own + kEpochWord;
    a.ticket = own + kTicket;
    a.timeout_ns = (uint64_t)timeout_ms * 1000000ull;
}

// kernel start: publish "done with the slots" for `phase`, wait for every peer's
void set_pre(ShardArgs& a, const taco_peers* peers, uint64_t flags_offset, uint32_t phase, uint32_t timeout_ms) {
    set_common(a, peers, flags_offset, timeout_ms);
    phase_words(peers, flags_offset, phase, a.pre_wait, a.pre_sig);
    a.npre = peers->nranks;
}

// kernel end: the last CTA opens the next epoch, publishes `phase`, waits for every peer's
void set_post(ShardArgs& a, const taco_peers* peers, uint64_t flags_offset, uint32_t phase, uint32_t timeout_ms) {
    set_common(a, peers, flags_offset, timeout_ms);
    phase_words(peers, flags_offset, phase, a.post_wait, a.post_sig);
    a.npost = peers->nranks;
}

int check_fused(const taco_config* cfg, const taco_peers* peers, uint64_t flags_offset) {
    if (int rc = check_push_cfg(cfg)) return rc;
    if (int rc = check_peers(peers)) return rc;
    if (flags_offset % 16) return fail(TACO_ERR_USAGE, "peer flag offset must be 16-byte aligned");
    if (cfg->format != 0 || cfg->block_size < 64 || cfg->block_size > 512 || !taco_impl::xk_family())
        return fail(TACO_ERR_USAGE, "fused peer signalling needs E4M3 and 64 <= B <= 512 "
                                    "(use the push kernels with taco_peer_barrier_dev)");
    return TACO_OK;
}
}  // namespace

int taco_peer_fused_supported(const taco_config* cfg) {
    if (check_push_cfg(cfg)) return 0;
    return cfg->format == 0 && cfg->block_size >= 64 && cfg->block_size <= 512 && taco_impl::xk_family();
}

int taco_peer_allreduce_dev(const taco_config* cfg, const void* x, int dtype, uint64_t n, const taco_peers* peers,
                            uint64_t recv_offset, uint64_t gath_offset, uint64_t slot_stride, uint64_t flags_offset,
                            void* out, int out_dtype, uint32_t timeout_ms, int* d_flags, void* stream) {
    if (int rc = check_fused(cfg, peers, flags_offset)) return rc;
    if (int rc = check_dtype(dtype)) return rc;
    if (int rc = check_dtype(out_dtype)) return rc;
    if (n == 0) return fail(TACO_ERR_INPUT, "input tensor is empty");
    const uint32_t P = peers->nranks, me = peers->rank;
    const uint64_t b = cfg->block_size, S = div_up(n, P), m = div_up(S, b);
    const taco_layout lay = layout_of(b, m);
    if (P > 1 && slot_stride < lay.msg_bytes) return fail(TACO_ERR_USAGE, "message stride too small");
    if ((recv_offset | gath_offset | slot_stride) % 16) return fail(TACO_ERR_USAGE, "peer slots must be 16-byte aligned");
    cudaStream_t st = (cudaStream_t)stream;
    // K1: push shard p into rank p's receive slot [me]; its last CTA opens the epoch,
    // publishes phase A and waits for every peer's (all P copies of my shard have landed)
    ShardArgs a1{n, S, P, 0, m, lay.msg_stride, lay.scal_offset, ((P == 1 || S % 8 == 0) ? vec_align(x) : 0), d_flags};
    taco_dev::with_full_blocks(a1, b);
    for (uint32_t q = 0; q < P; ++q) a1.dst[q] = static_cast<uint8_t*>(peers->base[q]) + recv_offset + me * slot_stride;
    a1.ndst = P;
    set_post(a1, peers, flags_offset, kPhaseA, timeout_ms);
    Launch l1{cfg->block_size, dtype, (int)cfg->format, x, a1.dst[0], nullptr, st};
    if (cudaError_t e = taco_impl::launch_compress(l1, a1, consts_of(cfg))) return cuda_fail(e, "K1 compress launch");
    // K3 (plain): reduce + re-encode into every rank's gather slot [me]
    ShardArgs a3{S, S, P, 0, m, slot_stride, lay.scal_offset, 0, d_flags};
    taco_dev::with_full_blocks(a3, b);
    a3.full_last = a3.full_mid;
    for (uint32_t q = 0; q < P; ++q) a3.dst[q] = static_cast<uint8_t*>(peers->base[q]) + gath_offset + me * slot_stride;
    a3.ndst = P;
    const uint8_t* own = static_cast<const uint8_t*>(peers->base[me]);
    Launch l3{cfg->block_size, TACO_DT_F32, (int)cfg->format, own + recv_offset, a3.dst[0], nullptr, st};
    if (cudaError_t e = taco_impl::launch_reduce_encode(l3, a3, consts_of(cfg)))
        return cuda_fail(e, "K3 reduce-encode launch");
    // K2: publish phase B (my K3 is done: my receive slots are free, my gather pushes are
    // out), wait for every peer's, decode locally
    ShardArgs a2{n, S, P, 0, m, slot_stride, lay.scal_offset, ((P == 1 || S % 8 == 0) ? vec_align(out) : 0), d_flags};
    taco_dev::with_full_blocks(a2, b);
    set_pre(a2, peers, flags_offset, kPhaseB, timeout_ms);
    Launch l2{cfg->block_size, out_dtype, (int)cfg->format, own + gath_offset, out, nullptr, st};
    if (cudaError_t e = taco_impl::launch_decompress(l2, a2, consts_of(cfg))) return cuda_fail(e, "K2 decompress launch");
    return TACO_OK;
}

int taco_peer_reduce_scatter_dev(const taco_config* cfg, const void* x, int dtype, uint64_t n,
                                 const taco_peers* peers, uint64_t recv_offset, uint64_t slot_stride,
                                 uint64_t flags_offset, void* out, int out_dtype, uint32_t timeout_ms, int* d_flags,
                                 void* stream) {
    if (int rc = check_fused(cfg, peers, flags_offset)) return rc;
    if (int rc = check_dtype(dtype)) return rc;
    if (int rc = check_dtype(out_dtype)) return rc;
    if (n == 0) return fail(TACO_ERR_INPUT, "input tensor is empty");
    const uint32_t P = peers->nranks, me = peers->rank;
    const uint64_t b = cfg->block_size, S = div_up(n, P), m = div_up(S, b);
    const taco_layout lay = layout_of(b, m);
    if (P > 1 && slot_stride < lay.msg_bytes) return fail(TACO_ERR_USAGE, "message stride too small");
    if ((recv_offset | slot_stride) % 16) return fail(TACO_ERR_USAGE, "peer slots must be 16-byte aligned");
    cudaStream_t st = (cudaStream_t)stream;
    ShardArgs a1{n, S, P, 0, m, lay.msg_stride, lay.scal_offset, ((P == 1 || S % 8 == 0) ? vec_align(x) : 0), d_flags};
    taco_dev::with_full_blocks(a1, b);
    for (uint32_t q = 0; q < P; ++q) a1.dst[q] = static_cast<uint8_t*>(peers->base[q]) + recv_offset + me * slot_stride;
    a1.ndst = P;
    // K1: phase B first (my previous K3 is done with my receive slots; wait until every
    // peer's is), push, then phase A (every rank's pushes have landed)
    set_pre(a1, peers, flags_offset, kPhaseB, timeout_ms);
    set_post(a1, peers, flags_offset, kPhaseA, timeout_ms);
    Launch l1{cfg->block_size, dtype, (int)cfg->format, x, a1.dst[0], nullptr, st};
    if (cudaError_t e = taco_impl::launch_compress(l1, a1, consts_of(cfg))) return cuda_fail(e, "K1 compress launch");
    // K3 (plain) with the fp32 (or bf16) stage-1 sum as the product
    ShardArgs a3{S, S, P, 0, m, slot_stride, lay.scal_offset, vec_align(out), d_flags};
    taco_dev::with_full_blocks(a3, b);
    a3.full_last = a3.full_mid;
    const uint8_t* own = static_cast<const uint8_t*>(peers->base[me]);
    Launch l3{cfg->block_size, out_dtype, (int)cfg->format, own + recv_offset, nullptr, out, st};
    if (cudaError_t e = taco_impl::launch_reduce_encode(l3, a3, consts_of(cfg)))
        return cuda_fail(e, "K3 reduce-encode launch");
    return TACO_OK;
}

int taco_peer_all_gather_dev(const taco_config* cfg, const void* x, int dtype, uint64_t n_local,
                             const taco_peers* peers, uint64_t gath_offset, uint64_t slot_stride, uint64_t flags_offset,
                             void* out, int out_dtype, uint32_t timeout_ms, int* d_flags, void* stream) {
    if (int rc = check_fused(cfg, peers, flags_offset)) return rc;
    if (int rc = check_dtype(dtype)) return rc;
    if (int rc = check_dtype(out_dtype)) return rc;
    if (n_local == 0) return fail(TACO_ERR_INPUT, "input tensor is empty");
    const uint32_t P = peers->nranks, me = peers->rank;
    const uint64_t b = cfg->block_size, m = div_up(n_local, b);
    const taco_layout lay = layout_of(b, m);
    if (P > 1 && slot_stride < lay.msg_bytes) return fail(TACO_ERR_USAGE, "message stride too small");
    if ((gath_offset | slot_stride) % 16) return fail(TACO_ERR_USAGE, "peer slots must be 16-byte aligned");
    cudaStream_t st = (cudaStream_t)stream;
    // K1 broadcast of the own slice into every rank's gather slot [me]: phase B first (every
    // peer's K2 of the previous call is done with the gather slots), then phase A (every
    // rank's broadcast has landed)
    ShardArgs a1{n_local, n_local, 1, 0, m, lay.msg_stride, lay.scal_offset, vec_align(x), d_flags};
    taco_dev::with_full_blocks(a1, b);
    for (uint32_t q = 0; q < P; ++q) a1.dst[q] = static_cast<uint8_t*>(peers->base[q]) + gath_offset + me * slot_stride;
    a1.ndst = P;
    a1.bcast = 1;
    set_pre(a1, peers, flags_offset, kPhaseB, timeout_ms);
    set_post(a1, peers, flags_offset, kPhaseA, timeout_ms);
    Launch l1{cfg->block_size, dtype, (int)cfg->format, x, a1.dst[0], nullptr, st};
    if (cudaError_t e = taco_impl::launch_compress(l1, a1, consts_of(cfg))) return cuda_fail(e, "K1 compress launch");
    // K2 (plain) of the P gathered slices
    const uint64_t n = (uint64_t)P * n_local;
    ShardArgs a2{n, n_local, P, 0, m, slot_stride, lay.scal_offset, ((P == 1 || n_local % 8 == 0) ? vec_align(out) : 0),
                 d_flags};
    taco_dev::with_full_blocks(a2, b);
    const uint8_t* own = static_cast<const uint8_t*>(peers->base[me]);
    Launch l2{cfg->block_size, out_dtype, (int)cfg->format, own + gath_offset, out, nullptr, st};
    if (cudaError_t e = taco_impl::launch_decompress(l2, a2, consts_of(cfg))) return cuda_fail(e, "K2 decompress launch");
    return TACO_OK;
}

int taco_reduce_encode_ptrs_dev(const taco_config* cfg, const void* const* msgs, uint32_t nranks,
                                uint64_t shard_len, uint64_t blk_begin, uint64_t blk_end, void* out_msg, void* acc_out,
                                int acc_dtype, int* d_flags, void* stream) {
    if (!msgs) return fail(TACO_ERR_USAGE, "null message pointer array");
    if (nranks == 0 || nranks > TACO_MAX_PEERS) return fail(TACO_ERR_USAGE, "pointer-array reduction takes 1 to 8 ranks");
    for (uint32_t r = 0; r < nranks; ++r) {
        if (!msgs[r]) return fail(TACO_ERR_USAGE, "null message pointer");
        if (int rc = check_msg_buffer(msgs[r], 0, 1, "messages")) return rc;
    }
    if (out_msg)
        if (int rc = check_msg_buffer(out_msg, 0, 1, "out_msg")) return rc;
    if (int rc = check_config(cfg)) return rc;
    if (acc_out)
        if (int rc = check_dtype(acc_dtype)) return rc;
    if (!out_msg && !acc_out) return fail(TACO_ERR_USAGE, "reduce-encode needs out_msg or acc_out");
    if (shard_len == 0) return fail(TACO_ERR_INPUT, "input tensor is empty");
    if (cfg->kind != 0)
        return fail(TACO_ERR_USAGE, "the fused reduce-encode serves CodecKind::Taco (use decompress + compress)");
    const uint64_t b = cfg->block_size, m = div_up(shard_len, b);
    if (int rc = check_range(m, blk_begin, blk_end)) return rc;
    if (b > 1024) return fail(TACO_ERR_USAGE, "pointer-array reduction supports block sizes up to 1024");
    const taco_layout lay = layout_of(b, blk_end - blk_begin);
    ShardArgs a{shard_len, shard_len, nranks, blk_begin, blk_end - blk_begin, lay.msg_stride, lay.scal_offset,
                acc_out ? vec_align(acc_out) : 0, d_flags};
    taco_dev::with_full_blocks(a, b);
    a.full_last = a.full_mid;
    for (uint32_t r = 0; r < nranks; ++r) a.src[r] = static_cast<const uint8_t*>(msgs[r]);
    a.nsrc = nranks;
    Launch l{cfg->block_size, acc_dtype, (int)cfg->format, msgs[0], out_msg, acc_out, (cudaStream_t)stream};
    if (cudaError_t e = taco_impl::launch_reduce_encode(l, a, consts_of(cfg)))
        return cuda_fail(e, "K3 reduce-encode launch");
    return TACO_OK;
}

uint64_t taco_allreduce_sim_workspace(const taco_config* cfg, uint32_t nranks, uint64_t n) {
    if (!cfg || nranks == 0 || n == 0) return 0;
    const uint64_t S = div_up(n, nranks);
    const taco_layout lay = layout_of(payload_of(cfg), div_up(S, cfg->block_size));
    // phase-1 messages [rank][shard] + re-encoded shards [shard] (+ fp32 sum and decode
    // scratch of one shard for the codec kinds without a fused reduce-encode)
    uint64_t w = (uint64_t)nranks * nranks * lay.msg_stride + (uint64_t)nranks * lay.msg_stride;
    if (cfg->kind != 0) w += 2 * align16(S * sizeof(float));
    return w;
}

// collective.cpp:75-111 on one device: K1 per rank into its P shard messages, K3 per
// shard over the P ranks' messages (ascending), K2 of the P re-encoded shards.  Codec
// kinds other than Taco decode each rank's copy, add in fp32 (ascending rank) and
// compress the sum with their own codec, like the reference's run_twoshot.
int taco_allreduce_sim_dev(const taco_config* cfg, const void* inputs, int dtype, uint32_t nranks, uint64_t n,
                           void* out, int out_dtype, float* stage1, void* work, int* d_flags, void* stream) {
    if (nranks < 2) return fail(TACO_ERR_USAGE, "allreduce needs at least 2 ranks");
    if (n == 0) return fail(TACO_ERR_INPUT, "input tensor is empty");
    if (int rc = check_config(cfg)) return rc;
    if (int rc = check_dtype(dtype)) return rc;
    const uint64_t P = nranks, S = div_up(n, P), m = div_up(S, cfg->block_size);
    const taco_layout lay = layout_of(payload_of(cfg), m);
    uint8_t* sent = static_cast<uint8_t*>(work);
    uint8_t* reduced = sent + P * P * lay.msg_stride;
    const uint8_t* in = static_cast<const uint8_t*>(inputs);
    for (uint64_t r = 0; r < P; ++r) {
        if (int rc = taco_compress_dev(cfg, in + r * n * dtype_size(dtype), dtype, n, nranks, 0, m,
                                       sent + r * P * lay.msg_stride, lay.msg_stride, d_flags, stream))
            return rc;
    }
    float* acc = reinterpret_cast<float*>(reduced + P * lay.msg_stride);
    float* tmp = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(acc) + align16(S * sizeof(float)));
    for (uint64_t s = 0; s < P; ++s) {
        if (cfg->kind == 0) {
            if (int rc = taco_reduce_encode_dev(cfg, sent + s * lay.msg_stride, P * lay.msg_stride, nranks, S, 0, m,
                                                reduced + s * lay.msg_stride, stage1 ? stage1 + s * S : nullptr,
                                                TACO_DT_F32, d_flags, stream))
                return rc;
            continue;
        }
        for (uint64_t r = 0; r < P; ++r) {  // acc = dec(rank 0); acc += dec(rank r)
            if (int rc = taco_decompress_dev(cfg, sent + (r * P + s) * lay.msg_stride, lay.msg_stride, 1, S, 0, m,
                                             r == 0 ? acc : tmp, TACO_DT_F32, d_flags, stream))
                return rc;
            if (r > 0)
                if (cudaError_t e = taco_impl::launch_add_f32(acc, tmp, S, (cudaStream_t)stream))
                    return cuda_fail(e, "fp32 sum launch");
        }
        if (stage1)
            if (cudaError_t e = cudaMemcpyAsync(stage1 + s * S, acc, S * sizeof(float), cudaMemcpyDeviceToDevice,
                                                (cudaStream_t)stream))
                return cuda_fail(e, "stage-1 copy");
        if (int rc = taco_compress_dev(cfg, acc, TACO_DT_F32, S, 1, 0, m, reduced + s * lay.msg_stride,
                                       lay.msg_stride, d_flags, stream))
            return rc;
    }
    return taco_decompress_dev(cfg, reduced, lay.msg_stride, nranks, n, 0, m, out, out_dtype, d_flags, stream);
}

int taco_scaled_spectrum_dev(const taco_config* cfg, const void* x, int dtype, uint64_t n, float* out, int* d_flags,
                             void* stream) {
    if (int rc = check_config(cfg)) return rc;
    if (int rc = check_dtype(dtype)) return rc;
    if (n == 0) return fail(TACO_ERR_INPUT, "input tensor is empty");
    const uint64_t b = cfg->block_size, m = div_up(n, b);
    ShardArgs a{n, n, 1, 0, m, 0, 0, 0, d_flags};
    taco_dev::with_full_blocks(a, b);
    Launch l{cfg->block_size, dtype, (int)cfg->format, x, out, nullptr, (cudaStream_t)stream};
    const double qtop = cfg->kind == 4 ? 127.0 : (cfg->format ? 57344.0 : 448.0);  // codec.cpp:311-313
    if (cudaError_t e = taco_impl::launch_scaled_spectrum(l, a, consts_of(cfg), qtop))
        return cuda_fail(e, "scaled spectrum launch");
    return TACO_OK;
}

int taco_error_report_dev(const void* original, int orig_dtype, const void* reconstructed, int recon_dtype,
                          uint64_t n, uint32_t bins, taco_error_report* out, uint64_t* counts, void* stream) {
    if (int rc = check_dtype(orig_dtype)) return rc;
    if (int rc = check_dtype(recon_dtype)) return rc;
    if (n == 0) return fail(TACO_ERR_INPUT, "input tensor is empty");
    if (bins == 0) return fail(TACO_ERR_CONFIG, "histogram needs at least one bin");
    double r[8];
    static_assert(sizeof(unsigned long long) == sizeof(uint64_t), "");
    if (int e = taco_impl::error_report_dev(original, orig_dtype, reconstructed, recon_dtype, n, bins, r,
                                            reinterpret_cast<unsigned long long*>(counts), (cudaStream_t)stream))
        return cuda_fail((cudaError_t)e, "error report");
    out->mse = r[0];
    out->relative_l2 = r[1];
    out->max_abs_error = r[2];
    out->zero_collapse_fraction = r[3];
    out->kurtosis = r[4];
    out->kurtosis_defined = r[5] != 0.0;
    out->hist_lo = r[6];
    out->hist_hi = r[7];
    return TACO_OK;
}

// ------------------------------------------------ TACOCMP1 archive (serialize.cpp) ----
// magic "TACOCMP1", kind u8, format id u8, block size u32 LE, length u64 LE, then per
// block [payload][alpha f32][scale f32] (serialize.cpp:109-124).
static uint8_t format_id(const taco_config* cfg) {  // serialize.cpp:79-89
    if (cfg->kind == 2 || cfg->kind == 4) return 2;
    if (cfg->kind == 3) return 3;
    return (uint8_t)cfg->format;
}

int taco_archive_header(const taco_config* cfg, uint64_t n, uint8_t* out22) {
    if (int rc = check_config(cfg)) return rc;
    static const char magic[8] = {'T', 'A', 'C', 'O', 'C', 'M', 'P', '1'};
    std::memcpy(out22, magic, 8);
    out22[8] = (uint8_t)cfg->kind;
    out22[9] = format_id(cfg);
    const uint32_t b = cfg->block_size;
    std::memcpy(out22 + 10, &b, 4);  // little-endian host (x86-64 / aarch64)
    std::memcpy(out22 + 14, &n, 8);
    return TACO_OK;
}

int taco_archive_export_dev(const taco_config* cfg, const void* msg, uint64_t n, void* archive, void* stream) {
    if (int rc = check_config(cfg)) return rc;
    if (n == 0) return fail(TACO_ERR_CORRUPT, "compressed tensor declares zero elements");
    const uint64_t m = div_up(n, cfg->block_size);
    const taco_layout lay = layout_of(payload_of(cfg), m);
    uint8_t hdr[22];
    taco_archive_header(cfg, n, hdr);
    if (cudaError_t e = taco_impl::launch_archive(static_cast<const uint8_t*>(msg), static_cast<uint8_t*>(archive),
                                                  m, payload_of(cfg), lay.scal_offset, hdr, 0, nullptr,
                                                  (cudaStream_t)stream))
        return cuda_fail(e, "archive export launch");
    return TACO_OK;
}

int taco_archive_import_dev(const taco_config* cfg, const void* archive, uint64_t n, void* msg, int* d_flags,
                            void* stream) {
    if (int rc = check_config(cfg)) return rc;
    if (n == 0) return fail(TACO_ERR_CORRUPT, "archive declares zero elements");
    const uint64_t m = div_up(n, cfg->block_size);
    const taco_layout lay = layout_of(payload_of(cfg), m);
    if (cudaError_t e = taco_impl::launch_archive(static_cast<const uint8_t*>(archive), static_cast<uint8_t*>(msg),
                                                  m, payload_of(cfg), lay.scal_offset, nullptr, 1, d_flags,
                                                  (cudaStream_t)stream))
        return cuda_fail(e, "archive import launch");
    return TACO_OK;
}

// archive_parse (serialize.cpp:126-160) header checks, in the reference's order and with its
// messages (the Reader's end-of-data message is "unexpected end of archive", :35).  A body
// shorter than the header declares reports "unexpected end of archive" (the caller scans
// the complete blocks' scalars first, as the reference's sequential reader would).
int taco_archive_parse_header(const uint8_t* bytes, uint64_t size, taco_config* cfg_out, uint64_t* n_out) {
    static const char magic[8] = {'T', 'A', 'C', 'O', 'C', 'M', 'P', '1'};
    static const char* eof = "unexpected end of archive";
    if (size < 8) return fail(TACO_ERR_CORRUPT, eof);
    if (std::memcmp(bytes, magic, 8) != 0) return fail(TACO_ERR_CORRUPT, "bad magic, not a compressed archive");
    if (size < 9) return fail(TACO_ERR_CORRUPT, eof);
    if (bytes[8] > 4) return fail(TACO_ERR_CORRUPT, "unknown codec kind in archive");
    if (size < 10) return fail(TACO_ERR_CORRUPT, eof);
    if (bytes[9] > 3) return fail(TACO_ERR_CORRUPT, "unknown payload format in archive");
    if (size < 14) return fail(TACO_ERR_CORRUPT, eof);
    taco_config c = taco_default_config();
    c.kind = bytes[8];
    c.format = bytes[9] == 1 ? 1u : 0u;
    uint32_t b;
    uint64_t n;
    std::memcpy(&b, bytes + 10, 4);
    if (!pow2(b) || b < 2 || b > 32768) return fail(TACO_ERR_CORRUPT, "archive block size is not a valid power of two");
    if (size < 22) return fail(TACO_ERR_CORRUPT, eof);
    std::memcpy(&n, bytes + 14, 8);
    if (n == 0) return fail(TACO_ERR_CORRUPT, "archive declares zero elements");
    c.block_size = b;
    *cfg_out = c;
    *n_out = n;
    const uint64_t need = 22 + div_up(n, b) * (payload_of(&c) + 8);
    if (size < need) return fail(TACO_ERR_CORRUPT, eof);
    if (size > need) return fail(TACO_ERR_CORRUPT, "trailing bytes after archive payload");
    return TACO_OK;
}

}  // extern "C"

// =================================================================== host API ====
// Pipelined host <-> device path.  Chunks of whole blocks rotate over kSlots streams;
// each slot has its own device buffers, so chunk i's H2D, kernels and D2H overlap
// with its neighbours' (two copy engines + SMs).  Pageable user memory is staged
// through pinned slot buffers; pinned user memory is copied directly.

// Host pipeline: three role streams (H2D, kernels, D2H) so the two copy engines stream
// back to back; per-slot events order buffer reuse between them.
struct taco_ctx {
    static constexpr int kSlots = 3;
    int device = 0;
    cudaStream_t st[kSlots] = {};  // st[0] H2D, st[1] kernels, st[2] D2H
    cudaEvent_t ev_in[kSlots] = {}, ev_k[kSlots] = {}, ev_out[kSlots] = {};
    void* d_in[kSlots] = {};
    void* d_msg[kSlots] = {};
    void* d_out[kSlots] = {};
    int* d_flags = nullptr;
    size_t cap_in = 0, cap_msg = 0, cap_out = 0;
    void* h_stage_in[kSlots] = {};
    void* h_stage_out[kSlots] = {};
    size_t cap_stage_in = 0, cap_stage_out = 0;
    void* d_scratch = nullptr;  // grow-only workspace of the one-shot host calls (allreduce_sim, spectrum)
    size_t cap_scratch = 0;
    std::mutex mu;
};

namespace {

bool is_pinned(const void* p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

int grow_dev(void** bufs, size_t& cap, size_t need) {
    if (need <= cap) return TACO_OK;
    for (int i = 0; i < taco_ctx::kSlots; ++i) {
        if (bufs[i]) cudaFree(bufs[i]);
        bufs[i] = nullptr;
        TACO_CUDA(cudaMalloc(&bufs[i], need));
    }
    cap = need;
    return TACO_OK;
}

int grow_host(void** bufs, size_t& cap, size_t need) {
    if (need <= cap) return TACO_OK;
    for (int i = 0; i < taco_ctx::kSlots; ++i) {
        if (bufs[i]) cudaFreeHost(bufs[i]);
        bufs[i] = nullptr;
        TACO_CUDA(cudaMallocHost(&bufs[i], need));
    }
    cap = need;
    return TACO_OK;
}

// chunk = whole blocks, ~TACO_HOST_CHUNK_KB (default 8 MiB) of input per chunk
uint64_t chunk_blocks(uint64_t b, size_t elt) {
    static const uint64_t bytes = [] {
        const char* v = std::getenv("TACO_HOST_CHUNK_KB");
        const long kb = v ? std::atol(v) : 0;
        return kb > 0 ? (uint64_t)kb << 10 : (8ull << 20);
    }();
    const uint64_t target = bytes / elt;
    return std::max<uint64_t>(1, target / b);
}

int finish(taco_ctx* ctx) {
    for (int i = 0; i < taco_ctx::kSlots; ++i) TACO_CUDA(cudaStreamSynchronize(ctx->st[i]));
    int flags = 0;
    TACO_CUDA(cudaMemcpy(&flags, ctx->d_flags, sizeof(int), cudaMemcpyDeviceToHost));
    return taco_flags_status(flags);
}

}  // namespace

extern "C" {

int taco_ctx_create(int device, taco_ctx** out) {
    auto* c = new taco_ctx();
    c->device = device;
    DeviceGuard dg(device);
    cudaError_t e = dg.err;
    for (int i = 0; i < taco_ctx::kSlots && e == cudaSuccess; ++i) {
        e = cudaStreamCreateWithFlags(&c->st[i], cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_in[i], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_k[i], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_out[i], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaMalloc(&c->d_flags, sizeof(int));
    if (e != cudaSuccess) {
        delete c;
        return cuda_fail(e, "taco_ctx_create");
    }
    *out = c;
    return TACO_OK;
}

void taco_ctx_destroy(taco_ctx* c) {
    if (!c) return;
    DeviceGuard dg(c->device);
    for (int i = 0; i < taco_ctx::kSlots; ++i) {
        if (c->st[i]) cudaStreamSynchronize(c->st[i]);
        cudaFree(c->d_in[i]);
        cudaFree(c->d_msg[i]);
        cudaFree(c->d_out[i]);
        if (c->h_stage_in[i]) cudaFreeHost(c->h_stage_in[i]);
        if (c->h_stage_out[i]) cudaFreeHost(c->h_stage_out[i]);
        if (c->st[i]) cudaStreamDestroy(c->st[i]);
        if (c->ev_in[i]) cudaEventDestroy(c->ev_in[i]);
        if (c->ev_k[i]) cudaEventDestroy(c->ev_k[i]);
        if (c->ev_out[i]) cudaEventDestroy(c->ev_out[i]);
    }
    cudaFree(c->d_flags);
    cudaFree(c->d_scratch);
    delete c;
}

namespace {
// Carves `count` 256-byte-aligned regions of the given sizes out of the context's grow-only
// scratch buffer: repeated host calls of the same (or a smaller) size never allocate, and
// the buffer is reallocated only after the context's streams drained.
int ctx_scratch(taco_ctx* ctx, const size_t* sizes, void** out, int count) {
    size_t total = 0;
    for (int i = 0; i < count; ++i) total += (sizes[i] + 255) & ~size_t(255);
    if (total > ctx->cap_scratch) {
        for (int i = 0; i < taco_ctx::kSlots; ++i) TACO_CUDA(cudaStreamSynchronize(ctx->st[i]));
        cudaFree(ctx->d_scratch);
        ctx->d_scratch = nullptr;
        ctx->cap_scratch = 0;
        TACO_CUDA(cudaMalloc(&ctx->d_scratch, total));
        ctx->cap_scratch = total;
    }
    auto* p = static_cast<uint8_t*>(ctx->d_scratch);
    for (int i = 0; i < count; ++i) {
        out[i] = sizes[i] ? p : nullptr;
        p += (sizes[i] + 255) & ~size_t(255);
    }
    return TACO_OK;
}
}  // namespace

// Shared driver of the three host calls.  mode 0 = compress, 1 = decompress, 2 = round trip.
static int host_pipeline(taco_ctx* ctx, const taco_config* cfg, int mode, const void* src, int in_dtype,
                         uint64_t n, void* dst, int out_dtype) {
    if (!ctx) return fail(TACO_ERR_USAGE, "null taco context");
    if (int rc = check_config(cfg)) return rc;
    if (mode != 1)
        if (int rc = check_dtype(in_dtype)) return rc;
    if (mode != 0)
        if (int rc = check_dtype(out_dtype)) return rc;
    if (n == 0) return mode == 1 ? fail(TACO_ERR_CORRUPT, "compressed tensor declares zero elements")
                                 : fail(TACO_ERR_INPUT, "input tensor is empty");
    std::lock_guard<std::mutex> lock(ctx->mu);
    DeviceGuard dg(ctx->device);
    TACO_CUDA(dg.err);
    const uint64_t b = cfg->block_size, m = div_up(n, b), pb = payload_of(cfg);
    const size_t ein = mode == 1 ? 1 : dtype_size(in_dtype);
    const size_t eout = mode == 0 ? 1 : dtype_size(out_dtype);
    // tensor-wide scales (DirectFp8 GlobalMax, Int8Uniform: codec.cpp:223-229) need the
    // whole tensor in one launch; everything else pipelines in chunks of whole blocks
    const bool whole = cfg->kind == 2 || (cfg->kind == 1 && cfg->direct_scale == 0);
    const uint64_t cb = whole ? m : chunk_blocks(b, mode == 1 ? 4 : ein);
    const taco_layout full = layout_of(pb, m);
    const taco_layout cl = layout_of(pb, std::min(cb, m));
    const size_t in_bytes = mode == 1 ? cl.msg_stride : cb * b * ein;  // (payload-aware via cl)
    const size_t out_bytes = mode == 0 ? cl.msg_stride : cb * b * eout;
    if (int rc = grow_dev(ctx->d_in, ctx->cap_in, in_bytes)) return rc;
    if (int rc = grow_dev(ctx->d_msg, ctx->cap_msg, cl.msg_stride)) return rc;
    if (int rc = grow_dev(ctx->d_out, ctx->cap_out, out_bytes)) return rc;
    const bool pin_in = is_pinned(src), pin_out = is_pinned(dst);
    if (!pin_in)
        if (int rc = grow_host(ctx->h_stage_in, ctx->cap_stage_in, in_bytes)) return rc;
    if (!pin_out)
        if (int rc = grow_host(ctx->h_stage_out, ctx->cap_stage_out, out_bytes)) return rc;
    cudaStream_t s_in = ctx->st[0], s_k = ctx->st[1], s_out = ctx->st[2];
    TACO_CUDA(cudaMemsetAsync(ctx->d_flags, 0, sizeof(int), s_k));

    const uint8_t* s8 = static_cast<const uint8_t*>(src);
    uint8_t* d8 = static_cast<uint8_t*>(dst);
    // chunk schedule: cb-block chunks, with the first and last ~1/8 of a chunk ramped
    // (cb/8, cb/4, cb/2 ... cb/2, cb/4, cb/8) so the un-overlapped pipeline fill (first H2D)
    // and drain (last kernels + D2H) are short; every chunk is whole blocks
    std::vector<std::pair<uint64_t, uint64_t>> chunks;
    {
        std::vector<uint64_t> head, tail;
        uint64_t left = m;
        if (!whole && m >= 4 * cb)
            for (uint64_t r = cb / 8; r >= 1 && r < cb; r *= 2) {
                head.push_back(r);
                tail.push_back(r);
                left -= 2 * r;
            }
        uint64_t b0 = 0;
        for (uint64_t r : head) chunks.push_back({b0, b0 + r}), b0 += r;
        const uint64_t mid_end = b0 + left;
        for (; b0 < mid_end; b0 += cb) chunks.push_back({b0, std::min(mid_end, b0 + cb)});
        b0 = mid_end;
        for (auto it = tail.rbegin(); it != tail.rend(); ++it) chunks.push_back({b0, b0 + *it}), b0 += *it;
    }
    const uint64_t nchunks = chunks.size();
    // staged output copies still in flight per slot: (host dst, bytes) pairs
    std::vector<std::pair<uint8_t*, size_t>> pending[taco_ctx::kSlots];
    auto drain = [&](int slot) -> int {
        if (pin_out || pending[slot].empty()) return TACO_OK;
        TACO_CUDA(cudaEventSynchronize(ctx->ev_out[slot]));
        size_t off = 0;
        for (auto& pr : pending[slot]) {
            std::memcpy(pr.first, static_cast<uint8_t*>(ctx->h_stage_out[slot]) + off, pr.second);
            off += pr.second;
        }
        pending[slot].clear();
        return TACO_OK;
    };
    for (uint64_t ci = 0; ci < nchunks; ++ci) {
        const int slot = (int)(ci % taco_ctx::kSlots);
        const bool reuse = ci >= (uint64_t)taco_ctx::kSlots;
        const uint64_t b0 = chunks[ci].first, b1 = chunks[ci].second, nb = b1 - b0;
        const uint64_t e0 = b0 * b, e1 = std::min<uint64_t>(n, b1 * b), ne = e1 - e0;
        const taco_layout lay = layout_of(pb, nb);
        if (int rc = drain(slot)) return rc;  // staged output of chunk ci - kSlots copied out
        // ---- H2D (s_in): d_in[slot] is free once the kernels of chunk ci - kSlots ran
        if (reuse) TACO_CUDA(cudaStreamWaitEvent(s_in, ctx->ev_k[slot], 0));
        if (!pin_in && reuse) TACO_CUDA(cudaEventSynchronize(ctx->ev_in[slot]));  // staging slot free
        auto h2d = [&](void* d, const uint8_t* h, size_t bytes, size_t stage_off) -> int {
            if (pin_in) {
                TACO_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s_in));
            } else {
                uint8_t* stage = static_cast<uint8_t*>(ctx->h_stage_in[slot]) + stage_off;
                std::memcpy(stage, h, bytes);
                TACO_CUDA(cudaMemcpyAsync(d, stage, bytes, cudaMemcpyHostToDevice, s_in));
            }
            return TACO_OK;
        };
        if (mode == 1) {  // chunk of the full message -> chunk message layout
            uint8_t* d = static_cast<uint8_t*>(ctx->d_in[slot]);
            if (int rc = h2d(d, s8 + b0 * pb, nb * pb, 0)) return rc;
            if (int rc = h2d(d + lay.scal_offset, s8 + full.scal_offset + b0 * 8, nb * 8, lay.scal_offset)) return rc;
        } else {
            if (int rc = h2d(ctx->d_in[slot], s8 + e0 * ein, ne * ein, 0)) return rc;
        }
        TACO_CUDA(cudaEventRecord(ctx->ev_in[slot], s_in));
        // ---- kernels (s_k): the chunk is a standalone tensor of ne elements (blocks never
        // span chunks); d_out[slot] is free once the D2H of chunk ci - kSlots finished
        TACO_CUDA(cudaStreamWaitEvent(s_k, ctx->ev_in[slot], 0));
        if (reuse) TACO_CUDA(cudaStreamWaitEvent(s_k, ctx->ev_out[slot], 0));
        void* msg = mode == 1 ? ctx->d_in[slot] : (mode == 0 ? ctx->d_out[slot] : ctx->d_msg[slot]);
        if (mode != 1)
            if (int rc = taco_compress_dev(cfg, ctx->d_in[slot], in_dtype, ne, 1, 0, nb, msg, lay.msg_stride,
                                           ctx->d_flags, s_k))
                return rc;
        if (mode != 0)
            if (int rc = taco_decompress_dev(cfg, msg, lay.msg_stride, 1, ne, 0, nb, ctx->d_out[slot], out_dtype,
                                             ctx->d_flags, s_k))
                return rc;
        TACO_CUDA(cudaEventRecord(ctx->ev_k[slot], s_k));
        // ---- D2H (s_out)
        TACO_CUDA(cudaStreamWaitEvent(s_out, ctx->ev_k[slot], 0));
        auto d2h = [&](uint8_t* h, const void* d, size_t bytes, size_t stage_off) -> int {
            if (pin_out) {
                TACO_CUDA(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s_out));
            } else {
                uint8_t* stage = static_cast<uint8_t*>(ctx->h_stage_out[slot]) + stage_off;
                TACO_CUDA(cudaMemcpyAsync(stage, d, bytes, cudaMemcpyDeviceToHost, s_out));
                pending[slot].push_back({h, bytes});
            }
            return TACO_OK;
        };
        if (mode == 0) {
            const uint8_t* d = static_cast<const uint8_t*>(ctx->d_out[slot]);
            if (int rc = d2h(d8 + b0 * pb, d, nb * pb, 0)) return rc;
            if (int rc = d2h(d8 + full.scal_offset + b0 * 8, d + lay.scal_offset, nb * 8, nb * pb)) return rc;
        } else {
            if (int rc = d2h(d8 + e0 * eout, ctx->d_out[slot], ne * eout, 0)) return rc;
        }
        TACO_CUDA(cudaEventRecord(ctx->ev_out[slot], s_out));
    }
    for (int i = 0; i < taco_ctx::kSlots; ++i)
        if (int rc = drain(i)) return rc;
    return finish(ctx);
}

int taco_compress_host(taco_ctx* ctx, const taco_config* cfg, const void* x_host, int dtype, uint64_t n,
                       void* msg_host) {
    return host_pipeline(ctx, cfg, 0, x_host, dtype, n, msg_host, 0);
}

int taco_decompress_host(taco_ctx* ctx, const taco_config* cfg, const void* msg_host, uint64_t n, void* out_host,
                         int out_dtype) {
    return host_pipeline(ctx, cfg, 1, msg_host, 0, n, out_host, out_dtype);
}

int taco_roundtrip_host(taco_ctx* ctx, const taco_config* cfg, const void* x_host, int dtype, uint64_t n,
                        void* out_host, int out_dtype) {
    return host_pipeline(ctx, cfg, 2, x_host, dtype, n, out_host, out_dtype);
}

int taco_scaled_spectrum_host(taco_ctx* ctx, const taco_config* cfg, const float* x_host, uint64_t n,
                              float* out_host) {
    if (!ctx) return fail(TACO_ERR_USAGE, "null taco context");
    if (int rc = check_config(cfg)) return rc;
    if (n == 0) return fail(TACO_ERR_INPUT, "input tensor is empty");
    std::lock_guard<std::mutex> lock(ctx->mu);
    DeviceGuard dg(ctx->device);
    TACO_CUDA(dg.err);
    const uint64_t out_n = div_up(n, cfg->block_size) * cfg->block_size;
    void* bufs[2] = {};
    const size_t sizes[2] = {n * 4, out_n * 4};
    if (int rc = ctx_scratch(ctx, sizes, bufs, 2)) return rc;
    void *d_in = bufs[0], *d_out = bufs[1];
    cudaStream_t st = ctx->st[0];
    int rc = TACO_OK;
    cudaError_t e = cudaMemsetAsync(ctx->d_flags, 0, sizeof(int), st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_in, x_host, n * 4, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) rc = cuda_fail(e, "scaled spectrum staging");
    if (rc == TACO_OK) rc = taco_scaled_spectrum_dev(cfg, d_in, TACO_DT_F32, n, static_cast<float*>(d_out), ctx->d_flags, st);
    if (rc == TACO_OK) {
        e = cudaMemcpyAsync(out_host, d_out, out_n * 4, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) rc = cuda_fail(e, "scaled spectrum readback");
    }
    if (rc == TACO_OK) {
        int flags = 0;
        e = cudaMemcpy(&flags, ctx->d_flags, sizeof(int), cudaMemcpyDeviceToHost);
        rc = e != cudaSuccess ? cuda_fail(e, "flags readback") : taco_flags_status(flags);
    }
    return rc;
}

int taco_allreduce_sim_host(taco_ctx* ctx, const taco_config* cfg, const float* inputs_host, uint32_t nranks,
                            uint64_t n, float* result_host, float* stage1_host) {
    if (!ctx) return fail(TACO_ERR_USAGE, "null taco context");
    if (nranks < 2) return fail(TACO_ERR_USAGE, "allreduce needs at least 2 ranks");
    if (n == 0) return fail(TACO_ERR_INPUT, "input tensor is empty");
    if (int rc = check_config(cfg)) return rc;
    std::lock_guard<std::mutex> lock(ctx->mu);
    DeviceGuard dg(ctx->device);
    TACO_CUDA(dg.err);
    const uint64_t S = div_up(n, nranks);
    const size_t in_bytes = (size_t)nranks * n * 4, st_bytes = stage1_host ? (size_t)nranks * S * 4 : 0;
    const size_t ws = taco_allreduce_sim_workspace(cfg, nranks, n);
    void* bufs[4] = {};
    const size_t sizes[4] = {in_bytes, n * 4, st_bytes, ws};
    if (int rc = ctx_scratch(ctx, sizes, bufs, 4)) return rc;
    void *d_in = bufs[0], *d_out = bufs[1], *d_st = bufs[2], *d_ws = bufs[3];
    cudaStream_t st = ctx->st[0];
    int rc = TACO_OK;
    cudaError_t e = cudaMemsetAsync(ctx->d_flags, 0, sizeof(int), st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_in, inputs_host, in_bytes, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) rc = cuda_fail(e, "allreduce staging");
    if (rc == TACO_OK)
        rc = taco_allreduce_sim_dev(cfg, d_in, TACO_DT_F32, nranks, n, d_out, TACO_DT_F32,
                                    static_cast<float*>(d_st), d_ws, ctx->d_flags, st);
    if (rc == TACO_OK) {
        e = cudaMemcpyAsync(result_host, d_out, n * 4, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess && st_bytes) e = cudaMemcpyAsync(stage1_host, d_st, st_bytes, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) rc = cuda_fail(e, "allreduce readback");
    }
    if (rc == TACO_OK) {
        int flags = 0;
        e = cudaMemcpy(&flags, ctx->d_flags, sizeof(int), cudaMemcpyDeviceToHost);
        rc = e != cudaSuccess ? cuda_fail(e, "flags readback") : taco_flags_status(flags);
    }
    return rc;
}

// taco::allreduce (collective.cpp:75-254) for all three schedules on host rank tensors,
// computed on the device.  Every "rank" tensor lives in one [P][padded] fp32 array; a ring
// or tree transfer is a compress + decompress of the moved range in place (the codec grid
// starts at the range start, as the reference's through_codec of a slice), and every fp32
// sum is a device add in ascending-origin order.  The host only walks the schedule's range
// bookkeeping.  exact_host receives the ascending-rank fp32 sum; rel_l2 (optional) the
// relative L2 of result vs exact (taco_error_report_dev's definition, analysis.cpp:97-124).
int taco_allreduce_schedule_host(taco_ctx* ctx, const taco_config* cfg, int algorithm, const float* inputs_host,
                                 uint32_t nranks, uint64_t n, float* result_host, float* exact_host,
                                 double* rel_l2) {
    if (!ctx) return fail(TACO_ERR_USAGE, "null taco context");
    if (nranks < 2) return fail(TACO_ERR_USAGE, "allreduce needs at least 2 ranks");
    if (n == 0) return fail(TACO_ERR_INPUT, "input tensor is empty");
    if (algorithm < 0 || algorithm > 2) return fail(TACO_ERR_USAGE, "unknown allreduce algorithm");
    if (!inputs_host || !result_host || !exact_host) return fail(TACO_ERR_USAGE, "allreduce needs host buffers");
    if (int rc = check_config(cfg)) return rc;
    std::lock_guard<std::mutex> lock(ctx->mu);
    DeviceGuard dg(ctx->device);
    TACO_CUDA(dg.err);
    const uint64_t P = nranks;
    uint64_t q = 1;
    while (2 * q <= P) q *= 2;
    const uint64_t padded = div_up(n, q) * q, slice = padded / q;
    const taco_layout lay = layout_of(payload_of(cfg), div_up(padded, cfg->block_size));
    void* bufs[6] = {};
    const size_t sizes[6] = {P * padded * 4, P * padded * 4, padded * 4, padded * 4, q * lay.msg_stride,
                             algorithm == 0 ? taco_allreduce_sim_workspace(cfg, nranks, n) : 0};
    if (int rc = ctx_scratch(ctx, sizes, bufs, 6)) return rc;
    float* in = static_cast<float*>(bufs[0]);    // [P][padded] rank inputs, zero-padded
    float* data = static_cast<float*>(bufs[1]);  // [P][padded] per-origin working copies
    float* exact = static_cast<float*>(bufs[2]);
    float* result = static_cast<float*>(bufs[3]);
    uint8_t* msg = static_cast<uint8_t*>(bufs[4]);
    cudaStream_t st = ctx->st[0];
    TACO_CUDA(cudaMemsetAsync(ctx->d_flags, 0, sizeof(int), st));
    TACO_CUDA(cudaMemsetAsync(in, 0, sizes[0], st));
    TACO_CUDA(cudaMemcpy2DAsync(in, padded * 4, inputs_host, n * 4, n * 4, P, cudaMemcpyHostToDevice, st));
    auto add = [&](float* a, const float* b, uint64_t len) -> int {
        if (cudaError_t e = taco_impl::launch_add_f32(a, b, len, st)) return cuda_fail(e, "fp32 sum launch");
        return TACO_OK;
    };
    // what the receiving rank reconstructs from one transfer of x[0, len): in place
    auto through_codec = [&](float* x, uint64_t len) -> int {
        const uint64_t m = div_up(len, cfg->block_size);
        if (int rc = taco_compress_dev(cfg, x, TACO_DT_F32, len, 1, 0, m, msg, lay.msg_stride, ctx->d_flags, st))
            return rc;
        return taco_decompress_dev(cfg, msg, lay.msg_stride, 1, len, 0, m, x, TACO_DT_F32, ctx->d_flags, st);
    };
    auto copy = [&](float* dst, const float* src, uint64_t len) -> int {
        TACO_CUDA(cudaMemcpyAsync(dst, src, len * 4, cudaMemcpyDeviceToDevice, st));
        return TACO_OK;
    };
    // exact: fp32 sum over ranks in ascending rank order (collective.cpp:36-41)
    int rc = copy(exact, in, padded);
    for (uint64_t r = 1; r < P && rc == TACO_OK; ++r) rc = add(exact, in + r * padded, padded);
    if (rc == TACO_OK && algorithm == 0) {
        // two-shot: the fused K1 -> K3 -> K2 simulation over a dense [P][n] copy
        TACO_CUDA(cudaMemcpy2DAsync(data, n * 4, in, padded * 4, n * 4, P, cudaMemcpyDeviceToDevice, st));
        rc = taco_allreduce_sim_dev(cfg, data, TACO_DT_F32, nranks, n, result, TACO_DT_F32, nullptr, bufs[5],
                                    ctx->d_flags, st);
    } else if (rc == TACO_OK && algorithm == 1) {
        // ring: the partial climbs the ranks; every hop crosses the codec, then the next
        // rank adds its own input; the total is compressed once and forwarded unchanged
        rc = copy(result, in, n);
        for (uint64_t r = 1; r < P && rc == TACO_OK; ++r) {
            rc = through_codec(result, n);
            if (rc == TACO_OK) rc = add(result, in + r * padded, n);
        }
        if (rc == TACO_OK) rc = through_codec(result, n);
    } else if (rc == TACO_OK) {
        // tree: origin o's values stay in data[o]; at[r] is where rank r's current range
        // starts and held[r] the origins it carries.  A halving round moves every carried
        // origin's far half to the partner through the codec.
        rc = copy(data, in, P * padded);
        std::vector<std::vector<uint32_t>> held(q);
        std::vector<uint64_t> at(q, 0);
        for (uint64_t r = 0; r < q; ++r) held[r].push_back((uint32_t)r);
        for (uint64_t j = q; j < P && rc == TACO_OK; ++j) {  // fold the excess ranks into rank j - q
            rc = through_codec(data + j * padded, padded);
            held[j - q].push_back((uint32_t)j);
        }
        for (uint64_t h = q / 2, len = padded; h >= 1 && rc == TACO_OK; h /= 2, len /= 2) {
            const uint64_t half = len / 2;
            std::vector<std::vector<uint32_t>> next = held;
            for (uint64_t r = 0; r < q && rc == TACO_OK; ++r) {
                const uint64_t far = at[r] + ((r & h) ? 0 : half);
                for (uint32_t o : held[r]) {
                    if ((rc = through_codec(data + o * padded + far, half))) break;
                    next[r ^ h].push_back(o);
                }
            }
            for (uint64_t r = 0; r < q; ++r) at[r] += (r & h) ? half : 0;
            held.swap(next);
        }
        // every rank holds all P origins over slice r: one ascending-origin sum for all
        // slices at once, then every slice is compressed at its owner and decoded once
        if (rc == TACO_OK) rc = copy(result, data, padded);
        for (uint64_t o = 1; o < P && rc == TACO_OK; ++o) rc = add(result, data + o * padded, padded);
        const uint64_t ms = div_up(slice, cfg->block_size);
        const taco_layout sl = layout_of(payload_of(cfg), ms);
        if (rc == TACO_OK)
            rc = taco_compress_dev(cfg, result, TACO_DT_F32, padded, (uint32_t)q, 0, ms, msg, sl.msg_stride,
                                   ctx->d_flags, st);
        if (rc == TACO_OK)
            rc = taco_decompress_dev(cfg, msg, sl.msg_stride, (uint32_t)q, padded, 0, ms, result, TACO_DT_F32,
                                     ctx->d_flags, st);
    }
    if (rc != TACO_OK) {
        cudaStreamSynchronize(st);
        return rc;
    }
    TACO_CUDA(cudaMemcpyAsync(exact_host, exact, n * 4, cudaMemcpyDeviceToHost, st));
    TACO_CUDA(cudaMemcpyAsync(result_host, result, n * 4, cudaMemcpyDeviceToHost, st));
    TACO_CUDA(cudaStreamSynchronize(st));
    int flags = 0;
    TACO_CUDA(cudaMemcpy(&flags, ctx->d_flags, sizeof(int), cudaMemcpyDeviceToHost));
    if (int frc = taco_flags_status(flags)) return frc;
    if (rel_l2) {
        taco_error_report rep;
        uint64_t count = 0;
        if (int erc = taco_error_report_dev(exact, TACO_DT_F32, result, TACO_DT_F32, n, 1, &rep, &count, st))
            return erc;
        *rel_l2 = rep.relative_l2;
    }
    return TACO_OK;
}

}  // extern "C"

// ============================================================= diagnostics ====
// Element-wise access to the exact FP8 conversion instructions the kernels use
// (enc2 / dec2 in taco_device.cuh), so tests can prove them equal to the reference's
// fp8_encode / decode table (fp8.cpp:16-91) over every fp32 bit pattern.
namespace {
template <int FMT>
__global__ void k_fp8_encode(const float* __restrict__ x, uint64_t n, uint8_t* __restrict__ out) {
    const uint64_t i = 2 * ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x);
    if (i + 1 < n) {
        *reinterpret_cast<uint16_t*>(out + i) = (uint16_t)taco_dev::enc2<FMT>(make_float2(x[i], x[i + 1]));
    } else if (i < n) {
        out[i] = (uint8_t)taco_dev::enc2<FMT>(make_float2(x[i], 0.0f));
    }
}
template <int FMT>
__global__ void k_fp8_decode(const uint8_t* __restrict__ c, uint64_t n, float* __restrict__ out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        out[i] = taco_dev::dec2<FMT>(c[i]).x;
    }
}
}  // namespace

extern "C" int taco_fp8_encode_dev(const float* x, uint64_t n, int format, uint8_t* out, void* stream) {
    if (n == 0) return TACO_OK;
    const unsigned grid = (unsigned)div_up(div_up(n, 2), 256);
    if (format) k_fp8_encode<1><<<grid, 256, 0, (cudaStream_t)stream>>>(x, n, out);
    else k_fp8_encode<0><<<grid, 256, 0, (cudaStream_t)stream>>>(x, n, out);
    if (cudaError_t e = cudaGetLastError()) return cuda_fail(e, "fp8 encode launch");
    return TACO_OK;
}

extern "C" int taco_fp8_decode_dev(const uint8_t* codes, uint64_t n, int format, float* out, void* stream) {
    if (n == 0) return TACO_OK;
    const unsigned grid = (unsigned)div_up(n, 256);
    if (format) k_fp8_decode<1><<<grid, 256, 0, (cudaStream_t)stream>>>(codes, n, out);
    else k_fp8_decode<0><<<grid, 256, 0, (cudaStream_t)stream>>>(codes, n, out);
    if (cudaError_t e = cudaGetLastError()) return cuda_fail(e, "fp8 decode launch");
    return TACO_OK;
}
