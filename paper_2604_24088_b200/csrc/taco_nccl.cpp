// taco_nccl.cpp -- the compressed collectives over a caller's NCCL communicator, as C ABI
// (include/taco_b200.h, SURVEY §8b "taco_allreduce_twoshot(..., ncclComm_t, cudaStream_t)").
//
// The schedule is the reference's two-shot (proj/src/collective.cpp:75-111) across real
// ranks, the same one collective.py runs through torch.distributed:
//   K1 compress the P shards -> grouped ncclSend/ncclRecv (all-to-all of FP8 messages)
//   -> K3 decode + ascending-rank fp32 sum + re-encode -> ncclAllGather -> K2 decode.
// NCCL is resolved at run time (dlopen of the already-loaded libnccl.so.2, else the
// system one): the library never links NCCL, and the communicator a caller passes is
// always served by the NCCL instance that created it.
#include <dlfcn.h>
#include <nccl.h>

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "taco_b200.h"

namespace {

struct Nccl {
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    // NCCL >= 2.28: the native all-to-all (optional; grouped send/recv otherwise)
    ncclResult_t (*all_to_all)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*count)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*user_rank)(const ncclComm_t, int*) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    std::string load_error;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the caller's NCCL, if loaded
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            n.load_error = std::string("libnccl.so.2 not found: ") + dlerror();
            return;
        }
        auto sym = [&](const char* name) { return dlsym(h, name); };
        n.group_start = reinterpret_cast<decltype(n.group_start)>(sym("ncclGroupStart"));
        n.group_end = reinterpret_cast<decltype(n.group_end)>(sym("ncclGroupEnd"));
        n.send = reinterpret_cast<decltype(n.send)>(sym("ncclSend"));
        n.recv = reinterpret_cast<decltype(n.recv)>(sym("ncclRecv"));
        n.all_gather = reinterpret_cast<decltype(n.all_gather)>(sym("ncclAllGather"));
        n.all_to_all = reinterpret_cast<decltype(n.all_to_all)>(sym("ncclAlltoAll"));
        if (const char* v = std::getenv("TACO_NCCL_ALLTOALL"); v && std::strcmp(v, "0") == 0) n.all_to_all = nullptr;
        n.count = reinterpret_cast<decltype(n.count)>(sym("ncclCommCount"));
        n.user_rank = reinterpret_cast<decltype(n.user_rank)>(sym("ncclCommUserRank"));
        n.error_string = reinterpret_cast<decltype(n.error_string)>(sym("ncclGetErrorString"));
        if (!n.group_start || !n.group_end || !n.send || !n.recv || !n.all_gather || !n.count || !n.user_rank ||
            !n.error_string)
            n.load_error = "libnccl.so.2 lacks the point-to-point / all-gather API (NCCL >= 2.7 needed)";
    });
    return n;
}

}  // namespace

namespace taco_impl {
int set_error(int code, const char* msg);  // taco_abi.cu: the message taco_last_error() returns
}

namespace {

int nfail(int code, const std::string& msg) { return taco_impl::set_error(code, msg.c_str()); }

uint64_t div_up(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

constexpr uint32_t kMaxChunks = 16;
constexpr uint32_t kDefaultChunks = 2;  // collective.py / bench.py default: two chunks per shard

struct Geo {
    int P = 0, rank = 0;
    taco_layout lay{};
};

// ranks of the communicator (the shard count) + config checks
int comm_geo(const taco_config* cfg, void* comm, Geo& g) {
    const Nccl& n = nccl();
    if (!n.load_error.empty()) return nfail(TACO_ERR_USAGE, n.load_error);
    if (!comm) return nfail(TACO_ERR_USAGE, "null NCCL communicator");
    if (int rc = taco_validate_config(cfg)) return rc;
    if (cfg->kind != 0) return nfail(TACO_ERR_USAGE, "the NCCL collectives serve CodecKind::Taco");
    ncclResult_t r = n.count(static_cast<ncclComm_t>(comm), &g.P);
    if (r == ncclSuccess) r = n.user_rank(static_cast<ncclComm_t>(comm), &g.rank);
    if (r != ncclSuccess) return nfail(TACO_ERR_CUDA, std::string("NCCL: ") + n.error_string(r));
    return TACO_OK;
}

int nccl_check(ncclResult_t r) {
    if (r == ncclSuccess) return TACO_OK;
    return nfail(TACO_ERR_CUDA, std::string("NCCL: ") + nccl().error_string(r));
}

// all-to-all of P messages of `bytes` each (send[r] -> rank r, recv[r] <- rank r)
int all_to_all(const uint8_t* send, uint8_t* recv, uint64_t stride, uint64_t bytes, const Geo& g, void* comm,
               void* stream) {
    const Nccl& n = nccl();
    auto c = static_cast<ncclComm_t>(comm);
    auto st = static_cast<cudaStream_t>(stream);
    if (n.all_to_all && bytes == stride)  // dense [P][stride] buffers: the native collective
        return nccl_check(n.all_to_all(send, recv, bytes, ncclUint8, c, st));
    if (int rc = nccl_check(n.group_start())) return rc;
    for (int r = 0; r < g.P; ++r) {
        if (int rc = nccl_check(n.send(send + r * stride, bytes, ncclUint8, r, c, st))) return rc;
        if (int rc = nccl_check(n.recv(recv + r * stride, bytes, ncclUint8, r, c, st))) return rc;
    }
    return nccl_check(n.group_end());
}

// Block-aligned chunks of every shard (blocks never span chunks, so numerics are unchanged,
// test_collective.cpp:225-238) -- the same split as collective.py's _Chunking.
struct Chunks {
    int count = 0;
    uint64_t b0[kMaxChunks] = {}, b1[kMaxChunks] = {};
    taco_layout lay[kMaxChunks] = {};
    uint64_t bytes_per_rank_slot = 0;  // sum of the chunk strides
};

int make_chunks(const taco_config* cfg, uint64_t m, uint32_t chunks, Chunks& ch) {
    if (chunks == 0) chunks = kDefaultChunks;
    if (chunks > kMaxChunks) return nfail(TACO_ERR_USAGE, "at most 16 pipelined chunks");
    const uint64_t c = std::max<uint64_t>(1, std::min<uint64_t>(chunks, m));
    const uint64_t per = div_up(m, c);
    ch = Chunks{};
    for (uint64_t b = 0; b < m; b += per) {
        const int k = ch.count++;
        ch.b0[k] = b;
        ch.b1[k] = std::min(m, b + per);
        if (int rc = taco_msg_layout(cfg, ch.b1[k] - ch.b0[k], &ch.lay[k])) return rc;
        ch.bytes_per_rank_slot += ch.lay[k].msg_stride;
    }
    return TACO_OK;
}

// The communication side stream of a device and a pool of ordering events.  The codec
// kernels stay on the caller's stream; every NCCL call goes to this stream, fenced by
// events both ways, so chunk c's transfer overlaps chunk c +- 1's kernels.  Under CUDA-graph
// capture of the caller's stream the event waits fork this stream into the capture and the
// final wait joins it back.
struct CommLane {
    std::mutex mu;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[4 * kMaxChunks] = {};
    int ready = 0;  // 1 ok, -1 failed
};

CommLane* comm_lane(int device) {
    static std::mutex mu;
    static CommLane* lanes[64] = {};
    if (device < 0 || device >= 64) return nullptr;
    std::lock_guard<std::mutex> lock(mu);
    CommLane*& l = lanes[device];
    if (!l) {
        l = new CommLane();
        bool ok = cudaStreamCreateWithFlags(&l->stream, cudaStreamNonBlocking) == cudaSuccess;
        for (auto& e : l->ev) ok = ok && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
        l->ready = ok ? 1 : -1;
    }
    return l->ready == 1 ? l : nullptr;
}

int cuda_check(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return TACO_OK;
    return nfail(TACO_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// `from` -> `to` ordering through event k
int order(cudaStream_t from, cudaStream_t to, cudaEvent_t ev) {
    if (int rc = cuda_check(cudaEventRecord(ev, from), "event record")) return rc;
    return cuda_check(cudaStreamWaitEvent(to, ev, 0), "stream wait");
}

struct Lane {
    CommLane* l = nullptr;
    std::unique_lock<std::mutex> lock;
    int open() {
        int dev = 0;
        if (int rc = cuda_check(cudaGetDevice(&dev), "current device")) return rc;
        l = comm_lane(dev);
        if (!l) return nfail(TACO_ERR_CUDA, "communication stream creation failed");
        lock = std::unique_lock<std::mutex>(l->mu);
        return TACO_OK;
    }
};

}  // namespace

extern "C" {

uint64_t taco_collective_nccl_workspace_chunked(const taco_config* cfg, uint32_t nranks, uint64_t n,
                                                uint32_t chunks) {
    if (!cfg || nranks == 0 || n == 0 || cfg->block_size == 0 || chunks > kMaxChunks) return 0;
    Chunks ch;
    if (make_chunks(cfg, div_up(div_up(n, nranks), cfg->block_size), chunks, ch)) return 0;
    return (3ull * nranks + 1) * ch.bytes_per_rank_slot;  // send, recv, gath [P][msg] + red [msg] per chunk
}

uint64_t taco_collective_nccl_workspace(const taco_config* cfg, uint32_t nranks, uint64_t n) {
    return taco_collective_nccl_workspace_chunked(cfg, nranks, n, kDefaultChunks);
}

int taco_allreduce_nccl_chunked(const taco_config* cfg, const void* x, int dtype, uint64_t n, void* out,
                                int out_dtype, void* work, void* comm, int* d_flags, void* stream, uint32_t chunks) {
    if (n == 0) return nfail(TACO_ERR_INPUT, "input tensor is empty");
    Geo g;  // P is the communicator's size: query it first, then size the shards
    if (int rc = comm_geo(cfg, comm, g)) return rc;
    const uint64_t P = (uint64_t)g.P, S = div_up(n, P), m = div_up(S, cfg->block_size);
    Chunks ch;
    if (int rc = make_chunks(cfg, m, chunks, ch)) return rc;
    if (!work) return nfail(TACO_ERR_USAGE, "workspace required (taco_collective_nccl_workspace bytes)");
    Lane lane;
    if (int rc = lane.open()) return rc;
    cudaStream_t cs = static_cast<cudaStream_t>(stream), ns = lane.l->stream;
    cudaEvent_t* ev = lane.l->ev;
    // per chunk: send [P][st], recv [P][st], gath [P][st], red [st]
    uint8_t *send[kMaxChunks], *recv[kMaxChunks], *gath[kMaxChunks], *red[kMaxChunks];
    uint8_t* at = static_cast<uint8_t*>(work);
    for (int c = 0; c < ch.count; ++c) {
        const uint64_t st = ch.lay[c].msg_stride;
        send[c] = at, recv[c] = at + P * st, gath[c] = at + 2 * P * st, red[c] = at + 3 * P * st;
        at += (3 * P + 1) * st;
    }
    auto nc = static_cast<ncclComm_t>(comm);
    // phase 1: K1 of every chunk, its all-to-all in flight on the comm lane
    for (int c = 0; c < ch.count; ++c) {
        const uint64_t st = ch.lay[c].msg_stride;
        if (int rc = taco_compress_dev(cfg, x, dtype, n, g.P, ch.b0[c], ch.b1[c], send[c], st, d_flags, stream))
            return rc;
        if (int rc = order(cs, ns, ev[c])) return rc;
        if (int rc = all_to_all(send[c], recv[c], st, st, g, comm, ns)) return rc;
    }
    // owner reduce + re-encode as each chunk lands, the all-gather in flight
    for (int c = 0; c < ch.count; ++c) {
        const uint64_t st = ch.lay[c].msg_stride;
        if (int rc = order(ns, cs, ev[kMaxChunks + c])) return rc;
        if (int rc = taco_reduce_encode_dev(cfg, recv[c], st, g.P, S, ch.b0[c], ch.b1[c], red[c], nullptr, 0,
                                            d_flags, stream))
            return rc;
        if (int rc = order(cs, ns, ev[2 * kMaxChunks + c])) return rc;
        if (int rc = nccl_check(nccl().all_gather(red[c], gath[c], st, ncclUint8, nc, ns))) return rc;
    }
    for (int c = 0; c < ch.count; ++c) {
        if (int rc = order(ns, cs, ev[3 * kMaxChunks + c])) return rc;
        if (int rc = taco_decompress_dev(cfg, gath[c], ch.lay[c].msg_stride, g.P, n, ch.b0[c], ch.b1[c], out,
                                         out_dtype, d_flags, stream))
            return rc;
    }
    return TACO_OK;
}

int taco_allreduce_nccl(const taco_config* cfg, const void* x, int dtype, uint64_t n, void* out, int out_dtype,
                        void* work, void* comm, int* d_flags, void* stream) {
    return taco_allreduce_nccl_chunked(cfg, x, dtype, n, out, out_dtype, work, comm, d_flags, stream,
                                       kDefaultChunks);
}

int taco_reduce_scatter_nccl_chunked(const taco_config* cfg, const void* x, int dtype, uint64_t n, void* out,
                                     int out_dtype, void* work, void* comm, int* d_flags, void* stream,
                                     uint32_t chunks) {
    if (n == 0) return nfail(TACO_ERR_INPUT, "input tensor is empty");
    Geo g;
    if (int rc = comm_geo(cfg, comm, g)) return rc;
    const uint64_t P = (uint64_t)g.P, S = div_up(n, P), m = div_up(S, cfg->block_size);
    Chunks ch;
    if (int rc = make_chunks(cfg, m, chunks, ch)) return rc;
    if (!work) return nfail(TACO_ERR_USAGE, "workspace required (taco_collective_nccl_workspace bytes)");
    Lane lane;
    if (int rc = lane.open()) return rc;
    cudaStream_t cs = static_cast<cudaStream_t>(stream), ns = lane.l->stream;
    cudaEvent_t* ev = lane.l->ev;
    uint8_t *send[kMaxChunks], *recv[kMaxChunks];
    uint8_t* at = static_cast<uint8_t*>(work);
    for (int c = 0; c < ch.count; ++c) {
        const uint64_t st = ch.lay[c].msg_stride;
        send[c] = at, recv[c] = at + P * st;
        at += 2 * P * st;
    }
    for (int c = 0; c < ch.count; ++c) {
        const uint64_t st = ch.lay[c].msg_stride;
        if (int rc = taco_compress_dev(cfg, x, dtype, n, g.P, ch.b0[c], ch.b1[c], send[c], st, d_flags, stream))
            return rc;
        if (int rc = order(cs, ns, ev[c])) return rc;
        if (int rc = all_to_all(send[c], recv[c], st, st, g, comm, ns)) return rc;
    }
    for (int c = 0; c < ch.count; ++c) {
        if (int rc = order(ns, cs, ev[kMaxChunks + c])) return rc;
        if (int rc = taco_reduce_encode_dev(cfg, recv[c], ch.lay[c].msg_stride, g.P, S, ch.b0[c], ch.b1[c], nullptr,
                                            out, out_dtype, d_flags, stream))
            return rc;
    }
    return TACO_OK;
}

int taco_reduce_scatter_nccl(const taco_config* cfg, const void* x, int dtype, uint64_t n, void* out,
                             int out_dtype, void* work, void* comm, int* d_flags, void* stream) {
    return taco_reduce_scatter_nccl_chunked(cfg, x, dtype, n, out, out_dtype, work, comm, d_flags, stream,
                                            kDefaultChunks);
}

int taco_all_gather_nccl_chunked(const taco_config* cfg, const void* x, int dtype, uint64_t n_local, void* out,
                                 int out_dtype, void* work, void* comm, int* d_flags, void* stream,
                                 uint32_t chunks) {
    if (n_local == 0) return nfail(TACO_ERR_INPUT, "input tensor is empty");
    Geo g;
    if (int rc = comm_geo(cfg, comm, g)) return rc;
    const uint64_t P = (uint64_t)g.P, m = div_up(n_local, cfg->block_size);
    Chunks ch;
    if (int rc = make_chunks(cfg, m, chunks, ch)) return rc;
    if (!work) return nfail(TACO_ERR_USAGE, "workspace required (taco_collective_nccl_workspace bytes)");
    Lane lane;
    if (int rc = lane.open()) return rc;
    cudaStream_t cs = static_cast<cudaStream_t>(stream), ns = lane.l->stream;
    cudaEvent_t* ev = lane.l->ev;
    uint8_t *mine[kMaxChunks], *gath[kMaxChunks];
    uint8_t* at = static_cast<uint8_t*>(work);
    for (int c = 0; c < ch.count; ++c) {
        const uint64_t st = ch.lay[c].msg_stride;
        mine[c] = at, gath[c] = at + st;
        at += (P + 1) * st;
    }
    auto nc = static_cast<ncclComm_t>(comm);
    for (int c = 0; c < ch.count; ++c) {
        const uint64_t st = ch.lay[c].msg_stride;
        if (int rc = taco_compress_dev(cfg, x, dtype, n_local, 1, ch.b0[c], ch.b1[c], mine[c], st, d_flags, stream))
            return rc;
        if (int rc = order(cs, ns, ev[c])) return rc;
        if (int rc = nccl_check(nccl().all_gather(mine[c], gath[c], st, ncclUint8, nc, ns))) return rc;
    }
    for (int c = 0; c < ch.count; ++c) {
        if (int rc = order(ns, cs, ev[kMaxChunks + c])) return rc;
        // the gathered tensor is P shards of n_local: shard geometry S = n_local exactly
        if (int rc = taco_decompress_dev(cfg, gath[c], ch.lay[c].msg_stride, g.P, P * n_local, ch.b0[c], ch.b1[c],
                                         out, out_dtype, d_flags, stream))
            return rc;
    }
    return TACO_OK;
}

int taco_all_gather_nccl(const taco_config* cfg, const void* x, int dtype, uint64_t n_local, void* out,
                         int out_dtype, void* work, void* comm, int* d_flags, void* stream) {
    return taco_all_gather_nccl_chunked(cfg, x, dtype, n_local, out, out_dtype, work, comm, d_flags, stream,
                                        kDefaultChunks);
}

}  // extern "C"
