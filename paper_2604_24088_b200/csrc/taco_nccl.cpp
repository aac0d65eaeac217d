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

#include <cstdint>
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
    if (int rc = nccl_check(n.group_start())) return rc;
    for (int r = 0; r < g.P; ++r) {
        if (int rc = nccl_check(n.send(send + r * stride, bytes, ncclUint8, r, c, st))) return rc;
        if (int rc = nccl_check(n.recv(recv + r * stride, bytes, ncclUint8, r, c, st))) return rc;
    }
    return nccl_check(n.group_end());
}

}  // namespace

extern "C" {

uint64_t taco_collective_nccl_workspace(const taco_config* cfg, uint32_t nranks, uint64_t n) {
    if (!cfg || nranks == 0 || n == 0 || cfg->block_size == 0) return 0;
    taco_layout lay{};
    if (taco_msg_layout(cfg, div_up(div_up(n, nranks), cfg->block_size), &lay)) return 0;
    return (3ull * nranks + 1) * lay.msg_stride;  // send, recv, gath [P][msg] + red [msg]
}

int taco_allreduce_nccl(const taco_config* cfg, const void* x, int dtype, uint64_t n, void* out, int out_dtype,
                        void* work, void* comm, int* d_flags, void* stream) {
    if (n == 0) return nfail(TACO_ERR_INPUT, "input tensor is empty");
    Geo g;  // P is the communicator's size: query it first, then size the shards
    if (int rc = comm_geo(cfg, comm, g)) return rc;
    const uint64_t S = div_up(n, (uint64_t)g.P), m = div_up(S, cfg->block_size);
    if (int rc = taco_msg_layout(cfg, m, &g.lay)) return rc;
    const uint64_t st = g.lay.msg_stride, P = (uint64_t)g.P;
    if (!work) return nfail(TACO_ERR_USAGE, "workspace required (taco_collective_nccl_workspace bytes)");
    uint8_t* send = static_cast<uint8_t*>(work);
    uint8_t* recv = send + P * st;
    uint8_t* gath = recv + P * st;
    uint8_t* red = gath + P * st;
    if (int rc = taco_compress_dev(cfg, x, dtype, n, g.P, 0, m, send, st, d_flags, stream)) return rc;
    if (int rc = all_to_all(send, recv, st, st, g, comm, stream)) return rc;
    if (int rc = taco_reduce_encode_dev(cfg, recv, st, g.P, S, 0, m, red, nullptr, 0, d_flags, stream)) return rc;
    if (int rc = nccl_check(nccl().all_gather(red, gath, st, ncclUint8, static_cast<ncclComm_t>(comm),
                                              static_cast<cudaStream_t>(stream))))
        return rc;
    return taco_decompress_dev(cfg, gath, st, g.P, n, 0, m, out, out_dtype, d_flags, stream);
}

int taco_reduce_scatter_nccl(const taco_config* cfg, const void* x, int dtype, uint64_t n, void* out,
                             int out_dtype, void* work, void* comm, int* d_flags, void* stream) {
    if (n == 0) return nfail(TACO_ERR_INPUT, "input tensor is empty");
    Geo g;
    if (int rc = comm_geo(cfg, comm, g)) return rc;
    const uint64_t S = div_up(n, (uint64_t)g.P), m = div_up(S, cfg->block_size);
    if (int rc = taco_msg_layout(cfg, m, &g.lay)) return rc;
    const uint64_t st = g.lay.msg_stride, P = (uint64_t)g.P;
    if (!work) return nfail(TACO_ERR_USAGE, "workspace required (taco_collective_nccl_workspace bytes)");
    uint8_t* send = static_cast<uint8_t*>(work);
    uint8_t* recv = send + P * st;
    if (int rc = taco_compress_dev(cfg, x, dtype, n, g.P, 0, m, send, st, d_flags, stream)) return rc;
    if (int rc = all_to_all(send, recv, st, st, g, comm, stream)) return rc;
    return taco_reduce_encode_dev(cfg, recv, st, g.P, S, 0, m, nullptr, out, out_dtype, d_flags, stream);
}

int taco_all_gather_nccl(const taco_config* cfg, const void* x, int dtype, uint64_t n_local, void* out,
                         int out_dtype, void* work, void* comm, int* d_flags, void* stream) {
    if (n_local == 0) return nfail(TACO_ERR_INPUT, "input tensor is empty");
    Geo g;
    if (int rc = comm_geo(cfg, comm, g)) return rc;
    const uint64_t m = div_up(n_local, cfg->block_size);
    if (int rc = taco_msg_layout(cfg, m, &g.lay)) return rc;
    const uint64_t st = g.lay.msg_stride;
    if (!work) return nfail(TACO_ERR_USAGE, "workspace required (taco_collective_nccl_workspace bytes)");
    uint8_t* mine = static_cast<uint8_t*>(work);
    uint8_t* gath = mine + st;
    if (int rc = taco_compress_dev(cfg, x, dtype, n_local, 1, 0, m, mine, st, d_flags, stream)) return rc;
    if (int rc = nccl_check(nccl().all_gather(mine, gath, st, ncclUint8, static_cast<ncclComm_t>(comm),
                                              static_cast<cudaStream_t>(stream))))
        return rc;
    return taco_decompress_dev(cfg, gath, st, g.P, (uint64_t)g.P * n_local, 0, m, out, out_dtype, d_flags, stream);
}

}  // extern "C"
