/*
 * taco_b200.h -- C ABI of the B200-native TACO compression path (sm_100a).
 *
 * The reference (arxiv/paper_2604_24088, /root/reference/proj) exposes the codec as a
 * C++ header API over host spans; this ABI is what sits underneath the drop-in
 * C++ layer (include/taco/{codec,fp8,...}.hpp, csrc/taco_cxx.cpp) and what
 * non-C++ callers (ctypes, the NCCL collective driver) bind directly.  Each entry
 * point names the reference interface it replaces.
 *
 * Conventions
 *  - Plain pointers and sizes only; no torch / CUDA types in signatures
 *    (streams are passed as `void*` = cudaStream_t, NULL = legacy default stream).
 *  - The device entry points never allocate and never synchronise: every buffer is
 *    caller-owned device memory, work is enqueued on `stream`.
 *  - Every function returns a taco_status; on error taco_last_error() holds the
 *    reference's exact message (proj/include/taco/error.hpp:10-40 codes + 1).
 *  - Data-dependent errors found by kernels (NaN/Inf input, bad block scalars) are
 *    OR-ed into a caller-owned device int `d_flags` (may be NULL) and turned into
 *    the reference's errors by taco_flags_status() once the stream is synchronised.
 *
 * Wire message layout (one per shard, or per shard-chunk), replacing the
 * reference's AoS CompressedTensor (codec.hpp:37-49) / TACOCMP1 blocks
 * (serialize.hpp:12-14) with an SoA that vector loads/stores can stream:
 *      [ codes: nblocks*B bytes ][ pad to 16 ][ (alpha, scale) f32 pairs: nblocks*8 bytes ]
 * msg_bytes = scal_offset + 8*nblocks (== nblocks*(B+8) whenever B >= 16, i.e. the
 * reference's per-block wire cost, collective.cpp:50-58 minus the 22-byte archive
 * header); msg_stride = msg_bytes rounded up to 16.
 * Alignment rule: the kernels move messages with 16-byte vector / TMA accesses, so every
 * message buffer passed to the device API must be 16-byte aligned and, when it holds more
 * than one message, its stride a multiple of 16 (use taco_layout.msg_stride); otherwise
 * the call returns TACO_ERR_USAGE before any launch.
 */
#ifndef TACO_B200_H
#define TACO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TACO_B200_ABI_VERSION 3

typedef enum {
    TACO_OK = 0,
    TACO_ERR_USAGE = 1,   /* taco::ErrorCode::Usage   */
    TACO_ERR_CONFIG = 2,  /* taco::ErrorCode::Config  */
    TACO_ERR_INPUT = 3,   /* taco::ErrorCode::Input   */
    TACO_ERR_IO = 4,      /* taco::ErrorCode::Io      */
    TACO_ERR_CORRUPT = 5, /* taco::ErrorCode::Corrupt */
    TACO_ERR_CUDA = 6     /* launch / runtime failure (no reference counterpart) */
} taco_status;

typedef enum { TACO_DT_F32 = 0, TACO_DT_BF16 = 1 } taco_dtype;

/* d_flags bits */
#define TACO_FLAG_NONFINITE_INPUT 1 /* -> Input,   "input tensor contains NaN or Inf"         */
#define TACO_FLAG_BAD_SCALARS 2     /* -> Corrupt, "block scalars must be finite and nonzero" */
#define TACO_FLAG_PEER_TIMEOUT 4    /* -> Cuda,    "peer barrier timed out" (no counterpart)  */

/* taco::CodecConfig (codec.hpp:24-33).
 * kind (codec.hpp:11-17): 0 = Taco (the fused sm_100a hot path), 1 = DirectFp8,
 *   2 = Int8Uniform, 3 = Identity (payload = 4B raw bytes per block), 4 = AshInt8;
 * format: 0 = E4M3, 1 = E5M2 (fp8.hpp:8);
 * direct_scale (codec.hpp:22, DirectFp8 only): 0 = GlobalMax, 1 = Unit, 2 = PerBlockMax.
 * GlobalMax and Int8Uniform derive one scale per shard (the reference compresses each
 * shard slice separately, collective.cpp:82-88). */
typedef struct {
    uint32_t block_size;
    float target_energy;
    float stability_epsilon;
    uint32_t format;
    uint32_t kind;
    uint32_t direct_scale;
} taco_config;

typedef struct {
    uint64_t nblocks;
    uint64_t codes_bytes; /* nblocks * payload (B, or 4B for Identity) */
    uint64_t scal_offset; /* codes_bytes rounded up to 16 */
    uint64_t msg_bytes;   /* scal_offset + 8 * nblocks */
    uint64_t msg_stride;  /* msg_bytes rounded up to 16 */
} taco_layout;

int taco_abi_version(void);
const char* taco_last_error(void);
/* thread-safe defaults: B=256, tau=1, eps=1e-12, E4M3, Taco (codec.hpp:24-33) */
taco_config taco_default_config(void);

/* taco::validate_config (codec.hpp:35; codec.cpp:189-197, transform.cpp:13-20) */
int taco_validate_config(const taco_config* cfg);

/* message geometry for `nblocks` blocks */
int taco_msg_layout(const taco_config* cfg, uint64_t nblocks, taco_layout* out);

/* ratio of the reference's wire layout, taco::compressed_ratio (codec.hpp:66) */
double taco_compressed_ratio(const taco_config* cfg, uint64_t n);

/* taco::archive_size_bytes (serialize.hpp:24): 22 + ceil(n/B)*(payload+8) */
uint64_t taco_archive_size(const taco_config* cfg, uint64_t n);

/* Map the device flags word to the reference's error (TACO_OK if 0). */
int taco_flags_status(int flags);

/* ---------------------------------------------------------------- device API -------
 * Shard geometry shared by the three kernels.  A logical input of n elements is cut
 * into `shards` contiguous shards of S = ceil(n/shards) elements, zero-padded past n
 * (collective.cpp:76-87); shard p is cut into ceil(S/B) blocks, zero-padded past S
 * (codec.cpp:20-28).  [blk_begin, blk_end) selects a chunk of blocks of every shard
 * (block-aligned chunking never changes numerics, test_collective.cpp:225-238).
 * shards == 1 is the plain taco::compress / taco::decompress of one tensor.
 */

/* K1 -- fused ASH transform + dual-scale FP8 encode.  Replaces taco::compress
 * (codec.hpp:57; codec.cpp:208-254 + rotate_block :45-62 + compress_block_taco
 * :64-76).  Message for shard p goes to msgs + p*msg_stride. */
int taco_compress_dev(const taco_config* cfg, const void* x, int dtype, uint64_t n,
                      uint32_t shards, uint64_t blk_begin, uint64_t blk_end, void* msgs,
                      uint64_t msg_stride, int* d_flags, void* stream);

/* K2 -- fused dequantise + inverse Hadamard + 1/alpha.  Replaces taco::decompress
 * (codec.hpp:61-62; codec.cpp:264-296 + decompress_block :144-155).  Writes only
 * the valid prefix of every shard (codec.cpp:151-153, collective.cpp:109). */
int taco_decompress_dev(const taco_config* cfg, const void* msgs, uint64_t msg_stride,
                        uint32_t shards, uint64_t n, uint64_t blk_begin, uint64_t blk_end,
                        void* out, int out_dtype, int* d_flags, void* stream);

/* K3 -- fused decode of `nranks` messages of one shard, fp32 sum in ascending rank
 * order, re-encode.  Replaces the owner loop of run_twoshot (collective.cpp:95-101):
 * acc = dec(msg 0); acc += dec(msg r) for r = 1..P-1; compress(acc).
 * Message r is read from msgs + r*rank_stride.  `shard_len` = S (positions >= S in
 * the last block are re-zeroed before re-encoding).  acc_out (optional, may be NULL)
 * receives the fp32 stage-1 sum for positions < S of the chunk (the SP reduce-scatter
 * output and the stage-isolated parity hook), in acc_dtype.  out_msg may be NULL
 * (reduce-scatter: no re-encode); at least one of out_msg / acc_out must be given. */
int taco_reduce_encode_dev(const taco_config* cfg, const void* msgs, uint64_t rank_stride,
                           uint32_t nranks, uint64_t shard_len, uint64_t blk_begin,
                           uint64_t blk_end, void* out_msg, void* acc_out, int acc_dtype,
                           int* d_flags, void* stream);

/* K3 with the P rank messages at arbitrary device addresses (SURVEY §8b
 * taco_decode_reduce_encode(const uint8_t* const* in, int P, ...)): msgs is a HOST array of
 * nranks (<= TACO_MAX_PEERS) device pointers, each a message of blk_end - blk_begin blocks
 * (e.g. the peers' send buffers mapped over NVLink: a pull-style owner reduction).  Same
 * results as taco_reduce_encode_dev on the same bytes.  B <= 1024. */
int taco_reduce_encode_ptrs_dev(const taco_config* cfg, const void* const* msgs, uint32_t nranks,
                                uint64_t shard_len, uint64_t blk_begin, uint64_t blk_end, void* out_msg,
                                void* acc_out, int acc_dtype, int* d_flags, void* stream);

/* In-process P-rank two-shot all-reduce on ONE device: the reference's RankSet
 * simulation (taco::allreduce, collective.hpp:28, Algorithm::TwoShot,
 * collective.cpp:75-111) with every "rank" a slice of `inputs` ([P][n], dtype).
 * `work` must hold taco_allreduce_sim_workspace() bytes.  out: n elements in
 * out_dtype (identical on every rank, so written once).  stage1 (optional): P*S fp32. */
uint64_t taco_allreduce_sim_workspace(const taco_config* cfg, uint32_t nranks, uint64_t n);
int taco_allreduce_sim_dev(const taco_config* cfg, const void* inputs, int dtype,
                           uint32_t nranks, uint64_t n, void* out, int out_dtype, float* stage1,
                           void* work, int* d_flags, void* stream);

/* taco::scaled_spectrum (codec.hpp:70; codec.cpp:306-326): Z/s of every block slot of
 * the Taco (q_top = q_max) or AshInt8 (q_top = 127) rotation, ceil(n/B)*B fp32 values. */
int taco_scaled_spectrum_dev(const taco_config* cfg, const void* x, int dtype, uint64_t n,
                             float* out, int* d_flags, void* stream);

/* --------------------------------------------- collectives over a caller's NCCL communicator ---
 * The two-shot across real ranks (collective.cpp:75-111; SURVEY §8b taco_allreduce_twoshot),
 * one rank per GPU: K1 -> grouped ncclSend/ncclRecv (all-to-all of the FP8 messages) -> K3
 * -> ncclAllGather -> K2.  `comm` is an ncclComm_t of P ranks (P = the shard count); NCCL is
 * resolved at run time from the process (the library does not link it).
 * Overlap: every shard is cut into `chunks` block-aligned chunks
 * (numerics unchanged, test_collective.cpp:225-238; 0 = the default, 2; at most 16).  The codec
 * kernels run on `stream`; the NCCL calls run on the library's communication stream of the
 * device, ordered against `stream` by events both ways, so chunk c's transfer overlaps chunk
 * c +- 1's kernels.  The call is CUDA-graph capturable (the communication stream is forked into
 * and joined back from the capture).  The unsuffixed entry points use the default chunking.
 * work: taco_collective_nccl_workspace[_chunked](cfg, P, n_total[, chunks]) bytes of device
 * memory, n_total = the full tensor (all-gather: P * n_local), for the same chunk count. */
uint64_t taco_collective_nccl_workspace(const taco_config* cfg, uint32_t nranks, uint64_t n_total);
uint64_t taco_collective_nccl_workspace_chunked(const taco_config* cfg, uint32_t nranks, uint64_t n_total,
                                                uint32_t chunks);
/* all-reduce: x[n] (dtype) -> out[n] (out_dtype), identical on every rank */
int taco_allreduce_nccl(const taco_config* cfg, const void* x, int dtype, uint64_t n, void* out, int out_dtype,
                        void* work, void* comm, int* d_flags, void* stream);
int taco_allreduce_nccl_chunked(const taco_config* cfg, const void* x, int dtype, uint64_t n, void* out,
                                int out_dtype, void* work, void* comm, int* d_flags, void* stream, uint32_t chunks);
/* sequence-parallel reduce-scatter: x[n] -> this rank's shard out[ceil(n/P)], the ascending-
 * rank fp32 sum of the decoded shard copies (collective.cpp:95-100), in out_dtype */
int taco_reduce_scatter_nccl(const taco_config* cfg, const void* x, int dtype, uint64_t n, void* out,
                             int out_dtype, void* work, void* comm, int* d_flags, void* stream);
int taco_reduce_scatter_nccl_chunked(const taco_config* cfg, const void* x, int dtype, uint64_t n, void* out,
                                     int out_dtype, void* work, void* comm, int* d_flags, void* stream,
                                     uint32_t chunks);
/* sequence-parallel all-gather: x[n_local] -> out[P * n_local] (every rank's slice decoded) */
int taco_all_gather_nccl(const taco_config* cfg, const void* x, int dtype, uint64_t n_local, void* out,
                         int out_dtype, void* work, void* comm, int* d_flags, void* stream);
int taco_all_gather_nccl_chunked(const taco_config* cfg, const void* x, int dtype, uint64_t n_local, void* out,
                                 int out_dtype, void* work, void* comm, int* d_flags, void* stream,
                                 uint32_t chunks);

/* ------------------------------------ peer-memory two-shot (SURVEY §8e, B200 extras) -----
 * The two-shot of collective.cpp:75-111 with the exchange folded into the kernels, no
 * NCCL call on the data path: K1 stores shard p's message straight into rank p's
 * receive slot, K3 stores its re-encoded shard into every rank's gather slot (NVLink
 * stores into CUDA-IPC mapped peer memory, then a system-scope fence), and a device
 * barrier (system-scope release/acquire flags) separates the phases.  Each rank owns
 * one region from taco_peer_alloc; the others map it with taco_peer_open on the
 * exported handle.  taco_peers.base[q] = rank q's region as mapped in this process. */
#define TACO_MAX_PEERS 8
typedef struct {
    unsigned char bytes[64]; /* cudaIpcMemHandle_t */
} taco_ipc_handle;
typedef struct {
    uint32_t nranks, rank;
    void* base[TACO_MAX_PEERS];
} taco_peers;

/* device memory on `device` (zeroed, synchronously) that peers can map; *handle exports it */
int taco_peer_alloc(int device, uint64_t bytes, void** ptr, taco_ipc_handle* handle);
/* map a peer's exported region into this process (on `device`, this rank's GPU) */
int taco_peer_open(int device, const taco_ipc_handle* handle, void** ptr);
int taco_peer_close(void* ptr);
/* TACO_OK when `device` can map memory of `peer_device` (cudaDeviceCanAccessPeer; the same
 * device always can); else TACO_ERR_USAGE naming both.  The opened mappings enable peer
 * access lazily (cudaIpcMemLazyEnablePeerAccess). */
int taco_peer_check_access(int device, int peer_device);
int taco_peer_free(void* ptr);
/* bytes of the barrier state at flags_offset: P arrival slots + this rank's epoch */
uint64_t taco_peer_flags_bytes(void);

/* Device barrier over the ranks of `peers`.  Bumps this rank's epoch (a counter in its
 * own region, so CUDA-graph replays keep counting), stores it into slot `rank` of every
 * rank's flag array (base[q] + flags_offset) with release semantics at system scope,
 * then waits until every slot of its own array has reached it.  Gives up after
 * timeout_ms, setting TACO_FLAG_PEER_TIMEOUT in d_flags (a dead peer never hangs). */
int taco_peer_barrier_dev(const taco_peers* peers, uint64_t flags_offset, uint32_t timeout_ms, int* d_flags,
                          void* stream);

/* Fused peer collectives: the phases are signalled by the codec kernels themselves, no
 * barrier kernels (all-reduce: 3 launches K1 -> K3 -> K2; reduce-scatter K1 -> K3 and
 * all-gather K1 -> K2: 2).  K1's last CTA fences (fence.sc.sys after every CTA's GPU-scope
 * release), opens the call's epoch, releases it into every peer's phase-A word
 * (st.release.sys) and waits (ld.acquire.sys) for every peer's: K1 completes only when every
 * rank's pushes have landed, so K3 runs unmodified.  In the all-reduce, K2's CTA 0 publishes
 * phase B (this rank's K3 is done) and every K2 CTA waits for all peers' before decoding;
 * the reduce-scatter / all-gather K1 starts with phase B instead (the previous call's K3 / K2
 * is done with the slots).  Slot reuse is therefore safe across calls and CUDA-graph replays.
 * Region per rank: receive slots at recv_offset and gather slots at gath_offset (P x
 * slot_stride each; slot [rank] is written by that rank only), the sync words at flags_offset
 * (taco_peer_flags_bytes(); regions zeroed by taco_peer_alloc).  Do not mix fused calls and
 * taco_peer_barrier_dev on one region.  E4M3, 64 <= B <= 512 (else TACO_ERR_USAGE: use the
 * push kernels + barrier).  A peer that never signals raises TACO_FLAG_PEER_TIMEOUT after
 * timeout_ms instead of hanging.  Results are bit-identical to the barrier-separated push
 * kernels and to the NCCL transport.
 * Reference: run_twoshot (collective.cpp:75-111) -- phase 1 exchange + owner reduce, phase 2
 * broadcast of the re-encoded shard. */
/* 1 when the fused peer collectives serve cfg (else use the push kernels + barrier) */
int taco_peer_fused_supported(const taco_config* cfg);
int taco_peer_allreduce_dev(const taco_config* cfg, const void* x, int dtype, uint64_t n, const taco_peers* peers,
                            uint64_t recv_offset, uint64_t gath_offset, uint64_t slot_stride, uint64_t flags_offset,
                            void* out, int out_dtype, uint32_t timeout_ms, int* d_flags, void* stream);
/* sequence-parallel reduce-scatter: x[n] -> out[ceil(n/P)] (the ascending-rank sum of this
 * rank's shard, out_dtype) */
int taco_peer_reduce_scatter_dev(const taco_config* cfg, const void* x, int dtype, uint64_t n,
                                 const taco_peers* peers, uint64_t recv_offset, uint64_t slot_stride,
                                 uint64_t flags_offset, void* out, int out_dtype, uint32_t timeout_ms, int* d_flags,
                                 void* stream);
/* sequence-parallel all-gather: x[n_local] -> out[P * n_local] */
int taco_peer_all_gather_dev(const taco_config* cfg, const void* x, int dtype, uint64_t n_local,
                             const taco_peers* peers, uint64_t gath_offset, uint64_t slot_stride, uint64_t flags_offset,
                             void* out, int out_dtype, uint32_t timeout_ms, int* d_flags, void* stream);

/* K1 into the peers: shard p's message (layout of blk_end - blk_begin blocks) goes to
 * base[p] + dst_offset + rank*slot_stride.  Taco kind, B <= 1024. */
int taco_compress_push_dev(const taco_config* cfg, const void* x, int dtype, uint64_t n, const taco_peers* peers,
                           uint64_t blk_begin, uint64_t blk_end, uint64_t dst_offset, uint64_t slot_stride,
                           int* d_flags, void* stream);

/* K1 broadcast (the SP all-gather): ONE message of this rank's n-element tensor (layout of
 * blk_end - blk_begin blocks) stored to base[q] + dst_offset + rank*slot_stride of EVERY
 * rank q.  Taco kind, B <= 1024. */
int taco_compress_bcast_dev(const taco_config* cfg, const void* x, int dtype, uint64_t n, const taco_peers* peers,
                            uint64_t blk_begin, uint64_t blk_end, uint64_t dst_offset, uint64_t slot_stride,
                            int* d_flags, void* stream);

/* K3 into the peers: reduce the P local messages (rank r at msgs + r*rank_stride) and
 * store the re-encoded shard to base[q] + dst_offset + rank*slot_stride of EVERY rank q
 * (the phase-2 all-gather done by K3's stores).  acc_out as in taco_reduce_encode_dev. */
int taco_reduce_encode_push_dev(const taco_config* cfg, const void* msgs, uint64_t rank_stride,
                                const taco_peers* peers, uint64_t shard_len, uint64_t blk_begin, uint64_t blk_end,
                                uint64_t dst_offset, uint64_t slot_stride, void* acc_out, int acc_dtype,
                                int* d_flags, void* stream);

/* ------------------------------------------------- TACOCMP1 archive -----
 * serialize.cpp:109-177: "TACOCMP1", kind u8, format id u8, block size u32, length u64,
 * then per block [payload][alpha f32][scale f32], little endian.  The device functions
 * convert between that byte stream and the SoA message of one tensor (n elements). */
int taco_archive_header(const taco_config* cfg, uint64_t n, uint8_t* out22);
/* archive_bytes (serialize.hpp:15): msg (device) -> archive (device, taco_archive_size bytes) */
int taco_archive_export_dev(const taco_config* cfg, const void* msg, uint64_t n, void* archive, void* stream);
/* archive_parse (serialize.hpp:16) header checks, exact reference messages; fills cfg/n */
int taco_archive_parse_header(const uint8_t* bytes, uint64_t size, taco_config* cfg_out, uint64_t* n_out);
/* archive (device) -> msg (device); non-finite scalars set TACO_FLAG_BAD_SCALARS */
int taco_archive_import_dev(const taco_config* cfg, const void* archive, uint64_t n, void* msg, int* d_flags,
                            void* stream);

/* ------------------------------------------------------------------ host API -------
 * Synchronous calls on host buffers, the shape of the reference's API (host spans in,
 * host vectors out).  A context owns a stream, device buffers and pinned staging; the
 * transfer is pipelined in chunks so H2D, kernels and D2H overlap. */
typedef struct taco_ctx taco_ctx;

int taco_ctx_create(int device, taco_ctx** out);
void taco_ctx_destroy(taco_ctx* ctx);

/* taco::compress on a host tensor: writes one message (layout for ceil(n/B) blocks)
 * into msg_host (>= taco_msg_layout(...).msg_bytes).  Raises the reference's errors. */
int taco_compress_host(taco_ctx* ctx, const taco_config* cfg, const void* x_host, int dtype,
                       uint64_t n, void* msg_host);

/* taco::decompress of one message into a host tensor of n elements */
int taco_decompress_host(taco_ctx* ctx, const taco_config* cfg, const void* msg_host,
                         uint64_t n, void* out_host, int out_dtype);

/* compress -> decompress of a host tensor (the reference round trip, acceptance.cpp
 * criterion 3) with H2D, K1, K2 and D2H pipelined over chunks */
int taco_roundtrip_host(taco_ctx* ctx, const taco_config* cfg, const void* x_host, int dtype,
                        uint64_t n, void* out_host, int out_dtype);

/* taco::allreduce(RankSet{TwoShot}) on host buffers: inputs [P][n] f32 -> result[n] f32
 * (collective.cpp:75-111), computed on the device by taco_allreduce_sim_dev.
 * stage1_host (optional): P*ceil(n/P) f32 ascending-rank sums before re-encoding. */
int taco_allreduce_sim_host(taco_ctx* ctx, const taco_config* cfg, const float* inputs_host,
                            uint32_t nranks, uint64_t n, float* result_host, float* stage1_host);

/* taco::allreduce (collective.hpp:28) for every Algorithm (0 TwoShot, 1 Ring, 2 Tree;
 * collective.cpp:75-111, :116-134, :153-254) on host rank tensors inputs [P][n] f32,
 * computed on the device: result[n] (identical on every rank), exact[n] = the fp32 sum in
 * ascending rank order (collective.cpp:36-41), rel_l2 (optional) = relative L2 of result
 * against exact (the error_vs_frequency column, collective.cpp:270-294). */
int taco_allreduce_schedule_host(taco_ctx* ctx, const taco_config* cfg, int algorithm,
                                 const float* inputs_host, uint32_t nranks, uint64_t n,
                                 float* result_host, float* exact_host, double* rel_l2);

/* taco::scaled_spectrum (codec.hpp:70) of a host tensor: ceil(n/B)*B fp32 values */
int taco_scaled_spectrum_host(taco_ctx* ctx, const taco_config* cfg, const float* x_host, uint64_t n,
                              float* out_host);

/* taco::error_report (analysis.hpp:42; analysis.cpp:97-132) on the device:
 * synchronous, deterministic.  Histogram edges are hist_lo + (hist_hi-hist_lo)/bins * i
 * (the last edge exactly hist_hi); counts[bins] receives the bin counts. */
typedef struct {
    double mse;
    double relative_l2;
    double max_abs_error;
    double zero_collapse_fraction;
    double kurtosis;
    int kurtosis_defined;
    double hist_lo, hist_hi;
} taco_error_report;
int taco_error_report_dev(const void* original, int orig_dtype, const void* reconstructed, int recon_dtype,
                          uint64_t n, uint32_t bins, taco_error_report* out, uint64_t* counts, void* stream);

/* ---------------------------------------------------------------- diagnostics ------
 * Element-wise FP8 conversion with exactly the instructions K1/K2/K3 use
 * (cvt.rn.satfinite.{e4m3,e5m2}x2.f32 / cvt.f16x2.{e4m3,e5m2}x2), replacing
 * taco::fp8_encode / fp8_decode (fp8.hpp:28-34) for bulk checks on the device. */
int taco_fp8_encode_dev(const float* x, uint64_t n, int format, uint8_t* out, void* stream);
int taco_fp8_decode_dev(const uint8_t* codes, uint64_t n, int format, float* out, void* stream);

/* ----------------------------------------------------------------- inputs ---------
 * taco::generate (analysis.hpp:40; analysis.cpp:70-95, rng.cpp): the reference's synthetic
 * tensors with identical values -- kind 0 = Gaussian N(0,1), 1 = near-zero mixture
 * (dense_sigma body, tail_sigma tail of tail_fraction*n elements, shuffled).  Host
 * routine (one sequential xoshiro256++ stream); fills out[0..n). */
int taco_generate_host(int kind, uint64_t n, uint64_t seed, double dense_sigma, double tail_sigma,
                       double tail_fraction, float* out);

#ifdef __cplusplus
}
#endif
#endif
