"""Compressed tensor-parallel collectives over torch.distributed (NCCL on NVLink).

The schedule is the reference's two-shot all-reduce (proj/src/collective.cpp:75-111),
run for real across ranks instead of simulated in one process:

    phase 1  K1 compress every shard of the local tensor   -> send [P][msg]
             all-to-all of FP8 messages                    -> recv [P][msg]  (rank r's copy of my shard)
             K3 decode + ascending-rank fp32 sum + encode  -> my reduced shard (one msg)
    phase 2  all-gather of the reduced messages            -> [P][msg]
             K2 decode every shard                         -> the all-reduced tensor

The sequence-parallel reduce-scatter is phase 1 with K3 emitting the fp32 sum (no
re-encode); the sequence-parallel all-gather is K1 of the own shard -> all-gather -> K2.

Overlap: each shard is cut into `chunks` block-aligned chunks (blocks never span
chunks, so numerics are unchanged -- test_collective.cpp:225-238).  Chunk c's
collective runs on NCCL's stream while the codec kernels of chunk c+1 / c-1 run on
the compute stream (async_op work handles order the two streams).

The codec is injected: the product passes nothing and gets the CUDA kernels
(CudaCodec, C ABI); the multi-process CPU tests inject a host implementation of the
same message format so the schedule itself is exercised under gloo.
"""
from __future__ import annotations

import ctypes as _ct

import torch
import torch.distributed as dist

from . import _abi, codec as dev
from ._abi import Config


def cdiv(a: int, b: int) -> int:
    return -(-a // b)


class CudaCodec:
    """K1/K2/K3 on the current CUDA stream (the product path; no fallback)."""

    def __init__(self, device=None):
        self.flags = dev.Flags(device)

    def layout(self, cfg: Config, nblocks: int) -> _abi.Layout:
        return _abi.msg_layout(cfg, nblocks)

    def compress(self, cfg, x, shards, b0, b1, out):
        dev.compress(x, cfg, shards=shards, blk=(b0, b1), out=out, flags=self.flags)

    def reduce_encode(self, cfg, recv, nranks, shard_len, rank_stride, b0, b1, out_msg, acc_out):
        dev.reduce_encode(recv, nranks, shard_len, cfg, rank_stride, out_msg, acc_out=acc_out, blk=(b0, b1),
                          flags=self.flags)

    def decompress(self, cfg, msgs, n, shards, b0, b1, out, msg_stride):
        dev.decompress(msgs, n, cfg, shards=shards, blk=(b0, b1), out=out, flags=self.flags, msg_stride=msg_stride)

    def check(self):
        self.flags.check()
        self.flags.reset()


class _Chunking:
    """Block ranges [b0, b1) of every shard for `chunks` pipelined chunks."""

    def __init__(self, cfg: Config, n: int, nranks: int, chunks: int, lay_fn):
        self.S = cdiv(n, nranks)
        self.m = cdiv(self.S, cfg.block_size)
        chunks = max(1, min(chunks, self.m))
        per = cdiv(self.m, chunks)
        self.ranges = [(b, min(self.m, b + per)) for b in range(0, self.m, per)]
        self.layouts = [lay_fn(cfg, b1 - b0) for b0, b1 in self.ranges]


class TwoShotAllReduce:
    """FP8 two-shot compressed all-reduce of a fixed-size tensor on `group`.

    x: [n] (any shape, flattened) bf16/fp32 on this rank's device.  Returns the
    all-reduced tensor (identical on every rank) in `out_dtype` (default x's dtype).
    Wire bytes per rank per direction: 2 (P-1)/P * n * (1 + 8/B).
    """

    def __init__(self, n: int, cfg: Config | None = None, group=None, dtype=torch.bfloat16, out_dtype=None,
                 chunks: int = 1, device=None, codec=None):
        self.group = group
        self.P = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.cfg = cfg if cfg is not None else _abi.make_config()
        self.n, self.dtype = n, dtype
        self.out_dtype = out_dtype or dtype
        self.device = torch.device(device) if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu"))
        self.codec = codec if codec is not None else CudaCodec(self.device)
        self.ch = _Chunking(self.cfg, n, self.P, chunks, self.codec.layout)
        P, dv = self.P, self.device
        u8 = dict(dtype=torch.uint8, device=dv)
        self.send = [torch.empty((P, lay.msg_stride), **u8) for lay in self.ch.layouts]
        self.recv = [torch.empty((P, lay.msg_stride), **u8) for lay in self.ch.layouts]
        self.red = [torch.empty((lay.msg_stride,), **u8) for lay in self.ch.layouts]
        self.gath = [torch.empty((P * lay.msg_stride,), **u8) for lay in self.ch.layouts]  # flat: gloo-compatible
        self.stage1 = None  # optional fp32 [S] hook for stage-isolated parity

    @property
    def shard_len(self) -> int:
        return self.ch.S

    def wire_bytes_per_rank(self) -> int:
        """bytes this rank sends (== receives) per call, both phases"""
        return sum(2 * (self.P - 1) * lay.msg_bytes for lay in self.ch.layouts)

    def __call__(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        x = x.reshape(-1)
        if x.numel() != self.n:
            raise _abi.TacoError(_abi.ERR_INPUT, "all rank inputs must have the same length")
        if out is None:
            out = torch.empty(self.n, dtype=self.out_dtype, device=self.device)
        cfg, P, S = self.cfg, self.P, self.ch.S
        works = []
        # phase 1: compress every chunk and put its all-to-all in flight
        for c, (b0, b1) in enumerate(self.ch.ranges):
            self.codec.compress(cfg, x, P, b0, b1, self.send[c])
            works.append(dist.all_to_all_single(self.recv[c], self.send[c], group=self.group, async_op=True))
        # owner reduce + re-encode as each chunk lands; phase 2 all-gather in flight
        gworks = []
        for c, (b0, b1) in enumerate(self.ch.ranges):
            works[c].wait()
            lay = self.ch.layouts[c]
            acc = None if self.stage1 is None else self.stage1
            self.codec.reduce_encode(cfg, self.recv[c], P, S, lay.msg_stride, b0, b1, self.red[c], acc)
            gworks.append(dist.all_gather_into_tensor(self.gath[c], self.red[c], group=self.group, async_op=True))
        for c, (b0, b1) in enumerate(self.ch.ranges):
            gworks[c].wait()
            self.codec.decompress(cfg, self.gath[c].view(P, -1), self.n, P, b0, b1, out, self.ch.layouts[c].msg_stride)
        return out


class CompressedReduceScatter:
    """Sequence-parallel reduce-scatter: phase 1 of the two-shot.  Returns this rank's
    shard ([S], S = ceil(n/P)) of the ascending-rank fp32 sum of the decoded shards."""

    def __init__(self, n: int, cfg: Config | None = None, group=None, dtype=torch.bfloat16, out_dtype=None,
                 chunks: int = 1, device=None, codec=None):
        self.ar = TwoShotAllReduce(n, cfg, group, dtype, out_dtype, chunks, device, codec)
        self.out_dtype = out_dtype or dtype

    @property
    def shard_len(self) -> int:
        return self.ar.ch.S

    def wire_bytes_per_rank(self) -> int:
        return sum((self.ar.P - 1) * lay.msg_bytes for lay in self.ar.ch.layouts)

    def __call__(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        a = self.ar
        x = x.reshape(-1)
        if x.numel() != a.n:
            raise _abi.TacoError(_abi.ERR_INPUT, "all rank inputs must have the same length")
        if out is None:
            out = torch.empty(a.ch.S, dtype=self.out_dtype, device=a.device)
        works = []
        for c, (b0, b1) in enumerate(a.ch.ranges):
            a.codec.compress(a.cfg, x, a.P, b0, b1, a.send[c])
            works.append(dist.all_to_all_single(a.recv[c], a.send[c], group=a.group, async_op=True))
        for c, (b0, b1) in enumerate(a.ch.ranges):
            works[c].wait()
            a.codec.reduce_encode(a.cfg, a.recv[c], a.P, a.ch.S, a.ch.layouts[c].msg_stride, b0, b1, None, out)
        return out


class CompressedAllGather:
    """Sequence-parallel all-gather of [n_local] shards: K1 of the own shard ->
    all-gather of the FP8 messages -> K2 of every shard.  Returns [P * n_local]."""

    def __init__(self, n_local: int, cfg: Config | None = None, group=None, dtype=torch.bfloat16, out_dtype=None,
                 chunks: int = 1, device=None, codec=None):
        self.group = group
        self.P = dist.get_world_size(group)
        self.cfg = cfg if cfg is not None else _abi.make_config()
        self.n_local = n_local
        self.out_dtype = out_dtype or dtype
        self.device = torch.device(device) if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu"))
        self.codec = codec if codec is not None else CudaCodec(self.device)
        self.ch = _Chunking(self.cfg, n_local, 1, chunks, self.codec.layout)
        u8 = dict(dtype=torch.uint8, device=self.device)
        self.mine = [torch.empty((lay.msg_stride,), **u8) for lay in self.ch.layouts]
        self.gath = [torch.empty((self.P * lay.msg_stride,), **u8) for lay in self.ch.layouts]

    def wire_bytes_per_rank(self) -> int:
        return sum((self.P - 1) * lay.msg_bytes for lay in self.ch.layouts)

    def __call__(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        x = x.reshape(-1)
        if x.numel() != self.n_local:
            raise _abi.TacoError(_abi.ERR_INPUT, "all rank inputs must have the same length")
        n = self.P * self.n_local
        if out is None:
            out = torch.empty(n, dtype=self.out_dtype, device=self.device)
        works = []
        for c, (b0, b1) in enumerate(self.ch.ranges):
            self.codec.compress(self.cfg, x, 1, b0, b1, self.mine[c].view(1, -1))
            works.append(dist.all_gather_into_tensor(self.gath[c], self.mine[c], group=self.group, async_op=True))
        for c, (b0, b1) in enumerate(self.ch.ranges):
            works[c].wait()
            # the gathered tensor is P shards of n_local: shard geometry S = n_local exactly
            self.codec.decompress(self.cfg, self.gath[c].view(self.P, -1), n, self.P, b0, b1, out,
                                  self.ch.layouts[c].msg_stride)
        return out


class Graphed:
    """CUDA-graph replay of a collective call on static buffers: the ~3*chunks codec
    launches and 2*chunks NCCL calls of a step are captured once, so a step costs one
    graph launch instead of a Python round trip per op (latency-bound at small sizes)."""

    def __init__(self, op, x: torch.Tensor, out: torch.Tensor, warmup: int = 2):
        self.op, self.x, self.out = op, x, out
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):  # NCCL communicators / workspaces exist before capture
                op(x, out)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            op(x, out)

    def __call__(self):
        self.graph.replay()
        return self.out


def nccl_comm_ptr(group=None, device=None) -> int:
    """The ncclComm_t behind a torch.distributed NCCL group (ProcessGroupNCCL._comm_ptr), the
    communicator is created first if torch has not used it yet."""
    pg = group if group is not None else dist.group.WORLD
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    backend = pg._get_backend(dev)
    ptr = int(backend._comm_ptr())
    if ptr == 0:  # lazily initialised communicator: one tiny collective creates it
        t = torch.zeros(1, device=dev)
        dist.all_reduce(t, group=pg)
        torch.cuda.synchronize(dev)
        ptr = int(backend._comm_ptr())
    if ptr == 0:
        raise _abi.TacoError(_abi.ERR_USAGE, "the group has no NCCL communicator")
    return ptr


class _AbiCollective:
    """Base of the C-ABI collectives on torch's own NCCL communicator: one library call per
    collective issues every codec kernel on the caller's stream and every NCCL call on the
    library's communication stream (include/taco_b200.h taco_*_nccl_chunked), so a step
    costs one host call instead of a Python round trip per chunk and op."""

    def __init__(self, n_total: int, cfg: Config | None, group, dtype, out_dtype, chunks: int, device):
        self.group = group
        self.P = dist.get_world_size(group)
        self.cfg = cfg if cfg is not None else _abi.make_config()
        self.dtype = dtype
        self.out_dtype = out_dtype or dtype
        self.chunks = chunks
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.comm = nccl_comm_ptr(group, self.device)
        lib = _abi.lib()
        ws = int(lib.taco_collective_nccl_workspace_chunked(_ct.byref(self.cfg), self.P, n_total, chunks))
        if ws == 0:
            raise _abi.TacoError(_abi.ERR_USAGE, "no workspace for this geometry (chunks must be 1 to 16)")
        self.work = torch.empty(ws, dtype=torch.uint8, device=self.device)
        self.flags = dev.Flags(self.device)

    def _call(self, fn: str, x: torch.Tensor, n: int, out: torch.Tensor, stream=None):
        st = _ct.c_void_p(stream.cuda_stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream)
        _abi.check(getattr(_abi.lib(), fn)(_ct.byref(self.cfg), _ct.c_void_p(x.data_ptr()), dev._dtype_code(x.dtype), n,
                                           _ct.c_void_p(out.data_ptr()), dev._dtype_code(out.dtype),
                                           _ct.c_void_p(self.work.data_ptr()), _ct.c_void_p(self.comm),
                                           self.flags.ptr(), st, self.chunks))
        return out

    def _check_in(self, x: torch.Tensor, n: int) -> torch.Tensor:
        x = x.reshape(-1)
        if x.device != self.device:
            raise _abi.TacoError(_abi.ERR_USAGE, f"input must live on {self.device}")
        if x.numel() != n:
            raise _abi.TacoError(_abi.ERR_INPUT, "all rank inputs must have the same length")
        return x.contiguous()

    def _out(self, out, numel):
        if out is None:
            return torch.empty(numel, dtype=self.out_dtype, device=self.device)
        if not out.is_contiguous() or out.numel() != numel or out.device != self.device:
            raise _abi.TacoError(_abi.ERR_USAGE, f"out must be a contiguous tensor of {numel} elements on {self.device}")
        return out

    def check(self):
        self.flags.check()


class AbiTwoShotAllReduce(_AbiCollective):
    """TwoShotAllReduce through taco_allreduce_nccl_chunked on the group's own communicator
    (bit-identical to TwoShotAllReduce with the same chunking)."""

    def __init__(self, n: int, cfg: Config | None = None, group=None, dtype=torch.bfloat16, out_dtype=None,
                 chunks: int = 2, device=None):
        super().__init__(n, cfg, group, dtype, out_dtype, chunks, device)
        self.n = n

    def __call__(self, x: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        x = self._check_in(x, self.n)
        return self._call("taco_allreduce_nccl_chunked", x, self.n, self._out(out, self.n), stream)


class AbiReduceScatter(_AbiCollective):
    """CompressedReduceScatter through taco_reduce_scatter_nccl_chunked: [n] -> [ceil(n/P)]."""

    def __init__(self, n: int, cfg: Config | None = None, group=None, dtype=torch.bfloat16, out_dtype=None,
                 chunks: int = 2, device=None):
        super().__init__(n, cfg, group, dtype, out_dtype, chunks, device)
        self.n = n
        self.shard_len = cdiv(n, self.P)

    def __call__(self, x: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        x = self._check_in(x, self.n)
        return self._call("taco_reduce_scatter_nccl_chunked", x, self.n, self._out(out, self.shard_len), stream)


class AbiAllGather(_AbiCollective):
    """CompressedAllGather through taco_all_gather_nccl_chunked: [n_local] -> [P * n_local]."""

    def __init__(self, n_local: int, cfg: Config | None = None, group=None, dtype=torch.bfloat16, out_dtype=None,
                 chunks: int = 2, device=None):
        P = dist.get_world_size(group)
        super().__init__(P * n_local, cfg, group, dtype, out_dtype, chunks, device)
        self.n_local = n_local

    def __call__(self, x: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        x = self._check_in(x, self.n_local)
        return self._call("taco_all_gather_nccl_chunked", x, self.n_local, self._out(out, self.P * self.n_local),
                          stream)
