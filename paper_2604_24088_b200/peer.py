"""Peer-memory two-shot all-reduce: the exchange folded into the codec kernels.

The reference's two-shot (proj/src/collective.cpp:75-111) needs two exchanges: every rank
sends shard p of its compressed tensor to rank p, and every owner sends its re-encoded
shard to everyone.  `collective.TwoShotAllReduce` does them with NCCL (all-to-all and
all-gather between the kernels).  Here the kernels do them with their own stores:

    K1 push   compress shard p straight into rank p's receive slot [my rank]   (NVLink stores)
    barrier   system-scope release/acquire flags: every K1 has landed
    K3 push   decode the P local copies of my shard, fp32 ascending-rank sum, re-encode,
              store the message into EVERY rank's gather slot [my rank]          (NVLink stores)
    barrier   every K3 has landed (and nobody still reads a receive slot)
    K2        decode the P gathered shards from local memory

Fused mode (the default where the exchange-butterfly kernels serve the config: E4M3,
64 <= B <= 512): no barrier kernels.  Each kernel that reads peer-written slots waits for
the phase words of the call's epoch itself, and the last CTA of each writing kernel
publishes its phase (taco_peer_allreduce_dev / _reduce_scatter_dev / _all_gather_dev):
3 launches per all-reduce (K1 -> K3 -> K2), 2 per reduce-scatter or all-gather.

Each rank owns one region (CUDA-IPC exportable, include/taco_b200.h taco_peer_alloc):

    [ recv: P x msg_stride ][ gath: P x msg_stride ][ barrier flags ]

mapped by every other rank of the group.  The arithmetic is exactly the NCCL path's
(same K1/K3/K2 code), so results are bit-identical to it and to
`codec.allreduce_sim`.  Two barriers per call make buffer reuse safe: a rank's next K1
can only write a receive slot after the second barrier proved every K3 finished
reading it, and its next K3 can only write a gather slot after the next call's first
barrier proved every K2 of this call finished.  Barriers give up after `timeout_ms`
and raise "peer barrier timed out" instead of hanging.
"""
from __future__ import annotations

import ctypes as C

import torch
import torch.distributed as dist

from . import _abi
from ._abi import Config, IpcHandle, Peers, TacoError
from .codec import Flags, _dtype_code, _ptr, _stream, cdiv


def _align16(v: int) -> int:
    return (v + 15) & ~15


class PeerRegion:
    """One rank's exportable device region (receive slots, gather slots, barrier flags)."""

    def __init__(self, nbytes: int, device: int):
        self.nbytes = nbytes
        self.ptr = C.c_void_p()
        self.handle = IpcHandle()
        _abi.check(_abi.lib().taco_peer_alloc(device, nbytes, C.byref(self.ptr), C.byref(self.handle)))

    def handle_bytes(self) -> bytes:
        return bytes(self.handle.bytes)

    def free(self):
        if self.ptr:
            _abi.check(_abi.lib().taco_peer_free(self.ptr))
            self.ptr = C.c_void_p()


def open_handle(raw: bytes, device: int) -> C.c_void_p:
    h = IpcHandle()
    C.memmove(C.byref(h), raw, 64)
    p = C.c_void_p()
    _abi.check(_abi.lib().taco_peer_open(device, C.byref(h), C.byref(p)))
    return p


class PeerLayout:
    """Region geometry for an n-element all-reduce over P ranks (one chunk per shard)."""

    def __init__(self, cfg: Config, n: int, P: int):
        self.S = cdiv(n, P)
        self.m = cdiv(self.S, cfg.block_size)
        self.lay = _abi.msg_layout(cfg, self.m)
        self.stride = self.lay.msg_stride
        self.recv_off = 0
        self.gath_off = P * self.stride
        self.flags_off = _align16(2 * P * self.stride)
        self.nbytes = self.flags_off + int(_abi.lib().taco_peer_flags_bytes())


def peers_struct(bases, rank: int) -> Peers:
    ps = Peers()
    ps.nranks, ps.rank = len(bases), rank
    for q, b in enumerate(bases):
        ps.base[q] = b.value if isinstance(b, C.c_void_p) else int(b)
    return ps


def push_step(cfg: Config, x: torch.Tensor, n: int, geo: PeerLayout, peers: Peers, out: torch.Tensor,
              flags: Flags, timeout_ms: int, stream=None, barriers: bool = True) -> None:
    """One all-reduce on this rank: K1 push, barrier, K3 push, barrier, K2 (all enqueued on
    `stream`, nothing synchronises -- CUDA-graph capturable)."""
    lib, st, fl = _abi.lib(), C.c_void_p(_stream(stream)), flags.ptr()
    own = peers.base[peers.rank]
    _abi.check(lib.taco_compress_push_dev(C.byref(cfg), _ptr(x), _dtype_code(x.dtype), n, C.byref(peers), 0, geo.m,
                                          geo.recv_off, geo.stride, fl, st))
    if barriers:
        _abi.check(lib.taco_peer_barrier_dev(C.byref(peers), geo.flags_off, timeout_ms, fl, st))
    _abi.check(lib.taco_reduce_encode_push_dev(C.byref(cfg), C.c_void_p(own + geo.recv_off), geo.stride,
                                               C.byref(peers), geo.S, 0, geo.m, geo.gath_off, geo.stride, None,
                                               _abi.DT_F32, fl, st))
    if barriers:
        _abi.check(lib.taco_peer_barrier_dev(C.byref(peers), geo.flags_off, timeout_ms, fl, st))
    decode(cfg, peers, geo, n, out, flags, stream)


def decode(cfg: Config, peers: Peers, geo: PeerLayout, n: int, out: torch.Tensor, flags: Flags, stream=None):
    own = peers.base[peers.rank]
    _abi.check(_abi.lib().taco_decompress_dev(C.byref(cfg), C.c_void_p(own + geo.gath_off), geo.stride,
                                              peers.nranks, n, 0, geo.m, _ptr(out), _dtype_code(out.dtype),
                                              flags.ptr(), C.c_void_p(_stream(stream))))


class _Mapped:
    """This rank's region, every peer's region mapped here, and the taco_peers view."""

    def __init__(self, nbytes: int, group, device: torch.device):
        self.group = group
        self.P = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.P > _abi.MAX_PEERS:
            raise TacoError(_abi.ERR_USAGE, "peer collectives support 1 to 8 ranks")
        dix = device.index if device.index is not None else torch.cuda.current_device()
        self.region = PeerRegion(nbytes, dix)
        handles = [None] * self.P
        dist.all_gather_object(handles, (self.region.handle_bytes(), dix), group=group)
        self.devices = [d for _, d in handles]
        self.bases, self.opened = [], []
        err = ""
        try:
            for q in range(self.P):
                _abi.check(_abi.lib().taco_peer_check_access(dix, self.devices[q]))
            for q in range(self.P):
                if q == self.rank:
                    self.bases.append(self.region.ptr)
                else:
                    p = open_handle(handles[q][0], dix)
                    self.opened.append(p)
                    self.bases.append(p)
        except TacoError as e:  # e.g. no P2P path between two GPUs
            err = f"rank {self.rank}: {e}"
        # every rank learns whether every mapping worked (nobody is left waiting in a barrier),
        # and every region is zeroed and mapped before the first signal
        errs = [None] * self.P
        dist.all_gather_object(errs, err, group=group)
        bad = [e for e in errs if e]
        if bad:
            self._unmap()
            self.region.free()
            raise TacoError(_abi.ERR_CUDA, "peer mapping failed: " + "; ".join(bad))
        self.peers = peers_struct(self.bases, self.rank)

    @property
    def own(self) -> int:
        return self.peers.base[self.rank]

    def _unmap(self):
        for p in self.opened:
            _abi.lib().taco_peer_close(p)
        self.opened = []

    def close(self, device):
        """Collective: unmap the peers' regions, then free this rank's own."""
        torch.cuda.synchronize(device)
        dist.barrier(group=self.group)
        self._unmap()
        dist.barrier(group=self.group)
        self.region.free()


def _input(x: torch.Tensor, n: int, device) -> torch.Tensor:
    """The kernels read x through a raw pointer: make it a dense 1-D tensor on this
    transport's device (a strided view such as buf[::2] would otherwise be read as if dense,
    unlike the NCCL transport, which also goes through .contiguous())."""
    if x.device != device:
        raise TacoError(_abi.ERR_USAGE, f"input must live on {device}, got {x.device}")
    x = x.reshape(-1).contiguous()
    if x.numel() != n:
        raise TacoError(_abi.ERR_INPUT, "all rank inputs must have the same length")
    return x


def _output(out: torch.Tensor | None, numel: int, dtype, device) -> torch.Tensor:
    if out is None:
        return torch.empty(numel, dtype=dtype, device=device)
    if not out.is_contiguous() or out.numel() != numel or out.device != device:
        raise TacoError(_abi.ERR_USAGE, f"out must be a contiguous tensor of {numel} elements on {device}")
    _dtype_code(out.dtype)
    return out


def _device(device):
    return torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())


def fused_supported(cfg: Config) -> bool:
    """Whether the kernel-signalled (barrier-free) peer collectives serve cfg."""
    return bool(_abi.lib().taco_peer_fused_supported(C.byref(cfg)))


def _fused(cfg: Config, fused) -> bool:
    ok = fused_supported(cfg)
    if fused and not ok:
        raise TacoError(_abi.ERR_USAGE, "fused peer signalling needs E4M3 and 64 <= B <= 512")
    return ok if fused is None else bool(fused)


class PeerTwoShotAllReduce:
    """FP8 two-shot all-reduce of a fixed-size tensor over peer memory (one process per GPU).

    Same contract as collective.TwoShotAllReduce (bit-identical results); the group is
    only used once, to exchange the IPC handles of the regions."""

    def __init__(self, n: int, cfg: Config | None = None, group=None, dtype=torch.bfloat16, out_dtype=None,
                 device=None, timeout_ms: int = 10_000, fused: bool | None = None):
        self.cfg = cfg if cfg is not None else _abi.make_config()
        self.n, self.dtype = n, dtype
        self.out_dtype = out_dtype or dtype
        self.device = _device(device)
        self.timeout_ms = timeout_ms
        self.fused = _fused(self.cfg, fused)
        self.P = dist.get_world_size(group)
        self.geo = PeerLayout(self.cfg, n, self.P)
        self.flags = Flags(self.device)
        self.map = _Mapped(self.geo.nbytes, group, self.device)
        self.peers = self.map.peers

    def launches(self) -> int:
        return 3 if self.fused else 5

    @property
    def shard_len(self) -> int:
        return self.geo.S

    def wire_bytes_per_rank(self) -> int:
        return 2 * (self.P - 1) * self.geo.lay.msg_bytes

    def __call__(self, x: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        x = _input(x, self.n, self.device)
        out = _output(out, self.n, self.out_dtype, self.device)
        if self.fused:
            g = self.geo
            _abi.check(_abi.lib().taco_peer_allreduce_dev(
                C.byref(self.cfg), _ptr(x), _dtype_code(x.dtype), self.n, C.byref(self.peers), g.recv_off,
                g.gath_off, g.stride, g.flags_off, _ptr(out), _dtype_code(out.dtype), self.timeout_ms,
                self.flags.ptr(), C.c_void_p(_stream(stream))))
        else:
            push_step(self.cfg, x, self.n, self.geo, self.peers, out, self.flags, self.timeout_ms, stream)
        return out

    def check(self):
        self.flags.check()

    def close(self):
        self.map.close(self.device)


class PeerReduceScatter:
    """Sequence-parallel reduce-scatter over peer memory: K1 pushes shard p into rank p's
    receive slot, barrier, K3 writes the ascending-rank fp32 sum of this rank's shard
    (no re-encode), barrier (the receive slots are free again).  Bit-identical to
    collective.CompressedReduceScatter."""

    def __init__(self, n: int, cfg: Config | None = None, group=None, dtype=torch.bfloat16, out_dtype=None,
                 device=None, timeout_ms: int = 10_000, fused: bool | None = None):
        self.cfg = cfg if cfg is not None else _abi.make_config()
        self.n, self.dtype = n, dtype
        self.out_dtype = out_dtype or dtype
        self.device = _device(device)
        self.timeout_ms = timeout_ms
        self.fused = _fused(self.cfg, fused)
        self.P = dist.get_world_size(group)
        self.geo = PeerLayout(self.cfg, n, self.P)
        self.flags = Flags(self.device)
        self.map = _Mapped(self.geo.nbytes, group, self.device)

    @property
    def shard_len(self) -> int:
        return self.geo.S

    def wire_bytes_per_rank(self) -> int:
        return (self.P - 1) * self.geo.lay.msg_bytes

    def __call__(self, x: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        x = _input(x, self.n, self.device)
        out = _output(out, self.geo.S, self.out_dtype, self.device)
        g, ps, lib = self.geo, self.map.peers, _abi.lib()
        st, fl = C.c_void_p(_stream(stream)), self.flags.ptr()
        if self.fused:
            _abi.check(lib.taco_peer_reduce_scatter_dev(C.byref(self.cfg), _ptr(x), _dtype_code(x.dtype), self.n,
                                                        C.byref(ps), g.recv_off, g.stride, g.flags_off, _ptr(out),
                                                        _dtype_code(out.dtype), self.timeout_ms, fl, st))
            return out
        _abi.check(lib.taco_compress_push_dev(C.byref(self.cfg), _ptr(x), _dtype_code(x.dtype), self.n, C.byref(ps),
                                              0, g.m, g.recv_off, g.stride, fl, st))
        _abi.check(lib.taco_peer_barrier_dev(C.byref(ps), g.flags_off, self.timeout_ms, fl, st))
        _abi.check(lib.taco_reduce_encode_dev(C.byref(self.cfg), C.c_void_p(self.map.own + g.recv_off), g.stride,
                                              self.P, g.S, 0, g.m, None, _ptr(out), _dtype_code(out.dtype), fl, st))
        _abi.check(lib.taco_peer_barrier_dev(C.byref(ps), g.flags_off, self.timeout_ms, fl, st))
        return out

    def check(self):
        self.flags.check()

    def close(self):
        self.map.close(self.device)


class PeerAllGather:
    """Sequence-parallel all-gather over peer memory: K1 of the own [n_local] slice stored
    into EVERY rank's gather slot [my rank], barrier, K2 of the P gathered messages,
    barrier (the gather slots are free again).  Bit-identical to collective.CompressedAllGather."""

    def __init__(self, n_local: int, cfg: Config | None = None, group=None, dtype=torch.bfloat16, out_dtype=None,
                 device=None, timeout_ms: int = 10_000, fused: bool | None = None):
        self.cfg = cfg if cfg is not None else _abi.make_config()
        self.n_local = n_local
        self.out_dtype = out_dtype or dtype
        self.device = _device(device)
        self.timeout_ms = timeout_ms
        self.fused = _fused(self.cfg, fused)
        self.P = dist.get_world_size(group)
        self.m = cdiv(n_local, self.cfg.block_size)
        self.lay = _abi.msg_layout(self.cfg, self.m)
        self.stride = self.lay.msg_stride
        self.flags_off = _align16(self.P * self.stride)
        self.flags = Flags(self.device)
        self.map = _Mapped(self.flags_off + int(_abi.lib().taco_peer_flags_bytes()), group, self.device)

    def wire_bytes_per_rank(self) -> int:
        return (self.P - 1) * self.lay.msg_bytes

    def __call__(self, x: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        x = _input(x, self.n_local, self.device)
        n = self.P * self.n_local
        out = _output(out, n, self.out_dtype, self.device)
        ps, lib = self.map.peers, _abi.lib()
        st, fl = C.c_void_p(_stream(stream)), self.flags.ptr()
        if self.fused:
            _abi.check(lib.taco_peer_all_gather_dev(C.byref(self.cfg), _ptr(x), _dtype_code(x.dtype), self.n_local,
                                                    C.byref(ps), 0, self.stride, self.flags_off, _ptr(out),
                                                    _dtype_code(out.dtype), self.timeout_ms, fl, st))
            return out
        _abi.check(lib.taco_compress_bcast_dev(C.byref(self.cfg), _ptr(x), _dtype_code(x.dtype), self.n_local,
                                               C.byref(ps), 0, self.m, 0, self.stride, fl, st))
        _abi.check(lib.taco_peer_barrier_dev(C.byref(ps), self.flags_off, self.timeout_ms, fl, st))
        _abi.check(lib.taco_decompress_dev(C.byref(self.cfg), C.c_void_p(self.map.own), self.stride, self.P, n, 0,
                                           self.m, _ptr(out), _dtype_code(out.dtype), fl, st))
        _abi.check(lib.taco_peer_barrier_dev(C.byref(ps), self.flags_off, self.timeout_ms, fl, st))
        return out

    def check(self):
        self.flags.check()

    def close(self):
        self.map.close(self.device)


def allreduce_sim_peer(inputs: torch.Tensor, cfg: Config, out_dtype=torch.float32) -> torch.Tensor:
    """The peer-memory schedule for P simulated ranks in ONE process (P regions on this
    device, the ranks' kernels enqueued in phase order on one stream, so no barrier is
    needed).  Exercises every push address computation; returns [P, n] (one result per
    rank, all of which must equal codec.allreduce_sim)."""
    P, n = inputs.shape
    geo = PeerLayout(cfg, n, P)
    dix = inputs.device.index if inputs.device.index is not None else torch.cuda.current_device()
    regions = [PeerRegion(geo.nbytes, dix) for _ in range(P)]
    try:
        bases = [r.ptr for r in regions]
        peers = [peers_struct(bases, r) for r in range(P)]
        flags = Flags(inputs.device)
        lib, st = _abi.lib(), C.c_void_p(_stream(None))
        outs = torch.empty((P, n), dtype=out_dtype, device=inputs.device)
        for r in range(P):
            x = inputs[r].contiguous()
            _abi.check(lib.taco_compress_push_dev(C.byref(cfg), _ptr(x), _dtype_code(x.dtype), n,
                                                  C.byref(peers[r]), 0, geo.m, geo.recv_off, geo.stride,
                                                  flags.ptr(), st))
        for r in range(P):
            own = peers[r].base[r]
            _abi.check(lib.taco_reduce_encode_push_dev(C.byref(cfg), C.c_void_p(own + geo.recv_off), geo.stride,
                                                       C.byref(peers[r]), geo.S, 0, geo.m, geo.gath_off,
                                                       geo.stride, None, _abi.DT_F32, flags.ptr(), st))
        for r in range(P):
            decode(cfg, peers[r], geo, n, outs[r], flags)
        torch.cuda.synchronize(inputs.device)
        flags.check()
        return outs
    finally:
        torch.cuda.synchronize(inputs.device)
        for r in regions:
            r.free()


def reduce_scatter_sim_peer(inputs: torch.Tensor, cfg: Config, out_dtype=torch.float32) -> torch.Tensor:
    """PeerReduceScatter's kernels for P simulated ranks in one process: [P, S]."""
    P, n = inputs.shape
    geo = PeerLayout(cfg, n, P)
    dix = inputs.device.index if inputs.device.index is not None else torch.cuda.current_device()
    regions = [PeerRegion(geo.nbytes, dix) for _ in range(P)]
    try:
        bases = [r.ptr for r in regions]
        peers = [peers_struct(bases, r) for r in range(P)]
        flags = Flags(inputs.device)
        lib, st = _abi.lib(), C.c_void_p(_stream(None))
        outs = torch.empty((P, geo.S), dtype=out_dtype, device=inputs.device)
        for r in range(P):
            x = inputs[r].contiguous()
            _abi.check(lib.taco_compress_push_dev(C.byref(cfg), _ptr(x), _dtype_code(x.dtype), n, C.byref(peers[r]),
                                                  0, geo.m, geo.recv_off, geo.stride, flags.ptr(), st))
        for r in range(P):
            _abi.check(lib.taco_reduce_encode_dev(C.byref(cfg), C.c_void_p(peers[r].base[r] + geo.recv_off),
                                                  geo.stride, P, geo.S, 0, geo.m, None, _ptr(outs[r]),
                                                  _dtype_code(out_dtype), flags.ptr(), st))
        torch.cuda.synchronize(inputs.device)
        flags.check()
        return outs
    finally:
        torch.cuda.synchronize(inputs.device)
        for r in regions:
            r.free()


def all_gather_sim_peer(inputs: torch.Tensor, cfg: Config, out_dtype=torch.float32) -> torch.Tensor:
    """PeerAllGather's kernels for P simulated ranks in one process: inputs [P, n_local]
    -> [P, P * n_local]."""
    P, nl = inputs.shape
    m = cdiv(nl, cfg.block_size)
    stride = _abi.msg_layout(cfg, m).msg_stride
    dix = inputs.device.index if inputs.device.index is not None else torch.cuda.current_device()
    regions = [PeerRegion(_align16(P * stride) + int(_abi.lib().taco_peer_flags_bytes()), dix) for _ in range(P)]
    try:
        bases = [r.ptr for r in regions]
        peers = [peers_struct(bases, r) for r in range(P)]
        flags = Flags(inputs.device)
        lib, st = _abi.lib(), C.c_void_p(_stream(None))
        outs = torch.empty((P, P * nl), dtype=out_dtype, device=inputs.device)
        for r in range(P):
            x = inputs[r].contiguous()
            _abi.check(lib.taco_compress_bcast_dev(C.byref(cfg), _ptr(x), _dtype_code(x.dtype), nl,
                                                   C.byref(peers[r]), 0, m, 0, stride, flags.ptr(), st))
        for r in range(P):
            _abi.check(lib.taco_decompress_dev(C.byref(cfg), C.c_void_p(peers[r].base[r]), stride, P, P * nl, 0, m,
                                               _ptr(outs[r]), _dtype_code(out_dtype), flags.ptr(), st))
        torch.cuda.synchronize(inputs.device)
        flags.check()
        return outs
    finally:
        torch.cuda.synchronize(inputs.device)
        for r in regions:
            r.free()
