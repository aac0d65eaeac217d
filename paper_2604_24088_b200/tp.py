"""Framework caller of the compressed collectives: where TACO sits in training.

TACO compresses the tensor-parallel communication of Megatron-style layers (PAPER.md:185-190,
485-493): the forward all-reduce after a row-parallel linear (activations) and the backward
all-reduce before a column-parallel linear (activation gradients), and, with sequence
parallelism, the reduce-scatter / all-gather pair that replaces them.  This module wires the
FP8 two-shot collectives of ``collective.py`` into autograd with the usual region semantics:

    reduce_from_tp   fwd: compressed all-reduce        bwd: identity
    copy_to_tp       fwd: identity                     bwd: compressed all-reduce
    reduce_scatter_to_sp   fwd: compressed RS          bwd: compressed AG
    gather_from_sp         fwd: compressed AG          bwd: compressed RS

plus ``RowParallelLinear`` / ``ColumnParallelLinear`` modules and ``torch.library`` custom
ops (``taco_b200::compress`` / ``decompress``) so the codec is an opaque op under
``torch.compile`` / FX.  The collective objects (buffers, chunking, optional CUDA graphs)
live in a bounded per-context LRU keyed on (group, size, dtype) and are released by
``TpContext.close()``; the codec is injectable like in ``collective.py``.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import _abi, collective
from ._abi import Config

from collections import OrderedDict

# Collective objects own device buffers (and, for the peer transport, a CUDA-IPC region
# mapped by every rank), so each TpContext keeps a bounded LRU of them keyed on the group
# OBJECT (held by the key, so a collected group's id() cannot be reused for a stale entry).
# Evicting or closing is collective for the peer transport: every rank makes the same calls
# in the same order (SPMD), so they evict the same entries together.
_MAX_CACHED = 8


def _key(kind, group, n, dtype, cfg: Config, chunks, codec, transport):
    return (kind, group, n, dtype, cfg.block_size, cfg.format, cfg.kind, chunks, id(codec), transport)


def _close(op) -> None:
    close = getattr(op, "close", None)
    if close is not None:
        close()


class TpContext:
    """Settings shared by the regions of one model: group, codec config, chunking, codec."""

    def __init__(self, group=None, cfg: Config | None = None, chunks: int = 1, codec=None, transport: str = "nccl"):
        """transport: "nccl" (K1 -> NCCL all-to-all -> K3 -> NCCL all-gather -> K2, chunked overlap)
        or "peer" (K1/K3 store into the peers' CUDA-IPC mapped buffers, device barriers;
        bit-identical results, no NCCL call on the data path)."""
        if transport not in ("nccl", "peer"):
            raise ValueError("transport must be 'nccl' or 'peer'")
        if transport == "peer" and codec is not None:
            raise ValueError("the peer transport runs the CUDA kernels only")
        self.group = group
        self.cfg = cfg if cfg is not None else _abi.make_config()
        self.chunks = chunks
        self.codec = codec
        self.transport = transport
        self._ops: OrderedDict = OrderedDict()

    def _get(self, kind, n, dtype, device):
        k = _key(kind, self.group, n, dtype, self.cfg, self.chunks, self.codec, self.transport)
        op = self._ops.get(k)
        if op is not None:
            self._ops.move_to_end(k)
            return op
        if self.transport == "peer":  # exchange inside the kernels (peer.py)
            from . import peer
            cls = {"ar": peer.PeerTwoShotAllReduce, "rs": peer.PeerReduceScatter, "ag": peer.PeerAllGather}[kind]
            op = cls(n, self.cfg, self.group, dtype=dtype, device=device)
        else:
            op = None
            if self.codec is None and device.type == "cuda" and dist.get_backend(self.group) == "nccl":
                # the C-ABI schedule on the group's own communicator: one library call per
                # collective instead of a Python call per chunk and op (same numerics)
                abi_cls = {"ar": collective.AbiTwoShotAllReduce, "rs": collective.AbiReduceScatter,
                           "ag": collective.AbiAllGather}[kind]
                try:
                    op = abi_cls(n, self.cfg, self.group, dtype=dtype, chunks=max(1, self.chunks), device=device)
                except (AttributeError, RuntimeError, _abi.TacoError):
                    op = None  # no communicator handle in this torch build: the Python schedule
            if op is None:
                cls = {"ar": collective.TwoShotAllReduce, "rs": collective.CompressedReduceScatter,
                       "ag": collective.CompressedAllGather}[kind]
                op = cls(n, self.cfg, self.group, dtype=dtype, chunks=self.chunks, device=device, codec=self.codec)
        self._ops[k] = op
        while len(self._ops) > _MAX_CACHED:
            _close(self._ops.popitem(last=False)[1])
        return op

    def close(self) -> None:
        """Release every cached collective (collective call for the peer transport)."""
        while self._ops:
            _close(self._ops.popitem(last=False)[1])

    @property
    def world(self) -> int:
        return dist.get_world_size(self.group)

    def all_reduce(self, x: torch.Tensor) -> torch.Tensor:
        op = self._get("ar", x.numel(), x.dtype, x.device)
        return op(x.contiguous()).view(x.shape)

    def reduce_scatter(self, x: torch.Tensor) -> torch.Tensor:
        """x: [T, ...] with T % world == 0 -> this rank's token slice [T/world, ...]"""
        w = self.world
        if x.shape[0] % w:
            raise _abi.TacoError(_abi.ERR_USAGE, "sequence length must divide by the tensor-parallel size")
        op = self._get("rs", x.numel(), x.dtype, x.device)
        return op(x.contiguous()).view(x.shape[0] // w, *x.shape[1:])

    def all_gather(self, x: torch.Tensor) -> torch.Tensor:
        """x: this rank's token slice [t, ...] -> [world * t, ...]"""
        op = self._get("ag", x.numel(), x.dtype, x.device)
        return op(x.contiguous()).view(self.world * x.shape[0], *x.shape[1:])


class _ReduceFromTP(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, tp):
        return tp.all_reduce(x)

    @staticmethod
    def backward(ctx, g):
        return g, None


class _CopyToTP(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, tp):
        ctx.tp = tp
        return x.view_as(x)

    @staticmethod
    def backward(ctx, g):
        return ctx.tp.all_reduce(g), None


class _ReduceScatterToSP(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, tp):
        ctx.tp = tp
        return tp.reduce_scatter(x)

    @staticmethod
    def backward(ctx, g):
        return ctx.tp.all_gather(g), None


class _GatherFromSP(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, tp):
        ctx.tp = tp
        return tp.all_gather(x)

    @staticmethod
    def backward(ctx, g):
        return ctx.tp.reduce_scatter(g), None


def reduce_from_tp(x, tp: TpContext):
    return _ReduceFromTP.apply(x, tp)


def copy_to_tp(x, tp: TpContext):
    return _CopyToTP.apply(x, tp)


def reduce_scatter_to_sp(x, tp: TpContext):
    return _ReduceScatterToSP.apply(x, tp)


def gather_from_sp(x, tp: TpContext):
    return _GatherFromSP.apply(x, tp)


class ColumnParallelLinear(torch.nn.Module):
    """Y_local = X W_local^T (W split by output features).  Input enters the TP region through
    copy_to_tp (backward: compressed all-reduce of dX), or, with sequence parallelism, through
    gather_from_sp (the SP all-gather of the token slices)."""

    def __init__(self, in_features, out_features_per_rank, tp: TpContext, sequence_parallel=False, bias=False,
                 device=None, dtype=None):
        super().__init__()
        self.tp, self.sp = tp, sequence_parallel
        self.linear = torch.nn.Linear(in_features, out_features_per_rank, bias=bias, device=device, dtype=dtype)

    def forward(self, x):
        x = gather_from_sp(x, self.tp) if self.sp else copy_to_tp(x, self.tp)
        return self.linear(x)


class RowParallelLinear(torch.nn.Module):
    """Y = sum_ranks X_local W_local^T (W split by input features): the partial products are
    combined with the compressed all-reduce (or the SP reduce-scatter)."""

    def __init__(self, in_features_per_rank, out_features, tp: TpContext, sequence_parallel=False, bias=False,
                 device=None, dtype=None):
        super().__init__()
        self.tp, self.sp = tp, sequence_parallel
        self.linear = torch.nn.Linear(in_features_per_rank, out_features, bias=False, device=device, dtype=dtype)
        self.bias = torch.nn.Parameter(torch.zeros(out_features, device=device, dtype=dtype)) if bias else None

    def forward(self, x):
        y = self.linear(x)
        y = reduce_scatter_to_sp(y, self.tp) if self.sp else reduce_from_tp(y, self.tp)
        return y + self.bias if self.bias is not None else y


# ------------------------------------------------------------- torch.library ops ---
def _register_ops():
    """taco_b200::compress / decompress as torch custom ops (opaque to torch.compile)."""
    from . import codec as dev

    @torch.library.custom_op("taco_b200::compress", mutates_args=())
    def compress_op(x: torch.Tensor, block_size: int, fmt: int) -> torch.Tensor:
        return dev.compress(x, _abi.make_config(block_size, fmt))[0].clone()

    @compress_op.register_fake
    def _(x, block_size, fmt):
        n = x.numel()
        m = -(-n // block_size)
        return x.new_empty(_abi.msg_layout(_abi.make_config(block_size, fmt), m).msg_stride, dtype=torch.uint8)

    @torch.library.custom_op("taco_b200::decompress", mutates_args=())
    def decompress_op(msg: torch.Tensor, n: int, block_size: int, fmt: int, out_dtype: torch.dtype) -> torch.Tensor:
        return dev.decompress(msg.view(1, -1), n, _abi.make_config(block_size, fmt), out_dtype=out_dtype)

    @decompress_op.register_fake
    def _(msg, n, block_size, fmt, out_dtype):
        return msg.new_empty(n, dtype=out_dtype)

    return compress_op, decompress_op


try:
    compress_op, decompress_op = _register_ops()
except Exception:  # already registered (module reload) or an older torch without custom_op
    compress_op = decompress_op = None
