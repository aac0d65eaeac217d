"""Torch-facing device API of the TACO codec (K1 / K2 / K3) over the C ABI.

Mirrors the reference's operator API (proj/include/taco/codec.hpp:57-62):
``compress`` / ``decompress`` keep their names and argument meaning, but take
and return CUDA tensors and never leave the device.  Messages are uint8 CUDA
tensors laid out as include/taco_b200.h documents (codes, then (alpha, scale)).
Errors raise TacoError with the reference's code and message; data-dependent
ones (NaN/Inf input, bad scalars) are raised when ``check`` synchronises.

torch is plumbing only: device memory, the current stream, dtypes.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _abi
from ._abi import (ASH_INT8, DIRECT_FP8, DT_BF16, DT_F32, E4M3, E5M2, GLOBAL_MAX, IDENTITY,  # noqa: F401
                   INT8_UNIFORM, PER_BLOCK_MAX, TACO, UNIT, Config, TacoError, make_config)

_DT = {torch.float32: DT_F32, torch.bfloat16: DT_BF16}


def _dtype_code(t: torch.dtype) -> int:
    try:
        return _DT[t]
    except KeyError:
        raise TacoError(_abi.ERR_USAGE, f"unsupported element dtype {t} (float32 or bfloat16)") from None


def _stream(stream) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _require_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise TacoError(_abi.ERR_USAGE, "tensors must live on a CUDA device (no CPU fallback)")


def cdiv(a: int, b: int) -> int:
    return -(-a // b)


def _require_buffer(t: torch.Tensor, what: str, min_numel: int, dtype=None, device=None) -> None:
    """Caller-supplied buffers are forwarded to the kernels as raw pointers: check that they
    are dense, large enough, of the right dtype and on the right device before any launch
    (an undersized buffer would otherwise be an out-of-bounds device access)."""
    if not t.is_contiguous():
        raise TacoError(_abi.ERR_USAGE, f"{what} must be contiguous")
    if dtype is not None and t.dtype != dtype:
        raise TacoError(_abi.ERR_USAGE, f"{what} must be {dtype}, got {t.dtype}")
    if device is not None and t.device != device:
        raise TacoError(_abi.ERR_USAGE, f"{what} must live on {device}, got {t.device}")
    if t.numel() < min_numel:
        raise TacoError(_abi.ERR_USAGE, f"{what} holds {t.numel()} elements, needs {min_numel}")


def generate(kind: int, n: int, seed: int, dense_sigma: float = 1e-3, tail_sigma: float = 1.0,
             tail_fraction: float = 0.01) -> torch.Tensor:
    """taco::generate (analysis.hpp:40): the reference's synthetic tensor, value for value
    (kind 0 Gaussian, 1 near-zero mixture), as a CPU float32 tensor (SURVEY §8d inputs)."""
    out = torch.empty(int(n), dtype=torch.float32)
    _abi.check(_abi.lib().taco_generate_host(int(kind), int(n), int(seed), float(dense_sigma), float(tail_sigma),
                                             float(tail_fraction), _ptr(out)))
    return out


GAUSSIAN, NEAR_ZERO_MIXTURE = 0, 1


@dataclass
class Geometry:
    """Shard / block / message geometry of one call (collective.cpp:76-87)."""

    n: int
    shards: int
    block_size: int

    @property
    def shard_len(self) -> int:
        return cdiv(self.n, self.shards)

    @property
    def blocks(self) -> int:
        return cdiv(self.shard_len, self.block_size)

    def layout(self, cfg: Config, nblocks: int | None = None) -> _abi.Layout:
        return _abi.msg_layout(cfg, self.blocks if nblocks is None else nblocks)


class Flags:
    """A device int of error flags (TACO_FLAG_*), checked on demand."""

    def __init__(self, device=None):
        self.t = torch.zeros(1, dtype=torch.int32, device=device or "cuda")

    def ptr(self):
        return C.c_void_p(self.t.data_ptr())

    def reset(self):
        self.t.zero_()

    def check(self):
        _abi.check(_abi.lib().taco_flags_status(int(self.t.item())))


def compress(x: torch.Tensor, cfg: Config, shards: int = 1, blk: tuple[int, int] | None = None,
             out: torch.Tensor | None = None, flags: Flags | None = None, stream=None) -> torch.Tensor:
    """K1: taco::compress of a CUDA tensor (flattened), cut into ``shards`` shards.

    Returns a uint8 tensor [shards, msg_stride] (message p = shard p)."""
    _require_cuda(x)
    x = x.reshape(-1)
    if not x.is_contiguous():
        x = x.contiguous()
    n = x.numel()
    g = Geometry(n, shards, cfg.block_size)
    b0, b1 = blk if blk is not None else (0, g.blocks if n else 0)
    lay = _abi.msg_layout(cfg, b1 - b0)
    if out is None:
        out = torch.empty((shards, lay.msg_stride), dtype=torch.uint8, device=x.device)
    _require_cuda(out)
    _require_buffer(out, "compress out", (shards - 1) * lay.msg_stride + lay.msg_bytes, torch.uint8, x.device)
    _abi.check(_abi.lib().taco_compress_dev(C.byref(cfg), _ptr(x), _dtype_code(x.dtype), n, shards, b0, b1,
                                            _ptr(out), lay.msg_stride, flags.ptr() if flags else None,
                                            C.c_void_p(_stream(stream))))
    return out


def decompress(msgs: torch.Tensor, n: int, cfg: Config, shards: int = 1, out_dtype=torch.float32,
               blk: tuple[int, int] | None = None, out: torch.Tensor | None = None,
               flags: Flags | None = None, stream=None, msg_stride: int | None = None) -> torch.Tensor:
    """K2: taco::decompress of ``shards`` messages into a flat tensor of n elements."""
    _require_cuda(msgs)
    g = Geometry(n, shards, cfg.block_size)
    b0, b1 = blk if blk is not None else (0, g.blocks if n else 0)
    lay = _abi.msg_layout(cfg, b1 - b0)
    stride = msg_stride if msg_stride is not None else lay.msg_stride
    if not msgs.is_contiguous() or msgs.dtype != torch.uint8:
        raise TacoError(_abi.ERR_USAGE, "messages must be a contiguous uint8 tensor")
    if msgs.numel() < (shards - 1) * stride + lay.msg_bytes:
        # codec.cpp:272-273: the message holds fewer blocks than the declared length needs
        raise TacoError(_abi.ERR_CORRUPT, "block count does not match the declared length")
    if out is None:
        out = torch.empty(n, dtype=out_dtype, device=msgs.device)
    _require_cuda(out)
    _require_buffer(out, "decompress out", n, device=msgs.device)
    _abi.check(_abi.lib().taco_decompress_dev(C.byref(cfg), _ptr(msgs), stride, shards, n, b0, b1, _ptr(out),
                                              _dtype_code(out.dtype), flags.ptr() if flags else None,
                                              C.c_void_p(_stream(stream))))
    return out


def reduce_encode(msgs: torch.Tensor, nranks: int, shard_len: int, cfg: Config, rank_stride: int,
                  out_msg: torch.Tensor | None, acc_out: torch.Tensor | None = None,
                  blk: tuple[int, int] | None = None, flags: Flags | None = None, stream=None) -> torch.Tensor:
    """K3: ascending-rank fp32 sum of ``nranks`` decoded messages of one shard, re-encoded.

    ``msgs`` points at rank 0's message; rank r's is ``rank_stride`` bytes further."""
    _require_cuda(msgs, out_msg, acc_out)
    m = cdiv(shard_len, cfg.block_size)
    b0, b1 = blk if blk is not None else (0, m)
    lay = _abi.msg_layout(cfg, b1 - b0)
    _require_buffer(msgs, "reduce_encode messages", (nranks - 1) * rank_stride + lay.msg_bytes, torch.uint8)
    if out_msg is not None:
        _require_buffer(out_msg, "reduce_encode out_msg", lay.msg_bytes, torch.uint8, msgs.device)
    if acc_out is not None:
        _require_buffer(acc_out, "reduce_encode acc_out", min(shard_len, b1 * cfg.block_size), device=msgs.device)
    _abi.check(_abi.lib().taco_reduce_encode_dev(
        C.byref(cfg), _ptr(msgs), rank_stride, nranks, shard_len, b0, b1, _ptr(out_msg), _ptr(acc_out),
        _dtype_code(acc_out.dtype) if acc_out is not None else DT_F32, flags.ptr() if flags else None,
        C.c_void_p(_stream(stream))))
    return out_msg


def allreduce_sim(inputs: torch.Tensor, cfg: Config, out_dtype=torch.float32, stage1: torch.Tensor | None = None,
                  flags: Flags | None = None, stream=None) -> torch.Tensor:
    """taco::allreduce(RankSet{TwoShot}) with all P ranks on this device: inputs [P, n]."""
    _require_cuda(inputs, stage1)
    p, n = inputs.shape
    inputs = inputs.contiguous()
    ws = torch.empty(max(1, _abi.lib().taco_allreduce_sim_workspace(C.byref(cfg), p, n)), dtype=torch.uint8,
                     device=inputs.device)
    out = torch.empty(n, dtype=out_dtype, device=inputs.device)
    _abi.check(_abi.lib().taco_allreduce_sim_dev(C.byref(cfg), _ptr(inputs), _dtype_code(inputs.dtype), p, n,
                                                 _ptr(out), _dtype_code(out_dtype), _ptr(stage1), _ptr(ws),
                                                 flags.ptr() if flags else None, C.c_void_p(_stream(stream))))
    return out


def scaled_spectrum(x: torch.Tensor, cfg: Config, flags: Flags | None = None, stream=None) -> torch.Tensor:
    """taco::scaled_spectrum (codec.hpp:70): Z/s of every block slot, ceil(n/B)*B fp32 values."""
    _require_cuda(x)
    x = x.reshape(-1).contiguous()
    n = x.numel()
    out = torch.empty(cdiv(n, cfg.block_size) * cfg.block_size, dtype=torch.float32, device=x.device)
    _abi.check(_abi.lib().taco_scaled_spectrum_dev(C.byref(cfg), _ptr(x), _dtype_code(x.dtype), n, _ptr(out),
                                                   flags.ptr() if flags else None, C.c_void_p(_stream(stream))))
    return out


def archive_export(msg: torch.Tensor, n: int, cfg: Config, stream=None) -> torch.Tensor:
    """taco::archive_bytes (serialize.hpp:15) of one message: a uint8 CUDA tensor of
    taco_archive_size bytes (TACOCMP1 header + [payload][alpha][scale] per block)."""
    _require_cuda(msg)
    size = _abi.lib().taco_archive_size(C.byref(cfg), n)
    out = torch.empty(size, dtype=torch.uint8, device=msg.device)
    _abi.check(_abi.lib().taco_archive_export_dev(C.byref(cfg), _ptr(msg), n, _ptr(out),
                                                  C.c_void_p(_stream(stream))))
    return out


def archive_import(archive: torch.Tensor, flags: Flags | None = None, stream=None):
    """taco::archive_parse (serialize.hpp:16): (config, n, message) from a TACOCMP1 byte
    stream held in a uint8 CUDA tensor; every malformed input raises the reference's error."""
    _require_cuda(archive)
    size = archive.numel()
    head = archive[: min(size, 22)].cpu().numpy().tobytes()
    hb = (C.c_uint8 * 22).from_buffer_copy(head + bytes(22 - len(head)))
    cfg, n = Config(), C.c_uint64()
    rc = _abi.lib().taco_archive_parse_header(C.cast(hb, C.c_void_p), size, C.byref(cfg), C.byref(n))
    if rc != _abi.OK:
        msg = _abi.lib().taco_last_error().decode()
        if msg == "unexpected end of archive" and n.value and size > 22:
            # the reference reads blocks in order: a bad scalar before the cut wins
            _scan_scalars(archive.cpu().numpy(), cfg, (size - 22) // (_payload(cfg) + 8))
        raise TacoError(rc, msg)
    msg = torch.empty(_abi.msg_layout(cfg, cdiv(n.value, cfg.block_size)).msg_stride, dtype=torch.uint8,
                      device=archive.device)
    own = flags or Flags(archive.device)
    _abi.check(_abi.lib().taco_archive_import_dev(C.byref(cfg), _ptr(archive), n.value, _ptr(msg), own.ptr(),
                                                  C.c_void_p(_stream(stream))))
    if flags is None and int(own.t.item()) & _abi.FLAG_BAD_SCALARS:
        raise TacoError(_abi.ERR_CORRUPT, "block scalars must be finite")
    return cfg, n.value, msg


def _payload(cfg: Config) -> int:
    return 4 * cfg.block_size if cfg.kind == IDENTITY else cfg.block_size


def _scan_scalars(raw, cfg: Config, complete: int) -> None:
    import numpy as np
    rec = _payload(cfg) + 8
    for k in range(complete):
        at = 22 + k * rec + _payload(cfg)
        ab = np.frombuffer(raw[at: at + 8].tobytes(), np.float32)
        if not np.all(np.isfinite(ab)):
            raise TacoError(_abi.ERR_CORRUPT, "block scalars must be finite")


def error_report(original: torch.Tensor, reconstructed: torch.Tensor, bins: int = 64, stream=None) -> dict:
    """taco::error_report (analysis.hpp:42) on the device: mse, relative_l2, max_abs_error,
    zero_collapse_fraction, kurtosis (excess, of the elementwise error), histogram."""
    _require_cuda(original, reconstructed)
    x, y = original.reshape(-1).contiguous(), reconstructed.reshape(-1).contiguous()
    if x.numel() != y.numel():
        raise TacoError(_abi.ERR_INPUT, "original and reconstructed lengths differ")
    rep = _abi.ErrorReportC()
    counts = (C.c_uint64 * max(bins, 1))()
    _abi.check(_abi.lib().taco_error_report_dev(_ptr(x), _dtype_code(x.dtype), _ptr(y), _dtype_code(y.dtype),
                                                x.numel(), bins, C.byref(rep), C.cast(counts, C.c_void_p),
                                                C.c_void_p(_stream(stream))))
    width = (rep.hist_hi - rep.hist_lo) / bins
    edges = [rep.hist_lo + width * i for i in range(bins)] + [rep.hist_hi]
    return {"mse": rep.mse, "relative_l2": rep.relative_l2, "max_abs_error": rep.max_abs_error,
            "zero_collapse_fraction": rep.zero_collapse_fraction,
            "kurtosis": rep.kurtosis if rep.kurtosis_defined else float("nan"),
            "kurtosis_defined": bool(rep.kurtosis_defined), "bin_edges": edges, "counts": list(counts)}


def split_message(msg: torch.Tensor, cfg: Config, nblocks: int):
    """(codes [nblocks*payload] uint8, alpha [nblocks] f32, scale [nblocks] f32) views of one message."""
    lay = _abi.msg_layout(cfg, nblocks)
    codes = msg[: lay.codes_bytes]
    scal = msg[lay.scal_offset: lay.scal_offset + 8 * nblocks].view(torch.float32).view(nblocks, 2)
    return codes, scal[:, 0], scal[:, 1]


class HostContext:
    """taco_ctx: synchronous host-buffer API (the shape of the reference's calls)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _abi.check(_abi.lib().taco_ctx_create(device, C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            _abi.lib().taco_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _host(t: torch.Tensor, what: str, numel: int | None = None) -> None:
        if t.is_cuda:
            raise TacoError(_abi.ERR_USAGE, f"{what} must be a host (CPU) tensor")
        if not t.is_contiguous():
            raise TacoError(_abi.ERR_USAGE, f"{what} must be contiguous")
        if numel is not None and t.numel() != numel:
            raise TacoError(_abi.ERR_USAGE, f"{what} holds {t.numel()} elements, expected {numel}")

    def roundtrip(self, x: torch.Tensor, cfg: Config, out: torch.Tensor) -> torch.Tensor:
        """compress -> decompress of a host tensor; out is a host tensor of x's size."""
        self._host(x, "roundtrip input")
        self._host(out, "roundtrip out", x.numel())
        _abi.check(_abi.lib().taco_roundtrip_host(self.h, C.byref(cfg), _ptr(x), _dtype_code(x.dtype), x.numel(),
                                                  _ptr(out), _dtype_code(out.dtype)))
        return out

    def compress(self, x: torch.Tensor, cfg: Config) -> torch.Tensor:
        self._host(x, "compress input")
        m = cdiv(x.numel(), cfg.block_size)
        msg = torch.empty(_abi.msg_layout(cfg, m).msg_bytes, dtype=torch.uint8)
        _abi.check(_abi.lib().taco_compress_host(self.h, C.byref(cfg), _ptr(x), _dtype_code(x.dtype), x.numel(),
                                                 _ptr(msg)))
        return msg

    def decompress(self, msg: torch.Tensor, n: int, cfg: Config, out_dtype=torch.float32) -> torch.Tensor:
        self._host(msg, "compressed message")
        if msg.dtype != torch.uint8 or msg.numel() < _abi.msg_layout(cfg, cdiv(n, cfg.block_size)).msg_bytes:
            raise TacoError(_abi.ERR_CORRUPT, "block count does not match the declared length")
        out = torch.empty(n, dtype=out_dtype)
        _abi.check(_abi.lib().taco_decompress_host(self.h, C.byref(cfg), _ptr(msg), n, _ptr(out),
                                                   _dtype_code(out_dtype)))
        return out

    def allreduce_sim(self, inputs: torch.Tensor, cfg: Config, want_stage1: bool = False):
        self._host(inputs, "rank inputs")
        if inputs.dtype != torch.float32:
            raise TacoError(_abi.ERR_USAGE, "rank inputs must be float32 (taco::RankSet)")
        p, n = inputs.shape
        res = torch.empty(n, dtype=torch.float32)
        st = torch.empty(p * cdiv(n, p), dtype=torch.float32) if want_stage1 else None
        _abi.check(_abi.lib().taco_allreduce_sim_host(self.h, C.byref(cfg), _ptr(inputs.contiguous()), p, n,
                                                      _ptr(res), _ptr(st)))
        return (res, st) if want_stage1 else res

    def allreduce(self, inputs: torch.Tensor, cfg: Config, algorithm: int = 0):
        """taco::allreduce(RankSet) for Algorithm 0 TwoShot / 1 Ring / 2 Tree on host rank tensors
        [P][n] f32, computed on the device: (result, exact, relative_l2)."""
        self._host(inputs, "rank inputs")
        if inputs.dtype != torch.float32 or inputs.dim() != 2:
            raise TacoError(_abi.ERR_USAGE, "rank inputs must be a [P][n] float32 tensor (taco::RankSet)")
        p, n = inputs.shape
        res = torch.empty(n, dtype=torch.float32)
        exact = torch.empty(n, dtype=torch.float32)
        rel = C.c_double(0.0)
        _abi.check(_abi.lib().taco_allreduce_schedule_host(self.h, C.byref(cfg), int(algorithm),
                                                           _ptr(inputs.contiguous()), p, n, _ptr(res), _ptr(exact),
                                                           C.byref(rel)))
        return res, exact, rel.value
