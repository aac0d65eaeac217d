"""ctypes binding of libtaco_b200.so (include/taco_b200.h).

This is the Python face of the drop-in boundary: the same C ABI the C++ layer
(include/taco/*.hpp) and the NCCL collective driver use.  Loading fails loudly
when the library was not built -- there is no CPU fallback anywhere in the
package.
"""
from __future__ import annotations

import ctypes as C
import os
import re

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TACO_B200_LIB") or os.path.join(PKG_DIR, "libtaco_b200.so")  # override: A/B builds
HEADER = os.path.join(os.path.dirname(PKG_DIR), "include", "taco_b200.h")

OK, ERR_USAGE, ERR_CONFIG, ERR_INPUT, ERR_IO, ERR_CORRUPT, ERR_CUDA = range(7)
DT_F32, DT_BF16 = 0, 1
E4M3, E5M2 = 0, 1
# taco::CodecKind (codec.hpp:11-17) and DirectScaleScope (codec.hpp:22)
TACO, DIRECT_FP8, INT8_UNIFORM, IDENTITY, ASH_INT8 = range(5)
GLOBAL_MAX, UNIT, PER_BLOCK_MAX = range(3)
FLAG_NONFINITE_INPUT, FLAG_BAD_SCALARS, FLAG_PEER_TIMEOUT = 1, 2, 4
MAX_PEERS = 8

# taco::ErrorCode names (proj/include/taco/error.hpp:10-16)
ERROR_NAMES = {ERR_USAGE: "usage", ERR_CONFIG: "config", ERR_INPUT: "input", ERR_IO: "io",
               ERR_CORRUPT: "corrupt", ERR_CUDA: "cuda"}


class TacoError(RuntimeError):
    """Mirror of taco::Error: ``code`` is the ErrorCode name, str(e) the reference message."""

    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status
        self.code = ERROR_NAMES.get(status, str(status))


class Config(C.Structure):
    """taco_config == taco::CodecConfig (proj/include/taco/codec.hpp:24-33)."""

    _fields_ = [("block_size", C.c_uint32), ("target_energy", C.c_float),
                ("stability_epsilon", C.c_float), ("format", C.c_uint32), ("kind", C.c_uint32),
                ("direct_scale", C.c_uint32)]

    def __repr__(self):
        return (f"Config(block_size={self.block_size}, target_energy={self.target_energy}, "
                f"stability_epsilon={self.stability_epsilon}, format={self.format}, kind={self.kind}, "
                f"direct_scale={self.direct_scale})")


class ErrorReportC(C.Structure):
    """taco_error_report == taco::ErrorReport (analysis.hpp:18-26) without the histogram vectors."""

    _fields_ = [("mse", C.c_double), ("relative_l2", C.c_double), ("max_abs_error", C.c_double),
                ("zero_collapse_fraction", C.c_double), ("kurtosis", C.c_double), ("kurtosis_defined", C.c_int),
                ("hist_lo", C.c_double), ("hist_hi", C.c_double)]


class Layout(C.Structure):
    _fields_ = [("nblocks", C.c_uint64), ("codes_bytes", C.c_uint64), ("scal_offset", C.c_uint64),
                ("msg_bytes", C.c_uint64), ("msg_stride", C.c_uint64)]


class IpcHandle(C.Structure):
    """taco_ipc_handle (cudaIpcMemHandle_t bytes, exchanged between ranks)."""

    _fields_ = [("bytes", C.c_ubyte * 64)]


class Peers(C.Structure):
    """taco_peers: rank q's peer region as mapped in this process, q < nranks."""

    _fields_ = [("nranks", C.c_uint32), ("rank", C.c_uint32), ("base", C.c_void_p * MAX_PEERS)]


def make_config(block_size=256, fmt=E4M3, target_energy=1.0, stability_epsilon=1e-12, kind=TACO,
                direct_scale=GLOBAL_MAX) -> Config:
    return Config(int(block_size), float(target_energy), float(stability_epsilon), int(fmt), int(kind),
                  int(direct_scale))


_P, _U64, _U32, _I = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int

_SIGNATURES = {
    "taco_abi_version": (C.c_int, []),
    "taco_last_error": (C.c_char_p, []),
    "taco_default_config": (Config, []),
    "taco_validate_config": (C.c_int, [C.POINTER(Config)]),
    "taco_msg_layout": (C.c_int, [C.POINTER(Config), _U64, C.POINTER(Layout)]),
    "taco_compressed_ratio": (C.c_double, [C.POINTER(Config), _U64]),
    "taco_archive_size": (_U64, [C.POINTER(Config), _U64]),
    "taco_flags_status": (C.c_int, [C.c_int]),
    "taco_compress_dev": (C.c_int, [C.POINTER(Config), _P, _I, _U64, _U32, _U64, _U64, _P, _U64, _P, _P]),
    "taco_decompress_dev": (C.c_int, [C.POINTER(Config), _P, _U64, _U32, _U64, _U64, _U64, _P, _I, _P, _P]),
    "taco_reduce_encode_dev": (C.c_int, [C.POINTER(Config), _P, _U64, _U32, _U64, _U64, _U64, _P, _P, _I,
                                         _P, _P]),
    "taco_reduce_encode_ptrs_dev": (C.c_int, [C.POINTER(Config), C.POINTER(C.c_void_p), _U32, _U64, _U64, _U64, _P,
                                              _P, _I, _P, _P]),
    "taco_allreduce_sim_workspace": (_U64, [C.POINTER(Config), _U32, _U64]),
    "taco_allreduce_sim_dev": (C.c_int, [C.POINTER(Config), _P, _I, _U32, _U64, _P, _I, _P, _P, _P, _P]),
    "taco_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "taco_ctx_destroy": (None, [_P]),
    "taco_compress_host": (C.c_int, [_P, C.POINTER(Config), _P, _I, _U64, _P]),
    "taco_decompress_host": (C.c_int, [_P, C.POINTER(Config), _P, _U64, _P, _I]),
    "taco_roundtrip_host": (C.c_int, [_P, C.POINTER(Config), _P, _I, _U64, _P, _I]),
    "taco_allreduce_sim_host": (C.c_int, [_P, C.POINTER(Config), _P, _U32, _U64, _P, _P]),
    "taco_allreduce_schedule_host": (C.c_int, [_P, C.POINTER(Config), C.c_int, _P, _U32, _U64, _P, _P, _P]),
    "taco_scaled_spectrum_dev": (C.c_int, [C.POINTER(Config), _P, _I, _U64, _P, _P, _P]),
    "taco_archive_header": (C.c_int, [C.POINTER(Config), _U64, _P]),
    "taco_archive_export_dev": (C.c_int, [C.POINTER(Config), _P, _U64, _P, _P]),
    "taco_archive_parse_header": (C.c_int, [_P, _U64, C.POINTER(Config), C.POINTER(C.c_uint64)]),
    "taco_archive_import_dev": (C.c_int, [C.POINTER(Config), _P, _U64, _P, _P, _P]),
    "taco_scaled_spectrum_host": (C.c_int, [_P, C.POINTER(Config), _P, _U64, _P]),
    "taco_error_report_dev": (C.c_int, [_P, _I, _P, _I, _U64, _U32, C.POINTER(ErrorReportC), _P, _P]),
    "taco_collective_nccl_workspace": (_U64, [C.POINTER(Config), _U32, _U64]),
    "taco_allreduce_nccl": (C.c_int, [C.POINTER(Config), _P, _I, _U64, _P, _I, _P, _P, _P, _P]),
    "taco_reduce_scatter_nccl": (C.c_int, [C.POINTER(Config), _P, _I, _U64, _P, _I, _P, _P, _P, _P]),
    "taco_all_gather_nccl": (C.c_int, [C.POINTER(Config), _P, _I, _U64, _P, _I, _P, _P, _P, _P]),
    "taco_peer_fused_supported": (C.c_int, [C.POINTER(Config)]),
    "taco_peer_check_access": (C.c_int, [C.c_int, C.c_int]),
    "taco_peer_allreduce_dev": (C.c_int, [C.POINTER(Config), _P, _I, _U64, _P, _U64, _U64, _U64, _U64, _P, _I, _U32,
                                          _P, _P]),
    "taco_peer_reduce_scatter_dev": (C.c_int, [C.POINTER(Config), _P, _I, _U64, _P, _U64, _U64, _U64, _P, _I, _U32,
                                               _P, _P]),
    "taco_peer_all_gather_dev": (C.c_int, [C.POINTER(Config), _P, _I, _U64, _P, _U64, _U64, _U64, _P, _I, _U32,
                                           _P, _P]),
    "taco_collective_nccl_workspace_chunked": (_U64, [C.POINTER(Config), _U32, _U64, _U32]),
    "taco_allreduce_nccl_chunked": (C.c_int, [C.POINTER(Config), _P, _I, _U64, _P, _I, _P, _P, _P, _P, _U32]),
    "taco_reduce_scatter_nccl_chunked": (C.c_int, [C.POINTER(Config), _P, _I, _U64, _P, _I, _P, _P, _P, _P, _U32]),
    "taco_all_gather_nccl_chunked": (C.c_int, [C.POINTER(Config), _P, _I, _U64, _P, _I, _P, _P, _P, _P, _U32]),
    "taco_peer_alloc": (C.c_int, [_I, _U64, C.POINTER(C.c_void_p), C.POINTER(IpcHandle)]),
    "taco_peer_open": (C.c_int, [_I, C.POINTER(IpcHandle), C.POINTER(C.c_void_p)]),
    "taco_peer_close": (C.c_int, [_P]),
    "taco_peer_free": (C.c_int, [_P]),
    "taco_peer_flags_bytes": (_U64, []),
    "taco_peer_barrier_dev": (C.c_int, [C.POINTER(Peers), _U64, _U32, _P, _P]),
    "taco_compress_push_dev": (C.c_int, [C.POINTER(Config), _P, _I, _U64, C.POINTER(Peers), _U64, _U64, _U64,
                                         _U64, _P, _P]),
    "taco_compress_bcast_dev": (C.c_int, [C.POINTER(Config), _P, _I, _U64, C.POINTER(Peers), _U64, _U64, _U64,
                                          _U64, _P, _P]),
    "taco_reduce_encode_push_dev": (C.c_int, [C.POINTER(Config), _P, _U64, C.POINTER(Peers), _U64, _U64, _U64,
                                              _U64, _U64, _P, _I, _P, _P]),
    "taco_fp8_encode_dev": (C.c_int, [_P, _U64, _I, _P, _P]),
    "taco_fp8_decode_dev": (C.c_int, [_P, _U64, _I, _P, _P]),
    "taco_generate_host": (C.c_int, [_I, _U64, _U64, C.c_double, C.c_double, C.c_double, _P]),
}

_lib = None


def header_symbols() -> list[str]:
    """Every function the C header declares (for the export check)."""
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(taco_[a-z0-9_]+)\s*\(", src)))


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: the CUDA extension was not built "
                               "(run `python -c 'import __graft_entry__ as g; g.build()'`). "
                               "There is no CPU fallback.")
        handle = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(rc: int) -> None:
    if rc != OK:
        raise TacoError(rc, lib().taco_last_error().decode())


def msg_layout(cfg: Config, nblocks: int) -> Layout:
    out = Layout()
    check(lib().taco_msg_layout(C.byref(cfg), int(nblocks), C.byref(out)))
    return out
