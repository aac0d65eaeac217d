"""ctypes face of the test oracles -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl
reference` leg may import this module.  Two oracles are exposed:

* ``Port``  -- oracle/_build/libtaco_oracle.so, the plain-C restatement
  (taco_oracle.c) of the reference codec path.
* ``Ref``   -- oracle/_ref/libtaco_ref.so, the unmodified reference sources
  (/root/reference/proj/src) compiled by oracle/Makefile behind ref_shim.cpp.

Both operate on numpy float32 / uint8 arrays.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libtaco_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtaco_ref.so")

E4M3, E5M2 = 0, 1
QMAX = {E4M3: 448.0, E5M2: 57344.0}
ERROR_NAMES = {1: "usage", 2: "config", 3: "input", 4: "io", 5: "corrupt"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = ERROR_NAMES.get(code, str(code))


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _f32p(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _u8p(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def _f32(x):
    return np.ascontiguousarray(x, dtype=np.float32)


class _Cfg(C.Structure):
    _fields_ = [("block_size", C.c_uint32), ("target_energy", C.c_float),
                ("stability_epsilon", C.c_float), ("format", C.c_int)]


class Port:
    """The C restatement (oracle/taco_oracle.c)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build()
        lib = C.CDLL(path)
        lib.tor_last_error.restype = C.c_char_p
        lib.tor_fp8_encode.restype = C.c_uint8
        lib.tor_fp8_encode.argtypes = [C.c_float, C.c_int]
        lib.tor_gaussian.argtypes = [C.c_size_t, C.c_uint64, C.c_double, C.POINTER(C.c_float)]
        lib.tor_mixture.argtypes = [C.c_size_t, C.c_uint64, C.c_double, C.c_double, C.c_double,
                                    C.POINTER(C.c_float)]
        lib.tor_compress.argtypes = [C.POINTER(C.c_float), C.c_size_t, C.POINTER(_Cfg),
                                     C.POINTER(C.c_uint8), C.POINTER(C.c_float), C.POINTER(C.c_float)]
        lib.tor_decompress.argtypes = [C.POINTER(C.c_uint8), C.POINTER(C.c_float),
                                       C.POINTER(C.c_float), C.c_size_t, C.POINTER(_Cfg),
                                       C.POINTER(C.c_float)]
        lib.tor_allreduce_twoshot.argtypes = [C.POINTER(C.c_float), C.c_size_t, C.c_size_t,
                                              C.POINTER(_Cfg), C.POINTER(C.c_float),
                                              C.POINTER(C.c_float), C.POINTER(C.c_float),
                                              C.POINTER(C.c_uint64)]
        lib.tor_fwht_inplace.argtypes = [C.POINTER(C.c_double), C.c_size_t]
        lib.tor_fp8_decode_table.argtypes = [C.c_int, C.POINTER(C.c_float)]
        self.lib = lib

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.lib.tor_last_error().decode())

    @staticmethod
    def cfg(block_size=256, fmt=E4M3, tau=1.0, eps=1e-12):
        return _Cfg(block_size, tau, eps, fmt)

    def encode(self, x: float, fmt=E4M3) -> int:
        return int(self.lib.tor_fp8_encode(float(x), fmt))

    def decode_table(self, fmt=E4M3) -> np.ndarray:
        t = np.zeros(256, np.float32)
        self.lib.tor_fp8_decode_table(fmt, _f32p(t))
        return t

    def fwht(self, v) -> np.ndarray:
        w = np.ascontiguousarray(v, dtype=np.float64).copy()
        self._check(self.lib.tor_fwht_inplace(w.ctypes.data_as(C.POINTER(C.c_double)), w.size))
        return w

    def gaussian(self, n, seed, sigma=1.0) -> np.ndarray:
        out = np.empty(n, np.float32)
        self.lib.tor_gaussian(n, seed, sigma, _f32p(out))
        return out

    def mixture(self, n, seed, dense_sigma=1e-3, tail_sigma=1.0, tail_fraction=0.01):
        out = np.empty(n, np.float32)
        self._check(self.lib.tor_mixture(n, seed, dense_sigma, tail_sigma, tail_fraction, _f32p(out)))
        return out

    def compress(self, x, block_size=256, fmt=E4M3, tau=1.0, eps=1e-12):
        x = _f32(x)
        m = -(-x.size // block_size) if block_size > 0 else 0
        codes = np.zeros(max(m, 1) * max(block_size, 1), np.uint8)
        al = np.zeros(max(m, 1), np.float32)
        sc = np.zeros(max(m, 1), np.float32)
        cfg = self.cfg(block_size, fmt, tau, eps)
        self._check(self.lib.tor_compress(_f32p(x), x.size, C.byref(cfg), _u8p(codes), _f32p(al),
                                          _f32p(sc)))
        return codes[: m * block_size], al[:m], sc[:m]

    def decompress(self, codes, alpha, scale, n, block_size=256, fmt=E4M3):
        codes = np.ascontiguousarray(codes, np.uint8)
        out = np.zeros(max(n, 1), np.float32)
        cfg = self.cfg(block_size, fmt)
        self._check(self.lib.tor_decompress(_u8p(codes), _f32p(_f32(alpha)), _f32p(_f32(scale)), n,
                                            C.byref(cfg), _f32p(out)))
        return out[:n]

    def allreduce_twoshot(self, inputs, block_size=256, fmt=E4M3, want_stage1=False):
        inputs = _f32(inputs)
        p, n = inputs.shape
        res = np.zeros(n, np.float32)
        exact = np.zeros(n, np.float32)
        shard = -(-n // p)
        st = np.zeros(p * shard, np.float32) if want_stage1 else None
        nbytes = C.c_uint64(0)
        cfg = self.cfg(block_size, fmt)
        self._check(self.lib.tor_allreduce_twoshot(
            _f32p(inputs), p, n, C.byref(cfg), _f32p(res), _f32p(exact),
            _f32p(st) if st is not None else None, C.byref(nbytes)))
        out = {"result": res, "exact": exact, "bytes_on_wire": nbytes.value}
        if want_stage1:
            out["stage1"] = st
        return out


class Ref:
    """The unmodified reference library (oracle/_ref/libtaco_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        lib = C.CDLL(path)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_worker_count.restype = C.c_uint
        lib.ref_set_threads.argtypes = [C.c_int]
        lib.ref_compress.argtypes = [C.POINTER(C.c_float), C.c_uint64, C.c_uint32, C.c_float,
                                     C.c_float, C.c_int, C.c_int, C.POINTER(C.c_uint8),
                                     C.POINTER(C.c_float), C.POINTER(C.c_float)]
        lib.ref_decompress.argtypes = [C.POINTER(C.c_uint8), C.POINTER(C.c_float),
                                       C.POINTER(C.c_float), C.c_uint64, C.c_uint32, C.c_int,
                                       C.c_int, C.POINTER(C.c_float)]
        lib.ref_roundtrip.argtypes = [C.POINTER(C.c_float), C.c_uint64, C.c_uint32, C.c_int,
                                      C.POINTER(C.c_float)]
        lib.ref_allreduce.argtypes = [C.POINTER(C.c_float), C.c_uint32, C.c_uint64, C.c_uint32,
                                      C.c_int, C.c_int, C.c_int, C.c_uint64,
                                      C.POINTER(C.c_float), C.POINTER(C.c_float),
                                      C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        lib.ref_generate.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_double, C.c_double,
                                     C.c_double, C.POINTER(C.c_float)]
        lib.ref_archive.argtypes = [C.POINTER(C.c_float), C.c_uint64, C.c_uint32, C.c_int,
                                    C.POINTER(C.c_uint8), C.c_uint64, C.POINTER(C.c_uint64)]
        lib.ref_archive_size.restype = C.c_uint64
        lib.ref_archive_size.argtypes = [C.c_uint32, C.c_int, C.c_uint64]
        lib.ref_compressed_ratio.restype = C.c_double
        lib.ref_compressed_ratio.argtypes = [C.c_uint32, C.c_int, C.c_uint64]
        lib.ref_compress2.argtypes = [C.POINTER(C.c_float), C.c_uint64, C.c_uint32, C.c_float, C.c_float,
                                      C.c_int, C.c_int, C.c_int, C.POINTER(C.c_uint8), C.POINTER(C.c_float),
                                      C.POINTER(C.c_float)]
        lib.ref_archive2.argtypes = [C.POINTER(C.c_float), C.c_uint64, C.c_uint32, C.c_int, C.c_int, C.c_int,
                                     C.POINTER(C.c_uint8), C.c_uint64, C.POINTER(C.c_uint64)]
        lib.ref_archive_decode.argtypes = [C.POINTER(C.c_uint8), C.c_uint64, C.POINTER(C.c_float), C.c_uint64,
                                           C.POINTER(C.c_uint64)]
        lib.ref_scaled_spectrum.argtypes = [C.POINTER(C.c_float), C.c_uint64, C.c_uint32, C.c_int, C.c_int,
                                            C.POINTER(C.c_float)]
        lib.ref_error_report.argtypes = [C.POINTER(C.c_float), C.POINTER(C.c_float), C.c_uint64, C.c_uint32,
                                         C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
        lib.ref_fp8_encode.restype = C.c_uint8
        lib.ref_fp8_encode.argtypes = [C.c_float, C.c_int]
        self.lib = lib

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def set_threads(self, t: int) -> None:
        self.lib.ref_set_threads(int(t))

    def worker_count(self) -> int:
        return int(self.lib.ref_worker_count())

    def encode(self, x, fmt=E4M3):
        return int(self.lib.ref_fp8_encode(float(x), fmt))

    def generate(self, kind, n, seed, dense_sigma=1e-3, tail_sigma=1.0, tail_fraction=0.01):
        out = np.empty(n, np.float32)
        self._check(self.lib.ref_generate(kind, n, seed, dense_sigma, tail_sigma, tail_fraction,
                                          _f32p(out)))
        return out

    def compress(self, x, block_size=256, fmt=E4M3, tau=1.0, eps=1e-12, kind=0):
        x = _f32(x)
        m = -(-x.size // block_size) if block_size > 0 else 0
        pay = 4 * block_size if kind == 3 else block_size
        codes = np.zeros(max(m * pay, 1), np.uint8)
        al = np.zeros(max(m, 1), np.float32)
        sc = np.zeros(max(m, 1), np.float32)
        self._check(self.lib.ref_compress(_f32p(x), x.size, block_size, tau, eps, fmt, kind,
                                          _u8p(codes), _f32p(al), _f32p(sc)))
        return codes[: m * pay], al[:m], sc[:m]

    def decompress(self, codes, alpha, scale, n, block_size=256, fmt=E4M3, kind=0):
        out = np.zeros(max(n, 1), np.float32)
        self._check(self.lib.ref_decompress(_u8p(np.ascontiguousarray(codes, np.uint8)),
                                            _f32p(_f32(alpha)), _f32p(_f32(scale)), n, block_size,
                                            fmt, kind, _f32p(out)))
        return out[:n]

    def roundtrip(self, x, out, block_size=256, fmt=E4M3):
        self._check(self.lib.ref_roundtrip(_f32p(x), x.size, block_size, fmt, _f32p(out)))

    def allreduce(self, inputs, block_size=256, fmt=E4M3, kind=0, algorithm=0, chunk=0):
        inputs = _f32(inputs)
        p, n = inputs.shape
        res = np.zeros(n, np.float32)
        exact = np.zeros(n, np.float32)
        steps, nbytes = C.c_uint64(0), C.c_uint64(0)
        self._check(self.lib.ref_allreduce(_f32p(inputs), p, n, block_size, fmt, kind, algorithm,
                                           chunk, _f32p(res), _f32p(exact), C.byref(steps),
                                           C.byref(nbytes)))
        return {"result": res, "exact": exact, "steps": steps.value, "bytes_on_wire": nbytes.value}

    def archive(self, x, block_size=256, fmt=E4M3) -> bytes:
        x = _f32(x)
        cap = 22 + (-(-x.size // block_size)) * (block_size + 8)
        buf = np.zeros(cap, np.uint8)
        size = C.c_uint64(0)
        self._check(self.lib.ref_archive(_f32p(x), x.size, block_size, fmt, _u8p(buf), cap,
                                         C.byref(size)))
        return buf[: size.value].tobytes()

    def compress2(self, x, block_size=256, fmt=E4M3, kind=0, scope=0, tau=1.0, eps=1e-12):
        """compress with the DirectFp8 scope (codec.hpp:22): codes (payload bytes), alpha, scale"""
        x = _f32(x)
        m = -(-x.size // block_size)
        pay = 4 * block_size if kind == 3 else block_size
        codes = np.zeros(max(m * pay, 1), np.uint8)
        al = np.zeros(max(m, 1), np.float32)
        sc = np.zeros(max(m, 1), np.float32)
        self._check(self.lib.ref_compress2(_f32p(x), x.size, block_size, tau, eps, fmt, kind, scope, _u8p(codes),
                                           _f32p(al), _f32p(sc)))
        return codes[: m * pay], al[:m], sc[:m]

    def archive2(self, x, block_size=256, fmt=E4M3, kind=0, scope=0) -> bytes:
        x = _f32(x)
        pay = 4 * block_size if kind == 3 else block_size
        cap = 22 + (-(-x.size // block_size)) * (pay + 8)
        buf = np.zeros(cap, np.uint8)
        size = C.c_uint64(0)
        self._check(self.lib.ref_archive2(_f32p(x), x.size, block_size, fmt, kind, scope, _u8p(buf), cap,
                                          C.byref(size)))
        return buf[: size.value].tobytes()

    def archive_decode(self, data: bytes, cap: int):
        raw = np.frombuffer(data, np.uint8).copy()
        out = np.zeros(max(cap, 1), np.float32)
        n = C.c_uint64(0)
        self._check(self.lib.ref_archive_decode(_u8p(raw), raw.size, _f32p(out), cap, C.byref(n)))
        return out[: n.value]

    def scaled_spectrum(self, x, block_size=256, fmt=E4M3, kind=0):
        x = _f32(x)
        out = np.zeros(-(-x.size // block_size) * block_size, np.float32)
        self._check(self.lib.ref_scaled_spectrum(_f32p(x), x.size, block_size, fmt, kind, _f32p(out)))
        return out

    def error_report(self, x, y, bins=64) -> dict:
        x, y = _f32(x), _f32(y)
        out = np.zeros(8, np.float64)
        counts = np.zeros(bins, np.uint64)
        self._check(self.lib.ref_error_report(_f32p(x), _f32p(y), x.size, bins,
                                              out.ctypes.data_as(C.POINTER(C.c_double)),
                                              counts.ctypes.data_as(C.POINTER(C.c_uint64))))
        keys = ["mse", "relative_l2", "max_abs_error", "zero_collapse_fraction", "kurtosis", "kurtosis_defined",
                "lo", "hi"]
        d = dict(zip(keys, out.tolist()))
        d["counts"] = counts.tolist()
        return d

    def archive_size(self, n, block_size=256, kind=0) -> int:
        return int(self.lib.ref_archive_size(block_size, kind, n))

    def compressed_ratio(self, n, block_size=256, kind=0) -> float:
        return float(self.lib.ref_compressed_ratio(block_size, kind, n))


def ref_available() -> bool:
    return os.path.exists(REF_SO)
