"""Vectorised (torch, integer) restatement of the reference fp8_encode (proj/src/fp8.cpp:66-91).

Test infrastructure: runs on the GPU so the device conversion can be compared against the
reference algorithm over all 2^32 fp32 bit patterns in seconds.  It is itself pinned against
the C oracle (oracle/taco_oracle.c) by tests/test_fp8_ref.py on CPU.
"""
import torch

_FMT = {0: (3, 7, 448.0, 0x7E), 1: (2, 15, 57344.0, 0x7B)}  # mbits, bias, qmax, top code


def encode(x: torch.Tensor, fmt: int) -> torch.Tensor:
    m, bias, qmax, top = _FMT[fmt]
    bits = x.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    sign = (bits >> 24) & 0x80
    ax = x.abs()
    abits = ax.view(torch.int32).to(torch.int64)
    # normal range: re-bias, round mantissa to m bits ties-to-even with carry
    a = abits - ((127 - bias) << 23)
    shift = 23 - m
    a = a + ((1 << (shift - 1)) - 1) + ((a >> shift) & 1)
    normal = (a >> shift) & 0xFF
    # subnormal range: nearbyint(|x| / 2^(1-bias-m)) in double (half to even)
    sub = torch.round(ax.double() * (2.0 ** (bias + m - 1))).to(torch.int64)
    min_normal = 2.0 ** (1 - bias)
    mag = torch.where(ax < min_normal, sub, normal)
    mag = torch.where(ax > qmax, torch.full_like(mag, top), mag)
    code = sign | mag
    code = torch.where(torch.isnan(x), torch.full_like(code, 0x7F), code)
    return code.to(torch.uint8)
